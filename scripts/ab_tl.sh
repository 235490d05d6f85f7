#!/bin/bash
# A/B of the TL-SPH (C4 column, dp = 1/68) variants on one box: general
# pass-list kernels vs the lattice passes at several occupancy targets, FP64
# and the FP32-record mode.
cd "$(dirname "$0")/.."
for v in ${AB_VARIANTS:-"SPHB_TL_LATTICE=0" "SPHB_TLAT_MINB_A=4" "SPHB_TLAT_MINB_A=3 SPHB_TLAT_MINB_B=3" "SPHB_TLAT_MINB_A=2 SPHB_TLAT_MINB_B=2" "SPHB_TLAT_MINB_A=5 SPHB_TLAT_MINB_B=5"}; do
  env $v python - "$v" <<'PY'
import sys
import torch
import bench
torch.cuda.set_device(0)
r = bench.c4_leg(torch, 32, 8, float(bench.peaks()[0]["hbm_gbs"]))
f32 = r.get("fp32_mode_1p6h", {}).get("ms_per_step", float("nan"))
print(sys.argv[1], "1.6h %.4f ms/step (HBM frac %.3f, fp32 mode %.4f)  2h %.4f ms/step" % (
    r["1p6h"]["ms_per_step"], r["1p6h"]["roofline"]["frac"], f32, r["2h"]["ms_per_step"]),
    flush=True)
PY
done
