#!/bin/bash
# A/B of the TL-SPH (C4 column, dp = 1/68) variants on one box.  Each
# argument is one variant: a space-separated list of environment settings
# (e.g. "SPHB_TL_PZ_B=8 SPHB_TL_ZMINB_B=3"); default: a fixed list.
cd "$(dirname "$0")/.."
if [ $# -eq 0 ]; then
  set -- "SPHB_TL_LATTICE=0" "SPHB_TLAT_MINB_A=4" "SPHB_TL_PZ_B=1" "SPHB_TL_PZ_B=8 SPHB_TL_ZMINB_B=2"
fi
for v in "$@"; do
  env $v python - "$v" <<'PY'
import sys
import torch
import bench
torch.cuda.set_device(0)
r = bench.c4_leg(torch, 32, 8, float(bench.peaks()[0]["hbm_gbs"]))
f32 = r.get("fp32_mode_1p6h", {}).get("ms_per_step", float("nan"))
print(sys.argv[1], "| 1.6h %.4f ms/step (HBM frac %.3f, fp32 mode %.4f)  2h %.4f ms/step" % (
    r["1p6h"]["ms_per_step"], r["1p6h"]["roofline"]["frac"], f32, r["2h"]["ms_per_step"]),
    flush=True)
PY
done
