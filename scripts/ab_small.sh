#!/bin/bash
# A/B of the small WC configs (C2 TGV-2D 200^2, C5 at 64^3): persistent
# multi-step lattice kernel vs CUDA-graph replay of per-stage launches.
cd "$(dirname "$0")/.."
for v in "SPHB_WC_PERSIST_MAX=0" "SPHB_WC_PERSIST_MAX=1000000000"; do
  env $v python - "$v" <<'PY'
import sys
import torch
sys.path.insert(0, ".")
from paper_2405_05155_b200 import configs
from paper_2405_05155_b200.eulerian import WEAKLY_COMPRESSIBLE, EosParams, EulerianSolver, FluidState
torch.cuda.set_device(0)
out = []
for name, cfg, steps in (("c2", configs.c2_tgv2d(), 1000), ("c2-2h", configs.c2_tgv2d(kernel="2h"), 1000),
                         ("c5-64", configs.c5_tgv3d(n_side=64), 100)):
    n = cfg["pos"].shape[0]
    s = EulerianSolver(cfg["pos"], n, FluidState(cfg["vol"], cfg["rho"], cfg["mom"], None, n),
                       EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=cfg["c_art"]), cfg["spec"], None,
                       cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])
    s.advance(16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); s.advance(steps); e1.record(); torch.cuda.synchronize()
    out.append("%s %.2f us/step" % (name, 1000 * e0.elapsed_time(e1) / steps))
print(sys.argv[1], "  ".join(out), flush=True)
PY
done
