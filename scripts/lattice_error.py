"""Field error of the WC lattice kernel vs the general (reference-geometry)
kernel and the oracle: rel-L2 of rho - rho0 and mom after 1 and N steps,
TGV-3D at several sizes (GPU; the oracle only where it fits quickly)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2405_05155_b200 import configs  # noqa: E402
from paper_2405_05155_b200.approx import l2_error  # noqa: E402
from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams,  # noqa: E402
                                            EulerianSolver, FluidState)


def make(cfg):
    n = cfg["pos"].shape[0]
    st = FluidState(cfg["vol"].copy(), cfg["rho"].copy(), cfg["mom"].copy(), None, n)
    return EulerianSolver(cfg["pos"], n, st, EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0),
                          cfg["spec"], None, cfl=cfg["cfl"], mu=cfg["mu"], periodic_box=cfg["box"])


for n_side, steps, with_oracle in ((16, 100, True), (64, 100, True), (256, 1, False)):
    for key in ("1.6h", "2h"):
        cfg = configs.c5_tgv3d(kernel=key, n_side=n_side)
        os.environ["SPHB_WC_LATTICE"] = "1"
        a = make(cfg)
        os.environ["SPHB_WC_LATTICE"] = "0"
        b = make(cfg)
        assert a.lattice is not None and b.lattice is None
        ref = O.EulerianWC(cfg["pos"], cfg["vol"], cfg["rho"], cfg["mom"], cfg["spec"], 10.0, 1.0,
                           cfg["mu"], cfg["cfl"], cfg["box"]) if with_oracle else None
        out = {"n_side": n_side, "kernel": key}
        for k in (1, steps):
            if k == 1:
                a.step(); b.step()
                if ref: ref.step()
            else:
                a.advance(k - 1); b.advance(k - 1)
                if ref:
                    for _ in range(k - 1):
                        ref.step()
            sa, sb = a.state, b.state
            rec = {"lattice_vs_general": [l2_error(sa.rho - 1, sb.rho - 1), l2_error(sa.mom, sb.mom)]}
            if ref:
                rec["lattice_vs_oracle"] = [l2_error(sa.rho - 1, ref.rho - 1), l2_error(sa.mom, ref.mom)]
                rec["general_vs_oracle"] = [l2_error(sb.rho - 1, ref.rho - 1), l2_error(sb.mom, ref.mom)]
            out[f"step{k}"] = rec
            if steps == 1:
                break
        print(json.dumps(out), flush=True)
        del a, b, ref
