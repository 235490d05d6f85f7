"""Single-GPU projection of the C5 slab decomposition.

One rank's solver of a `world`-way z-slab split of TGV-3D 256^3 (owned planes
+ one cell layer of halo each side, the lattice kernel on the owned rows,
boundary-first stage launches) runs on this GPU with a stand-in for
torch.distributed whose exchanges and all-reduces do nothing.  The fields are
therefore wrong (halos never refresh) but the timing is that rank's compute
and launch structure, without the NCCL transfers (~8 MB per stage per rank
over NVLink) and without cross-rank skew.  Prints per-rank ms/step and the
compute-only scaling efficiency (T_1 / world) / T_world, T_1 the eager
one-GPU step (slab steps run eagerly too) and, beside it, the one-GPU step
replayed from a CUDA graph (bench.py's number).  This is a
projection, NOT a multi-GPU measurement.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_05155_b200 import configs  # noqa: E402
from paper_2405_05155_b200.eulerian import (WEAKLY_COMPRESSIBLE, EosParams,  # noqa: E402
                                            EulerianSolver, FluidState)
from paper_2405_05155_b200.slab import slab_eulerian  # noqa: E402


class NullDist:
    """Accepts the torch.distributed calls slab.py / eulerian.py make and
    moves no data."""

    class ReduceOp:
        MAX = "max"
        SUM = "sum"

    class P2POp:
        def __init__(self, fn, tensor, peer, group=None):
            self.fn, self.tensor, self.peer = fn, tensor, peer

    def isend(self, *a):
        return None

    def irecv(self, *a):
        return None

    def batch_isend_irecv(self, ops):
        return []

    def all_reduce(self, t, op=None):
        return None


def timed(solver, steps, warmup, graph):
    solver.advance(warmup, graph=graph)          # captures the step graph outside the timing
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    solver.advance(steps, graph=graph)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    n_side = int(os.environ.get("N_SIDE", "256"))
    steps, warmup = 24, 8
    torch.cuda.set_device(0)
    out = {}
    for key in ("1.6h", "2h"):
        cfg = configs.c5_tgv3d(kernel=key, n_side=n_side)
        n = cfg["pos"].shape[0]
        eos = EosParams(WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0)

        def state():
            return FluidState(cfg["vol"].copy(), cfg["rho"].copy(), cfg["mom"].copy(), None, n)

        one = EulerianSolver(cfg["pos"], n, state(), eos, cfg["spec"], None, cfl=cfg["cfl"],
                             mu=cfg["mu"], periodic_box=cfg["box"])
        t1g = timed(one, steps, warmup, True)
        t1 = timed(one, steps, warmup, False)
        del one
        torch.cuda.empty_cache()
        rec = {"1": {"ms_per_step": t1, "ms_per_step_graph": t1g}}
        for world in (2, 4, 8):
            s = slab_eulerian(cfg["pos"], state(), eos, cfg["spec"], rank=0, world=world,
                              dist=NullDist(), cfl=cfg["cfl"], mu=cfg["mu"],
                              periodic_box=cfg["box"])
            if s.lattice is not None and not s.lattice.uniform_b:
                # the stand-in moves no halo data, so the halo rows keep their
                # locally computed B (truncated stencils); a real exchange
                # gives them their owners' B, which on the TGV lattice is the
                # uniform b0: emulate that for B alone, then re-run the check
                nn = s.n
                r0 = int(s.params.row0)
                p0 = s.B[:4 * nn].view(nn, 4)
                p1 = s.B[4 * nn:].view(nn, 2)
                p0.copy_(p0[r0].expand_as(p0).clone())
                p1.copy_(p1[r0].expand_as(p1).clone())
                s._setup_uniform_b()
            tw = timed(s, steps, warmup, False)      # slab steps run eagerly
            rec[str(world)] = {"ms_per_step": tw, "rows_local": int(s.n),
                               "rows_owned": int(s._slab.rows.stop - s._slab.rows.start),
                               "lattice_path": s.lattice is not None,
                               "uniform_b": bool(s.lattice is not None and s.lattice.uniform_b),
                               "compute_only_efficiency": (t1 / world) / tw}
            del s
            torch.cuda.empty_cache()
        out[key] = rec
        print(json.dumps({"kernel": key, **rec}), flush=True)


if __name__ == "__main__":
    main()
