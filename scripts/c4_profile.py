"""C4 column (dp = 1/68, 1.6h) TL-SPH steps for profiling (GPU box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2405_05155_b200 import configs
    from paper_2405_05155_b200.tlsph import SolidSystem

    cfg = configs.c4_column(kernel=sys.argv[1] if len(sys.argv) > 1 else "1.6h")
    m = cfg["material"]
    s = SolidSystem(cfg["X0"], m, cfg["spec"], cfg["dp"], fixed=cfg["fixed"], cfl=cfg["cfl"])
    s.v = cfg["v0"].copy()
    s.advance(4, graph=False)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
