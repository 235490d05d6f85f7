"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container, where the reference is mounted read-only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports `sph_trunc` (pkg/src of arXiv 2405.05155's package), drives each
hot-path configuration through the reference's own public functions
(SURVEY Appendix B recipes, at parity-test sizes) and writes compressed
.npz fixtures next to this script.  The fixtures are committed; the GPU box
never needs the reference.  Neighbour lists are stored as SHA-256 digests of
the raw CSR bytes (starts, idx, r, e) — byte equality, not just set equality —
plus the arrays themselves for the small cases.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from sph_trunc import approx, correction, eulerian, neighbors, relaxation, tlsph  # noqa: E402
from sph_trunc.geometry import lattice_points  # noqa: E402
from sph_trunc.kernels import kernel_spec  # noqa: E402

from paper_2405_05155_b200 import configs  # noqa: E402  (input generation only)


def csr_digest(nl) -> str:
    h = hashlib.sha256()
    for a in (nl.starts, nl.idx, nl.r, nl.e):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def neighbor_cases():
    """Inputs of the reference's own neighbour tests (test_neighbors.py)."""
    out = {}
    rng = np.random.default_rng(20240817)
    pos = rng.uniform(0, 1, size=(500, 2))
    out["random500"] = (pos, 0.11, None)
    rng = np.random.default_rng(20240817)
    pos = rng.uniform(0, 1, size=(300, 2))
    out["periodic300"] = (pos, 0.13, (1.0, 1.0))
    rng = np.random.default_rng(20240817)
    out["random3d_200"] = (rng.uniform(0, 1, size=(200, 3)), 0.25, None)
    out["lattice_sw"] = (lattice_points((0, 0), (9, 9), 1.0), 2.6, None)
    out["lattice_tw"] = (lattice_points((0, 0), (9, 9), 1.0), 2.08, None)
    out["lattice3d"] = (lattice_points((0, 0, 0), (9, 9, 9), 1.0), 2.3, None)
    out["periodic_lattice8"] = (lattice_points((0, 0), (8, 8), 1.0), 2.08, (8.0, 8.0))
    out["exact_cutoff"] = (np.array([[0.0, 0.0], [1.0, 0.0]]), 1.0, None)
    rng = np.random.default_rng(7)
    out["random1d_100"] = (rng.uniform(-1, 1, size=(100, 1)), 0.3, None)
    return out


def _sections():
    """`make_golden.py [section ...]`: regenerate only the named fixture
    groups (default: all)."""
    chosen = set(sys.argv[1:])
    return lambda name: not chosen or name in chosen


def main():
    want = _sections()
    if want("neighbors"):
        # ---------------------------------------------------------- neighbours
        arrays = {}
        for name, (pos, cut, box) in neighbor_cases().items():
            nl = neighbors.build_neighbors(pos, cut, box=box)
            arrays[f"{name}__pos"] = pos
            arrays[f"{name}__cutoff"] = np.array(cut)
            arrays[f"{name}__box"] = np.array(box if box is not None else [])
            arrays[f"{name}__starts"] = nl.starts
            arrays[f"{name}__idx"] = nl.idx
            arrays[f"{name}__r"] = nl.r
            arrays[f"{name}__e"] = nl.e
            arrays[f"{name}__digest"] = np.array(csr_digest(nl))
        save("neighbors", **arrays)

    if want("operators"):
        # ------------------------------------------- operators on small inputs
        arrays = {}
        rng = np.random.default_rng(11)
        pos = rng.uniform(0, 1, size=(400, 2))
        vols = rng.uniform(0.5, 1.5, size=400) / 400
        for fam in ("wendland", "wendland-truncated", "laguerre-gauss"):
            spec = kernel_spec(fam, 0.05, 2)
            nl = neighbors.build_neighbors(pos, 2.0 * spec.h)   # 2h list, kappa skip exercised
            key = fam.replace("-", "_")
            arrays[f"{key}__unity"] = approx.sph_unity_sum(nl, vols, spec)
            arrays[f"{key}__accel"] = relaxation.relax_accelerations(nl, vols, spec, 1.3, 0.9)
            arrays[f"{key}__moments"] = correction.moment_matrices(nl, vols, spec)
            res = correction.correction_matrices(nl, vols, spec)
            arrays[f"{key}__B"] = res.B
            arrays[f"{key}__det"] = res.det_neg_m
            arrays[f"{key}__nreg"] = np.array(res.n_regularized)
            arrays[f"{key}__gw"] = correction.pair_gradients(nl, spec, res.B)
            arrays[f"{key}__gw0"] = correction.pair_gradients(nl, spec, None)
        arrays["pos"] = pos
        arrays["vols"] = vols
        pos3 = rng.uniform(0, 1, size=(300, 3))
        spec3 = kernel_spec("wendland", 0.1, 3)
        nl3 = neighbors.build_neighbors(pos3, spec3.kappa * spec3.h)
        res3 = correction.correction_matrices(nl3, np.full(300, 1.0 / 300), spec3)
        arrays["pos3"] = pos3
        arrays["B3"] = res3.B
        arrays["det3"] = res3.det_neg_m
        save("operators", **arrays)

    if want("c1"):
        # ------------------------------------------------------------- C1
        c1 = configs.c1_relax(seed=0)
        spec = kernel_spec("laguerre-gauss", c1["h"], 2)
        pos = c1["pos"].copy()
        n = pos.shape[0]
        vols = np.full(n, c1["vol"])
        box = np.asarray(c1["box"])
        dt2 = c1["step_scale"] * spec.h**2
        cap = 0.25 * c1["dp"]
        digests, residuals, snaps = [], [], {}
        for step in range(c1["n_updates"] + 1):
            nl = neighbors.build_neighbors(pos, spec.kappa * spec.h, box=box)
            if step in (0, 1, c1["n_updates"]):
                digests.append(csr_digest(nl))
                snaps[step] = pos.copy()
            acc = relaxation.relax_accelerations(nl, vols, spec)
            residuals.append(float(np.mean(np.linalg.norm(acc, axis=1)) * spec.h))
            if step == 0:
                acc0 = acc.copy()
            if step == c1["n_updates"]:
                break
            dx = acc * dt2
            norms = np.linalg.norm(dx, axis=1)
            over = norms > cap
            if np.any(over):
                dx[over] *= (cap / norms[over])[:, None]
            pos += dx
            pos %= box
        dens = {}
        for key, fam in configs.FAMILY.items():
            ds = kernel_spec(fam, c1["h"], 2)
            nl = neighbors.build_neighbors(pos, ds.kappa * ds.h, box=box)
            dens[key] = approx.sph_unity_sum(nl, vols, ds)
            dens[key + "_digest"] = csr_digest(nl)
        save("c1_relax", pos0=snaps[0], pos1=snaps[1], pos100=snaps[c1["n_updates"]],
             acc0=acc0, residuals=np.asarray(residuals), digests=np.array(digests),
             rho_1p6h=dens["1.6h"], rho_2h=dens["2h"],
             digest_1p6h=np.array(dens["1.6h_digest"]), digest_2h=np.array(dens["2h_digest"]))

    if want("wc"):
        # ---------------------------------------------------- C2 / C5 (reduced)
        for label, builder, size, nsteps in (("c2_tgv2d", configs.c2_tgv2d, 64, 100),
                                             ("c5_tgv3d", configs.c5_tgv3d, 16, 200)):
            arrays = {}
            for key in ("1.6h", "2h"):
                cfg = builder(kernel=key, n_side=size)
                n = cfg["pos"].shape[0]
                state = eulerian.FluidState(vol=cfg["vol"].copy(), rho=cfg["rho"].copy(),
                                            mom=cfg["mom"].copy(), etot=None, n_interior=n)
                eos = eulerian.EosParams(eulerian.WEAKLY_COMPRESSIBLE, rho0=cfg["rho0"],
                                         c_art=cfg["c_art"])
                solver = eulerian.EulerianSolver(cfg["pos"], n, state, eos, cfg["spec"], None,
                                                 correction=True, cfl=cfg["cfl"], mu=cfg["mu"],
                                                 periodic_box=cfg["box"])
                tag = key.replace(".", "p")
                drho, dmom, _ = solver.rhs()
                arrays[f"{tag}__drho0"] = drho.copy()
                arrays[f"{tag}__dmom0"] = dmom.copy()
                dts = []
                for s in range(1, nsteps + 1):
                    dts.append(solver.step())
                    if s in (1, 100, nsteps):
                        arrays[f"{tag}__rho{s}"] = solver.state.rho.copy()
                        arrays[f"{tag}__mom{s}"] = solver.state.mom.copy()
                arrays[f"{tag}__dts"] = np.asarray(dts)
                arrays[f"{tag}__digest"] = np.array(csr_digest(solver.nlist))
            arrays["n_side"] = np.array(size)
            arrays["steps"] = np.array(nsteps)
            save(label, **arrays)

    if want("ghosts"):
        # ------------------------------- ghost layers, WC
        from sph_trunc import cases

        for label, sides_fn in (("cavity", lambda: {
                "y+": cases.SideSpec(eulerian.G_WALL, wall_v=(1.0, 0.0)),
                "y-": cases.SideSpec(eulerian.G_WALL), "x-": cases.SideSpec(eulerian.G_WALL),
                "x+": cases.SideSpec(eulerian.G_WALL)}),
                                ("mixed", lambda: {
                "y+": cases.SideSpec(eulerian.G_WALL, wall_v=(0.5, 0.0)),
                "y-": cases.SideSpec(eulerian.G_MIRROR),
                "x-": cases.SideSpec(eulerian.G_FIXED, fixed=(1.002, 0.3, 0.05, 0.0)),
                "x+": cases.SideSpec(eulerian.G_COPY)})):
            arrays = {}
            for key in ("1.6h", "2h"):
                dp = 1.0 / 20
                spec = kernel_spec(configs.FAMILY[key], 1.3 * dp, 2)
                eos = eulerian.EosParams(eulerian.WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0)
                interior, gpos, ghosts = cases.build_rect_case(
                    (0, 0), (1, 1), dp, spec.kappa * spec.h, sides_fn(), eos)
                if label == "mixed":        # feather part of the mirror band (cases.py:408-413)
                    bottom = ghosts.kind == eulerian.G_MIRROR
                    ghosts.kind[bottom & (gpos[:, 0] > 0.5)] = eulerian.G_BLEND_MIRROR
                    ghosts.blend = np.clip(gpos[:, 0] - 0.4, 0.0, 1.0)
                pos = np.vstack([interior, gpos])
                n, ni = pos.shape[0], interior.shape[0]
                rng = np.random.default_rng(5)
                rho = 1.0 + 0.002 * rng.standard_normal(n)
                mom = 0.05 * rng.standard_normal((n, 2))
                state = eulerian.FluidState(vol=np.full(n, dp * dp), rho=rho.copy(), mom=mom.copy(),
                                            etot=None, n_interior=ni)
                solver = eulerian.EulerianSolver(pos, ni, state, eos, spec, ghosts, correction=True,
                                                 cfl=0.5, mu=0.0025)
                tag = key.replace(".", "p")
                if key == "1.6h":
                    arrays["pos"], arrays["n_int"] = pos, np.array(ni)
                    arrays["rho_init"], arrays["mom_init"] = rho, mom
                arrays[f"{tag}__kind"] = ghosts.kind
                arrays[f"{tag}__src"] = ghosts.src
                arrays[f"{tag}__normal"] = ghosts.normal
                arrays[f"{tag}__wall_v"] = ghosts.wall_v
                arrays[f"{tag}__fixed"] = ghosts.fixed
                arrays[f"{tag}__blend"] = (ghosts.blend if ghosts.blend is not None
                                           else np.zeros(n - ni))
                arrays[f"{tag}__pos"] = pos
                dts = []
                for s in range(1, 51):
                    dts.append(solver.step())
                    if s in (1, 50):
                        arrays[f"{tag}__rho{s}"] = solver.state.rho[:ni].copy()
                        arrays[f"{tag}__mom{s}"] = solver.state.mom[:ni].copy()
                arrays[f"{tag}__dts"] = np.asarray(dts)
            save(f"ghosts_{label}", **arrays)

    if want("hllc"):
        # ------------------------------ HLLC + DMR
        arrays = {}
        for key in ("1.6h", "2h"):
            cfg = cases.CaseConfig(name="dmr-golden", case="dmr", solver="euler-hllc", dp=1.0 / 16,
                                   t_end=0.2, kernel_family=configs.FAMILY[key], h_ratio=1.3,
                                   cfl=0.5, correction=True)
            case = cases.build_dmr(cfg)
            solver = case.solver
            st = solver.state
            tag = key.replace(".", "p")
            g = solver.ghosts
            arrays[f"{tag}__pos"] = solver.pos
            arrays[f"{tag}__n_int"] = np.array(solver.n_int)
            arrays[f"{tag}__rho_init"] = st.rho.copy()
            arrays[f"{tag}__mom_init"] = st.mom.copy()
            arrays[f"{tag}__etot_init"] = st.etot.copy()
            for f in ("kind", "src", "normal", "wall_v", "fixed", "blend"):
                arrays[f"{tag}__{f}"] = getattr(g, f)
            arrays[f"{tag}__dmr_x0"] = np.array(g.dmr["x0"])
            arrays[f"{tag}__dmr_ghost_x"] = g.dmr["ghost_x"]
            arrays[f"{tag}__dmr_post"] = g.dmr["post"]
            arrays[f"{tag}__dmr_pre"] = g.dmr["pre"]
            drho, dmom, de = solver.rhs()
            # rhs() returns the solver's own buffers: copy before stepping reuses them
            arrays[f"{tag}__drho0"], arrays[f"{tag}__dmom0"], arrays[f"{tag}__de0"] = (
                drho.copy(), dmom.copy(), de.copy())
            dts = []
            for s_ in range(1, 21):
                dts.append(solver.step())
                if s_ in (1, 20):
                    ni = solver.n_int
                    arrays[f"{tag}__rho{s_}"] = solver.state.rho[:ni].copy()
                    arrays[f"{tag}__mom{s_}"] = solver.state.mom[:ni].copy()
                    arrays[f"{tag}__etot{s_}"] = solver.state.etot[:ni].copy()
            arrays[f"{tag}__dts"] = np.asarray(dts)
            arrays[f"{tag}__retries"] = np.array(solver.retries)
        save("hllc_dmr", **arrays)

    if want("cylinder"):
        # ------------------ cylinder: wall ghosts + wall-force series (§8(f) rank 1)
        arrays = {}
        for key in ("1.6h", "2h"):
            cfg = cases.CaseConfig(name="cyl-golden", case="cylinder", solver="euler-wc", dp=0.1,
                                   t_end=1.0, kernel_family=configs.FAMILY[key], h_ratio=1.3,
                                   cfl=0.5, correction=True,
                                   physics={"u_inf": 1.0, "rho0": 1.0, "re": 20.0},
                                   geometry={"diameter": 1.0, "extent": (5.0, 3.0),
                                             "center": (1.5, 1.5)})
            solver = cases.build_cylinder(cfg).solver
            st = solver.state
            tag = key.replace(".", "p")
            g = solver.ghosts
            arrays[f"{tag}__pos"] = solver.pos
            arrays[f"{tag}__n_int"] = np.array(solver.n_int)
            arrays[f"{tag}__mu"] = np.array(solver.mu)
            arrays[f"{tag}__wall_tag"] = np.nonzero(solver.wall_tag)[0]
            arrays[f"{tag}__rho_init"] = st.rho.copy()
            arrays[f"{tag}__mom_init"] = st.mom.copy()
            for f in ("kind", "src", "normal", "wall_v", "fixed"):
                arrays[f"{tag}__{f}"] = getattr(g, f)
            dts = []
            for s_ in range(1, 31):
                dts.append(solver.step())
                if s_ in (1, 30):
                    ni = solver.n_int
                    arrays[f"{tag}__rho{s_}"] = solver.state.rho[:ni].copy()
                    arrays[f"{tag}__mom{s_}"] = solver.state.mom[:ni].copy()
            arrays[f"{tag}__dts"] = np.asarray(dts)
            arrays[f"{tag}__wf_t"] = np.array([t for t, _ in solver.wall_force_series])
            arrays[f"{tag}__wf"] = np.array([w for _, w in solver.wall_force_series])
        save("cylinder", **arrays)

    if want("shapes"):
        # ------------- shapes + shape-bounded relaxation
        from sph_trunc import geometry as rgeo
        from sph_trunc.kernels import LAGUERRE_GAUSS, WENDLAND

        arrays = {}
        shapes = {
            "circle": rgeo.Circle(center=(0.0, 0.0), diameter=2.0),
            "semicircle": rgeo.SemiCircle(center=(0.0, 0.0), radius=0.5, flat_normal=(0.0, 1.0)),
            "rectangle": rgeo.Rectangle(lo=(0.0, 0.0), hi=(1.0, 0.5)),
            "ball": rgeo.Circle(center=(0.1, 0.2, 0.3), diameter=1.0),
            "box3": rgeo.Box3(lo=(0.0, 0.0, 0.0), hi=(1.0, 0.5, 0.25)),
        }
        rng = np.random.default_rng(5)
        for name, shp in shapes.items():
            lo, hi = shp.bounds()
            x = rng.uniform(lo - 0.3, hi + 0.3, size=(400, len(lo)))
            arrays[f"sdf_{name}__x"] = x
            arrays[f"sdf_{name}__sd"] = rgeo.signed_distance(shp, x)
            arrays[f"sdf_{name}__grad"] = rgeo.sdf_gradient(shp, x)
        for fam, hr, dim in ((WENDLAND, 1.3, 2), (LAGUERRE_GAUSS, 1.1, 2), (WENDLAND, 1.3, 3)):
            spec = kernel_spec(fam, hr * 0.1, dim)
            depth = np.linspace(-0.05, spec.kappa * spec.h + 0.05, 101)
            arrays[f"wall_{fam}_{dim}__depth"] = depth
            arrays[f"wall_{fam}_{dim}__w2"] = relaxation.wall_confinement(spec, depth)
        runs = (("circle_w", "circle", 0.1, WENDLAND, 1.3, 0.3),
                ("circle_lg", "circle", 0.1, LAGUERRE_GAUSS, 1.1, 0.1),
                ("semicircle_lg", "semicircle", 0.04, LAGUERRE_GAUSS, 1.1, 0.1),
                ("rectangle_w", "rectangle", 0.05, WENDLAND, 1.3, 0.2))
        for tag, shp, dp, fam, hr, ss in runs:
            cfg = relaxation.RelaxationConfig(shape=shapes[shp], dp=dp,
                                              kernel=kernel_spec(fam, hr * dp, 2), step_scale=ss,
                                              residual_tol=1e-12, max_steps=40, patience=None)
            res = relaxation.relax(cfg)
            arrays[f"{tag}__pos0"] = rgeo.lattice_fill(shapes[shp], dp)
            arrays[f"{tag}__positions"] = res.positions
            arrays[f"{tag}__residuals"] = res.residuals
            arrays[f"{tag}__meta"] = np.array([res.steps, res.best_step, res.n_isolated,
                                               int(res.converged)])
            arrays[f"{tag}__params"] = np.array([dp, hr, ss])
        save("relax_shapes", **arrays)

    if want("error_study"):
        # ------------------------------- error study (approx.py:61-246, §8(f) rank 3)
        arrays = {}
        rng = np.random.default_rng(9)
        pos = rng.uniform(-1, 1, size=(500, 2))
        spec = kernel_spec(WENDLAND, 0.13, 2)
        nl = neighbors.build_neighbors(pos, spec.kappa * spec.h)
        vols = np.full(500, 0.008)
        f = approx.exp_function(pos[:, 0])
        b = correction.correction_matrices(nl, vols, spec).B
        arrays["wg__pos"] = pos
        arrays["wg__plain"] = approx.weak_gradient(nl, f, vols, spec)
        arrays["wg__corrected"] = approx.weak_gradient(nl, f, vols, spec, b)
        for fam in (WENDLAND, "wendland-truncated", LAGUERRE_GAUSS):
            key = fam.replace("-", "_")
            for k, dp in enumerate((0.2, 0.1)):
                lat = approx.circle_distribution(approx.LATTICE, dp)
                arrays[f"unity__{key}__{k}"] = np.array(approx.unity_error(lat, dp, fam))
                for corr in (False, True):
                    arrays[f"grad__{key}__{k}__{int(corr)}"] = np.array(
                        approx.gradient_error(lat, dp, fam, corr))
            rows = approx.convergence_study(approx.LATTICE, fam, True)
            arrays[f"study__{key}"] = np.array([[r.dp, r.error, r.observed_order or 0.0]
                                                for r in rows])
            arrays[f"smooth__{key}"] = np.array([approx.smoothing_error(fam, h)
                                                 for h in (0.2, 0.1, 0.05)])
            arrays[f"order__{key}"] = np.array(approx.smoothing_order_check(fam))
        for dist in (approx.RELAXED_WENDLAND, approx.RELAXED_LAGUERRE_GAUSS):
            p_ = approx.circle_distribution(dist, 0.2, {"max_steps": 60, "patience": None,
                                                        "residual_tol": 1e-12})
            arrays[f"relaxed__{dist}"] = p_
            arrays[f"relaxed_grad__{dist}"] = np.array(approx.gradient_error(p_, 0.2, WENDLAND,
                                                                            True))
        save("error_study", **arrays)

    if want("harness"):
        # ------------------------------------- harness
        from sph_trunc import bench as rbench

        arrays = {}
        cfg = cases.CaseConfig(name="shear", case="shear-layer", solver="euler-wc", dp=1.0 / 32,
                               t_end=0.04, kernel_family=WENDLAND, h_ratio=1.3, cfl=0.5)
        pair, case_sw, case_tw = rbench.paired_run(cfg)
        for leg, rep in (("sw", pair.sw), ("tw", pair.tw)):
            arrays[f"shear_{leg}__steps"] = np.array(rep.steps)
            arrays[f"shear_{leg}__t_end"] = np.array(rep.t_end)
            arrays[f"shear_{leg}__nstats"] = np.array([rep.neighbor_stats[k] for k in
                                                       ("mean", "min", "max", "pairs")], float)
            arrays[f"shear_{leg}__mass_drift"] = np.array(rep.conservation["mass_rel_drift"])
            arrays[f"shear_{leg}__dt"] = np.array([rep.diagnostics["dt_min"],
                                                   rep.diagnostics["dt_max"]])
        arrays["shear__velocity_l2"] = np.array(pair.field_diff["velocity_l2"])
        arrays["shear__vorticity_l2"] = np.array(pair.field_diff["vorticity_l2"])
        arrays["shear_tw__vorticity"] = rbench.vorticity(case_tw)
        t = np.linspace(0.0, 40.0, 1600)
        f = np.column_stack([1.0 + 0.1 * np.sin(3.0 * t), 0.5 * np.sin(1.3 * t)])
        dl = rbench.drag_lift(t, f, 1.0, 1.0, 2.0)
        arrays["drag__t"], arrays["drag__f"] = t, f
        arrays["drag__cd"], arrays["drag__cl"] = dl["cd"], dl["cl"]
        arrays["drag__scalars"] = np.array([np.nan if dl["strouhal"] is None else dl["strouhal"],
                                            dl["cd_mean_tail"], dl["cl_amplitude_tail"]], float)
        save("harness", **arrays)

    if want("tl"):
        # ---------------------------------------------------- C3 / C4 (reduced)
        for label, builder, kwargs, nsteps in (("c3_plate", configs.c3_plate, {"dp": 0.002}, 100),
                                               ("c4_column", configs.c4_column, {"n_width": 6}, 200)):
            arrays = {}
            for key in ("1.6h", "2h"):
                cfg = builder(kernel=key, **kwargs)
                mat = tlsph.Material(cfg["material"].rho0, cfg["material"].E, cfg["material"].nu)
                system = tlsph.SolidSystem(cfg["X0"], mat, cfg["spec"], cfg["dp"],
                                           fixed=cfg["fixed"], correction=True, cfl=cfg["cfl"])
                system.v = cfg["v0"].copy()
                tag = key.replace(".", "p")
                arrays[f"{tag}__B0"] = system.B0.copy()
                arrays[f"{tag}__digest"] = np.array(csr_digest(system.nlist0))
                dts = []
                for s in range(1, nsteps + 1):
                    dts.append(system.step())
                    if s in (1, 100, nsteps):
                        arrays[f"{tag}__x{s}"] = system.x.copy()
                        arrays[f"{tag}__v{s}"] = system.v.copy()
                        arrays[f"{tag}__F{s}"] = system.F.copy()
                arrays[f"{tag}__dts"] = np.asarray(dts)
            arrays["steps"] = np.array(nsteps)
            save(label, **arrays)

    if want("retry"):
        # ---------------- retry-with-halving (eulerian.py:562-608), WC TGV-2D
        # step(dt) with dt a multiple of the CFL step: stages drive rho <= 0,
        # the reference halves, and (mult 20 at 1.6h, mult 40) a substep fails
        # after an accepted one, so the step restarts from its start state
        # while t keeps the accepted substep.
        arrays = {}
        for key in ("1.6h", "2h"):
            for mult in (20, 40):
                cfg = configs.c2_tgv2d(kernel=key, n_side=32)
                n = cfg["pos"].shape[0]
                state = eulerian.FluidState(vol=cfg["vol"].copy(), rho=cfg["rho"].copy(),
                                            mom=cfg["mom"].copy(), etot=None, n_interior=n)
                eos = eulerian.EosParams(eulerian.WEAKLY_COMPRESSIBLE, rho0=cfg["rho0"],
                                         c_art=cfg["c_art"])
                solver = eulerian.EulerianSolver(cfg["pos"], n, state, eos, cfg["spec"], None,
                                                 correction=True, cfl=cfg["cfl"], mu=cfg["mu"],
                                                 periodic_box=cfg["box"])
                dt = mult * solver.compute_dt()
                tag = f"{key.replace('.', 'p')}_x{mult}"
                retries, ts = [], []
                for s in range(1, 6):
                    solver.step(dt)
                    retries.append(solver.retries)
                    ts.append(solver.t)
                    arrays[f"{tag}__rho{s}"] = solver.state.rho.copy()
                    arrays[f"{tag}__mom{s}"] = solver.state.mom.copy()
                arrays[f"{tag}__dt"] = np.array(dt)
                arrays[f"{tag}__retries"] = np.asarray(retries)
                arrays[f"{tag}__t"] = np.asarray(ts)
        arrays["n_side"] = np.array(32)
        save("retry", **arrays)
        # HLLC (ideal gas, DMR at dp = 1/16): 8x the CFL step; stages leave
        # the admissible region (e < 0) and a substep fails after an accepted
        # one, so the step restarts with E restored too
        from sph_trunc import cases

        arrays = {}
        for key in ("wendland-truncated", "wendland"):
            case = cases.build_dmr(cases.CaseConfig(name="dmr", case="dmr", solver="euler-hllc",
                                                    dp=1.0 / 16, t_end=0.2, kernel_family=key))
            s_ = case.solver
            tag = "1p6h" if key == "wendland-truncated" else "2h"
            ni = s_.n_int
            dts, retries, ts = [], [], []
            for k in range(1, 7):
                dt = 8.0 * s_.compute_dt()
                s_.step(dt)
                dts.append(dt)
                retries.append(s_.retries)
                ts.append(s_.t)
                st = s_.state
                arrays[f"{tag}__rho{k}"] = st.rho[:ni].copy()
                arrays[f"{tag}__mom{k}"] = st.mom[:ni].copy()
                arrays[f"{tag}__etot{k}"] = st.etot[:ni].copy()
            arrays[f"{tag}__dt"] = np.asarray(dts)
            arrays[f"{tag}__retries"] = np.asarray(retries)
            arrays[f"{tag}__t"] = np.asarray(ts)
        save("retry_hllc", **arrays)

    if want("surface"):
        # ------ API surface beyond the hot path (eulerian.py:145-219, 366-447,
        # 645-653): pairwise Riemann helpers, module-level apply_boundaries,
        # dmr_shock_x, EulerianSolver.viscous_rhs
        arrays = {}
        rng = np.random.default_rng(17)
        lin, hll = [], []
        for k in range(40):
            d = 2 + k % 2
            e = rng.normal(size=d)
            e /= np.linalg.norm(e)
            st = []
            for _ in range(2):
                rho = 1.0 + 0.5 * rng.random()
                v = tuple(rng.normal(scale=0.8, size=d))
                p = 0.5 + rng.random()
                c = float(np.sqrt(1.4 * p / rho))
                etot = p / 0.4 + 0.5 * rho * float(np.dot(v, v))
                st.append(eulerian.InterfaceState(rho=rho, v=v, p=p, c=c, etot=etot))
            arrays[f"state{k}"] = np.array([[s_.rho, s_.p, s_.c, s_.etot] + list(s_.v) for s_ in st])
            arrays[f"e{k}"] = e
            for fn, out in ((eulerian.linearized_star, lin), (eulerian.hllc_star, hll)):
                r = fn(st[0], st[1], e)
                out.append([r.u_star, r.p_star, r.rho_star_l, r.rho_star_r, r.e_star_l,
                            r.e_star_r, r.s_l, r.s_r, r.s_star, r.beta] + list(r.v_star)
                           + [0.0] * (3 - d))
        arrays["linearized"], arrays["hllc"] = np.array(lin), np.array(hll)
        arrays["dmr_x"] = np.array([eulerian.dmr_shock_x(t) for t in (0.0, 0.05, 0.2)])
        # module-level apply_boundaries on a mixed WC frame and on the DMR frame
        from sph_trunc import cases

        dp = 1.0 / 20
        spec = kernel_spec("wendland-truncated", 1.3 * dp, 2)
        eos = eulerian.EosParams(eulerian.WEAKLY_COMPRESSIBLE, rho0=1.0, c_art=10.0)
        interior, gpos, ghosts = cases.build_rect_case(
            (0, 0), (1, 1), dp, spec.kappa * spec.h,
            {"y+": cases.SideSpec(eulerian.G_WALL, wall_v=(0.5, 0.0)),
             "y-": cases.SideSpec(eulerian.G_MIRROR),
             "x-": cases.SideSpec(eulerian.G_FIXED, fixed=(1.002, 0.3, 0.05, 0.0)),
             "x+": cases.SideSpec(eulerian.G_COPY)}, eos)
        bottom = ghosts.kind == eulerian.G_MIRROR
        ghosts.kind[bottom & (gpos[:, 0] > 0.5)] = eulerian.G_BLEND_MIRROR
        ghosts.blend = np.clip(gpos[:, 0] - 0.4, 0.0, 1.0)
        n, ni = interior.shape[0] + gpos.shape[0], interior.shape[0]
        rho = 1.0 + 0.002 * rng.standard_normal(n)
        mom = 0.05 * rng.standard_normal((n, 2))
        state = eulerian.FluidState(vol=np.full(n, dp * dp), rho=rho.copy(), mom=mom.copy(),
                                    etot=None, n_interior=ni)
        eulerian.apply_boundaries(state, ghosts, eos, 0.0)
        arrays["wc_rho_in"], arrays["wc_mom_in"] = rho, mom
        arrays["wc_rho_out"], arrays["wc_mom_out"] = state.rho, state.mom
        case = cases.build_dmr(cases.CaseConfig(name="dmr", case="dmr", solver="euler-hllc",
                                                dp=1.0 / 16, t_end=0.2,
                                                kernel_family="wendland-truncated"))
        st = case.solver.state
        st.rho[:st.n_interior] *= 1.0 + 0.01 * rng.standard_normal(st.n_interior)
        arrays["dmr_rho_in"], arrays["dmr_mom_in"] = st.rho.copy(), st.mom.copy()
        arrays["dmr_etot_in"] = st.etot.copy()
        eulerian.apply_boundaries(st, case.solver.ghosts, case.solver.eos, 0.07)
        arrays["dmr_rho_out"], arrays["dmr_mom_out"] = st.rho, st.mom
        arrays["dmr_etot_out"] = st.etot
        # viscous_rhs on C2 at 32^2
        cfg = configs.c2_tgv2d(kernel="1.6h", n_side=32)
        nn = cfg["pos"].shape[0]
        sv = eulerian.EulerianSolver(cfg["pos"], nn, eulerian.FluidState(
            vol=cfg["vol"].copy(), rho=cfg["rho"].copy(), mom=cfg["mom"].copy(), etot=None,
            n_interior=nn), eos, cfg["spec"], None, correction=True, cfl=cfg["cfl"],
            mu=cfg["mu"], periodic_box=cfg["box"])
        arrays["viscous_rhs"] = sv.viscous_rhs()
        save("surface", **arrays)


if __name__ == "__main__":
    main()
