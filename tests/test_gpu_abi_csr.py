"""The CSR-level C-ABI entries a reference maintainer would bind.

`sphb_rhs_wc_csr`, `sphb_tl_accelerations_csr` and
`sphb_tl_deformation_rates_csr` take exactly the arrays the reference's
numba kernels take (`_rhs_wc`, eulerian.py:224-266; `_accelerations`,
tlsph.py:88-102; `_deformation_rates`, tlsph.py:105-123): the reference CSR
(starts, idx, e), the per-pair gwv / viscv / g0 arrays, per-particle fields.
Here they are called through ctypes on device copies of the oracle's arrays
(the oracle's CSR is byte-identical to the reference's, test_oracle_golden.py)
and compared BIT FOR BIT with the oracle loops (both are compiled without
FMA contraction), plus the reference's own rhs golden.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2405_05155_b200 import _lib, configs
from paper_2405_05155_b200.approx import l2_error

pytestmark = pytest.mark.gpu


def dev(a, dtype=None):
    return _lib.to_device(np.ascontiguousarray(a), dtype)


@pytest.mark.parametrize("key", ["1.6h", "2h"])
def test_rhs_wc_csr_bitwise_vs_oracle_and_reference(gold, key):
    g = gold("c2_tgv2d")
    tag = key.replace(".", "p")
    cfg = configs.c2_tgv2d(kernel=key, n_side=int(g["n_side"]))
    ref = O.EulerianWC(cfg["pos"], cfg["vol"], cfg["rho"], cfg["mom"], cfg["spec"],
                       cfg["c_art"], cfg["rho0"], cfg["mu"], cfg["cfl"], cfg["box"])
    drho_o, dmom_o = ref.rhs()
    nl = ref.nl
    n, d = ref.n, ref.d
    p = cfg["c_art"] ** 2 * (ref.rho - ref.rho0)             # eos_eval (eulerian.py:67-75)
    v = ref.mom / ref.rho[:, None]                           # FluidState.velocity
    drho = torch.full((n,), np.nan, dtype=torch.float64, device="cuda")
    dmom = torch.zeros((n, d), dtype=torch.float64, device="cuda")   # caller-zeroed (:537)
    keep = [dev(nl.starts), dev(nl.idx), dev(nl.e), dev(ref.gwv), dev(ref.viscv),
            dev(ref.rho), dev(v), dev(p)]
    _lib.call("sphb_rhs_wc_csr", n, d, *[t.data_ptr() for t in keep[:8]], cfg["c_art"],
              cfg["mu"], None, drho.data_ptr(), dmom.data_ptr(), None, _lib.stream_ptr())
    drho_g, dmom_g = drho.cpu().numpy(), dmom.cpu().numpy()
    assert np.array_equal(drho_g, drho_o)
    assert np.array_equal(dmom_g, dmom_o)
    assert l2_error(drho_g, g[f"{tag}__drho0"]) < 1e-12
    assert l2_error(dmom_g, g[f"{tag}__dmom0"]) < 1e-12


@pytest.mark.parametrize("key", ["1.6h", "2h"])
def test_tl_csr_entries_bitwise_vs_oracle(key):
    cfg = configs.c3_plate(kernel=key, dp=0.004)
    m = cfg["material"]
    ref = O.SolidTL(cfg["X0"], m.rho0, m.E, m.nu, cfg["spec"], cfg["dp"], cfg["fixed"], True,
                    cfg["cfl"])
    ref.v = cfg["v0"].copy()
    for _ in range(3):                                       # a deformed state
        ref.step()
    nl, n, d = ref.nl, ref.n, ref.d
    # _deformation_rates: dF_i = [sum (v_j - v_i) (x) g0_ij] B0_i
    dF = torch.full((n, d, d), np.nan, dtype=torch.float64, device="cuda")
    keep = [dev(nl.starts), dev(nl.idx), dev(ref.g0), dev(ref.v), dev(ref.B0)]
    _lib.call("sphb_tl_deformation_rates_csr", n, d, *[t.data_ptr() for t in keep],
              dF.data_ptr(), _lib.stream_ptr())
    assert np.array_equal(dF.cpu().numpy(), ref.deformation_rates())
    # _accelerations: acc_i = sum (Q_i + Q_j) g0_ij / rho0, Q = P B0^T
    q = np.ascontiguousarray(np.concatenate(O._row_chunks(n, ref._first_pk_b0)))
    acc = torch.full((n, d), np.nan, dtype=torch.float64, device="cuda")
    keep = [dev(nl.starts), dev(nl.idx), dev(ref.g0), dev(q)]
    _lib.call("sphb_tl_accelerations_csr", n, d, *[t.data_ptr() for t in keep], m.rho0,
              acc.data_ptr(), _lib.stream_ptr())
    acc_o = np.empty((n, d))
    O.lib().orc_tl_accelerations(n, d, O._p(nl.starts), O._p(nl.idx), O._p(ref.g0), O._p(q),
                                 m.rho0, O._p(acc_o))
    assert np.array_equal(acc.cpu().numpy(), acc_o)
