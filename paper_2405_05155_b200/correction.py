"""Kernel-gradient correction matrices B_i on the GPU.

Drop-in for `sph_trunc.correction` (reference correction.py:1-122).
M_i = sum_j (alpha/h) dP(q) V_j r e (x) e (sphb_moment_matrices, the
_moment_matrices loop at correction.py:35-52), then B_i from M_i with the
reference's regularisation (correction.py:64-81): singular values clamped at
EPS_SV * s_max, pseudo-inverse, blend toward I by theta = clip(det(-M) /
EPS_DET, 0, 1).  The SVD is a per-particle one-sided Jacobi sweep on the
device (sphb_correction_from_moments) instead of batched LAPACK.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .kernels import KernelSpec
from .neighbors import NeighborList

EPS_SV = 1e-4     # correction.py:24
EPS_DET = 1e-6    # correction.py:25


@dataclass
class CorrectionResult:
    B: np.ndarray            # (n, d, d)
    det_neg_m: np.ndarray    # (n,) det(-M)
    n_regularized: int       # particles that hit the clamp or the blend


def _vols_dev(vols, n):
    torch = _lib.torch_cuda()
    v = _lib.to_device(np.asarray(vols, dtype=float) if not _is_t(vols) else vols, torch.float64)
    if v.ndim != 1 or v.shape[0] != n:
        raise ValueError(f"vols must have shape ({n},)")
    return v


def _is_t(a):
    import torch

    return isinstance(a, torch.Tensor)


def moment_matrices_device(nlist: NeighborList, vols, spec: KernelSpec):
    torch = _lib.torch_cuda()
    starts, idx, r, e = nlist.device_csr()
    n, d = nlist.n, e.shape[1]
    m = torch.empty((max(n, 1), d, d), dtype=torch.float64, device=starts.device)
    k = _lib.kernel_struct(spec)
    _lib.call("sphb_moment_matrices", n, d, starts.data_ptr(), idx.data_ptr(), r.data_ptr(),
              e.data_ptr(), _vols_dev(vols, n).data_ptr(), _lib.C.byref(k), m.data_ptr(),
              _lib.stream_ptr())
    return m[:n]


def moment_matrices(nlist: NeighborList, vols, spec: KernelSpec) -> np.ndarray:
    """M_i = sum_j r_ij (x) grad W_ij V_j (correction.py:55-61)."""
    return moment_matrices_device(nlist, vols, spec).cpu().numpy()


def correction_from_moments_device(m):
    """(B, det(-M), regularized flags) on the device from (n, d, d) moments."""
    torch = _lib.torch_cuda()
    n, d = m.shape[0], m.shape[1]
    m = m.contiguous()
    b = torch.empty((max(n, 1), d, d), dtype=torch.float64, device=m.device)
    det = torch.empty(max(n, 1), dtype=torch.float64, device=m.device)
    reg = torch.empty(max(n, 1), dtype=torch.int8, device=m.device)
    _lib.call("sphb_correction_from_moments", n, d, m.data_ptr(), b.data_ptr(), det.data_ptr(),
              reg.data_ptr(), _lib.stream_ptr())
    return b[:n], det[:n], reg[:n]


def correction_matrices_device(nlist: NeighborList, vols, spec: KernelSpec):
    return correction_from_moments_device(moment_matrices_device(nlist, vols, spec))


def correction_matrices(nlist: NeighborList, vols, spec: KernelSpec) -> CorrectionResult:
    """Per-particle correction matrices with regularised fallback."""
    b, det, reg = correction_matrices_device(nlist, vols, spec)
    return CorrectionResult(B=b.cpu().numpy(), det_neg_m=det.cpu().numpy(),
                            n_regularized=int(reg.sum().item()) if reg.numel() else 0)


def corrected_gradient(b_i, b_j, grad_w):
    """((B_i + B_j)/2) grad W_ij for one pair (correction.py:84-86)."""
    return 0.5 * (np.asarray(b_i) + np.asarray(b_j)) @ np.asarray(grad_w)


def pair_gradients_device(nlist: NeighborList, spec: KernelSpec, b=None):
    torch = _lib.torch_cuda()
    starts, idx, r, e = nlist.device_csr()
    n, d = nlist.n, e.shape[1]
    gw = torch.empty((max(e.shape[0], 1), d), dtype=torch.float64, device=starts.device)
    bd = None if b is None else _lib.to_device(b, torch.float64)
    k = _lib.kernel_struct(spec)
    _lib.call("sphb_pair_gradients", n, d, starts.data_ptr(), idx.data_ptr(), r.data_ptr(),
              e.data_ptr(), _lib.C.byref(k), _lib.ptr(bd), gw.data_ptr(), _lib.stream_ptr())
    return gw[:e.shape[0]]


def pair_gradients(nlist: NeighborList, spec: KernelSpec, b: np.ndarray | None = None) -> np.ndarray:
    """Per-pair (corrected) kernel gradients (correction.py:115-122)."""
    return pair_gradients_device(nlist, spec, b).cpu().numpy()
