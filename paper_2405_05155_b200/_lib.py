"""ctypes binding of libsphb.so, the C-ABI library of the CUDA hot path.

The library exports plain `extern "C"` functions over device pointers
(include/sphb.h).  This module loads it, declares the argument types, and
turns non-zero status codes into Python exceptions.  PyTorch is used only as
the device-memory / stream runtime: tensors are passed as raw pointers.

There is deliberately no fallback: if the library is missing or no CUDA
device is visible, every operator raises `BackendUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPHB_LIB selects another build of the same ABI (e.g. the bounds-checked
# `make debug` library, libsphb_debug.so)
LIB_PATH = os.environ.get("SPHB_LIB") or os.path.join(_HERE, "libsphb.so")


class BackendUnavailable(RuntimeError):
    """The CUDA extension is not built or no CUDA device is available."""


class SphbError(RuntimeError):
    """A C-ABI call returned an error status."""


# ----------------------------------------------------------------- structs
class Grid(C.Structure):
    _fields_ = [
        ("dim", C.c_int32),
        ("periodic", C.c_int32),
        ("ncell", C.c_int64 * 3),
        ("strides", C.c_int64 * 3),
        ("ntot", C.c_int64),
        ("inv_cell", C.c_double * 3),
        ("box", C.c_double * 3),
        ("lo", C.c_double * 3),
        ("cutoff", C.c_double),
        ("cut2", C.c_double),
        ("sstrides", C.c_int64 * 3),
        ("slow_axis", C.c_int32),
        ("reserved", C.c_int32),
    ]


class Kernel(C.Structure):
    _fields_ = [
        ("code", C.c_int32),
        ("dim", C.c_int32),
        ("h", C.c_double),
        ("alpha", C.c_double),
        ("kappa", C.c_double),
    ]


class Shape(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("dim", C.c_int32),
        ("center", C.c_double * 3),
        ("radius", C.c_double),
        ("lo", C.c_double * 3),
        ("hi", C.c_double * 3),
        ("normal", C.c_double * 3),
    ]


def shape_struct(kind, dim, *, center=None, radius=0.0, lo=None, hi=None, normal=None) -> Shape:
    s = Shape()
    s.kind, s.dim, s.radius = int(kind), int(dim), float(radius)
    for name, val in (("center", center), ("lo", lo), ("hi", hi), ("normal", normal)):
        if val is not None:
            arr = getattr(s, name)
            for a, v in enumerate(val):
                arr[a] = float(v)
    return s


class WCParams(C.Structure):
    _fields_ = [
        ("dim", C.c_int32),
        ("periodic", C.c_int32),
        ("uniform_vol", C.c_int32),
        ("width", C.c_int32),
        ("n", C.c_int64),
        ("row0", C.c_int64),
        ("nrows", C.c_int64),
        ("box", C.c_double * 3),
        ("h", C.c_double),
        ("alpha", C.c_double),
        ("kappa", C.c_double),
        ("c_art", C.c_double),
        ("rho0", C.c_double),
        ("mu", C.c_double),
        ("cfl", C.c_double),
        ("vol_const", C.c_double),
        ("reserved0", C.c_int32),
        ("reserved", C.c_int32),
        ("interior", C.c_void_p),
        ("gamma", C.c_double),
        ("wall_tag", C.c_void_p),
        ("wall_force", C.c_void_p),
        ("push_prev", C.c_void_p),
        ("push_next", C.c_void_p),
        ("push_lo0", C.c_int64),
        ("push_lo1", C.c_int64),
        ("push_prev_at", C.c_int64),
        ("push_hi0", C.c_int64),
        ("push_hi1", C.c_int64),
        ("push_next_at", C.c_int64),
    ]


class TLParams(C.Structure):
    _fields_ = [
        ("dim", C.c_int32),
        ("width", C.c_int32),
        ("n", C.c_int64),
        ("row0", C.c_int64),
        ("nrows", C.c_int64),
        ("h", C.c_double),
        ("alpha", C.c_double),
        ("kappa", C.c_double),
        ("vol0", C.c_double),
        ("rho0", C.c_double),
        ("lam", C.c_double),
        ("g", C.c_double),
        ("push_q_prev", C.c_void_p),
        ("push_q_next", C.c_void_p),
        ("push_a_prev", C.c_void_p),
        ("push_a_next", C.c_void_p),
        ("push_v_prev", C.c_void_p),
        ("push_v_next", C.c_void_p),
        ("push_lo0", C.c_int64),
        ("push_lo1", C.c_int64),
        ("push_prev_at", C.c_int64),
        ("push_hi0", C.c_int64),
        ("push_hi1", C.c_int64),
        ("push_next_at", C.c_int64),
        ("q_stride", C.c_int64),
        ("vh32", C.c_void_p),
        ("q32", C.c_void_p),
        ("law", C.c_int32),
        ("q_dense", C.c_int32),
    ]


LATTICE_MAXW = 80


class Lattice(C.Structure):
    """sphb_lattice: the lattice fast path's extents and per-slot geometry."""

    _fields_ = [
        ("width", C.c_int32),
        ("r2", C.c_int32),
        ("n", C.c_int32 * 3),
        ("uniform_b", C.c_int32),
        ("dx", (C.c_double * 3) * LATTICE_MAXW),
        ("inv_r", C.c_double * LATTICE_MAXW),
        ("g2", C.c_double * LATTICE_MAXW),
        ("mv", C.c_double * LATTICE_MAXW),
        ("b0", C.c_double * 6),
    ]


TL_LATTICE_MAXW = 56


class TLLattice(C.Structure):
    """sphb_tl_lattice: extents and per-slot g0 expansion of the TL lattice path."""

    _fields_ = [
        ("width", C.c_int32),
        ("r2", C.c_int32),
        ("n", C.c_int32 * 3),
        ("table", C.c_int32),
        ("n_interior", C.c_int64),
        ("shell", C.c_void_p),
        ("n_shell", C.c_int64),
        ("shell_nbr", C.c_void_p),
        ("shell_cnt", C.c_void_p),
        ("r2k", C.c_double * TL_LATTICE_MAXW),
        ("f", C.c_double * TL_LATTICE_MAXW),
        ("df", C.c_double * TL_LATTICE_MAXW),
        ("dx", (C.c_double * 3) * TL_LATTICE_MAXW),
        ("g", (C.c_double * 3) * TL_LATTICE_MAXW),
        ("uniform_b0", C.c_int32),
        ("reserved_b0", C.c_int32),
        ("b0", C.c_double * 6),
    ]


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
F64 = C.c_double
SZ = C.c_size_t

# name -> (restype, argtypes); the list IS the exported ABI (tests check it
# against include/sphb.h).
SIGNATURES = {
    "sphb_version": (C.c_char_p, []),
    "sphb_last_cuda_error": (C.c_char_p, []),
    "sphb_device_count": (C.c_int, []),
    "sphb_bin_workspace_bytes": (SZ, [I64, P]),
    "sphb_bin": (C.c_int, [P, P, I64, P, P, P, P, P, SZ, P]),
    "sphb_csr_workspace_bytes": (SZ, [I64]),
    "sphb_csr_starts": (C.c_int, [P, I64, P, P, P, P, P, P, SZ, P]),
    "sphb_csr_fill": (C.c_int, [P, I64, P, P, P, P, P, P, P, P, P]),
    "sphb_ell_count": (C.c_int, [P, I64, P, P, P, F64, F64, P, P, P]),
    "sphb_ell_fill": (C.c_int, [P, I64, P, P, P, F64, F64, I32, P, P]),
    "sphb_ell_moments": (C.c_int, [P, I64, P, P, P, P, P, P, P]),
    "sphb_unity_sums": (C.c_int, [I64, P, P, P, P, P, P, P]),
    "sphb_pressure_accel": (C.c_int, [I64, I32, P, P, P, P, P, P, F64, F64, P, P]),
    "sphb_moment_matrices": (C.c_int, [I64, I32, P, P, P, P, P, P, P, P]),
    "sphb_correction_from_moments": (C.c_int, [I64, I32, P, P, P, P, P]),
    "sphb_pair_gradients": (C.c_int, [I64, I32, P, P, P, P, P, P, P, P]),
    "sphb_rhs_wc_csr": (C.c_int, [I64, I32, P, P, P, P, P, P, P, P, F64, F64, P, P, P, P, P]),
    "sphb_tl_accelerations_csr": (C.c_int, [I64, I32, P, P, P, P, F64, P, P]),
    "sphb_tl_deformation_rates_csr": (C.c_int, [I64, I32, P, P, P, P, P, P, P]),
    "sphb_wc_stage": (C.c_int, [P, I32, I32, P, P, P, P, P, P, P, P, P, P, P, P]),
    "sphb_lattice_width": (C.c_int, [I32, I32]),
    "sphb_mirror_to_host": (C.c_int, [P, P, I64, P]),
    "sphb_tl_kick": (C.c_int, [P, P, P, P, P, P]),
    "sphb_tl_lattice_width": (C.c_int, [I32, I32]),
    "sphb_tl_lattice_check": (C.c_int, [P, P, P, P, P, F64, P, P]),
    "sphb_tl_pass_a_lattice": (C.c_int, [P, P, P, P, P, P, P, P, P, P, P, P, P]),
    "sphb_tl_pass_b_lattice": (C.c_int, [P, P, P, P, P, P, P, P, P, P, I32, P, P]),
    "sphb_lattice_offsets": (C.c_int, [I32, I32, P]),
    "sphb_wc_lattice_check": (C.c_int, [P, P, P, P, P, F64, P, P]),
    "sphb_wc_lattice_isotropic_b": (C.c_int, [I32, P]),
    "sphb_wc_uniform_b_check": (C.c_int, [P, P, P, F64, P, P]),
    "sphb_tl_uniform_b0_check": (C.c_int, [P, P, P, P, F64, P, P]),
    "sphb_wc_stage_lattice": (C.c_int, [P, P, I32, P, P, P, P, P, P, P, P, P]),
    "sphb_wc_stage_lattice_f32": (C.c_int, [P, P, I32, P, P, P, P, P, P, P, P, P, P]),
    "sphb_wc_speed_max": (C.c_int, [P, P, P, P]),
    "sphb_ell_sort_rows": (C.c_int, [P, I64, P, P, P, F64, P, P]),
    "sphb_weak_gradient": (C.c_int, [I64, I32, P, P, P, P, P, P, P]),
    "sphb_shape_sdf": (C.c_int, [P, I64, P, P, P, P]),
    "sphb_relax_confine": (C.c_int, [P, I64, P, F64, P, P, I32, F64, P, P, P]),
    "sphb_relax_update_shape": (C.c_int, [P, I64, P, F64, F64, F64, P, P]),
    "sphb_bounds": (C.c_int, [I64, I32, P, P, P]),
    "sphb_wall_record": (C.c_int, [I32, P, P, F64, P, P, I64, P]),
    "sphb_copy_records": (C.c_int, [I64, P, P, P, P, P, P, P, P]),
    "sphb_wc_ghosts": (C.c_int, [I32, I64, P, P, P, P, P, P, P, P, P, P, P]),
    "sphb_hllc_stage": (C.c_int, [P, I32, P, P, P, P, P, P, P, P, P, P, P, P, P, P]),
    "sphb_hllc_pack_state": (C.c_int, [I64, I32, P, P, F64, P, P, P, P, P, P, P, P, P]),
    "sphb_hllc_unpack_state": (C.c_int, [I64, I32, P, P, P, P, P, P, P, P]),
    "sphb_hllc_ghosts": (C.c_int, [I32, I64, P, P, P, P, P, P, P, P, F64, F64, P, P, F64, F64,
                                   P, P, P, P, P, P]),
    "sphb_wc_stage_f32": (C.c_int, [P, I32, P, P, P, P, P, P, P, P, P, P, P, P, P]),
    "sphb_wc_state_to_f32": (C.c_int, [I64, I32, F64, P, P, P]),
    "sphb_wc_geometry": (C.c_int, [P, I64, P, P, P, I32, P, P, P, P, P]),
    "sphb_wc_stage_geo": (C.c_int, [P, I32, P, P, P, P, P, P, P, P, P, P, P]),
    "sphb_wc_pack_state": (C.c_int, [I64, I32, P, P, P, P, P, P]),
    "sphb_wc_unpack_state": (C.c_int, [I64, I32, P, P, P, P, P, P]),
    "sphb_fp64_probe": (C.c_int, [P, I32, I32, I32, P]),
    "sphb_set_dt": (C.c_int, [F64, F64, F64, P, P, P]),
    "sphb_tl_pass_a": (C.c_int, [P, P, P, P, P, P, P, P, P, P, P, P, P, P, P]),
    "sphb_tl_pass_b": (C.c_int, [P, P, P, P, P, P, P, P, P, P, I32, P, P]),
    "sphb_tl_geometry": (C.c_int, [P, I64, P, P, P, I32, P, F64, P, P]),
    "sphb_tl_stress": (C.c_int, [P, P, P, P, P, P]),
    "sphb_tl_speed_max": (C.c_int, [P, P, P, P]),
    "sphb_relax_accel": (C.c_int, [P, I64, P, P, P, P, P, P, F64, F64, P, P, P]),
    "sphb_relax_update": (C.c_int, [I64, I32, P, F64, F64, P, P, P]),
}

_STATUS = {
    -1: "invalid argument",
    -2: "CUDA error",
    -3: "workspace too small",
    -4: "table overflow",
}


@lru_cache(maxsize=1)
def load_library() -> C.CDLL:
    """Load libsphb.so and declare every exported signature (no device needed)."""
    if not os.path.exists(LIB_PATH):
        raise BackendUnavailable(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2405_05155_b200/csrc`"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


@lru_cache(maxsize=1)
def _torch_cuda():
    import torch

    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device visible; the sphb operators are GPU-only")
    return torch


def torch_cuda():
    """torch module, after checking that a CUDA device exists."""
    return _torch_cuda()


def lib() -> C.CDLL:
    torch_cuda()
    return load_library()


def stream_ptr() -> int:
    torch = torch_cuda()
    return torch.cuda.current_stream().cuda_stream


def check(status: int, what: str) -> None:
    if status != 0:
        msg = _STATUS.get(status, f"status {status}")
        if status == -2:
            msg += ": " + load_library().sphb_last_cuda_error().decode()
        if status == -1:
            raise ValueError(f"{what}: {msg}")
        raise SphbError(f"{what}: {msg}")


# C-ABI entry points issued from the host (bench.py counts the launches of a
# step with it; graph replays do not pass through here)
CALLS: dict = {}


def call(name: str, *args) -> None:
    CALLS[name] = CALLS.get(name, 0) + 1
    check(getattr(lib(), name)(*args), name)


def ptr(t) -> int | None:
    """Raw device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def device():
    torch = torch_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def to_device(a, dtype=None):
    """numpy array / tensor -> contiguous CUDA tensor."""
    torch = torch_cuda()
    if isinstance(a, torch.Tensor):
        t = a
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if t.device.type != "cuda":
            t = t.to(device())
        return t.contiguous()
    arr = np.ascontiguousarray(a)
    t = torch.from_numpy(arr)
    if dtype is not None:
        t = t.to(dtype)
    return t.to(device(), non_blocking=False).contiguous()


def kernel_struct(spec) -> Kernel:
    k = Kernel()
    k.code = spec.code
    k.dim = spec.dim
    k.h = spec.h
    k.alpha = spec.alpha
    k.kappa = spec.kappa
    return k
