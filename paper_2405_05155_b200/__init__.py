"""B200-native truncated-Wendland SPH hot path (arXiv 2405.05155).

Drop-in for the reference package `sph_trunc` on the particle-interaction hot
path: the modules below carry the reference's module and function names
(kernels, neighbors, correction, approx, relaxation, eulerian, tlsph,
geometry) and run every pass as a hand-written sm_100a CUDA kernel behind the
C ABI in include/sphb.h (libsphb.so, loaded through `_lib`).  There is no CPU
fallback: operators raise `BackendUnavailable` without a GPU.
"""

from .kernels import (
    KernelSpec,
    cutoff_radius,
    kernel_grad_magnitude,
    kernel_spec,
    kernel_value,
)

__all__ = [
    "KernelSpec",
    "kernel_spec",
    "kernel_value",
    "kernel_grad_magnitude",
    "cutoff_radius",
]

__version__ = "0.1.0"
