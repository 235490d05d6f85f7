"""The C-ABI library loads and exports exactly what include/sphb.h declares.

CPU only: symbols are resolved, no compute entry point is called.
"""

import ctypes
import os
import re

from paper_2405_05155_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "sphb.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b(sphb_\w+)\s*\(", src, flags=re.M))


def test_header_declares_functions():
    names = declared_functions()
    assert "sphb_bin" in names and "sphb_wc_stage" in names and "sphb_tl_pass_a" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    for name in sorted(declared_functions()):
        assert hasattr(lib, name), f"libsphb.so does not export {name}"


def test_binding_table_matches_header():
    assert declared_functions() == set(_lib.SIGNATURES)


def test_version_string_without_gpu():
    lib = _lib.load_library()
    assert lib.sphb_version().decode().startswith("sphb")


def test_structs_match_header_layout(tmp_path):
    """ctypes mirrors of the ABI structs have the C compiler's size and offsets."""
    import shutil
    import subprocess

    import pytest

    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    checks = {
        "sphb_grid": (_lib.Grid, ["dim", "periodic", "ncell", "strides", "ntot", "inv_cell", "box",
                                  "lo", "cutoff", "cut2"]),
        "sphb_kernel": (_lib.Kernel, ["code", "dim", "h", "alpha", "kappa"]),
        "sphb_wc_params": (_lib.WCParams, [f for f, _ in _lib.WCParams._fields_]),
        "sphb_tl_params": (_lib.TLParams, [f for f, _ in _lib.TLParams._fields_]),
        "sphb_lattice": (_lib.Lattice, [f for f, _ in _lib.Lattice._fields_]),
        "sphb_tl_lattice": (_lib.TLLattice, [f for f, _ in _lib.TLLattice._fields_]),
    }
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "sphb.h"', "int main(void){"]
    for cname, (_, fields) in checks.items():
        lines.append(f'printf("%zu\\n", sizeof({cname}));')
        for f in fields:
            lines.append(f'printf("%zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(src), "-o", str(exe)],
                   check=True)
    vals = [int(x) for x in subprocess.run([str(exe)], check=True, capture_output=True,
                                           text=True).stdout.split()]
    k = 0
    for cname, (cls, fields) in checks.items():
        assert ctypes.sizeof(cls) == vals[k], cname
        k += 1
        for f in fields:
            assert getattr(cls, f).offset == vals[k], f"{cname}.{f}"
            k += 1


def test_product_path_fails_loudly_without_gpu():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2405_05155_b200.neighbors import build_neighbors

    with pytest.raises(_lib.BackendUnavailable):
        build_neighbors([[0.0, 0.0], [1.0, 0.0]], 1.5)


def test_lattice_host_queries_without_gpu():
    """Host-side lattice logic of the C ABI (no device work): stencil widths
    and canonical offsets (mirror-symmetric: slot W-1-k holds -o_k, which the
    mirror-order kernels rely on), and the isotropic-B test of the uniform-B
    form (b0 = beta I to 1e-12 of max|b0|)."""
    import numpy as np

    lib = _lib.load_library()
    for dim, r2, width in ((2, 4, 12), (2, 6, 20), (3, 4, 32), (3, 6, 80)):
        assert lib.sphb_lattice_width(dim, r2) == width
        off = np.zeros(3 * width, dtype=np.int32)
        assert lib.sphb_lattice_offsets(dim, r2, off.ctypes.data) == 0
        off = off.reshape(width, 3)
        assert np.array_equal(off[::-1], -off)
        assert np.all((off**2).sum(axis=1) <= r2) and np.all((off**2).sum(axis=1) > 0)
    L = _lib.Lattice()
    L.width, L.r2 = 32, 4
    beta = 1.0965629524
    for e, v in enumerate((beta, 3e-17, -2e-17, beta, 1e-17, beta * (1 + 1e-15))):
        L.b0[e] = v
    L.uniform_b = 0
    assert lib.sphb_wc_lattice_isotropic_b(3, ctypes.byref(L)) == 0      # not uniform
    L.uniform_b = 1
    assert lib.sphb_wc_lattice_isotropic_b(3, ctypes.byref(L)) == 1
    L.b0[1] = 1e-9                                                       # off-diagonal
    assert lib.sphb_wc_lattice_isotropic_b(3, ctypes.byref(L)) == 0
    L.b0[1], L.b0[3] = 0.0, beta * (1 + 1e-9)                            # unequal diagonal
    assert lib.sphb_wc_lattice_isotropic_b(3, ctypes.byref(L)) == 0
    L.width = 31
    assert lib.sphb_wc_lattice_isotropic_b(3, ctypes.byref(L)) < 0      # bad table
