"""CPU-side checks of the drop-in boundary: the library loads, exports every
symbol include/igs_capi.h declares, and the ctypes struct mirror has the
exact C layout (checked against the header compiled with gcc)."""

import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "igs_capi.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(igs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1809_05471_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = header_functions()
    assert declared, "no functions parsed from the header"
    for name in declared:
        assert hasattr(lib, name), f"{name} missing from libigs_b200.so"
    assert set(declared) == set(_lib.EXPORTED), "ctypes binding out of sync with the header"
    assert lib.igs_abi_version() == 1


def test_status_strings_and_errors_without_gpu():
    from paper_1809_05471_b200 import _lib
    from paper_1809_05471_b200.errors import CapacityError, DomainError, UnsupportedDerivativeError

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = _lib.load()
    assert lib.igs_status_string(0) == b"ok"
    # argument validation happens on the host: no GPU needed
    st = lib.igs_tabulate(3, None, 8, None, 4, 5, None, None, None)
    assert st == _lib.IGS_EDERIV
    with pytest.raises(UnsupportedDerivativeError):
        _lib.check(st)
    st = lib.igs_gauss_rule(0, None, 2, None, None, None)
    with pytest.raises(ValueError):
        _lib.check(st)
    prob = _lib.IgsProblem()
    prob.d = 4
    st = lib.igs_apply(ctypes.byref(prob), None, None, None, None, 0, 0, None)
    assert st == _lib.IGS_EARG
    assert issubclass(DomainError, ValueError) and issubclass(CapacityError, RuntimeError)


def test_struct_layout_matches_header():
    from paper_1809_05471_b200 import _lib

    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "igs_capi.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(igs_dir), sizeof(igs_problem),
         offsetof(igs_problem, test), offsetof(igs_problem, theta), offsetof(igs_problem, plane_of),
         offsetof(igs_problem, plane_stride), offsetof(igs_problem, dir_order),
         offsetof(igs_problem, num_pairs), offsetof(igs_problem, slab_lo));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(c, "w").write(src)
        r = subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        out = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    P = _lib.IgsProblem
    want = [ctypes.sizeof(_lib.IgsDir), ctypes.sizeof(P), P.test.offset, P.theta.offset, P.plane_of.offset,
            P.plane_stride.offset, P.dir_order.offset, P.num_pairs.offset, P.slab_lo.offset]
    assert out == want


def test_pullback_struct_layout_matches_header():
    from paper_1809_05471_b200 import _lib

    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "igs_capi.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(igs_pullback_args), offsetof(igs_pullback_args, npts),
         offsetof(igs_pullback_args, grad), offsetof(igs_pullback_args, wval),
         offsetof(igs_pullback_args, reaction_stride), offsetof(igs_pullback_args, convection),
         offsetof(igs_pullback_args, diffusion), offsetof(igs_pullback_args, rtol));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(c, "w").write(src)
        r = subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        out = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    A = _lib.IgsPullbackArgs
    want = [ctypes.sizeof(A), A.npts.offset, A.grad.offset, A.wval.offset, A.reaction_stride.offset,
            A.convection.offset, A.diffusion.offset, A.rtol.offset]
    assert out == want


def test_package_imports_without_gpu():
    import paper_1809_05471_b200 as pkg
    from paper_1809_05471_b200 import bspline, sharded, tensorspace

    kv = bspline.uniform_open_knots(4, 8)
    b = bspline.UnivariateBasis(kv)
    assert b.num_basis == 11 and b.max_smoothness
    assert tensorspace.nnz_count_exact(b, b) == 2 * 4 * 11 - (16 + 8 - 1)
    assert bspline.find_span(b, 1.0) == b.num_basis - 1
    with pytest.raises(pkg.DomainError):
        bspline.find_span(b, 1.5)
    assert bspline.overlap_param(b, [0.05, 0.55]) == 4 and bspline.overlap_param(b, [0.5]) == 5
    part = sharded.SlabPartition(128, 6, 8)
    assert part.elements(0) == (0, 16) and part.own_layers(7) == (112, 133)


def test_matrix_market_roundtrip_host():
    import numpy as np
    import scipy.io
    import scipy.sparse

    from paper_1809_05471_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = _lib.load()
    A = scipy.sparse.random(60, 45, density=0.15, format="csr", random_state=3)
    A.sort_indices()
    ip = A.indptr.astype(np.int64)
    ix = A.indices.astype(np.int64)
    v = A.data.astype(np.float64)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "a.mtx")
        st = lib.igs_write_matrix_market(path.encode(), 60, 45, ip.ctypes.data, ix.ctypes.data, v.ctypes.data)
        assert st == 0
        head = open(path).readline()
        assert head.startswith("%%MatrixMarket matrix coordinate real general")
        B = scipy.io.mmread(path).tocsr()
    assert B.shape == A.shape
    assert abs(B - A).max() == 0.0   # 17 significant digits round-trip exactly
