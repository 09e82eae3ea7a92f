"""The drop-in boundary: both C-ABI libraries load and export every symbol the
headers in include/ declare; without a GPU the CUDA path fails loudly (no CPU
fallback)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "include")
LIB = os.path.join(ROOT, "paper_1902_01715_b200", "lib")


def declared(header):
    txt = open(os.path.join(INC, header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(aspamg_[a-z0-9_]+)\s*\(", txt)))


def exported(lib):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    return {ln.split()[-1] for ln in out.splitlines() if " T " in ln}


@pytest.mark.parametrize("header,lib", [("aspamg_gpu.h", "libaspamg_gpu.so"), ("aspamg_host.h", "libaspamg_host.so")])
def test_every_declared_symbol_is_exported(header, lib):
    path = os.path.join(LIB, lib)
    assert os.path.exists(path), f"{lib} not built"
    C.CDLL(path)  # loads without a GPU
    names = declared(header)
    assert len(names) >= 10
    missing = [n for n in names if n not in exported(path)]
    assert not missing, missing


def test_gpu_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", os.path.join(LIB, "libaspamg_gpu.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product_path():
    """The product package never loads the oracle (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_1902_01715_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "pyoracle" not in txt and "liboracle" not in txt and "orc_" not in txt, f


def test_gpu_calls_fail_loudly_without_device(pkg):
    from paper_1902_01715_b200 import _native as N
    lib = N.gpu()
    n = C.c_int()
    assert lib.aspamg_gpu_device_count(C.byref(n)) == 0
    if n.value > 0:
        pytest.skip("a CUDA device is present")
    ctx = C.c_void_p()
    assert lib.aspamg_gpu_ctx_create(0, C.byref(ctx)) == 5
    assert b"no CUDA device" in lib.aspamg_gpu_last_error(None)
    p = pkg.Problem.hex_cube(2)
    h = pkg.Hierarchy.setup(p.K, p.coords)
    with pytest.raises(pkg.CudaError):
        pkg.GpuVcycle(h)


def test_null_context_is_config_error():
    from paper_1902_01715_b200 import _native as N
    lib = N.gpu()
    assert lib.aspamg_gpu_finalize(None) == 4
    assert lib.aspamg_gpu_vcycle(None, None, None) == 4


@pytest.mark.parametrize("rows,fold,gran", [(256, 1, 3), (128, 1, 4), (64, 1, 2), (32, 1, 1), (512, 2, 3), (256, 2, 4), (64, 2, 3)])
def test_xsell_layout_walk_is_bit_exact(pkg, rows, fold, gran):
    """Tile-local SELL (kernels.cuh DXsell): the arrays the upload builds, walked
    on the CPU with the kernel's indexing, reproduce the sequential ascending
    row sums of spmv (sparse_matrix.cpp:100-105) bit for bit — on G, G', P, P'
    and A_1 of a small hierarchy, and on a ragged matrix with empty rows, an
    empty tile and a row count that is not a multiple of the tile."""
    import numpy as np
    import scipy.sparse as sp
    from paper_1902_01715_b200 import _native as N
    lib = N.gpu()
    P_d = C.POINTER(C.c_double)
    rng = np.random.default_rng(rows + gran)

    def check(m):
        x = rng.standard_normal(m.n_cols)
        y = np.full(m.n_rows, np.nan)
        v = m.view()
        assert lib.aspamg_gpu_xsell_layout_spmv(C.byref(v), rows, fold, gran, x.ctypes.data_as(P_d), y.ctypes.data_as(P_d)) == 0, \
            lib.aspamg_gpu_last_error(None)
        ref = np.zeros(m.n_rows)
        rp, ci, va = np.asarray(m.row_offsets), np.asarray(m.col_indices), np.asarray(m.values)
        for i in range(m.n_rows):  # the reference order: ascending columns, separate multiply / add
            s = 0.0
            for k in range(rp[i], rp[i + 1]):
                s = s + va[k] * x[ci[k]]
            ref[i] = s
        assert np.array_equal(y, ref)

    p = pkg.Problem.hex_cube(5)
    h = pkg.Hierarchy.setup(p.K, p.coords)
    lv = h.level(0)
    for m in (lv.G, lv.Gt, lv.P, lv.Pt, h.level(1).A):
        check(m)
    n, nc = 700, 333
    A = sp.random(n, nc, density=0.03, random_state=5, format="lil")
    A[256:520, :] = 0          # an all-empty tile (rows 256..511) and more empty rows
    A[5, :] = rng.standard_normal(nc)  # one full row
    A = A.tocsr()
    A.eliminate_zeros()
    A.sort_indices()
    check(pkg.SparseMatrix.from_scipy(A))


def test_view_validation_without_a_device(pkg):
    """check_view (context.cu) through the host-only layout entry point: sizes past the int32
    device indexing are a ConfigError (status 4) before any array is scanned; malformed views
    (nnz mismatch, column out of range, unsorted row) are DimensionErrors (status 1)."""
    import numpy as np
    from paper_1902_01715_b200 import _native as N
    lib = N.gpu()
    P_d = C.POINTER(C.c_double)
    x = np.zeros(4)
    y = np.zeros(4)

    def status(n_rows, n_cols, nnz, rp, ci, va):
        rp = np.asarray(rp, np.int64)
        ci = np.asarray(ci, np.int64)
        va = np.asarray(va, np.float64)
        v = N.CsrView(n_rows, n_cols, nnz, rp.ctypes.data_as(C.POINTER(C.c_int64)),
                      ci.ctypes.data_as(C.POINTER(C.c_int64)), va.ctypes.data_as(P_d))
        return lib.aspamg_gpu_xsell_layout_spmv(C.byref(v), 32, 1, 1, x.ctypes.data_as(P_d), y.ctypes.data_as(P_d))

    big = 1 << 31
    assert status(1, 4, big, [0, big], [0], [1.0]) == 4          # nnz >= 2^31: exceeds device indexing
    assert status(2, 4, 3, [0, 2, 2], [0, 1], [1.0, 1.0]) == 1    # row_offsets[n] != nnz
    assert status(2, 4, 2, [0, 1, 2], [0, 7], [1.0, 1.0]) == 1    # column out of range
    assert status(1, 4, 2, [0, 2], [2, 1], [1.0, 1.0]) == 1       # columns not ascending
    assert status(2, 4, 2, [0, 1, 2], [0, 3], [1.0, 1.0]) == 0    # well-formed
