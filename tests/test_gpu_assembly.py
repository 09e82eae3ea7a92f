"""GPU setup components: the structured-hex stiffness
assembly on the device (aspamg_gpu_assemble_hex, fem.cpp:87-184 semantics)
behind the generator's assembly hook. Bar: K bit-identical to the host
assembly (which tests/test_golden.py pins against the reference's
from_triplets on its element-order triplet stream)."""
import ctypes as C

import numpy as np
import pytest


def _same(a, b):
    assert a.n_rows == b.n_rows and a.n_cols == b.n_cols and a.nnz == b.nnz
    assert np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    # bit for bit (also the sign of zeros)
    assert np.array_equal(a.values.view(np.int64), b.values.view(np.int64))


def test_assembly_hook_cpu(pkg):
    """Host logic of the hook: the backend is called with the mesh description, its
    status maps to the generator's errors, and un-registering restores the CPU path."""
    from paper_1902_01715_b200 import _native as N
    seen = {}

    class HexAssembly(C.Structure):
        _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64), ("n_free", C.c_int64),
                    ("cube", C.c_int32), ("h", C.c_double), ("node_xyz", C.c_void_p), ("free_index", C.c_void_p),
                    ("free_node", C.c_void_p), ("el_ke", C.c_void_p), ("n_ke", C.c_int64), ("young", C.c_void_p),
                    ("poisson", C.c_void_p)]

    FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(HexAssembly), C.c_void_p, C.c_void_p)

    def backend(user, inp, alloc, sink):
        m = inp.contents
        seen.update(nx=m.nx, ny=m.ny, nz=m.nz, n_free=m.n_free, cube=m.cube, n_ke=m.n_ke, h=m.h)
        return 4

    cb = FN(backend)
    lib = N.host()
    lib.aspamg_set_assembly_backend(C.cast(cb, C.c_void_p), None)
    try:
        with pytest.raises(pkg.ConfigError):
            pkg.Problem.config(2, 16)
    finally:
        lib.aspamg_set_assembly_backend(None, None)
    assert seen["nx"] == 4 and seen["n_free"] == 5 * 5 * 4 and seen["cube"] == 1 and 1 <= seen["n_ke"] <= 64
    p = pkg.Problem.config(2, 16)  # CPU path again
    assert p.K.n_rows == 3 * seen["n_free"]


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,scale", [(1, 1), (2, 4), (3, 4), (4, 8), (5, 4)])
def test_gpu_assembly_bit_identical_configs(pkg, cfg, scale):
    host = pkg.Problem.config(cfg, scale)
    dev = pkg.Problem.config(cfg, scale, assembly_device=0)
    _same(host.K, dev.K)
    assert np.array_equal(host.rhs, dev.rhs) and np.array_equal(host.coords, dev.coords)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,clamp", [((3, 2, 1), 0), ((1, 1, 1), 16), ((5, 4, 3), 63), ((6, 6, 2), 1 | 8 | 32)])
def test_gpu_assembly_bit_identical_clamps(pkg, dims, clamp):
    """Small meshes, every clamp-face combination class: none (K singular), one face, all
    faces (interior nodes only), mixed."""
    nx, ny, nz = dims
    host = pkg.Problem.hex_cube(nx, ny, nz, spacing=0.37, young=2.5, poisson=0.21, clamp=clamp)
    dev = pkg.Problem.hex_cube(nx, ny, nz, spacing=0.37, young=2.5, poisson=0.21, clamp=clamp, assembly_device=0)
    _same(host.K, dev.K)


@pytest.mark.gpu
def test_gpu_assembly_solves(pkg):
    """The device-assembled K drives the same setup + solve."""
    p = pkg.Problem.config(1, 2, assembly_device=0)
    h = pkg.Hierarchy.setup(p.K, p.coords)
    g = pkg.GpuVcycle(h, device=0)
    x, rep = g.pcg(p.rhs)
    assert rep.converged and rep.iterations <= 120
    g.close()
