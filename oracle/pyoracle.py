"""ctypes front-end of the CPU oracle. TEST INFRASTRUCTURE ONLY.

May be imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg — never by the product package.

* ``liboracle.so``          : oracle.c (C restatement of spmv / smoothing step /
                              V-cycle / PCG, see oracle.h for file:line anchors)
* ``_ref/libaspamg_ref.so`` : the reference's own sparse_matrix.cpp compiled
                              unmodified (+ ref_shim.cpp); optional.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
i64 = C.c_int64
P_i64 = C.POINTER(C.c_int64)
P_dbl = C.POINTER(C.c_double)


class OrcCsr(C.Structure):
    _fields_ = [("n_rows", i64), ("n_cols", i64), ("rp", P_i64), ("ci", P_i64), ("v", P_dbl), ("ref", C.c_void_p)]


class OrcLevel(C.Structure):
    _fields_ = [("A", OrcCsr), ("G", OrcCsr), ("Gt", OrcCsr), ("P", OrcCsr), ("Pt", OrcCsr), ("omega", C.c_double)]


class OrcHier(C.Structure):
    _fields_ = [("n_levels", i64), ("levels", C.POINTER(OrcLevel)), ("n_c", i64), ("Lcm", P_dbl),
                ("nu1", i64), ("nu2", i64)]


HOOK = C.CFUNCTYPE(None, C.c_void_p, P_dbl, P_dbl)

_lib = None
_ref = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = C.CDLL(os.path.join(HERE, "liboracle.so"))
        _lib.orc_set_threads.argtypes = [C.c_int]
        _lib.orc_set_dot_mode.argtypes = [C.c_int]
        _lib.orc_set_spmv_hook.argtypes = [C.c_void_p]
        _lib.orc_spmv.argtypes = [C.POINTER(OrcCsr), P_dbl, P_dbl]
        _lib.orc_smooth.argtypes = [C.POINTER(OrcHier), i64, P_dbl, P_dbl, P_dbl]
        _lib.orc_coarse_solve.argtypes = [C.POINTER(OrcHier), P_dbl, P_dbl]
        _lib.orc_vcycle.argtypes = [C.POINTER(OrcHier), P_dbl, P_dbl]
        _lib.orc_pcg.argtypes = [C.POINTER(OrcHier), P_dbl, P_dbl, C.c_double, i64, P_dbl, P_dbl, P_i64,
                                 C.POINTER(C.c_int), P_dbl]
    return _lib


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libaspamg_ref.so"))


def ref() -> C.CDLL:
    """The reference's own compiled sparse kernels (sparse_matrix.cpp)."""
    global _ref
    if _ref is None:
        _ref = C.CDLL(os.path.join(HERE, "_ref", "libaspamg_ref.so"))
        _ref.ref_csr_create.argtypes = [i64, i64, P_i64, P_i64, P_dbl]
        _ref.ref_csr_create.restype = C.c_void_p
        _ref.ref_csr_from_triplets.argtypes = [i64, i64, i64, P_i64, P_i64, P_dbl, C.c_int]
        _ref.ref_csr_from_triplets.restype = C.c_void_p
        _ref.ref_csr_free.argtypes = [C.c_void_p]
        _ref.ref_csr_shape.argtypes = [C.c_void_p, P_i64, P_i64, P_i64]
        _ref.ref_csr_copy.argtypes = [C.c_void_p, P_i64, P_i64, P_dbl]
        _ref.ref_set_threads.argtypes = [C.c_int]
        _ref.ref_spmv_checked.argtypes = [C.c_void_p, P_dbl, i64, P_dbl, i64]
        _ref.ref_spmv.argtypes = [C.c_void_p, P_dbl, P_dbl]
        _ref.ref_spmv_transpose.argtypes = [C.c_void_p, P_dbl, P_dbl]
        _ref.ref_transpose.argtypes = [C.c_void_p]
        _ref.ref_transpose.restype = C.c_void_p
        _ref.ref_galerkin_triple.argtypes = [C.c_void_p, C.c_void_p]
        _ref.ref_galerkin_triple.restype = C.c_void_p
        _ref.ref_sparse_multiply.argtypes = [C.c_void_p, C.c_void_p]
        _ref.ref_sparse_multiply.restype = C.c_void_p
        _ref.ref_lower_tri_solve_t.argtypes = [C.c_void_p, P_dbl, P_dbl]
    return _ref


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class RefCsr:
    """Handle to an aspamg::SparseMatrix living in the reference's own code."""

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def from_arrays(cls, n_rows, n_cols, rp, ci, v):
        rp = np.ascontiguousarray(rp, np.int64)
        ci = np.ascontiguousarray(ci, np.int64)
        v = np.ascontiguousarray(v, np.float64)
        return cls(ref().ref_csr_create(n_rows, n_cols, _p(rp, C.c_int64), _p(ci, C.c_int64), _p(v, C.c_double)))

    @classmethod
    def from_triplets(cls, n_rows, n_cols, r, c, v, symmetric=False):
        r = np.ascontiguousarray(r, np.int64)
        c = np.ascontiguousarray(c, np.int64)
        v = np.ascontiguousarray(v, np.float64)
        return cls(ref().ref_csr_from_triplets(n_rows, n_cols, len(v), _p(r, C.c_int64), _p(c, C.c_int64),
                                               _p(v, C.c_double), int(symmetric)))

    def arrays(self):
        nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        ref().ref_csr_shape(self.h, C.byref(nr), C.byref(nc), C.byref(nz))
        rp = np.empty(nr.value + 1, np.int64)
        ci = np.empty(nz.value, np.int64)
        v = np.empty(nz.value)
        ref().ref_csr_copy(self.h, _p(rp, C.c_int64), _p(ci, C.c_int64), _p(v, C.c_double))
        return nr.value, nc.value, rp, ci, v

    def spmv(self, x):
        x = np.ascontiguousarray(x, np.float64)
        nr, nc, _, _, _ = self.shape()
        y = np.empty(nr)
        ref().ref_spmv(self.h, _p(x, C.c_double), _p(y, C.c_double))
        return y

    def spmv_transpose(self, x):
        x = np.ascontiguousarray(x, np.float64)
        nr, nc, _, _, _ = self.shape()
        y = np.empty(nc)
        ref().ref_spmv_transpose(self.h, _p(x, C.c_double), _p(y, C.c_double))
        return y

    def shape(self):
        nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        ref().ref_csr_shape(self.h, C.byref(nr), C.byref(nc), C.byref(nz))
        return nr.value, nc.value, nz.value, None, None

    def transpose(self):
        return RefCsr(ref().ref_transpose(self.h))

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_csr_free(self.h)
            self.h = None


class OracleHierarchy:
    """Borrowed view of a product Hierarchy (the SAME arrays the GPU gets)."""

    def __init__(self, h, use_ref_spmv: bool = False, threads: int = 1):
        info = h.info()
        self._hier = h  # the views below borrow its arrays
        self._keep = []
        self._refs = []
        L = int(info.n_levels)
        self.levels = (OrcLevel * L)()
        for l in range(L):
            lv = h.level(l, copy=False)
            for name in ("A", "G", "Gt", "P", "Pt"):
                m = getattr(lv, name)
                oc = OrcCsr(m.n_rows, m.n_cols, _p(m.row_offsets, C.c_int64), _p(m.col_indices, C.c_int64),
                            _p(m.values, C.c_double), None)
                self._keep.append(m)
                if use_ref_spmv and m.n_rows > 0:
                    r = RefCsr.from_arrays(m.n_rows, m.n_cols, m.row_offsets, m.col_indices, m.values)
                    self._refs.append(r)
                    oc.ref = r.h
                setattr(self.levels[l], name, oc)
            self.levels[l].omega = lv.omega
        self.Lcm = np.asfortranarray(h.coarse_factor())
        self._Lflat = np.ascontiguousarray(self.Lcm.ravel(order="F"))
        self.h = OrcHier(L, self.levels, self.Lcm.shape[0], _p(self._Lflat, C.c_double), info.nu1, info.nu2)
        self.n = int(self.levels[0].A.n_rows)
        self.use_ref = use_ref_spmv
        self.threads = threads
        self._hook = HOOK(lambda h_, x, y: ref().ref_spmv(h_, x, y)) if use_ref_spmv else None

    def _activate(self):
        lib().orc_set_threads(self.threads)
        if self.use_ref:
            ref().ref_set_threads(self.threads)
            lib().orc_set_spmv_hook(C.cast(ref().ref_spmv, C.c_void_p))
        else:
            lib().orc_set_spmv_hook(None)

    def spmv(self, level: int, which: str, x):
        self._activate()
        m = getattr(self.levels[level], which)
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(m.n_rows)
        lib().orc_spmv(C.byref(m), _p(x, C.c_double), _p(y, C.c_double))
        return y

    def vcycle(self, y):
        self._activate()
        y = np.ascontiguousarray(y, np.float64)
        z = np.empty_like(y)
        lib().orc_vcycle(C.byref(self.h), _p(y, C.c_double), _p(z, C.c_double))
        return z

    def smooth(self, level, b, x):
        self._activate()
        b = np.ascontiguousarray(b, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(x)
        lib().orc_smooth(C.byref(self.h), level, _p(b, C.c_double), _p(x, C.c_double), _p(out, C.c_double))
        return out

    def coarse_solve(self, y):
        self._activate()
        y = np.ascontiguousarray(y, np.float64)
        z = np.empty_like(y)
        lib().orc_coarse_solve(C.byref(self.h), _p(y, C.c_double), _p(z, C.c_double))
        return z

    def pcg(self, b, x0: Optional[np.ndarray] = None, rel_tol=1e-8, max_it=1000):
        self._activate()
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        hist = np.empty(max(max_it, 1))
        n_it = C.c_int64()
        conv = C.c_int()
        trr = C.c_double()
        x0p = _p(np.ascontiguousarray(x0, np.float64), C.c_double) if x0 is not None else None
        st = lib().orc_pcg(C.byref(self.h), _p(b, C.c_double), x0p, rel_tol, max_it, _p(x, C.c_double),
                           _p(hist, C.c_double), C.byref(n_it), C.byref(conv), C.byref(trr))
        return st, x, hist[: n_it.value].copy(), bool(conv.value), float(trr.value)
