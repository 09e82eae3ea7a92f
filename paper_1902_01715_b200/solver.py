"""Host-side mirror of the reference's solver interface for the solve path.

The reference's (C++) surface on this path is ``amg_setup(A, coordinates, cfg)
-> Hierarchy``, ``vcycle_apply(h, y)`` and
``pcg(A, b, precond, rel_tol, max_it, x0) -> (x, SolveReport)``
 with ``SolveReport`` fields from SPEC.md:498-501. The same
names, argument meanings and error behaviour are kept here; every numeric
operation of the solve runs in ``lib/libaspamg_gpu.so`` (sm_100a) behind the
C-ABI of ``include/aspamg_gpu.h``. The setup runs in ``lib/libaspamg_host.so``
(CPU, as BASELINE.json's north_star prescribes).

Errors map to the reference's hierarchy (types.hpp:15-41): status 1 ->
DimensionError, 2 -> NotSpdError, 3 -> NumericalError, 4 -> ConfigError,
7 -> IoError; 5 is a CUDA/runtime failure; 6 is non-convergence (not raised:
``SolveReport.converged`` is False).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N


class AspamgError(RuntimeError):
    pass


class DimensionError(AspamgError, ValueError):
    pass


class NotSpdError(AspamgError):
    pass


class NumericalError(AspamgError):
    pass


class ConfigError(AspamgError, ValueError):
    pass


class IoError(AspamgError):
    pass


class CudaError(AspamgError):
    pass


_ERR = {1: DimensionError, 2: NotSpdError, 3: NumericalError, 4: ConfigError, 5: CudaError, 7: IoError}


def _raise(code: int, msg: str) -> None:
    raise _ERR.get(code, AspamgError)(msg)


def _chk_host(code: int) -> None:
    if code != 0:
        _raise(code, N.host().aspamg_host_last_error().decode())


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


# --------------------------------------------------------------------- CSR
@dataclass
class SparseMatrix:
    """CSR carrier, sparse_matrix.hpp:27-59 (int64 indices, fp64 values)."""

    n_rows: int
    n_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray
    symmetric: bool = False

    @property
    def nnz(self) -> int:
        return int(self.col_indices.shape[0])

    @classmethod
    def from_view(cls, v: N.CsrView, copy: bool = True, owner=None) -> "SparseMatrix":
        """copy=False borrows the native buffers; ``owner`` (the object whose
        lifetime bounds them) is then kept alive by every array."""
        if v.n_rows == 0 and v.nnz == 0 and not v.row_offsets:
            return cls(0, int(v.n_cols), np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
        rp = _borrow(v.row_offsets, (v.n_rows + 1,), owner)
        ci = _borrow(v.col_indices, (v.nnz,), owner) if v.nnz else np.zeros(0, np.int64)
        va = _borrow(v.values, (v.nnz,), owner) if v.nnz else np.zeros(0)
        if copy:
            rp, ci, va = rp.copy(), ci.copy(), va.copy()
        return cls(int(v.n_rows), int(v.n_cols), rp, ci, va)

    @classmethod
    def from_scipy(cls, m, symmetric: bool = False) -> "SparseMatrix":
        m = m.tocsr()
        m.sort_indices()
        return cls(m.shape[0], m.shape[1], m.indptr.astype(np.int64), m.indices.astype(np.int64),
                   m.data.astype(np.float64), symmetric)

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values, self.col_indices, self.row_offsets), shape=(self.n_rows, self.n_cols))

    def view(self) -> N.CsrView:
        self.row_offsets = np.ascontiguousarray(self.row_offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(self.col_indices, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)
        return N.CsrView(self.n_rows, self.n_cols, self.nnz, _ptr(self.row_offsets, C.c_int64),
                         _ptr(self.col_indices, C.c_int64), _ptr(self.values, C.c_double))


class _Borrowed:
    """Array-interface wrapper: a numpy view of native memory whose base holds
    the memory's owner, so `K = Problem.config(2).K` cannot outlive its buffers."""

    def __init__(self, arr: np.ndarray, owner):
        self.__array_interface__ = arr.__array_interface__
        self._arr = arr
        self._owner = owner


def _borrow(ptr, shape, owner) -> np.ndarray:
    a = np.ctypeslib.as_array(ptr, shape=shape)
    return a if owner is None else np.asarray(_Borrowed(a, owner))


# ------------------------------------------------------------------ problem
class Problem:
    """Generated elasticity problem (fem.hpp:43-66 restated; BASELINE configs 1-5)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        lib = N.host()
        v = N.CsrView()
        _chk_host(lib.aspamg_problem_matrix(self._h, C.byref(v)))
        self.K = SparseMatrix.from_view(v, copy=False, owner=self)
        self.K.symmetric = True
        rp = N.P_dbl()
        n = C.c_int64()
        _chk_host(lib.aspamg_problem_rhs(self._h, C.byref(rp), C.byref(n)))
        self.rhs = _borrow(rp, (n.value,), self) if n.value else np.zeros(0)
        _chk_host(lib.aspamg_problem_coords(self._h, C.byref(rp), C.byref(n)))
        self.coords = _borrow(rp, (n.value, 3), self) if n.value else np.zeros((0, 3))

    @staticmethod
    def _assembly_backend(device: Optional[int]):
        """Route the stiffness assembly (element matrices, pattern, fill) to the GPU
        assembler on that device; K is bit-identical."""
        lib = N.host()
        if device is None:
            lib.aspamg_set_assembly_backend(None, None)
        else:
            lib.aspamg_set_assembly_backend(C.cast(N.gpu().aspamg_gpu_assemble_hex, C.c_void_p),
                                            C.c_void_p(int(device)) if device else None)

    @classmethod
    def config(cls, cfg: int, scale: int = 1, assembly_device: Optional[int] = None) -> "Problem":
        h = C.c_void_p()
        if assembly_device is not None:
            cls._assembly_backend(assembly_device)
        try:
            _chk_host(N.host().aspamg_problem_config(cfg, scale, C.byref(h)))
        finally:
            if assembly_device is not None:
                cls._assembly_backend(None)
        return cls(h)

    @classmethod
    def hex_cube(cls, nx: int, ny: Optional[int] = None, nz: Optional[int] = None, spacing: float = 1.0,
                 young: float = 1.0, poisson: float = 0.3, clamp: int = 16,
                 assembly_device: Optional[int] = None) -> "Problem":
        h = C.c_void_p()
        if assembly_device is not None:
            cls._assembly_backend(assembly_device)
        try:
            _chk_host(N.host().aspamg_problem_hex(nx, ny or nx, nz or nx, spacing, young, poisson, clamp, C.byref(h)))
        finally:
            if assembly_device is not None:
                cls._assembly_backend(None)
        return cls(h)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                N.host().aspamg_problem_free(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


# ---------------------------------------------------------------- hierarchy
def default_config(**overrides) -> N.SetupConfig:
    """Table-3 / SPEC defaults."""
    cfg = N.SetupConfig()
    _chk_host(N.host().aspamg_setup_config_default(C.byref(cfg)))
    for k, v in overrides.items():
        if not hasattr(cfg, k):
            raise ConfigError(f"unknown config key {k!r}")
        setattr(cfg, k, v)
    return cfg


@dataclass
class LevelData:
    A: SparseMatrix
    G: SparseMatrix
    Gt: SparseMatrix
    P: SparseMatrix
    Pt: SparseMatrix
    omega: float
    lambda_hat: float
    refinement_passes: int
    smoother_exit: int
    n_tv: int
    t_smoother: float = 0.0


class Hierarchy:
    """Output of the CPU setup: levels + coarsest Cholesky factor."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    @classmethod
    def setup(cls, A: SparseMatrix, coords: Optional[np.ndarray] = None, cfg: Optional[N.SetupConfig] = None,
              threads: int = 0, setup_device: Optional[int] = None) -> "Hierarchy":
        """setup_device: run the GPU setup components (SRQCG) on
        that CUDA device; None keeps the whole setup on the CPU. Both give
        bit-identical hierarchies."""
        lib = N.host()
        lib.aspamg_host_set_threads(threads)
        cfg = cfg or default_config()
        h = C.c_void_p()
        v = A.view()
        if setup_device is not None:
            dev = C.c_void_p(int(setup_device)) if setup_device else None
            lib.aspamg_set_srqcg_backend(C.cast(N.gpu().aspamg_gpu_srqcg, C.c_void_p), dev)
            lib.aspamg_set_galerkin_backend(C.cast(N.gpu().aspamg_gpu_galerkin, C.c_void_p), dev)
            lib.aspamg_set_smoother_backend(C.cast(N.gpu().aspamg_gpu_smoother_setup, C.c_void_p), dev)
        try:
            if coords is not None and len(coords):
                xyz = np.ascontiguousarray(coords, dtype=np.float64)
                _chk_host(lib.aspamg_setup(C.byref(v), _ptr(xyz, C.c_double), xyz.shape[0], C.byref(cfg),
                                           C.byref(h)))
            else:
                _chk_host(lib.aspamg_setup(C.byref(v), None, 0, C.byref(cfg), C.byref(h)))
        finally:
            if setup_device is not None:
                lib.aspamg_set_srqcg_backend(None, None)
                lib.aspamg_set_galerkin_backend(None, None)
                lib.aspamg_set_smoother_backend(None, None)
        return cls(h)

    @classmethod
    def load(cls, path: str) -> "Hierarchy":
        h = C.c_void_p()
        _chk_host(N.host().aspamg_hierarchy_load(path.encode(), C.byref(h)))
        return cls(h)

    def save(self, path: str) -> None:
        _chk_host(N.host().aspamg_hierarchy_save(self._h, path.encode()))

    def info(self) -> N.HierarchyInfo:
        i = N.HierarchyInfo()
        _chk_host(N.host().aspamg_hierarchy_info_get(self._h, C.byref(i)))
        return i

    @property
    def n_levels(self) -> int:
        return int(self.info().n_levels)

    def level_view(self, l: int) -> N.LevelView:
        lv = N.LevelView()
        _chk_host(N.host().aspamg_hierarchy_level(self._h, l, C.byref(lv)))
        return lv

    def level(self, l: int, copy: bool = True) -> LevelData:
        lv = self.level_view(l)
        f = lambda v: SparseMatrix.from_view(v, copy, None if copy else self)  # noqa: E731
        return LevelData(f(lv.A), f(lv.G), f(lv.Gt), f(lv.P), f(lv.Pt), lv.omega, lv.lambda_hat,
                         int(lv.refinement_passes), int(lv.smoother_exit), int(lv.n_tv), float(lv.t_smoother))

    def signature(self, stride: int = 1009) -> str:
        """Content hash of the hierarchy (sizes, nnz, omega and every stride-th value /
        column of each operand, the coarse factor): golden fixtures recorded on one
        hierarchy (tests/golden) are only compared against the same hierarchy."""
        import hashlib
        hh = hashlib.sha1()
        for l in range(self.n_levels):
            d = self.level(l, copy=False)
            hh.update(np.float64(d.omega).tobytes())
            for m in (d.A, d.G, d.Gt, d.P, d.Pt):
                hh.update(np.array([m.n_rows, m.n_cols, m.nnz], dtype=np.int64).tobytes())
                if m.nnz:
                    hh.update(np.ascontiguousarray(m.values[::stride]).tobytes())
                    hh.update(np.ascontiguousarray(m.col_indices[::stride]).tobytes())
        hh.update(np.ascontiguousarray(self.coarse_factor().ravel()[::7]).tobytes())
        return hh.hexdigest()

    def coarse_factor(self) -> np.ndarray:
        n = C.c_int64()
        p = N.P_dbl()
        _chk_host(N.host().aspamg_hierarchy_coarse(self._h, C.byref(n), C.byref(p)))
        return np.ctypeslib.as_array(p, shape=(n.value * n.value,)).reshape(n.value, n.value, order="F").copy()

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                N.host().aspamg_hierarchy_free(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


# ---------------------------------------------------------------- GPU solve
@dataclass
class SolveReport:
    """SPEC.md:498-501."""

    iterations: int = 0
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    converged: bool = False
    true_rel_residual: float = float("nan")
    T_s: float = 0.0          # solve seconds (device time of the PCG, events)
    T_wall: float = 0.0       # host wall time of the C-ABI call (includes H2D/D2H)
    complexities: tuple = (1.0, 1.0, 0.0)


SPMV_A, SPMV_G, SPMV_GT, SPMV_P, SPMV_PT = 0, 1, 2, 3, 4


class GpuVcycle:
    """One device context holding an uploaded hierarchy.

    Usable as the ``precond`` operator of :func:`pcg`; ``apply(y)`` is
    ``vcycle_apply(h, y)`` on the GPU.
    """

    def __init__(self, hierarchy: Hierarchy, device: int = 0, options: Optional[dict] = None):
        lib = N.gpu()
        self._lib = lib
        self._ctx = C.c_void_p()
        self._chk(lib.aspamg_gpu_ctx_create(device, C.byref(self._ctx)))
        self.hierarchy = hierarchy
        info = hierarchy.info()
        self.complexities = (info.C_gd, info.C_op, info.C_fs)
        for k, v in (options or {}).items():
            self._chk(lib.aspamg_gpu_set_option(self._ctx, k.encode(), int(v)))
        self._chk(lib.aspamg_gpu_set_cycle(self._ctx, info.nu1, info.nu2))
        for l in range(info.n_levels):
            lv = hierarchy.level_view(l)
            self._chk(lib.aspamg_gpu_upload_level(self._ctx, l, C.byref(lv.A), C.byref(lv.G), C.byref(lv.Gt),
                                                  C.byref(lv.P), C.byref(lv.Pt), lv.omega))
        n_c = C.c_int64()
        L = N.P_dbl()
        _chk_host(N.host().aspamg_hierarchy_coarse(hierarchy._h, C.byref(n_c), C.byref(L)))
        self._chk(lib.aspamg_gpu_upload_coarse(self._ctx, n_c.value, L))
        self._chk(lib.aspamg_gpu_finalize(self._ctx))
        self.n = int(hierarchy.level_view(0).A.n_rows)

    def _chk(self, code: int) -> None:
        if code != 0:
            msg = self._lib.aspamg_gpu_last_error(self._ctx if self._ctx else None)
            _raise(code, (msg or b"").decode())

    def apply(self, y: np.ndarray) -> np.ndarray:
        y = np.ascontiguousarray(y, dtype=np.float64)
        if y.shape != (self.n,):
            raise DimensionError("vcycle_apply: y length mismatch")
        z = np.empty_like(y)
        self._chk(self._lib.aspamg_gpu_vcycle(self._ctx, _ptr(y, C.c_double), _ptr(z, C.c_double)))
        return z

    __call__ = apply

    def spmv(self, level: int, which: int, x: np.ndarray) -> np.ndarray:
        lv = self.hierarchy.level_view(level)
        mat = [lv.A, lv.G, lv.Gt, lv.P, lv.Pt][which]
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (mat.n_cols,):
            raise DimensionError("spmv: x length mismatch")
        y = np.empty(mat.n_rows)
        self._chk(self._lib.aspamg_gpu_spmv(self._ctx, level, which, _ptr(x, C.c_double), _ptr(y, C.c_double)))
        return y

    def smooth(self, level: int, b: np.ndarray, x: np.ndarray) -> np.ndarray:
        """apply_smoothing_step (fsai.hpp:78-80): x' = x + w G'(G(b - A x))."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._chk(self._lib.aspamg_gpu_smooth(self._ctx, level, _ptr(b, C.c_double), _ptr(x, C.c_double),
                                              _ptr(out, C.c_double)))
        return out

    def coarse_solve(self, y: np.ndarray) -> np.ndarray:
        y = np.ascontiguousarray(y, dtype=np.float64)
        z = np.empty_like(y)
        self._chk(self._lib.aspamg_gpu_coarse_solve(self._ctx, _ptr(y, C.c_double), _ptr(z, C.c_double)))
        return z

    def pcg(self, b: np.ndarray, x0: Optional[np.ndarray] = None, rel_tol: float = 1e-8,
            max_it: int = 1000) -> tuple[np.ndarray, SolveReport]:
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.shape != (self.n,):
            raise DimensionError("pcg: b length mismatch")
        x = np.empty_like(b)
        hist = np.empty(max(int(max_it), 1))
        n_it = C.c_int64()
        conv = C.c_int()
        trr = C.c_double()
        x0p = None
        if x0 is not None:
            x0 = np.ascontiguousarray(x0, dtype=np.float64)
            if x0.shape != b.shape:
                raise DimensionError("pcg: x0 length mismatch")
            x0p = _ptr(x0, C.c_double)
        t = time.perf_counter()
        code = self._lib.aspamg_gpu_pcg(self._ctx, _ptr(b, C.c_double), x0p, rel_tol, max_it,
                                        _ptr(x, C.c_double), _ptr(hist, C.c_double), C.byref(n_it),
                                        C.byref(conv), C.byref(trr))
        wall = time.perf_counter() - t
        if code not in (0, 6):
            self._chk(code)
        ms = C.c_double()
        self._lib.aspamg_gpu_last_solve_ms(self._ctx, C.byref(ms))
        rep = SolveReport(int(n_it.value), hist[: n_it.value].copy(), bool(conv.value), float(trr.value),
                          ms.value / 1e3, wall, self.complexities)
        return x, rep

    def level_info(self, l: int) -> N.GpuLevelInfo:
        i = N.GpuLevelInfo()
        self._chk(self._lib.aspamg_gpu_level_info(self._ctx, l, C.byref(i)))
        return i

    def profile_iteration(self) -> list[tuple[str, int, float, float]]:
        buf = (N.GpuKernelTime * 512)()
        cnt = C.c_int()
        self._chk(self._lib.aspamg_gpu_profile_iteration(self._ctx, buf, 512, C.byref(cnt)))
        return [(buf[i].name.decode(), int(buf[i].level), float(buf[i].ms), float(buf[i].alg_bytes))
                for i in range(cnt.value)]

    def profile_ops(self, reps: int = 20) -> list[tuple[str, int, float, float]]:
        """Graph-mode per-op times (each op replayed ``reps`` times in one graph)."""
        buf = (N.GpuKernelTime * 512)()
        cnt = C.c_int()
        self._chk(self._lib.aspamg_gpu_profile_ops(self._ctx, reps, buf, 512, C.byref(cnt)))
        return [(buf[i].name.decode(), int(buf[i].level), float(buf[i].ms), float(buf[i].alg_bytes))
                for i in range(cnt.value)]

    def time_vcycle(self, reps: int = 50) -> float:
        """Average device ms of one V-cycle (its CUDA graph, launched back to back)."""
        ms = C.c_double()
        self._chk(self._lib.aspamg_gpu_time_vcycle(self._ctx, reps, C.byref(ms)))
        return ms.value

    def time_kernel(self, name: str, level: int, reps: int = 20) -> tuple[float, float]:
        ms = C.c_double()
        by = C.c_double()
        self._chk(self._lib.aspamg_gpu_time_kernel(self._ctx, name.encode(), level, reps, C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def launch_count(self) -> int:
        v = C.c_int64()
        self._chk(self._lib.aspamg_gpu_launch_count(self._ctx, C.byref(v)))
        return int(v.value)

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            self._lib.aspamg_gpu_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def amg_setup(A: SparseMatrix, coordinates: Optional[np.ndarray] = None, cfg: Optional[N.SetupConfig] = None,
              threads: int = 0, setup_device: Optional[int] = None) -> Hierarchy:
    """SPEC.md:436-444 (produces the hierarchy uploaded once). The setup runs on
    the CPU; with ``setup_device`` its smoother set-up (aFSAI + Lanczos), SRQCG
    test space and Galerkin products run on that GPU (bit-identical hierarchy)."""
    return Hierarchy.setup(A, coordinates, cfg, threads, setup_device)


def gpu_srqcg(A: SparseMatrix, G: SparseMatrix, V0: np.ndarray, k_max: int, k_ritz: int = 1, tol: float = 1e-2,
              seed: int = 1234, device: int = 0, Gt: Optional[SparseMatrix] = None):
    """SRQCG (Alg. 4) on S = G A G' on the GPU (include/aspamg_gpu.h
    aspamg_gpu_srqcg). Returns (V, quotients, iterations, rank_collapse)."""
    Gt = Gt if Gt is not None else SparseMatrix.from_scipy(G.to_scipy().T.tocsr())
    n, m = V0.shape
    v0 = np.asfortranarray(V0, dtype=np.float64).ravel(order="F")
    V = np.empty(n * m)
    q = np.empty(m)
    mo, it, rc = C.c_int64(), C.c_int64(), C.c_int()
    av, gv, gtv = A.view(), G.view(), Gt.view()
    P = C.POINTER(C.c_double)
    st = N.gpu().aspamg_gpu_srqcg(C.c_void_p(device) if device else None, C.byref(av), C.byref(gv), C.byref(gtv),
                                  v0.ctypes.data_as(P), m, k_max, k_ritz, tol, seed, V.ctypes.data_as(P),
                                  q.ctypes.data_as(P), C.byref(mo), C.byref(it), C.byref(rc))
    if st != 0:
        _raise(st, N.gpu().aspamg_gpu_last_error(None).decode())
    k = mo.value
    return V[: n * k].reshape(n, k, order="F"), q[:k], it.value, bool(rc.value)


class _CsrSink:
    """Numpy-owned output for aspamg_csr_alloc_fn producers."""

    def __init__(self):
        self.arrays = None
        self.shape = None
        self.fn = N.CSR_ALLOC_FN(self._alloc)

    def _alloc(self, sink, n_rows, n_cols, nnz, rp, ci, v):
        self.shape = (n_rows, n_cols)
        self.arrays = (np.zeros(n_rows + 1, np.int64), np.zeros(max(nnz, 1), np.int64), np.zeros(max(nnz, 1)))
        self.nnz = nnz
        rp[0] = self.arrays[0].ctypes.data_as(N.P_i64)
        ci[0] = self.arrays[1].ctypes.data_as(N.P_i64)
        v[0] = self.arrays[2].ctypes.data_as(N.P_dbl)
        return 0

    def matrix(self) -> "SparseMatrix":
        rp, ci, v = self.arrays
        return SparseMatrix(self.shape[0], self.shape[1], rp, ci[: self.nnz], v[: self.nnz])


def gpu_galerkin(P: SparseMatrix, A: SparseMatrix, device: int = 0) -> SparseMatrix:
    """A_c = P' (A P) on the GPU (include/aspamg_gpu.h aspamg_gpu_galerkin),
    bit-identical to the host galerkin_triple."""
    Pt = SparseMatrix.from_scipy(P.to_scipy().T.tocsr())
    sink = _CsrSink()
    pv, ptv, av = P.view(), Pt.view(), A.view()
    st = N.gpu().aspamg_gpu_galerkin(C.c_void_p(device) if device else None, C.byref(pv), C.byref(ptv), C.byref(av),
                                     C.cast(sink.fn, C.c_void_p), None)
    if st != 0:
        _raise(st, N.gpu().aspamg_gpu_last_error(None).decode())
    return sink.matrix()


def gpu_afsai(A: SparseMatrix, k: int, rho: int, eps: float, device: int = 0):
    """aFSAI build from the identity start on the GPU (aspamg_gpu_afsai_build);
    returns (G, psi), bit-identical to the host afsai_build."""
    sink = _CsrSink()
    psi = np.empty(max(A.n_rows, 1))
    av = A.view()
    st = N.gpu().aspamg_gpu_afsai_build(C.c_void_p(device) if device else None, C.byref(av), k, rho, eps,
                                        C.cast(sink.fn, C.c_void_p), None, psi.ctypes.data_as(N.P_dbl))
    if st != 0:
        _raise(st, N.gpu().aspamg_gpu_last_error(None).decode())
    return sink.matrix(), psi[: A.n_rows]


def gpu_smoother_setup(A: SparseMatrix, cfg: Optional[N.SetupConfig] = None, rho_bar: float = 0.0,
                       device: int = 0) -> dict:
    """fsai.cpp smoother_setup (Alg. 3) on the GPU (aspamg_gpu_smoother_setup)."""
    cfg = cfg or default_config()
    if rho_bar <= 0.0:
        a = A.to_scipy().tocoo()
        rho_bar = 2.0 * float(np.count_nonzero(a.col <= a.row)) / A.n_rows if A.n_rows else 1.0
    prm = N.SmootherParams(cfg.k0, cfg.rho0, cfg.eps0, cfg.ki, cfg.rhoi, cfg.epsi, cfg.omega_bar, rho_bar,
                           cfg.lanczos_steps, cfg.seed)
    sink = _CsrSink()
    psi = np.empty(max(A.n_rows, 1))
    om, lam = C.c_double(), C.c_double()
    passes, ex = C.c_int64(), C.c_int()
    av = A.view()
    st = N.gpu().aspamg_gpu_smoother_setup(C.c_void_p(device) if device else None, C.byref(av), C.byref(prm),
                                           C.cast(sink.fn, C.c_void_p), None, psi.ctypes.data_as(N.P_dbl),
                                           C.byref(om), C.byref(lam), C.byref(passes), C.byref(ex))
    if st == -1:
        return None  # declined by the level policy (gpu_setup_policy)
    if st not in (0, -2):
        _raise(st, N.gpu().aspamg_gpu_last_error(None).decode())
    return {"G": sink.matrix(), "psi": psi[: A.n_rows], "omega": om.value, "lambda_hat": lam.value,
            "passes": passes.value, "exit": ex.value, "handed_back": st == -2}


def gpu_setup_policy(key: str, value: float) -> None:
    """Process-wide policy of the GPU setup phases (aspamg_gpu_set_setup_policy)."""
    st = N.gpu().aspamg_gpu_set_setup_policy(key.encode(), float(value))
    if st != 0:
        _raise(st, N.gpu().aspamg_gpu_last_error(None).decode())


def host_smoother_setup(A: SparseMatrix, cfg: Optional[N.SetupConfig] = None) -> dict:
    """fsai.cpp smoother_setup (Alg. 3) of one operator on the host."""
    cfg = cfg or default_config()
    h = C.c_void_p()
    gv = N.CsrView()
    om, lam = C.c_double(), C.c_double()
    passes, ex = C.c_int64(), C.c_int()
    av = A.view()
    _chk_host(N.host().aspamg_smoother_setup(C.byref(av), C.byref(cfg), C.byref(h), C.byref(gv), C.byref(om),
                                             C.byref(lam), C.byref(passes), C.byref(ex)))
    try:
        G = SparseMatrix.from_view(gv, copy=True)
    finally:
        N.host().aspamg_csr_free(h)
    return {"G": G, "omega": om.value, "lambda_hat": lam.value, "passes": passes.value, "exit": ex.value}


def host_galerkin(P: SparseMatrix, A: SparseMatrix) -> SparseMatrix:
    """The host restatement of galerkin_triple (sparse_matrix.cpp:191-199)."""
    pv, av = P.view(), A.view()
    h = C.c_void_p()
    out = N.CsrView()
    _chk_host(N.host().aspamg_galerkin(C.byref(pv), C.byref(av), C.byref(h), C.byref(out)))
    try:
        return SparseMatrix.from_view(out, True)
    finally:
        N.host().aspamg_csr_free(h)


def vcycle_apply(h: GpuVcycle, y: np.ndarray) -> np.ndarray:
    """SPEC.md:445-453 on the GPU."""
    return h.apply(y)


def _same_matrix(a: SparseMatrix, b: SparseMatrix) -> bool:
    if (a.n_rows, a.n_cols, a.nnz) != (b.n_rows, b.n_cols, b.nnz):
        return False
    return all(x is y or x.ctypes.data == y.ctypes.data or np.array_equal(x, y)
               for x, y in ((a.row_offsets, b.row_offsets), (a.col_indices, b.col_indices), (a.values, b.values)))


def pcg(A: SparseMatrix, b: np.ndarray, precond: GpuVcycle, rel_tol: float = 1e-8, max_it: int = 1000,
        x0: Optional[np.ndarray] = None) -> tuple[np.ndarray, SolveReport]:
    """SPEC.md:504-512. The operator A must be the finest level of ``precond``'s
    hierarchy (the GPU context owns it on the device); a size mismatch raises
    DimensionError, pᵀAp <= 0 raises NotSpdError, non-convergence returns
    converged=False."""
    if A.n_rows != precond.n or A.n_cols != precond.n:
        raise DimensionError("pcg: operator does not match the preconditioner's finest level")
    if not _same_matrix(A, precond.hierarchy.level(0, copy=False).A):
        # the Krylov operator on the device is the hierarchy's level 0, not A
        raise DimensionError("pcg: A differs from the finest operator of the preconditioner's hierarchy")
    x, rep = precond.pcg(b, x0=x0, rel_tol=rel_tol, max_it=max_it)
    return x, rep
