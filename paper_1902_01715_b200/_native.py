"""ctypes bindings for the two in-tree native libraries.

* ``lib/libaspamg_host.so`` — CPU setup + generator, C-ABI in ``include/aspamg_host.h``.
* ``lib/libaspamg_gpu.so``  — the sm_100a solve path, C-ABI in ``include/aspamg_gpu.h``.

Nothing here computes: it only declares signatures. The GPU library is loaded
lazily and a missing/unloadable library raises — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")

i64 = C.c_int64
i32 = C.c_int32
dbl = C.c_double
P_i64 = C.POINTER(C.c_int64)
P_dbl = C.POINTER(C.c_double)


class CsrView(C.Structure):
    _fields_ = [("n_rows", i64), ("n_cols", i64), ("nnz", i64),
                ("row_offsets", P_i64), ("col_indices", P_i64), ("values", P_dbl)]


class SmootherParams(C.Structure):
    """aspamg_smoother_params (include/aspamg_csr.h)."""
    _fields_ = [("k0", C.c_int64), ("rho0", C.c_int64), ("eps0", C.c_double), ("ki", C.c_int64),
                ("rhoi", C.c_int64), ("epsi", C.c_double), ("omega_bar", C.c_double), ("rho_bar", C.c_double),
                ("lanczos_steps", C.c_int64), ("seed", C.c_uint64)]


class SetupConfig(C.Structure):
    _fields_ = [("k0", i64), ("rho0", i64), ("eps0", dbl),
                ("ki", i64), ("rhoi", i64), ("epsi", dbl),
                ("omega_bar", dbl), ("rho_bar", dbl), ("lanczos_steps", i64),
                ("n_tv", i64), ("n_rq", i64), ("k_ritz", i64), ("srqcg_tol", dbl),
                ("theta", i64), ("d_p", i64), ("n_max", i64), ("eps_p", dbl), ("kappa_p", dbl),
                ("max_levels", i64), ("min_coarse_size", i64), ("nu1", i64), ("nu2", i64),
                ("seed", C.c_uint64)]


class LevelView(C.Structure):
    _fields_ = [("A", CsrView), ("G", CsrView), ("Gt", CsrView), ("P", CsrView), ("Pt", CsrView),
                ("omega", dbl), ("lambda_hat", dbl), ("kaporin_estimate", dbl),
                ("refinement_passes", i64), ("smoother_exit", i32), ("n_tv", i64), ("t_smoother", dbl)]


class HierarchyInfo(C.Structure):
    _fields_ = [("n_levels", i64), ("n_coarse", i64), ("nu1", i64), ("nu2", i64),
                ("C_gd", dbl), ("C_op", dbl), ("C_fs", dbl),
                ("T_ts", dbl), ("T_cs", dbl), ("T_sm", dbl), ("T_pl", dbl), ("T_rap", dbl), ("T_p", dbl)]


class GpuLevelInfo(C.Structure):
    _fields_ = [("n", i64), ("a_format", i32), ("a_nnz", i64), ("a_nnzb", i64), ("a_fill", dbl),
                ("g_nnz", i64), ("p_nnz", i64), ("omega", dbl),
                ("alg_bytes_A", dbl), ("alg_bytes_G", dbl), ("alg_bytes_Gt", dbl),
                ("alg_bytes_P", dbl), ("alg_bytes_Pt", dbl), ("device_bytes", dbl),
                ("fmt", i32 * 5), ("fill", dbl * 5)]


class GpuKernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("level", i32), ("ms", dbl), ("alg_bytes", dbl)]


class Status(RuntimeError):
    """Non-zero status from a C-ABI call; ``code`` follows SURVEY.md §8b."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_host = None
_gpu = None


def host() -> C.CDLL:
    global _host
    if _host is None:
        path = os.path.join(LIB_DIR, "libaspamg_host.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run __graft_entry__.build() (make)")
        lib = C.CDLL(path)
        lib.aspamg_host_last_error.restype = C.c_char_p
        lib.aspamg_host_set_threads.argtypes = [C.c_int]
        lib.aspamg_problem_config.argtypes = [C.c_int, i64, C.POINTER(C.c_void_p)]
        lib.aspamg_problem_hex.argtypes = [i64, i64, i64, dbl, dbl, dbl, C.c_uint32, C.POINTER(C.c_void_p)]
        lib.aspamg_problem_matrix.argtypes = [C.c_void_p, C.POINTER(CsrView)]
        lib.aspamg_problem_rhs.argtypes = [C.c_void_p, C.POINTER(P_dbl), P_i64]
        lib.aspamg_problem_coords.argtypes = [C.c_void_p, C.POINTER(P_dbl), P_i64]
        lib.aspamg_problem_free.argtypes = [C.c_void_p]
        lib.aspamg_problem_free.restype = None
        lib.aspamg_setup_config_default.argtypes = [C.POINTER(SetupConfig)]
        lib.aspamg_setup.argtypes = [C.POINTER(CsrView), P_dbl, i64, C.POINTER(SetupConfig), C.POINTER(C.c_void_p)]
        lib.aspamg_hierarchy_info_get.argtypes = [C.c_void_p, C.POINTER(HierarchyInfo)]
        lib.aspamg_hierarchy_level.argtypes = [C.c_void_p, i64, C.POINTER(LevelView)]
        lib.aspamg_hierarchy_coarse.argtypes = [C.c_void_p, P_i64, C.POINTER(P_dbl)]
        lib.aspamg_hierarchy_save.argtypes = [C.c_void_p, C.c_char_p]
        lib.aspamg_hierarchy_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        lib.aspamg_hierarchy_free.argtypes = [C.c_void_p]
        lib.aspamg_hierarchy_free.restype = None
        lib.aspamg_srqcg.argtypes = [C.POINTER(CsrView), C.POINTER(CsrView), P_dbl, i64, i64, i64, dbl, C.c_uint64,
                                     P_dbl, P_dbl, P_i64]
        lib.aspamg_afsai_build.argtypes = [C.POINTER(CsrView), i64, i64, dbl, C.POINTER(C.c_void_p), C.POINTER(CsrView)]
        lib.aspamg_smoother_setup.argtypes = [C.POINTER(CsrView), C.POINTER(SetupConfig), C.POINTER(C.c_void_p),
                                              C.POINTER(CsrView), P_dbl, P_dbl, P_i64, C.POINTER(C.c_int)]
        lib.aspamg_estimate_lambda_max.argtypes = [C.POINTER(CsrView), C.POINTER(CsrView), i64, C.c_uint64, P_dbl]
        lib.aspamg_csr_free.argtypes = [C.c_void_p]
        lib.aspamg_csr_free.restype = None
        lib.aspamg_set_srqcg_backend.argtypes = [C.c_void_p, C.c_void_p]
        lib.aspamg_set_galerkin_backend.argtypes = [C.c_void_p, C.c_void_p]
        lib.aspamg_set_smoother_backend.argtypes = [C.c_void_p, C.c_void_p]
        lib.aspamg_set_assembly_backend.argtypes = [C.c_void_p, C.c_void_p]
        lib.aspamg_galerkin.argtypes = [C.POINTER(CsrView), C.POINTER(CsrView), C.POINTER(C.c_void_p),
                                        C.POINTER(CsrView)]
        _host = lib
    return _host


def check_host(code: int) -> None:
    if code != 0:
        raise Status(code, host().aspamg_host_last_error().decode())


def gpu() -> C.CDLL:
    """Load the CUDA solve library. Raises if it is missing: no fallback path."""
    global _gpu
    if _gpu is None:
        path = os.path.join(LIB_DIR, "libaspamg_gpu.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: the CUDA extension is required (run make)")
        lib = C.CDLL(path)
        vp = C.c_void_p
        lib.aspamg_gpu_last_error.argtypes = [vp]
        lib.aspamg_gpu_last_error.restype = C.c_char_p
        lib.aspamg_gpu_device_count.argtypes = [C.POINTER(C.c_int)]
        lib.aspamg_gpu_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
        lib.aspamg_gpu_ctx_destroy.argtypes = [vp]
        lib.aspamg_gpu_upload_level.argtypes = [vp, i64, C.POINTER(CsrView), C.POINTER(CsrView), C.POINTER(CsrView),
                                                C.POINTER(CsrView), C.POINTER(CsrView), dbl]
        lib.aspamg_gpu_upload_coarse.argtypes = [vp, i64, P_dbl]
        lib.aspamg_gpu_set_cycle.argtypes = [vp, i64, i64]
        lib.aspamg_gpu_set_option.argtypes = [vp, C.c_char_p, i64]
        lib.aspamg_gpu_finalize.argtypes = [vp]
        lib.aspamg_gpu_vcycle.argtypes = [vp, P_dbl, P_dbl]
        lib.aspamg_gpu_vcycle_device.argtypes = [vp, vp, vp]
        lib.aspamg_gpu_spmv.argtypes = [vp, i64, C.c_int, P_dbl, P_dbl]
        lib.aspamg_gpu_smooth.argtypes = [vp, i64, P_dbl, P_dbl, P_dbl]
        lib.aspamg_gpu_coarse_solve.argtypes = [vp, P_dbl, P_dbl]
        lib.aspamg_gpu_pcg.argtypes = [vp, P_dbl, P_dbl, dbl, i64, P_dbl, P_dbl, P_i64, C.POINTER(C.c_int), P_dbl]
        lib.aspamg_gpu_pcg_device.argtypes = [vp, vp, vp, dbl, i64, vp, P_dbl, P_i64, C.POINTER(C.c_int), P_dbl]
        lib.aspamg_gpu_level_info.argtypes = [vp, i64, C.POINTER(GpuLevelInfo)]
        lib.aspamg_gpu_num_levels.argtypes = [vp, P_i64]
        lib.aspamg_gpu_profile_iteration.argtypes = [vp, C.POINTER(GpuKernelTime), C.c_int, C.POINTER(C.c_int)]
        lib.aspamg_gpu_profile_ops.argtypes = [vp, C.c_int, C.POINTER(GpuKernelTime), C.c_int, C.POINTER(C.c_int)]
        lib.aspamg_gpu_time_vcycle.argtypes = [vp, C.c_int, P_dbl]
        lib.aspamg_gpu_time_kernel.argtypes = [vp, C.c_char_p, i64, C.c_int, P_dbl, P_dbl]
        lib.aspamg_gpu_launch_count.argtypes = [vp, P_i64]
        lib.aspamg_gpu_last_solve_ms.argtypes = [vp, P_dbl]
        lib.aspamg_gpu_stream.argtypes = [vp, C.POINTER(vp)]
        lib.aspamg_gpu_xsell_layout_spmv.argtypes = [C.POINTER(CsrView), i64, i64, i64, P_dbl, P_dbl]
        lib.aspamg_gpu_srqcg.argtypes = [vp, C.POINTER(CsrView), C.POINTER(CsrView), C.POINTER(CsrView), P_dbl, i64, i64,
                                         i64, dbl, C.c_uint64, P_dbl, P_dbl, P_i64, P_i64, C.POINTER(C.c_int)]
        lib.aspamg_gpu_galerkin.argtypes = [vp, C.POINTER(CsrView), C.POINTER(CsrView), C.POINTER(CsrView), vp, vp]
        lib.aspamg_gpu_assemble_hex.argtypes = [vp, vp, vp, vp]
        lib.aspamg_gpu_set_setup_policy.argtypes = [C.c_char_p, dbl]
        lib.aspamg_gpu_afsai_build.argtypes = [vp, C.POINTER(CsrView), i64, i64, dbl, vp, vp, P_dbl]
        lib.aspamg_gpu_smoother_setup.argtypes = [vp, C.POINTER(CsrView), C.POINTER(SmootherParams), vp, vp, P_dbl,
                                                  P_dbl, P_dbl, P_i64, C.POINTER(C.c_int)]
        _gpu = lib
    return _gpu


# int (*)(void* sink, int64 n_rows, int64 n_cols, int64 nnz, int64** rp, int64** ci, double** v)
CSR_ALLOC_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, i64, i64, i64, C.POINTER(P_i64), C.POINTER(P_i64), C.POINTER(P_dbl))
