"""B200-native solve phase of aSP-AMG (arXiv 1902.01715): PCG + V(1,1)-cycle in sm_100a CUDA.

See DESIGN.md for the path, the boundary and the kernels.
"""
from .solver import (  # noqa: F401
    AspamgError, ConfigError, CudaError, DimensionError, GpuVcycle, Hierarchy, IoError, NotSpdError,
    NumericalError, Problem, SolveReport, SparseMatrix, amg_setup, default_config, gpu_afsai, gpu_galerkin,
    gpu_setup_policy, gpu_smoother_setup, gpu_srqcg,
    host_galerkin, host_smoother_setup, pcg, vcycle_apply,
    SPMV_A, SPMV_G, SPMV_GT, SPMV_P, SPMV_PT,
)

__all__ = [
    "AspamgError", "ConfigError", "CudaError", "DimensionError", "GpuVcycle", "Hierarchy", "IoError",
    "NotSpdError", "NumericalError", "Problem", "SolveReport", "SparseMatrix", "amg_setup", "default_config",
    "gpu_afsai", "gpu_galerkin", "gpu_setup_policy", "gpu_smoother_setup", "gpu_srqcg", "host_galerkin", "host_smoother_setup", "pcg", "vcycle_apply", "SPMV_A", "SPMV_G", "SPMV_GT", "SPMV_P", "SPMV_PT",
]
