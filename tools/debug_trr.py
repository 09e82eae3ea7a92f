import ctypes as C, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1902_01715_b200 as P
from paper_1902_01715_b200 import _native as N
for opts in ({}, {"pdl": 0}):
    p = P.Problem.config(1, 2)
    h = P.Hierarchy.setup(p.K, p.coords)
    g = P.GpuVcycle(h, options=opts)
    for i in range(3):
        x, rep = g.pcg(p.rhs)
        r = p.rhs - p.K.to_scipy() @ x
        print(opts, "host-path", rep.iterations, rep.converged, "trr", rep.true_rel_residual, "numpy trr", np.linalg.norm(r) / np.linalg.norm(p.rhs), flush=True)
    lib = N.gpu()
    n = p.K.n_rows
    bd, xd = C.c_void_p(), C.c_void_p()
    lib.aspamg_gpu_alloc_device(g._ctx, 8 * n, C.byref(bd)); lib.aspamg_gpu_alloc_device(g._ctx, 8 * n, C.byref(xd))
    b = np.ascontiguousarray(p.rhs)
    lib.aspamg_gpu_memcpy(g._ctx, bd, b.ctypes.data_as(C.c_void_p), 8 * n)
    hist = np.empty(1000); n_it = C.c_int64(); conv = C.c_int(); trr = C.c_double()
    code = lib.aspamg_gpu_pcg_device(g._ctx, bd, None, 1e-8, 1000, xd, hist.ctypes.data_as(C.POINTER(C.c_double)), C.byref(n_it), C.byref(conv), C.byref(trr))
    print(opts, "device-path", code, n_it.value, conv.value, "trr", trr.value, flush=True)
    x, rep = g.pcg(p.rhs)
    print(opts, "host-path again", rep.true_rel_residual, flush=True)
    g.close()
