"""GPU setup components: SRQCG test-space generation on
the device (aspamg_gpu_srqcg). The device run restates the host srqcg operation
for operation (setup_gpu.cu header), so the bar is bit-identity with the CPU
restatement, and hence an identical hierarchy and identical PCG."""
import ctypes as C

import numpy as np
import pytest
import scipy.sparse as sp


def _host_srqcg(pkg, A, G, V0, k_max, k_ritz=1, tol=1e-2, seed=1234):
    from paper_1902_01715_b200 import _native as N
    av, gv = A.view(), G.view()
    n, m = V0.shape
    v0 = np.asfortranarray(V0).ravel(order="F")
    V = np.empty(n * m)
    q = np.empty(m)
    mo = C.c_int64()
    P = C.POINTER(C.c_double)
    assert N.host().aspamg_srqcg(C.byref(av), C.byref(gv), v0.ctypes.data_as(P), m, k_max, k_ritz, tol, seed,
                                 V.ctypes.data_as(P), q.ctypes.data_as(P), C.byref(mo)) == 0
    return V[: n * mo.value].reshape(n, mo.value, order="F"), q[: mo.value]


def _afsai(pkg, A, k=4, rho=4, eps=1e-3):
    from paper_1902_01715_b200 import _native as N
    av = A.view()
    h = C.c_void_p()
    gv = N.CsrView()
    assert N.host().aspamg_afsai_build(C.byref(av), k, rho, eps, C.byref(h), C.byref(gv)) == 0
    G = pkg.SparseMatrix.from_view(gv)
    G = pkg.SparseMatrix.from_scipy(G.to_scipy())  # own the arrays
    N.host().aspamg_csr_free(h)
    return G


def _levels_equal(h1, h2):
    assert h1.n_levels == h2.n_levels
    for l in range(h1.n_levels):
        a, b = h1.level(l), h2.level(l)
        for name in ("A", "G", "P"):
            ma, mb = getattr(a, name), getattr(b, name)
            for arr in ("row_offsets", "col_indices", "values"):
                xa, xb = getattr(ma, arr), getattr(mb, arr)
                assert (xa is None) == (xb is None), (l, name, arr)
                if xa is not None:
                    assert np.array_equal(xa, xb), (l, name, arr)
        assert a.omega == b.omega and a.n_tv == b.n_tv
    assert np.array_equal(h1.coarse_factor(), h2.coarse_factor())


def _all_gpu(pkg):
    for k in ("smoother_max_mean_row", "smoother_min_rows", "smoother_max_pattern"):
        pkg.gpu_setup_policy(k, 0)


def _default_policy(pkg):
    pkg.gpu_setup_policy("smoother_max_mean_row", 0)
    pkg.gpu_setup_policy("smoother_min_rows", 20000)
    pkg.gpu_setup_policy("smoother_max_pattern", 0)


def test_srqcg_backend_hook_cpu(pkg):
    """The external test-space hook (aspamg_set_srqcg_backend) on the CPU: a
    backend that forwards to the host restatement reproduces the built-in path
    bit for bit, and a failing backend surfaces as an error."""
    from paper_1902_01715_b200 import _native as N
    lib = N.host()
    FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(N.CsrView), C.POINTER(N.CsrView), C.POINTER(N.CsrView),
                     C.POINTER(C.c_double), C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_uint64,
                     C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                     C.POINTER(C.c_int))
    calls = []

    def fwd(user, A, G, Gt, V0, m, k_max, k_ritz, tol, seed, V, q, m_out, iters, rc):
        calls.append(m)
        iters[0] = 0
        rc[0] = 0
        return lib.aspamg_srqcg(A, G, V0, m, k_max, k_ritz, tol, seed, V, q, m_out)

    def bad(*args):
        return 3

    p = pkg.Problem.config(1, 4)
    ref = pkg.amg_setup(p.K, p.coords)
    cb = FN(fwd)
    lib.aspamg_set_srqcg_backend(C.cast(cb, C.c_void_p), None)
    try:
        h = pkg.amg_setup(p.K, p.coords)
    finally:
        lib.aspamg_set_srqcg_backend(None, None)
    assert calls == [10]
    _levels_equal(ref, h)
    cbad = FN(bad)
    lib.aspamg_set_srqcg_backend(C.cast(cbad, C.c_void_p), None)
    try:
        with pytest.raises(pkg.NumericalError):
            pkg.amg_setup(p.K, p.coords)
    finally:
        lib.aspamg_set_srqcg_backend(None, None)


@pytest.mark.gpu
@pytest.mark.parametrize("k_max,k_ritz,tol", [(0, 1, 1e-2), (1, 1, 1e-2), (5, 1, 1e-2), (6, 2, 0.0), (4, 3, 1e-1)])
def test_gpu_srqcg_bit_identical(pkg, k_max, k_ritz, tol):
    p = pkg.Problem.config(1, 4)
    G = _afsai(pkg, p.K)
    V0 = np.random.default_rng(5).standard_normal((p.K.n_rows, 8))
    Vh, qh = _host_srqcg(pkg, p.K, G, V0, k_max, k_ritz, tol)
    Vd, qd, it, _ = pkg.gpu_srqcg(p.K, G, V0, k_max, k_ritz, tol)
    assert np.array_equal(qh, qd)
    assert np.array_equal(Vh, Vd)
    assert it <= k_max


@pytest.mark.gpu
def test_gpu_srqcg_large_chunks_and_rank_collapse(pkg):
    """n > 8192 (several dot chunks, host partial pass) and duplicated seed
    columns (entry rank collapse -> seeded random replacement)."""
    p = pkg.Problem.config(2, 4)
    G = _afsai(pkg, p.K)
    rng = np.random.default_rng(7)
    V0 = rng.standard_normal((p.K.n_rows, 6))
    V0[:, 3] = V0[:, 1]
    V0[:, 5] = 2.0 * V0[:, 0]
    assert p.K.n_rows > 8192
    Vh, qh = _host_srqcg(pkg, p.K, G, V0, 4)
    Vd, qd, _, rc = pkg.gpu_srqcg(p.K, G, V0, 4)
    assert rc
    assert np.array_equal(qh, qd)
    assert np.array_equal(Vh, Vd)


@pytest.mark.gpu
def test_gpu_srqcg_known_answers(pkg):
    """SPEC.md:265 / acceptance #10 (scaled spectrum, see test_setup_components)."""
    lam = np.linspace(0.05, 1.9, 10)
    A = pkg.SparseMatrix.from_scipy(sp.csr_matrix(np.diag(lam)))
    I = pkg.SparseMatrix.from_scipy(sp.identity(10, format="csr"))
    V0 = np.random.default_rng(1).standard_normal((10, 2))
    V, q, _, _ = pkg.gpu_srqcg(A, I, V0, 50, 1, 1e-10)
    assert np.allclose(np.sort(q), lam[:2], atol=1e-6)
    assert np.abs(V.T @ V - np.eye(2)).max() <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,scale", [(1, 2), (2, 4), (3, 4), (5, 6)])
def test_gpu_setup_hierarchy_identical(pkg, cfg, scale):
    """amg_setup(..., setup_device=0) == CPU amg_setup, level by level, bit for bit
    (with the default level policy and with every level's smoother on the GPU);
    the PCG on it therefore reproduces the CPU-setup solve exactly."""
    p = pkg.Problem.config(cfg, scale)
    h_cpu = pkg.amg_setup(p.K, p.coords)
    h_gpu = pkg.amg_setup(p.K, p.coords, setup_device=0)
    _levels_equal(h_cpu, h_gpu)
    _all_gpu(pkg)
    try:
        _levels_equal(h_cpu, pkg.amg_setup(p.K, p.coords, setup_device=0))
    finally:
        _default_policy(pkg)
    pkg.gpu_setup_policy("smoother_max_pattern", 24)  # hand back after the first refinement passes
    pkg.gpu_setup_policy("smoother_min_rows", 0)
    try:
        _levels_equal(h_cpu, pkg.amg_setup(p.K, p.coords, setup_device=0))
    finally:
        _default_policy(pkg)
    M1, M2 = pkg.GpuVcycle(h_cpu), pkg.GpuVcycle(h_gpu)
    x1, r1 = pkg.pcg(p.K, p.rhs, M1)
    x2, r2 = pkg.pcg(p.K, p.rhs, M2)
    assert r1.iterations == r2.iterations
    assert np.array_equal(x1, x2)


def _csr_equal(X, Y):
    assert (X.n_rows, X.n_cols) == (Y.n_rows, Y.n_cols)
    assert np.array_equal(X.row_offsets, Y.row_offsets)
    assert np.array_equal(X.col_indices, Y.col_indices)
    assert np.array_equal(X.values, Y.values)


def _random_pair(n, nc, p_per_row, a_per_row, seed):
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n), p_per_row)
    cols = rng.integers(0, nc, n * p_per_row)
    P = sp.csr_matrix((rng.standard_normal(n * p_per_row), (rows, cols)), shape=(n, nc))
    B = sp.random(n, n, density=a_per_row / n, random_state=seed, format="csr")
    A = (B + B.T + sp.identity(n) * 4.0).tocsr()
    return P, A


def test_host_galerkin_hook_cpu(pkg):
    """aspamg_set_galerkin_backend on the CPU: a backend forwarding to the host
    product gives the built-in hierarchy bit for bit."""
    from paper_1902_01715_b200 import _native as N
    lib = N.host()
    FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(N.CsrView), C.POINTER(N.CsrView), C.POINTER(N.CsrView),
                     C.c_void_p, C.c_void_p)
    calls = []

    def fwd(user, P, Pt, A, alloc, sink):
        calls.append(P.contents.n_rows)
        h = C.c_void_p()
        out = N.CsrView()
        st = lib.aspamg_galerkin(P, A, C.byref(h), C.byref(out))
        if st:
            return st
        rp, ci, v = N.P_i64(), N.P_i64(), N.P_dbl()
        st = N.CSR_ALLOC_FN(alloc)(sink, out.n_rows, out.n_cols, out.nnz, C.byref(rp), C.byref(ci), C.byref(v))
        C.memmove(rp, out.row_offsets, 8 * (out.n_rows + 1))
        C.memmove(ci, out.col_indices, 8 * out.nnz)
        C.memmove(v, out.values, 8 * out.nnz)
        lib.aspamg_csr_free(h)
        return st

    p = pkg.Problem.config(1, 4)
    ref = pkg.amg_setup(p.K, p.coords)
    cb = FN(fwd)
    lib.aspamg_set_galerkin_backend(C.cast(cb, C.c_void_p), None)
    try:
        h = pkg.amg_setup(p.K, p.coords)
    finally:
        lib.aspamg_set_galerkin_backend(None, None)
    assert len(calls) == ref.n_levels - 1
    _levels_equal(ref, h)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,scale", [(1, 2), (2, 4)])
def test_gpu_galerkin_hierarchy_levels(pkg, cfg, scale):
    """P_l' A_l P_l on the GPU == the host product, every level, bit for bit."""
    p = pkg.Problem.config(cfg, scale)
    h = pkg.amg_setup(p.K, p.coords)
    for l in range(h.n_levels - 1):
        L = h.level(l)
        _csr_equal(pkg.gpu_galerkin(L.P, L.A), pkg.host_galerkin(L.P, L.A))


@pytest.mark.gpu
def test_gpu_galerkin_wide_rows(pkg):
    """Rows with more distinct columns than a warp's table (1024) take the CTA
    path; explicit zeros, empty rows and empty columns are preserved."""
    P, A = _random_pair(3000, 2500, 12, 40, 11)
    P = P.tolil()
    P[5, :] = 0.0   # an empty fine row
    P = P.tocsr()
    P.eliminate_zeros()
    Ps, As = pkg.SparseMatrix.from_scipy(P), pkg.SparseMatrix.from_scipy(A)
    G = pkg.gpu_galerkin(Ps, As)
    H = pkg.host_galerkin(Ps, As)
    _csr_equal(G, H)
    assert np.diff(H.row_offsets).max() > 1024
    # exact cancellation keeps the entry (first-touch accumulator, no drop)
    P2 = sp.csr_matrix(np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 1.0]]))
    A2 = sp.csr_matrix(np.ones((3, 3)))
    G2 = pkg.gpu_galerkin(pkg.SparseMatrix.from_scipy(P2), pkg.SparseMatrix.from_scipy(A2))
    _csr_equal(G2, pkg.host_galerkin(pkg.SparseMatrix.from_scipy(P2), pkg.SparseMatrix.from_scipy(A2)))
    assert G2.nnz == 4 and G2.values[0] == 0.0


@pytest.mark.gpu
def test_gpu_galerkin_errors(pkg):
    P, A = _random_pair(50, 20, 2, 3, 1)
    with pytest.raises(pkg.DimensionError):
        pkg.gpu_galerkin(pkg.SparseMatrix.from_scipy(P[:40]), pkg.SparseMatrix.from_scipy(A))


@pytest.mark.gpu
@pytest.mark.parametrize("k,rho,eps", [(4, 4, 1e-3), (2, 8, 0.0), (0, 4, 1e-3), (6, 3, 1e-2)])
def test_gpu_afsai_bit_identical(pkg, k, rho, eps):
    """aspamg_gpu_afsai_build == the host afsai_build (fsai.cpp), bit for bit, on K
    and on a dense-row Galerkin operator."""
    p = pkg.Problem.config(2, 4)
    h = pkg.amg_setup(p.K, p.coords)
    for A in (p.K, h.level(1).A):
        G, psi = pkg.gpu_afsai(A, k, rho, eps)
        _csr_equal(G, _afsai(pkg, A, k, rho, eps))
        assert np.all(psi > 0)


@pytest.mark.gpu
def test_gpu_afsai_known_answers(pkg):
    """SPEC.md:178-180 on the device build."""
    D = pkg.SparseMatrix.from_scipy(sp.csr_matrix(np.diag(np.arange(1.0, 8.0))))
    G, _ = pkg.gpu_afsai(D, 3, 4, 1e-3)
    assert np.allclose(G.to_scipy().toarray(), np.diag(1 / np.sqrt(np.arange(1.0, 8.0))), rtol=1e-15)
    n = 10
    T = np.diag(np.full(n, 4.0)) + np.diag(np.full(n - 1, -1.0), 1) + np.diag(np.full(n - 1, -1.0), -1)
    G, _ = pkg.gpu_afsai(pkg.SparseMatrix.from_scipy(sp.csr_matrix(T)), 20, 20, 0.0)
    Gd = G.to_scipy().toarray()
    assert np.abs(Gd @ T @ Gd.T - np.eye(n)).max() <= 1e-10


@pytest.mark.gpu
def test_gpu_afsai_not_spd(pkg):
    A = pkg.SparseMatrix.from_scipy(sp.csr_matrix(np.array([[1.0, 2.0], [2.0, 1.0]])))
    with pytest.raises(pkg.NotSpdError):
        pkg.gpu_afsai(A, 2, 2, 0.0)


@pytest.mark.gpu
def test_gpu_smoother_policy_declines_long_rows(pkg):
    """Level policy: small operators are declined (-1 -> None); a pattern bound
    below the refinement growth hands the loop back after finished passes."""
    p = pkg.Problem.config(2, 4)
    assert pkg.gpu_smoother_setup(p.K) is None            # 13,872 rows < smoother_min_rows
    pkg.gpu_setup_policy("smoother_min_rows", 0)
    pkg.gpu_setup_policy("smoother_max_pattern", 20)
    try:
        r = pkg.gpu_smoother_setup(p.K)
    finally:
        _default_policy(pkg)
    assert r is not None and r["handed_back"] and r["passes"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,scale", [(2, 4), (5, 6)])
def test_gpu_smoother_setup_matches_host(pkg, cfg, scale):
    """Alg. 3 on the device (aFSAI passes, device transpose, Lanczos) reproduces
    every level's host smoother: G, omega, lambda_hat, passes, exit reason."""
    p = pkg.Problem.config(cfg, scale)
    h = pkg.amg_setup(p.K, p.coords)
    _all_gpu(pkg)  # never decline or hand back: exercise the device path on every level
    try:
        rs = [pkg.gpu_smoother_setup(h.level(l).A) for l in range(h.n_levels - 1)]
    finally:
        _default_policy(pkg)
    for l in range(h.n_levels - 1):
        L = h.level(l)
        r = rs[l]
        _csr_equal(r["G"], L.G)
        assert r["omega"] == L.omega and r["lambda_hat"] == L.lambda_hat
        assert r["passes"] == L.refinement_passes and r["exit"] == L.smoother_exit
