"""SPEC known answers for the setup components (CPU): aFSAI,
Lanczos lambda_max, SRQCG (acceptance #10)."""
import ctypes as C

import numpy as np
import pytest
import scipy.sparse as sp


def _lib():
    from paper_1902_01715_b200 import _native as N
    return N


def _view(pkg, M):
    sm = pkg.SparseMatrix.from_scipy(sp.csr_matrix(M))
    return sm, sm.view()


def _afsai(pkg, A, k, rho, eps):
    N = _lib()
    a, av = _view(pkg, A)
    h = C.c_void_p()
    gv = N.CsrView()
    assert N.host().aspamg_afsai_build(C.byref(av), k, rho, eps, C.byref(h), C.byref(gv)) == 0
    G = pkg.SparseMatrix.from_view(gv).to_scipy().toarray()
    N.host().aspamg_csr_free(h)
    return G


def test_afsai_diagonal_and_k0(pkg):
    D = np.diag(np.arange(1.0, 8.0))
    for k in (0, 3):
        G = _afsai(pkg, D, k, 4, 1e-3)
        assert np.allclose(G, np.diag(1 / np.sqrt(np.arange(1.0, 8.0))), rtol=1e-15)
    rng = np.random.default_rng(0)
    B = rng.standard_normal((12, 12))
    A = B @ B.T + 12 * np.eye(12)
    G0 = _afsai(pkg, A, 0, 4, 1e-3)
    assert np.allclose(G0, np.diag(1 / np.sqrt(np.diag(A))), rtol=1e-15)


def test_afsai_full_pattern_is_exact_inverse_cholesky(pkg):
    """10x10 SPD tridiagonal, k, rho large, eps 0 -> G A G' = I to 1e-10."""
    n = 10
    A = np.diag(np.full(n, 4.0)) + np.diag(np.full(n - 1, -1.0), 1) + np.diag(np.full(n - 1, -1.0), -1)
    G = _afsai(pkg, A, 20, 20, 0.0)
    assert np.abs(G @ A @ G.T - np.eye(n)).max() <= 1e-10
    assert np.allclose(np.triu(G, 1), 0)


def test_afsai_scaling_normalisation(pkg):
    p = pkg.Problem.config(1, 4)
    K = p.K.to_scipy()
    G = _afsai(pkg, K.toarray(), 4, 4, 1e-3)
    assert np.abs(np.diag(G @ K.toarray() @ G.T) - 1).max() <= 1e-12


def _lanczos(pkg, G, A, steps):
    N = _lib()
    g, gv = _view(pkg, G)
    a, av = _view(pkg, A)
    lam = C.c_double()
    assert N.host().aspamg_estimate_lambda_max(C.byref(gv), C.byref(av), steps, 1234, C.byref(lam)) == 0
    return lam.value


def test_lanczos_known_answers(pkg):
    assert _lanczos(pkg, np.eye(6), np.eye(6), 10) == pytest.approx(1.05, abs=1e-10)
    assert _lanczos(pkg, np.eye(2), np.diag([1.0, 4.0]), 2) == pytest.approx(4 * 1.05, rel=1e-8)
    rng = np.random.default_rng(3)
    B = rng.standard_normal((50, 50))
    A = B @ B.T + np.eye(50)
    lam = _lanczos(pkg, np.eye(50), A, 30)
    assert lam >= 0.99 * np.linalg.eigvalsh(A).max()


def _srqcg(pkg, A, G, V0, k_max, tol=1e-2):
    N = _lib()
    a, av = _view(pkg, A)
    g, gv = _view(pkg, G)
    n, m = V0.shape
    v0 = np.asfortranarray(V0).ravel(order="F")
    V = np.empty(n * m)
    q = np.empty(m)
    mo = C.c_int64()
    P = C.POINTER(C.c_double)
    assert N.host().aspamg_srqcg(C.byref(av), C.byref(gv), v0.ctypes.data_as(P), m, k_max, 1, tol, 1234,
                                 V.ctypes.data_as(P), q.ctypes.data_as(P), C.byref(mo)) == 0
    return V[: n * mo.value].reshape(n, mo.value, order="F"), q[: mo.value]


def test_srqcg_diagonal_oracle(pkg):
    """SPEC.md:265 / acceptance #10 on an operator scaled like G A G' (spectrum in
    (0, 2), as the aFSAI normalisation guarantees): the literal Alg. 4 pre-smoothing
    Z0 = (I - S) V0 annihilates an eigenvalue of exactly 1, so SPEC's diag(1..10)
    with G = I cannot reach lambda = 1; the scaled diagonal keeps the contract
    "quotients -> the two smallest eigenvalues" testable."""
    lam = np.linspace(0.05, 1.9, 10)
    A = np.diag(lam)
    V0 = np.random.default_rng(1).standard_normal((10, 2))
    V, q = _srqcg(pkg, A, np.eye(10), V0, 50, tol=1e-10)
    assert np.allclose(np.sort(q), lam[:2], atol=1e-6)
    assert np.abs(V.T @ V - np.eye(2)).max() <= 1e-10  # orthonormal output


def test_srqcg_converged_input(pkg):
    """V0 = exact eigenvectors of S -> residuals zero, V spans them."""
    lam = np.linspace(0.05, 1.9, 10)
    V0 = np.eye(10)[:, :3]
    V, q = _srqcg(pkg, np.diag(lam), np.eye(10), V0, 10)
    assert np.allclose(np.sort(q), lam[:3], atol=1e-12)
    assert np.linalg.matrix_rank(np.hstack([V, V0]), 1e-8) == 3


def test_srqcg_improves_rigid_body_seeds(pkg):
    """More SRQCG iterations lower the Rayleigh quotients of S (monotone minimisation)."""
    p = pkg.Problem.config(1, 4)
    K = p.K.to_scipy().toarray()
    G = _afsai(pkg, K, 4, 4, 1e-3)
    V0 = np.random.default_rng(2).standard_normal((K.shape[0], 6))
    _, q1 = _srqcg(pkg, K, G, V0, 1, tol=0.0)
    _, q5 = _srqcg(pkg, K, G, V0, 5, tol=0.0)
    assert np.sum(q5) <= np.sum(q1) * (1 + 1e-12)
