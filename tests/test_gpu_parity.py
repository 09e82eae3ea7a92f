"""GPU-vs-oracle parity through the C-ABI (include/aspamg_gpu.h).

The oracle (oracle/oracle.c) runs on the SAME hierarchy arrays the GPU
receives, so every difference is kernel arithmetic (FMA contraction, tree
reductions) — the north_star tolerances apply: PCG iteration count +-1,
first-20 relative residuals within 1e-9 relative, final solution 1e-8.
Per-product tolerances are written per test.
"""
import numpy as np
import pytest

from conftest import problem_and_hierarchy, rel_err

pytestmark = pytest.mark.gpu

RTOL_SPMV = 1e-13   # one fp64 product, different summation order
RTOL_VCYCLE = 1e-11  # a whole V-cycle (several levels of products)


def _gpu(pkg, h, **opt):
    return pkg.GpuVcycle(h, device=0, options=opt or None)


def _oracle(oracle, h):
    return oracle.OracleHierarchy(h, use_ref_spmv=False, threads=4)


@pytest.fixture(scope="module")
def c1_ctx(pkg, oracle):
    p, h = problem_and_hierarchy(1, 1)
    return p, h, _gpu(pkg, h), _oracle(oracle, h)


def test_k_is_bsr3_and_levels_uploaded(c1_ctx):
    p, h, g, o = c1_ctx
    info = g.level_info(0)
    assert info.a_format == 1 and 1.0 <= info.a_fill < 1.2
    assert info.a_nnzb * 9 == p.K.nnz
    assert h.n_levels >= 2


def test_k_spmv_bit_exact_vs_reference_golden(pkg):
    """Sliced BSR3 keeps the reference's per-row order with separate mul/add:
    y is bit-identical to the reference's own compiled spmv (tests/golden)."""
    import os
    gold = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_kernels.npz")))
    p, h = problem_and_hierarchy(1, 4)
    g = _gpu(pkg, h)
    assert np.array_equal(p.K.values, gold["K_v"])
    assert g.level_info(0).a_format == 1
    assert np.array_equal(g.spmv(0, 0, gold["K_x"]), gold["K_y"])


@pytest.mark.parametrize("which", ["A", "G", "Gt", "P", "Pt"])
def test_spmv_every_operand_every_level(c1_ctx, pkg, which):
    p, h, g, o = c1_ctx
    rng = np.random.default_rng(7)
    wi = ["A", "G", "Gt", "P", "Pt"].index(which)
    for l in range(h.n_levels - (0 if which == "A" else 1)):
        m = getattr(h.level(l, copy=False), which)
        x = rng.standard_normal(m.n_cols)
        yg = g.spmv(l, wi, x)
        yo = o.spmv(l, which, x)
        if g.level_info(l).fmt[wi] in (1, 2, 3):  # sliced formats: reference order, bit-exact
            assert np.array_equal(yg, yo), (which, l)
            continue
        # per-entry bound: |sum| error <= nnz_row * eps * sum|a_ij x_j|
        absrow = np.abs(m.to_scipy()) @ np.abs(x)
        assert np.all(np.abs(yg - yo) <= 1e-14 * absrow + 1e-300), (which, l)


def test_spmv_identity_and_zero(c1_ctx):
    p, h, g, o = c1_ctx
    n = p.K.n_rows
    assert np.array_equal(g.spmv(0, 0, np.zeros(n)), np.zeros(n))


def test_smoothing_step_matches_oracle_and_fixed_point(c1_ctx):
    p, h, g, o = c1_ctx
    rng = np.random.default_rng(3)
    n = p.K.n_rows
    b = rng.standard_normal(n)
    x = rng.standard_normal(n)
    assert rel_err(g.smooth(0, b, x), o.smooth(0, b, x)) < 1e-12
    # exact solution is a fixed point: b = A x -> x' = x
    bx = o.spmv(0, "A", x)
    assert rel_err(g.smooth(0, bx, x), x) < 1e-12


def test_coarse_solve_matches_oracle(c1_ctx):
    p, h, g, o = c1_ctx
    rng = np.random.default_rng(5)
    n_c = h.coarse_factor().shape[0]
    y = rng.standard_normal(n_c)
    zg = g.coarse_solve(y)
    zo = o.coarse_solve(y)
    assert rel_err(zg, zo) < 1e-10
    # L L' z = y
    L = h.coarse_factor()
    assert rel_err(L @ (L.T @ zg), y) < 1e-10


def test_vcycle_matches_oracle(c1_ctx):
    p, h, g, o = c1_ctx
    rng = np.random.default_rng(11)
    for _ in range(3):
        y = rng.standard_normal(p.K.n_rows)
        assert rel_err(g.apply(y), o.vcycle(y)) < RTOL_VCYCLE
    assert np.array_equal(g.apply(np.zeros(p.K.n_rows)), np.zeros(p.K.n_rows))


def test_vcycle_symmetric_positive_definite(c1_ctx):
    """<B^-1 u, v> = <u, B^-1 v> to 1e-10, <B^-1 u, u> > 0."""
    p, h, g, o = c1_ctx
    rng = np.random.default_rng(13)
    for _ in range(5):
        u = rng.standard_normal(p.K.n_rows)
        v = rng.standard_normal(p.K.n_rows)
        bu, bv = g.apply(u), g.apply(v)
        assert abs(bu @ v - u @ bv) <= 1e-10 * max(abs(bu @ v), 1e-300)
        assert bu @ u > 0


def test_vcycle_is_deterministic(c1_ctx):
    p, h, g, o = c1_ctx
    y = np.random.default_rng(17).standard_normal(p.K.n_rows)
    assert np.array_equal(g.apply(y), g.apply(y))


def _pcg_parity(p, h, g, o, tol=1e-8, max_it=1000):
    xg, rep = g.pcg(p.rhs, rel_tol=tol, max_it=max_it)
    st, xo, ho, conv_o, trr_o = o.pcg(p.rhs, rel_tol=tol, max_it=max_it)
    assert st == 0
    assert rep.converged and conv_o
    assert abs(rep.iterations - len(ho)) <= 1, (rep.iterations, len(ho))
    k = min(20, rep.iterations, len(ho))
    assert np.all(np.abs(rep.residual_history[:k] - ho[:k]) <= 1e-9 * ho[:k]), "first-20 residual history"
    assert rel_err(xg, xo) <= 1e-8
    assert rep.true_rel_residual <= 10 * tol
    assert len(rep.residual_history) == rep.iterations
    return rep, ho


def test_pcg_c1_full_size(c1_ctx):
    p, h, g, o = c1_ctx
    rep, ho = _pcg_parity(p, h, g, o)
    assert rep.iterations <= 120  # SPEC.md:657 acceptance #4 spirit


def test_pcg_deterministic_and_repeatable(c1_ctx):
    p, h, g, o = c1_ctx
    x1, r1 = g.pcg(p.rhs)
    x2, r2 = g.pcg(p.rhs)
    assert np.array_equal(x1, x2) and np.array_equal(r1.residual_history, r2.residual_history)


def test_pcg_host_loop_matches_device_loop(pkg, oracle):
    p, h = problem_and_hierarchy(1, 2)
    g1 = _gpu(pkg, h)
    g2 = _gpu(pkg, h, device_loop=0)
    x1, r1 = g1.pcg(p.rhs)
    x2, r2 = g2.pcg(p.rhs)
    assert r1.iterations == r2.iterations
    assert np.array_equal(x1, x2)


def test_pcg_with_x0_and_edge_cases(c1_ctx, pkg):
    p, h, g, o = c1_ctx
    n = p.K.n_rows
    # b = 0 -> x = 0, 0 iterations
    x, rep = g.pcg(np.zeros(n))
    assert rep.iterations == 0 and rep.converged and not np.any(x)
    # x0 = exact-ish solution -> 0 or few iterations
    xs, _ = g.pcg(p.rhs)
    x, rep = g.pcg(p.rhs, x0=xs)
    assert rep.iterations <= 1
    # random x0 agrees with the oracle
    x0 = np.random.default_rng(1).standard_normal(n)
    xg, rg = g.pcg(p.rhs, x0=x0)
    st, xo, ho, conv, trr = o.pcg(p.rhs, x0=x0)
    assert abs(rg.iterations - len(ho)) <= 1 and rel_err(xg, xo) < 1e-8
    # max_it cap -> not converged, history length == max_it
    x, rep = g.pcg(p.rhs, max_it=3)
    assert rep.iterations == 3 and not rep.converged
    # dimension mismatch -> DimensionError
    with pytest.raises(pkg.DimensionError):
        g.pcg(np.ones(n + 1))


def test_pcg_not_spd_raises(pkg):
    """p'Ap <= 0 -> NotSpdError: negate the operator."""
    p, h = problem_and_hierarchy(1, 4)
    import ctypes as C
    from paper_1902_01715_b200 import _native as N
    lib = N.gpu()
    ctx = C.c_void_p()
    assert lib.aspamg_gpu_ctx_create(0, C.byref(ctx)) == 0
    info = h.info()
    for l in range(info.n_levels):
        lv = h.level(l)
        if l == 0:
            lv.A.values = -lv.A.values
        views = [m.view() for m in (lv.A, lv.G, lv.Gt, lv.P, lv.Pt)]
        assert lib.aspamg_gpu_upload_level(ctx, l, *[C.byref(v) for v in views], lv.omega if l < info.n_levels - 1 else 1.0) == 0
    L = np.ascontiguousarray(h.coarse_factor().ravel(order="F"))
    assert lib.aspamg_gpu_upload_coarse(ctx, h.coarse_factor().shape[0], L.ctypes.data_as(C.POINTER(C.c_double))) == 0
    assert lib.aspamg_gpu_finalize(ctx) == 0
    n = p.K.n_rows
    b = np.ascontiguousarray(p.rhs)
    x = np.empty(n)
    hist = np.empty(100)
    n_it = C.c_int64()
    conv = C.c_int()
    trr = C.c_double()
    P_d = C.POINTER(C.c_double)
    code = lib.aspamg_gpu_pcg(ctx, b.ctypes.data_as(P_d), None, 1e-8, 100, x.ctypes.data_as(P_d),
                              hist.ctypes.data_as(P_d), C.byref(n_it), C.byref(conv), C.byref(trr))
    assert code == 2
    lib.aspamg_gpu_ctx_destroy(ctx)


@pytest.mark.parametrize("cfg,scale", [(2, 4), (3, 4), (4, 8), (5, 8)])
def test_pcg_configs_scaled(pkg, oracle, cfg, scale):
    """Same construction as BASELINE configs 2-5 at reduced element counts."""
    p, h = problem_and_hierarchy(cfg, scale)
    g = _gpu(pkg, h)
    o = _oracle(oracle, h)
    _pcg_parity(p, h, g, o)


def test_pcg_c2_full_size(pkg, oracle):
    """BASELINE config 2 at full size (0.8M dofs, 63.7M nnz)."""
    p, h = problem_and_hierarchy(2, 1)
    g = _gpu(pkg, h)
    o = oracle.OracleHierarchy(h, use_ref_spmv=False, threads=8)
    _pcg_parity(p, h, g, o)


def test_nu_variants_match_oracle(pkg, oracle):
    p, h = problem_and_hierarchy(1, 2, nu1=2, nu2=1)
    g = _gpu(pkg, h)
    o = _oracle(oracle, h)
    y = np.random.default_rng(2).standard_normal(p.K.n_rows)
    assert rel_err(g.apply(y), o.vcycle(y)) < RTOL_VCYCLE
    _pcg_parity(p, h, g, o)


def test_one_level_hierarchy_is_direct_solve(pkg, oracle):
    """n <= min_coarse_size -> the V-cycle is the exact solve."""
    p = pkg.Problem.hex_cube(3)
    h = pkg.Hierarchy.setup(p.K, p.coords)
    assert h.n_levels == 1
    g = _gpu(pkg, h)
    y = np.random.default_rng(4).standard_normal(p.K.n_rows)
    z = g.apply(y)
    K = p.K.to_scipy()
    assert rel_err(K @ z, y) < 1e-10
    x, rep = g.pcg(p.rhs)
    assert rep.iterations == 1 and rep.converged  # exact preconditioner


@pytest.mark.parametrize("tail_rows", [10000, 2000])
def test_coarse_tail_persistent_kernel_matches_oracle(pkg, oracle, tail_rows):
    """Levels below tail_rows run as one persistent cooperative kernel; same results."""
    p, h = problem_and_hierarchy(1, 1)
    g = _gpu(pkg, h, tail_rows=tail_rows, tail_dense=0)
    o = _oracle(oracle, h)
    y = np.random.default_rng(21).standard_normal(p.K.n_rows)
    assert rel_err(g.apply(y), o.vcycle(y)) < RTOL_VCYCLE
    ref = _gpu(pkg, h, tail_dense=0)
    assert np.array_equal(g.apply(y), ref.apply(y))  # same kernels' arithmetic, same bits
    _pcg_parity(p, h, g, o)


@pytest.mark.parametrize("opts", [{"sell_chh": 8}, {"sell_chh": 32, "sell_sort_fill_pct": 100000},
                                  {"sell_sort": 1}, {"sell_sort": 1, "sell_sigma": 256}, {"sell_u": 41}, {"sell_u": 21},
                                  {"sell_u": 44}, {"sell_u": 83}, {"pdl": 0}, {"idx16": 0}, {"idx16": 0, "sell_chh": 8}])
def test_sell_layout_variants_are_bit_identical(pkg, opts):
    """Every SELL layout/kernel variant sums each row sequentially in ascending
    column order, so the V-cycle output is bit-identical across variants."""
    p, h = problem_and_hierarchy(2, 2)
    y = np.random.default_rng(5).standard_normal(p.K.n_rows)
    ref = _gpu(pkg, h, sell_chh=32, sell_sort_fill_pct=100000, sell_min_mean=1, xsell=0).apply(y)
    opts = dict(opts, sell_min_mean=1, xsell=0)
    if "sell_sort" not in opts:  # keep every SELL-eligible operand in SELL (CSR trees differ in bits)
        opts.setdefault("sell_sort_fill_pct", 100000)
    g = _gpu(pkg, h, **opts)
    assert np.array_equal(g.apply(y), ref)
    if "pdl" in opts:
        g2 = _gpu(pkg, h, pdl=1, sell_chh=32, sell_sort_fill_pct=100000, sell_min_mean=1, xsell=0)  # restore the default
        assert np.array_equal(g2.apply(y), ref)


@pytest.mark.parametrize("opts", [{"csr_pf": 0}, {"csr_pf": 0, "idx16": 0}])
def test_csr_kernel_variants_are_bit_identical(pkg, opts):
    """CSR kernel variants (with / without the row-pointer prefetch) keep every
    thread's entries and their order, so the V-cycle output is bit-identical."""
    p, h = problem_and_hierarchy(2, 2)
    y = np.random.default_rng(9).standard_normal(p.K.n_rows)
    base = {"idx16": 0, "xsell": 0} if opts.get("idx16") == 0 else {"xsell": 0}
    ref = _gpu(pkg, h, csr_pf=1, **base).apply(y)
    assert np.array_equal(_gpu(pkg, h, xsell=0, **opts).apply(y), ref)


@pytest.mark.parametrize("opts", [{"csr_long": 1}, {"csr_long": 2}, {"csr_long": 4, "csr_pf": 0},
                                  {"csr_long": 1, "idx16": 0}])
def test_csr_long_row_split_matches_oracle(pkg, oracle, opts):
    """Long-row split (rows past the threshold computed warp-per-row by extra
    CTAs of the same launch): every operand within the CSR per-row bound, PCG
    within the north_star tolerances, deterministic run to run."""
    p, h = problem_and_hierarchy(2, 2)
    g = _gpu(pkg, h, xsell=0, **opts)
    o = _oracle(oracle, h)
    rng = np.random.default_rng(13)
    for l in range(h.n_levels - 1):
        for wi, which in enumerate(["A", "G", "Gt", "P", "Pt"]):
            m = getattr(h.level(l, copy=False), which)
            x = rng.standard_normal(m.n_cols)
            yg, yo = g.spmv(l, wi, x), o.spmv(l, which, x)
            absrow = np.abs(m.to_scipy()) @ np.abs(x)
            assert np.all(np.abs(yg - yo) <= 1e-14 * absrow + 1e-300), (opts, which, l)
    y = rng.standard_normal(p.K.n_rows)
    assert np.array_equal(g.apply(y), g.apply(y))
    assert rel_err(g.apply(y), o.vcycle(y)) < RTOL_VCYCLE
    _pcg_parity(p, h, g, o)


@pytest.mark.parametrize("cfg,scale,opts", [(2, 2, {}), (2, 2, {"bsr": 0}), (1, 1, {"tail_dense": 0}), (3, 4, {})])
def test_fused_residual_restriction_matches_oracle(pkg, oracle, cfg, scale, opts):
    """Restriction fused with the fine residual (fuse_rr):
    one cooperative launch per level computes r = y - A s, crosses a grid barrier and
    gathers r_c = P' r. Level 0 runs the sliced-BSR3 variant (k_resid_restrict), CSR
    levels the two-op table kernel. V-cycle within 1e-11 of the oracle and within
    rounding of the unfused path, deterministic, PCG inside the north_star gates."""
    p, h = problem_and_hierarchy(cfg, scale)
    g = _gpu(pkg, h, fuse_rr=1, **opts)
    g0 = _gpu(pkg, h, fuse_rr=0, **opts)
    o = _oracle(oracle, h)
    names = [(n, l) for n, l, _, _ in g.profile_iteration()]
    fused = [(n, l) for n, l in names if n.startswith("resid_restrict")]
    assert fused and (fused[0][1] == 0), names
    if "bsr" not in opts:
        assert fused[0][0].startswith("resid_restrict.sbsr3+csr")
    assert not any(n.startswith("restrict_Pt") and l == 0 for n, l in names)
    rng = np.random.default_rng(29)
    for _ in range(2):
        y = rng.standard_normal(p.K.n_rows)
        zf = g.apply(y)
        assert np.array_equal(zf, g.apply(y))
        assert rel_err(zf, o.vcycle(y)) < RTOL_VCYCLE
        assert rel_err(zf, g0.apply(y)) < 1e-13
    _pcg_parity(p, h, g, o)
    g.close()
    g0.close()


@pytest.mark.parametrize("rows", [0, 300, 2000, 8000])
def test_dense_coarse_tail_matches_oracle(pkg, oracle, rows):
    """Collapsed coarse tail (tail_dense): the V-cycle below the first level
    with <= rows rows replaced by its own matrix, formed on the device from the
    sub-cycle's kernels. Same operator up to rounding: V-cycle within 1e-11,
    PCG within the north_star tolerances."""
    p, h = problem_and_hierarchy(2, 2)
    g = _gpu(pkg, h, tail_dense=rows)
    o = _oracle(oracle, h)
    y = np.random.default_rng(17).standard_normal(p.K.n_rows)
    assert rel_err(g.apply(y), o.vcycle(y)) < RTOL_VCYCLE
    assert np.array_equal(g.apply(y), g.apply(y))
    _pcg_parity(p, h, g, o)


@pytest.mark.parametrize("opts", [{}, {"xsell_rows": 256}, {"xsell_rows": 128, "xsell_gran": 4}, {"xsell_rows": 64, "xsell_gran": 2},
                                  {"xsell_rows": 32, "xsell_gran": 1}, {"xsell_q": 14}, {"xsell_q": 16}, {"xsell_q": 23},
                                  {"xsell_fold": 1}, {"xsell_fold": 1, "xsell_rows": 256, "xsell_q": 23},
                                  {"xsell_fold": 1, "xsell_q": 14, "xsell_gran": 4}, {"xsell_fold": 1, "xsell_q": 16},
                                  {"xsell": 31, "xsell_max_mean": 100000, "xsell_rows": 64}, {"xsell_smem_kb": 8}])
def test_xsell_operands_bit_exact_and_pcg_parity(pkg, oracle, opts):
    """Tile-local SELL (x footprint staged in shared memory, 16-bit local columns):
    every operand uploaded in that format multiplies bit-identically to the
    oracle spmv (sequential ascending sums, sparse_matrix.cpp:100-105) for every
    tile height / granule / kernel variant; operands that do not fit the
    shared-memory budget fall back to SELL / CSR; V-cycle and PCG parity hold."""
    p, h = problem_and_hierarchy(2, 2)
    g = _gpu(pkg, h, xsell_min_rows=0, **{"xsell": 30, **opts})  # the format is opt-in (default mask 0)
    o = _oracle(oracle, h)
    rng = np.random.default_rng(29)
    n3 = 0
    for l in range(h.n_levels - 1):
        for wi, which in enumerate(["A", "G", "Gt", "P", "Pt"]):
            m = getattr(h.level(l, copy=False), which)
            x = rng.standard_normal(m.n_cols)
            yg, yo = g.spmv(l, wi, x), o.spmv(l, which, x)
            if g.level_info(l).fmt[wi] == 3:
                n3 += 1
                assert np.array_equal(yg, yo), (opts, which, l)
            else:
                absrow = np.abs(m.to_scipy()) @ np.abs(x)
                assert np.all(np.abs(yg - yo) <= 1e-14 * absrow + 1e-300), (opts, which, l)
    assert n3 >= (4 if opts.get("xsell_smem_kb") != 8 else 0), n3
    y = rng.standard_normal(p.K.n_rows)
    assert np.array_equal(g.apply(y), g.apply(y))
    assert rel_err(g.apply(y), o.vcycle(y)) < RTOL_VCYCLE
    # smoothing step and epilogues (resid / add / addscale) through the xsell operands
    b = rng.standard_normal(p.K.n_rows)
    assert rel_err(g.smooth(0, b, y), o.smooth(0, b, y)) < 1e-12
    _pcg_parity(p, h, g, o)


def test_sell_all_empty_row_groups(pkg):
    """A SELL-32 operand whose 32-row groups are alternately all-empty and
    populated, with more chunks than resident warps (each warp walks several
    chunks): the next chunk's column prefetch must not be skipped by an empty
    group. Products checked exactly against scipy (one entry per
    row or ascending sequential sums of exactly representable values)."""
    import ctypes as C
    import scipy.sparse as sp
    from paper_1902_01715_b200 import _native as N
    lib = N.gpu()
    rng = np.random.default_rng(23)
    n, nc = 32 * 12000, 64
    rows, cols, vals = [], [], []
    for g in range(n // 32):
        if g % 3 == 1:
            continue  # all 32 rows of this group empty
        for r in range(32 * g, 32 * g + 32):
            k = 1 + (r % 3)
            cs = np.sort(rng.choice(nc, size=k, replace=False))
            rows += [r] * k
            cols += list(cs)
            vals += list(rng.integers(1, 8, size=k).astype(float))
    Pm = sp.csr_matrix((vals, (rows, cols)), shape=(n, nc))
    Pm.sort_indices()
    I = sp.identity(n, format="csr")
    Ic = sp.identity(nc, format="csr")
    mats0 = [pkg.SparseMatrix.from_scipy(m) for m in (I, I, I, Pm, Pm.T.tocsr())]
    empty = pkg.SparseMatrix(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    mats1 = [pkg.SparseMatrix.from_scipy(Ic)] + [empty] * 4
    ctx = C.c_void_p()
    assert lib.aspamg_gpu_ctx_create(0, C.byref(ctx)) == 0
    try:
        for k, v in {"sell_min_rows": 0, "sell_min_mean": 0, "sell_chh": 32, "bsr": 0, "tail_dense": 0, "xsell": 0}.items():
            assert lib.aspamg_gpu_set_option(ctx, k.encode(), v) == 0
        for l, ms in enumerate((mats0, mats1)):
            views = [m.view() for m in ms]
            assert lib.aspamg_gpu_upload_level(ctx, l, *[C.byref(v) for v in views], 1.0) == 0
        L = np.ascontiguousarray(np.eye(nc).ravel(order="F"))
        assert lib.aspamg_gpu_upload_coarse(ctx, nc, L.ctypes.data_as(C.POINTER(C.c_double))) == 0
        assert lib.aspamg_gpu_finalize(ctx) == 0
        info = N.GpuLevelInfo()
        assert lib.aspamg_gpu_level_info(ctx, 0, C.byref(info)) == 0
        assert info.fmt[3] == 2, "P must be uploaded as SELL for this test"
        x = rng.integers(-4, 5, size=nc).astype(float)
        y = np.empty(n)
        P_d = C.POINTER(C.c_double)
        assert lib.aspamg_gpu_spmv(ctx, 0, 3, x.ctypes.data_as(P_d), y.ctypes.data_as(P_d)) == 0
        assert np.array_equal(y, Pm @ x)
    finally:
        lib.aspamg_gpu_ctx_destroy(ctx)


@pytest.mark.parametrize("u,extra", [(4, {}), (8, {}), (4, {"csr_blocked": 1}), (8, {"csr_blocked": 1, "csr_noalloc": 1,
                                                                                  "stream_bytes": 1})])
def test_csrw_pipelined_kernel_bit_identical(pkg, oracle, u, extra):
    """Warp-per-row pipelined CSR kernel (k_csrw: columns one round ahead across row
    boundaries, row pointers two rows ahead): same per-lane order, fma chain and shuffle
    tree as k_csr<32>, so every product and the whole V-cycle are bit-identical to the
    unpipelined kernel with the same thread groups; PCG inside the north_star gates."""
    p, h = problem_and_hierarchy(2, 2)
    base = dict(csr_max_group=32, csr_per_thread=1, sell_min_rows=1 << 40, csr_long=0, idx16=0)
    g0 = _gpu(pkg, h, csrw=0, **base)
    g1 = _gpu(pkg, h, csrw=u, **base, **extra)  # blocked rows / L1-bypassing matrix loads change no bits
    o = _oracle(oracle, h)
    names = [n for n, l, _, _ in g1.profile_iteration()]
    assert sum(".csrw" in n for n in names) >= 2, names
    rng = np.random.default_rng(31)
    for l in range(h.n_levels - 1):
        for wi, which in enumerate(["A", "G", "Gt", "P", "Pt"]):
            m = getattr(h.level(l, copy=False), which)
            x = rng.standard_normal(m.n_cols)
            assert np.array_equal(g1.spmv(l, wi, x), g0.spmv(l, wi, x)), (which, l)
    y = rng.standard_normal(p.K.n_rows)
    assert np.array_equal(g1.apply(y), g0.apply(y))
    assert rel_err(g1.apply(y), o.vcycle(y)) < RTOL_VCYCLE
    _pcg_parity(p, h, g1, o)
    g0.close()
    g1.close()


@pytest.mark.parametrize("u,blocked", [(4, 0), (8, 0), (4, 1), (8, 1)])
def test_csrw_ragged_and_empty_rows(pkg, u, blocked):
    """k_csrw on an operand with empty rows (single and in long runs, first and last
    row), rows of exactly one round, one entry more, and many rounds, with more rows
    than resident warps: exact products (small integers) against scipy."""
    import ctypes as C
    import scipy.sparse as sp
    from paper_1902_01715_b200 import _native as N
    lib = N.gpu()
    rng = np.random.default_rng(37)
    n, nc = 70000, 3000
    lens = rng.choice([0, 0, 1, 31, 32, 33, 32 * u, 32 * u + 1, 200, 700], size=n)
    lens[0] = 0
    lens[-1] = 0
    lens[1000:1400] = 0  # a run of empty rows longer than one warp stride window
    lens[5] = 2500
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    ci = np.concatenate([np.sort(rng.choice(nc, size=k, replace=False)) for k in lens if k] or [np.zeros(0, np.int64)])
    va = rng.integers(-3, 4, size=rp[-1]).astype(float)
    Pm = sp.csr_matrix((va, ci.astype(np.int64), rp), shape=(n, nc))
    I = sp.identity(n, format="csr")
    Ic = sp.identity(nc, format="csr")
    mats0 = [pkg.SparseMatrix.from_scipy(m) for m in (I, I, I, Pm, Pm.T.tocsr())]
    empty = pkg.SparseMatrix(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    mats1 = [pkg.SparseMatrix.from_scipy(Ic)] + [empty] * 4
    ctx = C.c_void_p()
    assert lib.aspamg_gpu_ctx_create(0, C.byref(ctx)) == 0
    try:
        for k, v in {"sell_min_rows": 1 << 40, "bsr": 0, "tail_dense": 0, "csr_long": 0, "idx16": 0, "csrw": u,
                     "csr_per_thread": 1, "csr_max_group": 32, "csr_blocked": blocked, "csr_noalloc": blocked,
                     "stream_bytes": 1 if blocked else 48 << 20}.items():
            assert lib.aspamg_gpu_set_option(ctx, k.encode(), v) == 0
        for l, ms in enumerate((mats0, mats1)):
            views = [m.view() for m in ms]
            assert lib.aspamg_gpu_upload_level(ctx, l, *[C.byref(v) for v in views], 1.0) == 0
        L = np.ascontiguousarray(np.eye(nc).ravel(order="F"))
        assert lib.aspamg_gpu_upload_coarse(ctx, nc, L.ctypes.data_as(C.POINTER(C.c_double))) == 0
        assert lib.aspamg_gpu_finalize(ctx) == 0
        cap, cnt = 64, C.c_int()
        buf = (N.GpuKernelTime * cap)()
        assert lib.aspamg_gpu_profile_iteration(ctx, buf, cap, C.byref(cnt)) == 0
        names = [buf[i].name.decode() for i in range(cnt.value)]
        assert any(nm.startswith("prolong_P.csrw") for nm in names), names
        x = rng.integers(-4, 5, size=nc).astype(float)
        y = np.empty(n)
        P_d = C.POINTER(C.c_double)
        assert lib.aspamg_gpu_spmv(ctx, 0, 3, x.ctypes.data_as(P_d), y.ctypes.data_as(P_d)) == 0
        assert np.array_equal(y, Pm @ x)
    finally:
        lib.aspamg_gpu_ctx_destroy(ctx)


def test_upload_rejects_unsorted_row(pkg):
    """check_view: columns must ascend within a row (sparse_matrix.hpp:27-33) —
    the 16-bit column mode would otherwise wrap silently. Status 1 (DimensionError)."""
    import ctypes as C
    from paper_1902_01715_b200 import _native as N
    lib = N.gpu()
    ctx = C.c_void_p()
    assert lib.aspamg_gpu_ctx_create(0, C.byref(ctx)) == 0
    A = pkg.SparseMatrix(3, 3, np.array([0, 2, 3, 5], np.int64), np.array([1, 0, 1, 0, 2], np.int64),
                         np.array([1.0, 4.0, 4.0, 1.0, 4.0]))
    e = pkg.SparseMatrix(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    v = A.view()
    ev = e.view()
    code = lib.aspamg_gpu_upload_level(ctx, 0, C.byref(v), C.byref(ev), C.byref(ev), C.byref(ev), C.byref(ev), 1.0)
    assert code == 1
    assert b"ascending" in lib.aspamg_gpu_last_error(ctx)
    lib.aspamg_gpu_ctx_destroy(ctx)
