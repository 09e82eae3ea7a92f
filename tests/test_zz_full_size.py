"""Full-size parity on the BASELINE.json configs 3, 4 (and 5), through the C-ABI.

The GPU solve and the oracle PCG (oracle/oracle.c, all host cores, on the
reference's compiled spmv when oracle/_ref is present) run on the SAME
hierarchy; the gates are the north_star's: iteration count +-1, first-20
relative residuals within 1e-9 relative, solution within 1e-8
(pcg contract SPEC.md:504-512,519-521; stopping rule PAPER.md:760-762).

The file sorts last so that its minutes of CPU setup + oracle solve come after
every other GPU test. C1 and C2 at full size live in test_gpu_parity.py.

C5 (6.39M dofs, 0.51B nnz) needs ~60 GB of host memory for K + the hierarchy
and ~5 minutes of GPU-assisted setup; it runs when ASPAMG_TEST_C5=1 or when the
box has >= 100 GB of RAM. Its oracle solve (936 iterations, ~11 minutes on 16
cores) is read from the recorded fixture tests/golden/c5_oracle.npz
(tools/make_full_golden.py, run on the same kind of box) when the hierarchy
built here has the recorded signature; otherwise the oracle runs.
"""
import os

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


def _setup(pkg, cfg):
    p = pkg.Problem.config(cfg, 1)
    # GPU-assisted setup: the bit-identical hierarchy of the CPU setup (tests/test_gpu_setup.py)
    h = pkg.Hierarchy.setup(p.K, p.coords, setup_device=0)
    return p, h


def _oracle(oracle, h):
    return oracle.OracleHierarchy(h, use_ref_spmv=oracle.ref_available(), threads=os.cpu_count() or 1)


def _gates(rep, xg, ho, xo):
    k = min(20, rep.iterations, len(ho))
    assert k > 0
    assert np.all(np.abs(rep.residual_history[:k] - ho[:k]) <= 1e-9 * ho[:k]), "first-20 residual history"
    assert abs(rep.iterations - len(ho)) <= 1, (rep.iterations, len(ho))
    assert rel_err(xg, xo) <= 1e-8
    assert len(rep.residual_history) == rep.iterations


def test_pcg_c3_full_size(pkg, oracle):
    """BASELINE config 3: distorted 96x96x24 box, aspect ratio 20, N(0,1) rhs."""
    p, h = _setup(pkg, 3)
    assert p.K.n_rows == 677448
    g = pkg.GpuVcycle(h, device=0)
    xg, rep = g.pcg(p.rhs, rel_tol=1e-8, max_it=1000)
    st, xo, ho, conv, trr = _oracle(oracle, h).pcg(p.rhs, rel_tol=1e-8, max_it=1000)
    assert st == 0 and conv and rep.converged
    assert rep.true_rel_residual <= 1e-7
    _gates(rep, xg, ho, xo)
    g.close()


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _fixture(cfg):
    """Recorded oracle solve of a full-size config (tools/make_full_golden.py), or None."""
    path = os.path.join(GOLDEN, f"c{cfg}_oracle.npz")
    if os.environ.get("ASPAMG_FULL_ORACLE") == "1" or not os.path.exists(path):
        return None
    return np.load(path)


def _gates_fixture(rep, xg, fx):
    """The same gates against the recorded oracle solve: the solution is compared on the
    recorded every-STRIDE-th sample (relative 2-norm error) and through ||x||_2."""
    ho = fx["history"]
    k = min(20, rep.iterations, len(ho))
    assert k > 0
    assert np.all(np.abs(rep.residual_history[:k] - ho[:k]) <= 1e-9 * ho[:k]), "first-20 residual history"
    assert abs(rep.iterations - len(ho)) <= 1, (rep.iterations, len(ho))
    xs = fx["x_sample"]
    assert rel_err(xg[::int(fx["x_stride"])], xs) <= 1e-8
    assert abs(np.linalg.norm(xg) - float(fx["x_norm"])) <= 1e-8 * float(fx["x_norm"])
    assert len(rep.residual_history) == rep.iterations


def test_pcg_c4_full_size(pkg, oracle):
    """BASELINE config 4: 400x400x4 plate, nu = 0.49, clamped sides. At full
    size the recursive residual needs ~2600 iterations; with the paper's
    max_it = 1000 BOTH solves stop unconverged at 1000 and must
    agree: same count, same `converged = false`, first-20 history within 1e-9,
    the WHOLE 1000-entry history within 1e-6 relative, iterates within 1e-8.
    The oracle's 1000 iterations (~4.5 min on 16 cores) come from the recorded
    fixture tests/golden/c4_oracle.npz when the hierarchy has its signature."""
    p, h = _setup(pkg, 4)
    assert p.K.n_rows == 2388015
    fx = _fixture(4)
    if fx is not None and str(fx["signature"]) != h.signature():
        fx = None
    g = pkg.GpuVcycle(h, device=0)
    xg, rep = g.pcg(p.rhs, rel_tol=1e-8, max_it=1000)
    if fx is not None:
        ho, conv = fx["history"], bool(fx["converged"])
        assert rep.converged == conv
        _gates_fixture(rep, xg, fx)
    else:
        st, xo, ho, conv, trr = _oracle(oracle, h).pcg(p.rhs, rel_tol=1e-8, max_it=1000)
        assert rep.converged == bool(conv)
        _gates(rep, xg, ho, xo)
    if not rep.converged:
        assert rep.iterations == 1000 and len(ho) == 1000
        hg = np.asarray(rep.residual_history)
        assert np.all(np.abs(hg - ho) <= 1e-6 * ho), "unconverged histories must agree"
    g.close()


def _c5_enabled():
    if os.environ.get("ASPAMG_TEST_C5") == "1":
        return True
    if os.environ.get("ASPAMG_TEST_C5") == "0":
        return False
    try:
        import psutil
        return psutil.virtual_memory().total >= 100 * 2 ** 30
    except Exception:
        return False


def test_pcg_c5_full_size(pkg, oracle):
    """BASELINE config 5: 128^3 cube with 200 stiff spheres (6.39M dofs). The oracle
    solve (936 iterations, ~11 min on 16 cores) is taken from the recorded fixture
    tests/golden/c5_oracle.npz when this run's hierarchy has the recorded signature
    (the setup is deterministic); ASPAMG_FULL_ORACLE=1 reruns the oracle instead."""
    if not _c5_enabled():
        pytest.skip("C5 needs >= 100 GB of host RAM (set ASPAMG_TEST_C5=1 to force)")
    p, h = _setup(pkg, 5)
    assert p.K.n_rows == 6390144
    fx = _fixture(5)
    if fx is not None and str(fx["signature"]) != h.signature():
        fx = None  # another hierarchy: the recorded solve does not apply
    g = pkg.GpuVcycle(h, device=0)
    xg, rep = g.pcg(p.rhs, rel_tol=1e-8, max_it=1000)
    assert rep.converged
    if fx is not None:
        assert bool(fx["converged"]) and int(fx["status"]) == 0
        _gates_fixture(rep, xg, fx)
    elif os.environ.get("ASPAMG_FULL_ORACLE") == "1":
        st, xo, ho, conv, trr = _oracle(oracle, h).pcg(p.rhs, rel_tol=1e-8, max_it=1000)
        assert st == 0 and conv
        _gates(rep, xg, ho, xo)
    else:
        # no applicable fixture and no time for 936 oracle iterations: the first-20 gate
        # against a 20-iteration oracle run, and the iterate after those 20 iterations
        st, xo, ho, conv, trr = _oracle(oracle, h).pcg(p.rhs, rel_tol=1e-8, max_it=20)
        x20, rep20 = g.pcg(p.rhs, rel_tol=1e-8, max_it=20)
        assert np.all(np.abs(rep20.residual_history[:20] - ho[:20]) <= 1e-9 * ho[:20])
        assert rel_err(x20, xo) <= 1e-8
        pytest.skip("hierarchy signature differs from tests/golden/c5_oracle.npz: checked 20 iterations only")
    g.close()
