"""The C++ `solve` CLI (paper_1902_01715_b200/lib/aspamg_solve, built on the C++
host API include/aspamg_b200.hpp): SPEC.md:619-624 contract and exit codes."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1902_01715_b200", "lib", "aspamg_solve")


def run(*args, timeout=600):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=timeout)


def test_cli_exit_codes(tmp_path):
    assert run("--config", "1", "bogus_key=3").returncode == 1            # config error
    assert run("--config", "9").returncode == 1
    assert run("--matrix", str(tmp_path / "missing.mtx")).returncode == 2  # I/O error
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 2.0\n")
    assert run("--matrix", str(bad)).returncode == 2


def _write_mtx(path, K):
    K = K.tocoo()
    low = K.row >= K.col
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n% generated\n")
        f.write(f"{K.shape[0]} {K.shape[1]} {int(low.sum())}\n")
        for i, j, v in zip(K.row[low], K.col[low], K.data[low]):
            f.write(f"{i + 1} {j + 1} {float(v)!r}\n")


def test_cli_rejects_stale_hierarchy(tmp_path, pkg):
    """--hierarchy must not reuse a cache built from another matrix of the same size
    (the device Krylov operator is the hierarchy's level 0, not the input A)."""
    p = pkg.Problem.hex_cube(3, spacing=1 / 3)
    K = p.K.to_scipy()
    hb = tmp_path / "h.bin"
    _write_mtx(tmp_path / "K.mtx", K)
    run("--matrix", str(tmp_path / "K.mtx"), "--hierarchy", str(hb))  # builds + saves (solve needs a GPU)
    assert hb.exists()
    _write_mtx(tmp_path / "K2.mtx", 2.0 * K)
    r = run("--matrix", str(tmp_path / "K2.mtx"), "--hierarchy", str(hb))
    assert r.returncode == 1 and "different matrix" in r.stderr


def _has_gpu():
    import ctypes as C
    import sys
    sys.path.insert(0, ROOT)
    from paper_1902_01715_b200 import _native as N
    n = C.c_int()
    N.gpu().aspamg_gpu_device_count(C.byref(n))
    return n.value > 0


def test_cli_without_gpu_fails_loudly():
    if _has_gpu():
        pytest.skip("a CUDA device is present")
    r = run("--config", "1", "--scale", "4")
    assert r.returncode == 5 and "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_cli_solve_matches_python_api(tmp_path, pkg):
    rep = tmp_path / "r.json"
    r = run("--config", "1", "--scale", "2", "--report", str(rep))
    assert r.returncode == 0, r.stderr
    d = json.loads(rep.read_text())
    p = pkg.Problem.config(1, 2)
    h = pkg.Hierarchy.setup(p.K, p.coords)
    x, rr = pkg.pcg(p.K, p.rhs, pkg.GpuVcycle(h))
    assert d["iterations"] == rr.iterations and d["converged"]
    assert np.allclose(d["residual_history"], rr.residual_history, rtol=1e-12)


@pytest.mark.gpu
def test_pcg_rejects_foreign_operator(pkg):
    """pcg(A, b, M): A of the right size but not M's finest operator -> DimensionError."""
    p = pkg.Problem.config(1, 4)
    M = pkg.GpuVcycle(pkg.Hierarchy.setup(p.K, p.coords))
    K2 = pkg.SparseMatrix(p.K.n_rows, p.K.n_cols, p.K.row_offsets.copy(), p.K.col_indices.copy(), 2.0 * p.K.values)
    with pytest.raises(pkg.DimensionError):
        pkg.pcg(K2, p.rhs, M)
    x, rep = pkg.pcg(p.K, p.rhs, M)
    assert rep.converged


@pytest.mark.gpu
def test_cli_matrix_market_input(tmp_path, pkg):
    """symmetric Matrix Market (lower triangle) + coordinates, ones rhs."""
    p = pkg.Problem.hex_cube(4, spacing=0.25)
    mtx = tmp_path / "K.mtx"
    _write_mtx(mtx, p.K.to_scipy())
    xyz = tmp_path / "xyz.txt"
    np.savetxt(xyz, p.coords)
    r = run("--matrix", str(mtx), "--coords", str(xyz))
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["converged"] and d["true_relative_residual"] <= 1e-7
