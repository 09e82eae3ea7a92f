"""bench.py contract on CPU: the reference arm prints one JSON line with the
required keys; the GPU arm fails loudly without a device (no CPU fallback)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          cwd=ROOT, env=env, timeout=600)


def test_reference_arm_json_line():
    r = _run(["--impl", "reference", "--config", "1", "--scale", "4", "--steps", "1", "--warmup", "0",
              "--ref-sample-s", "0.2"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is False and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0


def test_reference_arm_nonzero_rank_exits_quietly():
    r = _run(["--impl", "reference", "--config", "1", "--scale", "4", "--steps", "1"],
             {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and not r.stdout.strip()


def test_gpu_arm_fails_loudly_without_device():
    import ctypes as C
    sys.path.insert(0, ROOT)
    from paper_1902_01715_b200 import _native as N
    n = C.c_int()
    N.gpu().aspamg_gpu_device_count(C.byref(n))
    if n.value > 0:
        pytest.skip("a CUDA device is present")
    r = _run(["--config", "1", "--scale", "4", "--steps", "1", "--no-cpu"])
    assert r.returncode != 0
    assert "no CUDA device" in r.stderr


def test_both_arms_share_metric_and_unit():
    """The driver divides the two arms' values only when metric, unit and direction are
    identical (round 1 printed two different strings and got a null ratio)."""
    sys.path.insert(0, ROOT)
    import inspect

    import bench
    r = _run(["--impl", "reference", "--config", "1", "--scale", "4", "--steps", "1", "--warmup", "0", "--ref-sample-s", "0.2"])
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")][0])
    assert d["metric"] == bench.METRIC and d["unit"] == "s/iteration"
    src = inspect.getsource(bench.run_b200)
    assert '"metric": METRIC' in src and '"unit": "s/iteration"' in src and '"higher_is_better": False' in src


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """GPU arm on a small config: one JSON line with the contract's keys, e2e from host buffers
    (copies declared), kernel launches counted, the same metric string as the reference arm."""
    sys.path.insert(0, ROOT)
    import bench
    r = _run(["--config", "1", "--steps", "2", "--warmup", "3", "--ref-sample-s", "0.5"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["metric"] == bench.METRIC and d["unit"] == "s/iteration" and d["higher_is_better"] is False
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * d["config"]["n"] and d["e2e"]["d2h_bytes_per_step"] > 8 * d["config"]["n"]
    assert d["e2e"]["value"] >= d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 2
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["one_thread"]["cores"] == 1
    assert d["config"]["converged"] is True
