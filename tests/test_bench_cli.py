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
