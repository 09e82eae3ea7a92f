import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: large configurations (minutes of CPU setup)")


@pytest.fixture(scope="session")
def pkg():
    import paper_1902_01715_b200 as P
    return P


@pytest.fixture(scope="session")
def oracle():
    import pyoracle
    return pyoracle


_cache = {}


def problem_and_hierarchy(cfg: int, scale: int, **cfg_overrides):
    """Generated config + CPU setup, cached per session (same arrays go to GPU and oracle)."""
    import paper_1902_01715_b200 as P
    key = (cfg, scale, tuple(sorted(cfg_overrides.items())))
    if key not in _cache:
        p = P.Problem.config(cfg, scale)
        c = P.default_config(**cfg_overrides) if cfg_overrides else None
        h = P.Hierarchy.setup(p.K, p.coords, c)
        _cache[key] = (p, h)
    return _cache[key]


@pytest.fixture(scope="session")
def c1():
    return problem_and_hierarchy(1, 1)


def rel_err(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    d = np.linalg.norm(a - b)
    n = np.linalg.norm(b)
    return d / n if n > 0 else d
