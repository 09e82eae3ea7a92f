"""N > 1 host path of bench.py on CPU (gloo, world_size 2): replicas only
 — rank 0 runs the CPU setup and shares it through the
hierarchy dump; every rank then holds the identical hierarchy; timings are
reduced as the max over ranks."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, cache_root, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import bench
    import paper_1902_01715_b200 as P
    bench.ROOT = cache_root  # private cache dir for the test
    d = bench.Dist(ws, rank, rank, "gloo")
    prob, h, t_gen, t_setup, origin = bench.get_hierarchy(P, 1, 4, rank, d, 2)
    lv = h.level(1)
    chk = float(np.sum(lv.A.values)) + float(np.sum(h.level(0).G.values))
    import pyoracle as O
    st, x, hist, conv, trr = O.OracleHierarchy(h).pcg(prob.rhs)
    # staged turns (replicas of a large config load + upload one group of ranks at a time)
    import time

    def turn():
        t0 = time.time()
        time.sleep(0.3)
        return (t0, time.time())
    span = bench.staged(d, rank, ws, 1, turn)
    path_only = bench.get_hierarchy(P, 1, 4, rank, d, 2, load=False)[1]
    assert isinstance(path_only, str) and os.path.exists(path_only)
    t = d.max(float(rank + 1))
    tot = d.sum(float(len(hist)))
    assert origin == ("cpu" if rank == 0 else "cached: cpu")
    q.put((rank, chk, len(hist), conv, t, tot, span))
    d.close()


@pytest.mark.timeout(300)
def test_two_rank_replicas_gloo(tmp_path):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, str(tmp_path), q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    (_, c0, n0, v0, t0, s0, sp0), (_, c1, n1, v1, t1, s1, sp1) = res
    assert sp0[1] <= sp1[0], "staged(): rank 1's turn starts after rank 0's ended"
    assert c0 == c1 and n0 == n1 and v0 and v1
    assert t0 == t1 == 2.0  # max over ranks
    assert s0 == s1 == 2.0 * n0  # whole-job iterations (replicas)
    assert any(f.startswith("hier_c1_s4") for f in os.listdir(tmp_path / ".cache"))


def test_host_slots():
    sys.path.insert(0, ROOT)
    import bench
    gb = 1 << 30
    assert bench.host_slots(8, 47 * gb, 196 * gb) == 3   # C5 on the 196 GB box: 3 host copies at a time
    assert bench.host_slots(8, 4 * gb, 196 * gb) == 8    # C2: everyone at once
    assert bench.host_slots(2, 500 * gb, 196 * gb) == 1  # never zero
