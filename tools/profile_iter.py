#!/usr/bin/env python3
"""Run one warm-up + one profiled PCG iteration of the bench workload eagerly
(one launch per kernel, in V-cycle order) — the target command for ncu
captures. Prints the per-kernel event table.

usage: python tools/profile_iter.py [--config 2] [--scale 1] [--opt k=v ...]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1902_01715_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--gpu-setup", type=int, default=1, help="SRQCG / aFSAI / Galerkin on the GPU (the identical hierarchy)")
    ap.add_argument("--opt", nargs="*", default=[])
    args = ap.parse_args()

    class D:
        def barrier(self):
            pass

    prob, h, _, _, _ = bench.get_hierarchy(P, args.config, args.scale, 0, D(), os.cpu_count() or 1,
                                            0 if args.gpu_setup else None)
    opts = {k: int(v) for k, v in (o.split("=") for o in args.opt)}
    g = P.GpuVcycle(h, device=0, options=opts)
    # ncu runs this with --profile-from-start off: only the two body runs below are
    # captured (not the upload / finalize kernels, e.g. the dense-tail probe).
    # a short real solve first: the profiled iteration then runs on live vectors (on a fresh
    # context r = p = 0, p'Kp = 0 raises the not-SPD flag and the last op, pcg_xr, returns early)
    g.pcg(prob.rhs, max_it=3)
    import ctypes
    cu = ctypes.CDLL("libcuda.so.1")
    cu.cuProfilerStart()
    prof = g.profile_iteration()  # runs the body twice: warm + timed (ncu sees both)
    cu.cuProfilerStop()
    for name, lvl, ms, by in prof:
        print(f"{name:24s} L{lvl} {ms * 1e3:8.1f} us {by / 1e6:9.2f} MB {by / (ms * 1e-3) / 1e9 if ms else 0:8.1f} GB/s")


if __name__ == "__main__":
    main()
