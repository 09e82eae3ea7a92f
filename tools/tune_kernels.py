#!/usr/bin/env python3
"""Sweep device-format options on one hierarchy (GPU box): per option set, the
eager per-kernel profile of one PCG iteration and the graph solve time.

usage: python tools/tune_kernels.py [--config 2] [--scale 1] [--sets name=k:v,k:v ...]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1902_01715_b200 as P  # noqa: E402

DEFAULT_SETS = {
    "default": {},
    "sigma256": {"sell_sigma": 256},
    "sigma64": {"sell_sigma": 64},
    "nosort": {"sell_sort_fill_pct": 100000},
    "u4": {"sell_u": 4},
    "u2": {"sell_u": 2},
    "mean24": {"sell_max_mean": 24},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--gpu-setup", type=int, default=1, help="SRQCG / aFSAI / Galerkin on the GPU (the identical hierarchy)")
    ap.add_argument("--sets", nargs="*", default=None)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "tune.json"))
    ap.add_argument("--solves", type=int, default=3, help="timed solves per option set (after one warm-up)")
    ap.add_argument("--max-it", type=int, default=1000)
    args = ap.parse_args()
    sets = DEFAULT_SETS
    if args.sets:
        sets = {}
        for s in args.sets:
            name, _, kv = s.partition("=")
            sets[name] = {k: int(v) for k, v in (p.split(":") for p in kv.split(",") if p)}

    class D:
        def barrier(self):
            pass

    prob, h, _, _, _ = bench.get_hierarchy(P, args.config, args.scale, 0, D(), os.cpu_count() or 1,
                                            0 if args.gpu_setup else None)
    res = {}
    for name, opts in sets.items():
        g = P.GpuVcycle(h, device=0, options=opts)
        g.pcg(prob.rhs, max_it=args.max_it)  # warm
        t = []
        for _ in range(max(1, args.solves)):
            x, rep = g.pcg(prob.rhs, max_it=args.max_it)
            t.append(rep.T_s / max(rep.iterations, 1))
        vms = g.time_vcycle(50)
        prof = g.profile_ops(reps=20)
        res[name] = {"opts": opts, "s_per_it": min(t), "n_it": rep.iterations, "vcycle_ms": vms,
                     "graph_ops_ms": sum(p[2] for p in prof),
                     "kernels": [(p[0], p[1], round(p[2] * 1e3, 1), round(p[3] / (p[2] * 1e-3) / 1e9) if p[2] else 0)
                                 for p in prof]}
        print(f"{name:10s} {min(t)*1e3:.4f} ms/it  vcycle {vms:.4f} ms  ops {res[name]['graph_ops_ms']:.3f} ms  n_it {rep.iterations}",
              flush=True)
        g.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    # compact per-kernel comparison (us)
    names = list(res)
    rows = res[names[0]]["kernels"]
    for i, k in enumerate(rows):
        print(f"{k[0]:22s} L{k[1]} " + " ".join(f"{res[n]['kernels'][i][2]:7.1f}" if i < len(res[n]['kernels']) else "    -  " for n in names))


if __name__ == "__main__":
    main()
