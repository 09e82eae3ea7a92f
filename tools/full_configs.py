#!/usr/bin/env python3
"""Full-size parity + timing on all BASELINE configs (GPU box).

For each config: generate, CPU setup (cached in .cache/), GPU PCG (device time,
s/it) and the oracle PCG on the reference's compiled spmv on all host cores
(same hierarchy), then the north_star parity gates: iteration count +-1,
first-20 relative residuals within 1e-9 relative, final solution within 1e-8.

usage: python tools/full_configs.py [--configs 1 2 3 4 5] [--out gpurun_out/full_configs.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import bench  # noqa: E402
import paper_1902_01715_b200 as P  # noqa: E402
import pyoracle as O  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4, 5])
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "full_configs.json"))
    ap.add_argument("--oracle", type=int, default=1, help="run the CPU oracle solve (0 = GPU only)")
    ap.add_argument("--max-it", type=int, default=1000,
                    help="PCG iteration cap (the paper's 1000, PAPER.md:1211; C4 needs more at full size)")
    ap.add_argument("--gpu-reps", type=int, default=3, help="timed GPU solves (after one warm-up)")
    ap.add_argument("--gpu-setup", type=int, default=0, help="SRQCG + Galerkin on the GPU (bit-identical hierarchy)")
    args = ap.parse_args()

    class D:
        def barrier(self):
            pass

    results = {}
    if os.path.exists(args.out):
        results = json.load(open(args.out))
    threads = os.cpu_count() or 1
    for cfg in args.configs:
        t0 = time.perf_counter()
        prob, h, t_gen, t_setup, _origin = bench.get_hierarchy(P, cfg, args.scale, 0, D(), threads,
                                                      0 if args.gpu_setup else None)
        info = h.info()
        print(cfg, "setup", round(t_gen, 1), round(t_setup, 1), {k: round(getattr(info, k), 2) for k in
              ("T_ts", "T_sm", "T_cs", "T_pl", "T_rap")}, flush=True)
        rec = {"config": bench.CONFIG_DESC[cfg], "n": prob.K.n_rows, "nnz": prob.K.nnz, "setup_s": t_setup,
               "gen_s": t_gen, "gpu_setup": bool(args.gpu_setup),
               "setup_phases": {k: getattr(info, k) for k in ("T_ts", "T_sm", "T_cs", "T_pl", "T_rap")},
               "levels": int(info.n_levels), "C_gd": info.C_gd, "C_op": info.C_op, "C_fs": info.C_fs,
               "max_it": args.max_it, "level_sizes": [int(h.level_view(l).A.n_rows) for l in range(info.n_levels)]}
        g = P.GpuVcycle(h)
        g.pcg(prob.rhs, max_it=args.max_it)
        ts = []
        for _ in range(max(1, args.gpu_reps)):
            xg, rep = g.pcg(prob.rhs, max_it=args.max_it)
            ts.append(rep.T_s)
        rec.update({"gpu_n_it": rep.iterations, "gpu_converged": rep.converged, "gpu_T_s": min(ts),
                    "gpu_s_per_it": min(ts) / max(rep.iterations, 1), "gpu_true_rel_res": rep.true_rel_residual,
                    "gpu_e2e_s": rep.T_wall})
        print(cfg, "gpu", rep.iterations, round(min(ts), 4), flush=True)
        if args.oracle:
            oh = O.OracleHierarchy(h, use_ref_spmv=O.ref_available(), threads=threads)
            t = time.perf_counter()
            st, xo, ho, conv, trr = oh.pcg(prob.rhs, max_it=args.max_it)
            t_cpu = time.perf_counter() - t
            k = min(20, rep.iterations, len(ho))
            rel_hist = float(np.max(np.abs(rep.residual_history[:k] - ho[:k]) / ho[:k])) if k else 0.0
            sol = float(np.linalg.norm(xg - xo) / np.linalg.norm(xo))
            hg = np.asarray(rep.residual_history)
            rec["history"] = {"every": 50, "gpu": hg[::50].tolist(), "cpu": np.asarray(ho)[::50].tolist(),
                              "gpu_tail": hg[-12:].tolist(), "cpu_tail": np.asarray(ho)[-12:].tolist()}
            rec.update({"cpu_n_it": len(ho), "cpu_converged": conv, "cpu_T_s": t_cpu,
                        "cpu_s_per_it": t_cpu / max(len(ho), 1), "cpu_threads": threads,
                        "cpu_kind": "reference spmv (oracle/_ref)" if O.ref_available() else "oracle port",
                        "parity": {"iterations_diff": rep.iterations - len(ho),
                                   "first20_max_rel_diff": rel_hist, "solution_rel_err": sol,
                                   "pass": abs(rep.iterations - len(ho)) <= 1 and rel_hist <= 1e-9 and sol <= 1e-8}})
            print(cfg, "cpu", len(ho), round(t_cpu, 2), rec["parity"], flush=True)
        rec["wall_s"] = time.perf_counter() - t0
        results[f"c{cfg}_s{args.scale}" + ("" if args.max_it == 1000 else f"_it{args.max_it}")] = rec
        g.close()
        del h
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        json.dump(results, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
