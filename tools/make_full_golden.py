#!/usr/bin/env python3
"""Record the CPU oracle's PCG solve of a full-size BASELINE config as a golden
fixture (run on the GPU box, where the 16 host cores and the RAM are):

    python tools/make_full_golden.py --config 5 --out gpurun_out/c5_oracle.npz

The fixture holds the hierarchy signature (Hierarchy.signature), the oracle's
residual history, every STRIDE-th entry of its solution, ||x||_2 and the
convergence flags. tests/test_zz_full_size.py compares the GPU solve against it
when (and only when) the hierarchy it builds has the same signature — the
oracle solve of C5 takes ~11 minutes, the fixture makes the driver's GPU test
window enough. Oracle: oracle/oracle.c pcg on the reference's compiled spmv
(oracle/_ref), same hierarchy arrays as the GPU.
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_1902_01715_b200 as P  # noqa: E402
import pyoracle as O  # noqa: E402

STRIDE = 61


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--max-it", type=int, default=1000)
    ap.add_argument("--gpu-setup", type=int, default=1)
    ap.add_argument("--cached", type=int, default=1)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    out = args.out or os.path.join(ROOT, "gpurun_out", f"c{args.config}_oracle.npz")
    t0 = time.perf_counter()
    if args.cached:  # reuse bench.py's hierarchy cache (.cache/): a save/load round trip is bit-exact
        import bench

        class _D:
            def barrier(self):
                pass
        p, h, _, _, _ = bench.get_hierarchy(P, args.config, 1, 0, _D(), os.cpu_count() or 1,
                                            0 if args.gpu_setup else None)
    else:
        p = P.Problem.config(args.config, 1)
        h = P.Hierarchy.setup(p.K, p.coords, setup_device=0 if args.gpu_setup else None)
    t_setup = time.perf_counter() - t0
    sig = h.signature()
    print("setup", round(t_setup, 1), "s, signature", sig, flush=True)
    threads = os.cpu_count() or 1
    oh = O.OracleHierarchy(h, use_ref_spmv=O.ref_available(), threads=threads)
    t0 = time.perf_counter()
    st, xo, ho, conv, trr = oh.pcg(p.rhs, rel_tol=1e-8, max_it=args.max_it)
    t_cpu = time.perf_counter() - t0
    ho = np.asarray(ho)
    print("oracle", len(ho), "its", round(t_cpu, 1), "s conv", conv, "trr", trr, flush=True)
    rec = dict(signature=np.array(sig), config=args.config, n=p.K.n_rows, history=ho, x_stride=STRIDE,
               x_sample=np.asarray(xo)[::STRIDE].copy(), x_norm=float(np.linalg.norm(xo)), status=int(st),
               converged=bool(conv), true_rel_res=float(trr), cpu_seconds=t_cpu, cpu_threads=threads,
               ref_spmv=bool(O.ref_available()), max_it=args.max_it)
    # the GPU solve on the same hierarchy, for the record (the test repeats it)
    try:
        g = P.GpuVcycle(h, device=0)
        xg, rep = g.pcg(p.rhs, rel_tol=1e-8, max_it=args.max_it)
        hg = np.asarray(rep.residual_history)
        k = min(20, len(hg), len(ho))
        rec.update(gpu_history=hg, gpu_iterations=rep.iterations, gpu_T_s=rep.T_s,
                   gpu_first20=float(np.max(np.abs(hg[:k] - ho[:k]) / ho[:k])),
                   gpu_rel_err=float(np.linalg.norm(xg - xo) / np.linalg.norm(xo)))
        print("gpu", rep.iterations, "its", rep.T_s, "s first20", rec["gpu_first20"], "rel_err", rec["gpu_rel_err"], flush=True)
    except Exception as e:  # no GPU: fixture without the comparison
        print("gpu solve skipped:", e)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    np.savez_compressed(out, **rec)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
