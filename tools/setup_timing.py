"""Setup-phase timing, CPU vs GPU test space.

For each config: CPU amg_setup and amg_setup(setup_device=0); prints T_ts
(test-space phase) of both, the total setup time, and whether the two
hierarchies are bit-identical. Writes one JSON object per config."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_01715_b200 as P  # noqa: E402


def same(h1, h2):
    if h1.n_levels != h2.n_levels:
        return False
    for l in range(h1.n_levels):
        a, b = h1.level(l), h2.level(l)
        for name in ("A", "G", "P"):
            ma, mb = getattr(a, name), getattr(b, name)
            for arr in ("row_offsets", "col_indices", "values"):
                xa, xb = getattr(ma, arr), getattr(mb, arr)
                if (xa is None) != (xb is None) or (xa is not None and not np.array_equal(xa, xb)):
                    return False
    return bool(np.array_equal(h1.coarse_factor(), h2.coarse_factor()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2")
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--out", default=None)
    ap.add_argument("--smoother-max-mean-row", type=float, default=0.0,
                    help="GPU smoother level policy (0 = every level on the GPU)")
    a = ap.parse_args()
    res = []
    P.gpu_setup_policy("smoother_max_mean_row", a.smoother_max_mean_row)
    for cfg in [int(c) for c in a.configs.split(",")]:
        p = P.Problem.config(cfg, a.scale)
        warm = P.Problem.config(1, 4)
        P.amg_setup(warm.K, warm.coords, setup_device=0)  # CUDA context / module warm-up
        t = time.perf_counter()
        hc = P.amg_setup(p.K, p.coords)
        tc = time.perf_counter() - t
        t = time.perf_counter()
        hg = P.amg_setup(p.K, p.coords, setup_device=0)
        tg = time.perf_counter() - t
        ic, ig = hc.info(), hg.info()
        ph = ("T_ts", "T_sm", "T_cs", "T_pl", "T_rap")
        r = {"config": cfg, "scale": a.scale, "n": p.K.n_rows, "cpu_setup_s": tc, "gpu_setup_s": tg,
             "cpu": {k: getattr(ic, k) for k in ph}, "gpu": {k: getattr(ig, k) for k in ph},
             "identical": same(hc, hg), "threads": os.cpu_count(),
             "smoother_max_mean_row": a.smoother_max_mean_row,
             "levels": [{"n": int(hc.level(l).A.n_rows), "nnz_row": hc.level(l).A.nnz / max(hc.level(l).A.n_rows, 1),
                         "passes": hc.level(l).refinement_passes, "cpu_t_sm": hc.level(l).t_smoother,
                         "gpu_t_sm": hg.level(l).t_smoother} for l in range(hc.n_levels - 1)],
             "gpu_phases": "T_sm (aFSAI + Lanczos), T_ts (SRQCG), T_rap (Galerkin) on the GPU; T_cs, T_pl on the CPU"}
        print(json.dumps(r), flush=True)
        res.append(r)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
