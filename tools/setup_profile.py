"""Setup-phase profile of one config (per level: rows, refinement passes, t_smoother).

python tools/setup_profile.py --config 5 [--scale 1] [--gpu-setup 1] [--out f.json]
Writes one JSON object (setup phases T_ts/T_sm/T_cs/T_pl/T_rap, complexities,
per-level smoother statistics)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_01715_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--gpu-setup", type=int, default=1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    t = time.perf_counter()
    p = P.Problem.config(a.config, a.scale)
    t_gen = time.perf_counter() - t
    t = time.perf_counter()
    h = P.amg_setup(p.K, p.coords, setup_device=0 if a.gpu_setup else None)
    t_setup = time.perf_counter() - t
    i = h.info()
    r = {"config": a.config, "scale": a.scale, "n": p.K.n_rows, "nnz": p.K.nnz, "gen_s": t_gen,
         "setup_s": t_setup, "gpu_setup": bool(a.gpu_setup), "threads": os.cpu_count(),
         "phases": {k: getattr(i, k) for k in ("T_ts", "T_sm", "T_cs", "T_pl", "T_rap", "T_p")},
         "C_gd": i.C_gd, "C_op": i.C_op, "C_fs": i.C_fs, "levels": []}
    for l in range(h.n_levels - 1):
        lv = h.level_view(l)
        r["levels"].append({"n": int(lv.A.n_rows), "nnz_A": int(lv.A.nnz), "nnz_G": int(lv.G.nnz),
                            "passes": int(lv.refinement_passes), "exit": int(lv.smoother_exit),
                            "omega": lv.omega, "lambda_hat": lv.lambda_hat, "t_smoother": lv.t_smoother})
    print(json.dumps(r), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(r, f, indent=1)


if __name__ == "__main__":
    main()
