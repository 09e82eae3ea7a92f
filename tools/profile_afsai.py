"""Device aFSAI on level 1 of a config (for ncu): setup with the GPU phases,
then smoother_setup of A_1 alone on the device.

python tools/profile_afsai.py --config 5 --scale 2"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_01715_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--scale", type=int, default=2)
    ap.add_argument("--level", type=int, default=1)
    a = ap.parse_args()
    p = P.Problem.config(a.config, a.scale)
    h = P.amg_setup(p.K, p.coords, setup_device=0)
    A = h.level(a.level).A
    import torch
    torch.cuda.init()
    torch.cuda.profiler.start()  # ncu --profile-from-start off: only this call is captured
    t = time.perf_counter()
    r = P.gpu_smoother_setup(A)
    torch.cuda.profiler.stop()
    print(f"level {a.level}: n={A.n_rows} passes={r['passes']} omega={r['omega']:.4f} "
          f"nnz_r(G)={r['G'].nnz / A.n_rows:.1f} t={time.perf_counter() - t:.2f}s", flush=True)


if __name__ == "__main__":
    main()
