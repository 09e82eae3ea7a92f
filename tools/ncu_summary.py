#!/usr/bin/env python3
"""Summarise ncu artefacts into profiles/ (run here, after gpurun brings them back).

  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
      --ops gpurun_out/plain.log --tag r01 [--traffic-key c2]

Writes profiles/ncu_<tag>_full.csv (per captured kernel: duration, DRAM bytes,
achieved GB/s, occupancy, top stalls), profiles/ncu_<tag>_launches.csv (every
launch of one PCG iteration with its ncu duration and share), and merges the
per-op DRAM traffic into profiles/traffic.json (read by bench.py).
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw_rows(rep):
    """Raw page of a report: a .ncu-rep (read through ncu) or an already exported raw CSV."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


UNIT = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6,      # -> MB
        "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3, "second": 1e6}   # -> us


def ops_from_plain(path):
    ops = []
    for ln in open(path):
        m = re.match(r"(\S+)\s+L(\d+)\s+([\d.]+) us\s+([\d.]+) MB", ln)
        if m:
            ops.append((m.group(1), int(m.group(2)), float(m.group(3)), float(m.group(4)) * 1e6))
    return ops


def kernel_of(op):
    name = op.split(".")
    fmt = name[1] if len(name) > 1 else ""
    if op.startswith("pcg_p"):
        return "k_pcg_p"
    if op.startswith("pcg_xr"):
        return "k_pcg_xr"
    if fmt == "sbsr3":
        return "k_sbsr3"
    if fmt.startswith("sell"):
        return "k_sell"
    if fmt.startswith("csr"):
        return "k_csr"
    return ""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--ops")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--regex", default="k_sell|k_csr|k_sbsr3")
    ap.add_argument("--skip", type=int, default=0, help="-s used for the capture (filtered launches skipped)")
    ap.add_argument("--traffic-key", default="c2")
    ap.add_argument("--all-ops", action="store_true",
                    help="the capture holds every launch of one iteration in op order (tools/run_profile.sh)")
    ap.add_argument("--peak", type=float, default=6550.4, help="measured HBM copy peak, GB/s (MEASURED_PEAKS.json)")
    ap.add_argument("--build-tag", default=None, help="kernel build hash for traffic.json (bench.kernel_build_tag())")
    args = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    ops = ops_from_plain(args.ops) if args.ops else []
    body = ops[-(len(ops) // 2):] if ops else []  # profile_iter runs the body twice; plain.log prints one
    body = ops
    if args.rep:
        hdr, units, rows = raw_rows(args.rep)
        g = lambda row, n: row[hdr.index(n)] if n in hdr else ""  # noqa: E731

        def gs(row, n):
            """Metric scaled by the report's unit for that column (MB for bytes, us for times)."""
            if n not in hdr:
                return 0.0
            i = hdr.index(n)
            return float(row[i] or 0) * UNIT.get(units[i], 1.0)
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
                      and h.endswith("_per_issue_active.ratio")]
        # align captured kernels with the op sequence (filtered by the capture regex)
        rx = re.compile(args.regex)
        filt = [o for o in body if rx.search(kernel_of(o[0]) or "-")]
        seq = (filt * 3)[args.skip % max(len(filt), 1):]
        if args.all_ops:
            seq = body
        out = []
        traffic = {}
        for k, row in enumerate(rows):
            op = seq[k] if k < len(seq) else ("?", -1, 0, 0)
            dur = gs(row, "gpu__time_duration.sum")  # us
            rd = gs(row, "dram__bytes_read.sum")     # MB
            wr = gs(row, "dram__bytes_write.sum")
            stalls = sorted(((float(row[i] or 0), hdr[i].replace("smsp__average_warps_issue_stalled_", "")
                              .replace("_per_issue_active.ratio", "")) for i in stall_cols), reverse=True)[:3]
            rec = {"op": op[0], "level": op[1], "kernel": g(row, "Kernel Name").split("(")[0],
                   "us": dur, "dram_read_MB": rd, "dram_write_MB": wr,
                   "dram_GBs": (rd + wr) / dur * 1e3 if dur else 0.0,
                   "alg_MB": op[3] / 1e6, "alg_GBs": op[3] / 1e6 / dur * 1e3 if dur else 0.0,
                   "regs": g(row, "launch__registers_per_thread"),
                   "warps_active": g(row, "sm__warps_active.avg.per_cycle_active"),
                   "l2_hit_pct": g(row, "lts__t_sector_hit_rate.pct"),
                   "dram_over_alg": (rd + wr) * 1e6 / op[3] if op[3] else 0.0,
                   "frac_of_peak": (op[3] / 1e6 / dur * 1e3 / args.peak) if dur else 0.0,
                   "dram_pct": g(row, "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
                   "l1tex_pct": g(row, "l1tex__throughput.avg.pct_of_peak_sustained_active"),
                   "lts_pct": g(row, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                   "top_stalls": "; ".join(f"{n}={v:.1f}" for v, n in stalls)}
            out.append(rec)
            traffic[f"{op[0]}@L{op[1]}"] = (rd + wr) * 1e6
        path = os.path.join(prof, f"ncu_{args.tag}_full.csv")
        with open(path, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=list(out[0].keys()))
            w.writeheader()
            w.writerows(out)
        print("wrote", path)
        tpath = os.path.join(prof, "traffic.json")
        tj = json.load(open(tpath)) if os.path.exists(tpath) else {}
        if args.build_tag:
            tj.setdefault(args.build_tag, {}).setdefault(args.traffic_key, {}).update(traffic)
        else:
            tj.setdefault(args.traffic_key, {}).update(traffic)
        json.dump(tj, open(tpath, "w"), indent=1)
        print("updated", tpath)
    if args.launches:
        rows = list(csv.reader(open(args.launches)))
        hdr = None
        data = []
        for r in rows:
            if r and r[0] == "ID":
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                if d.get("Metric Name") == "gpu__time_duration.sum":
                    data.append((d["Kernel Name"].split("(")[0], float(d["Metric Value"]) / 1e3))
        it = data[-len(body):] if body else data
        tot = sum(v for _, v in it)
        path = os.path.join(prof, f"ncu_{args.tag}_launches.csv")
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["op", "level", "kernel", "ncu_us", "share", "event_us", "alg_MB"])
            for k, (kn, us) in enumerate(it):
                op = body[k] if k < len(body) else ("?", -1, 0, 0)
                w.writerow([op[0], op[1], kn, f"{us:.2f}", f"{us / tot:.4f}", f"{op[2]:.1f}", f"{op[3] / 1e6:.2f}"])
        print("wrote", path, "total ncu us per iteration", round(tot, 1))


if __name__ == "__main__":
    main()
