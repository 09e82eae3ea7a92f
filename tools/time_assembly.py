#!/usr/bin/env python3
"""Host vs device stiffness assembly on the BASELINE configs:
generation time with the CPU assembler and with aspamg_gpu_assemble_hex behind the
assembly hook, and bit-identity of the two K. Prints one JSON object."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1902_01715_b200 as P  # noqa: E402

out = {"threads": os.cpu_count()}
P.Problem.config(1, 1, assembly_device=0)  # context / module warm-up
for cfg in (2, 3, 4, 5):
    t0 = time.perf_counter()
    host = P.Problem.config(cfg, 1)
    t_host = time.perf_counter() - t0
    t0 = time.perf_counter()
    dev = P.Problem.config(cfg, 1, assembly_device=0)
    t_dev = time.perf_counter() - t0
    same = (np.array_equal(host.K.row_offsets, dev.K.row_offsets) and np.array_equal(host.K.col_indices, dev.K.col_indices)
            and np.array_equal(host.K.values.view(np.int64), dev.K.values.view(np.int64)))
    out[f"c{cfg}"] = {"n": host.K.n_rows, "nnz": host.K.nnz, "generate_host_s": t_host, "generate_device_s": t_dev,
                      "bit_identical": bool(same)}
    del host, dev
print(json.dumps(out, indent=1))
