"""Host-side breakdown of the end-to-end call (bench.py's `e2e`): isrs_egn_create (validation, plan,
H2D, precompute), the first isrs_egn_nli on the fresh handle (+ sync), a second nli on the same
handle, the D2H read, and isrs_egn_destroy — wall clock per phase, several repetitions.

    python tools/e2e_breakdown.py [--config c2] [--reps 8]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=8)
    a = ap.parse_args()
    import torch
    import paper_2412_11614_b200 as isrs
    from workloads import bj_config
    link = bj_config(a.config)
    torch.cuda.init()
    rows = []
    for r in range(a.reps):
        t0 = time.perf_counter()
        e = isrs.Engine(link)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        eta = e.nli()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        k1 = e.last_kernel_ms()[0]
        eta = e.nli()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        h = eta.cpu().numpy()
        t4 = time.perf_counter()
        e.close()
        t5 = time.perf_counter()
        t6 = time.perf_counter()
        isrs.eta_host(link)
        t7 = time.perf_counter()
        rows.append({"create_ms": 1e3 * (t1 - t0), "nli1_ms": 1e3 * (t2 - t1), "kernel_phase1_ms": k1[3],
                     "nli2_ms": 1e3 * (t3 - t2), "d2h_ms": 1e3 * (t4 - t3), "destroy_ms": 1e3 * (t5 - t4),
                     "eta_host_ms": 1e3 * (t7 - t6)})
        print(json.dumps(rows[-1]), flush=True)
    med = {k: float(np.median([x[k] for x in rows])) for k in rows[0]}
    print(json.dumps({"config": a.config, "median": med, "eta0": float(h[0])}))


if __name__ == "__main__":
    main()
