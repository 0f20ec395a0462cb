"""Every BASELINE.json config on the GPU ("5 BJ configs as seeded synthetic
inputs"): one warm-up + timed nli() over all COIs, point-spans/s, channels/s, kernel split, the
algorithmic FP64 roofline fraction, and eta statistics.  One JSON line per config.

    python tools/run_configs.py [--configs c1,c2,c3,c4,c5] [--precision 64]
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
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--precision", type=int, default=64)
    ap.add_argument("--warm", type=int, default=1)
    a = ap.parse_args()
    import torch
    import paper_2412_11614_b200 as isrs
    from bench import algorithmic_work_per_point, fp64_peak_tflops
    from workloads import bj_config
    for cfg in a.configs.split(","):
        link = bj_config(cfg)
        t0 = time.perf_counter()
        with isrs.Engine(link, precision=a.precision) as e:
            t_create = time.perf_counter() - t0
            for _ in range(a.warm):
                e.nli()
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            eta = e.nli()
            ev1.record()
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1)
            kms, kps = e.last_kernel_ms()
            pts, pspans, nreg = e.work()
            chain_g, k_s = e.span_chains()
            grp = e.chain_groups() if a.precision == 64 else None
        eta = eta.cpu().numpy()
        fl, sl = algorithmic_work_per_point(chain_g, k_s, grp)
        ach = kps[2] * fl / link.n_span / (kms[3] * 1e-3) / 1e12
        print(json.dumps({
            "config": cfg, "n_ch": link.n_ch, "n_span": link.n_span, "grid_n": link.grid_n,
            "precision": a.precision, "regions": nreg, "points": pts, "point_spans": pspans,
            "ms": ms, "kernel_ms": kms, "point_spans_per_s": pspans / (ms * 1e-3),
            "channels_per_s": link.n_ch / (ms * 1e-3), "create_s": t_create,
            "fp64_flops_frac": ach / fp64_peak_tflops() / (2.0 if a.precision == 32 else 1.0),
            "span_chains": [int(g) for g in chain_g],
            "chain_groups": None if grp is None else [int(g) for g in grp],
            "eta_db_min_max": [float(10 * np.log10(eta.min())), float(10 * np.log10(eta.max()))],
            "finite": bool(np.all(np.isfinite(eta)) and np.all(eta > 0))}), flush=True)


if __name__ == "__main__":
    main()
