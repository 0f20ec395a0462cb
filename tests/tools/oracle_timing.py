"""Time the oracle (oracle/, numpy fp64, closed mode = literal Eqs. 8-10) on whole small configs and
on bounded samples of the large ones, on this host's cores (SURVEY.md §8(d) "oracle timed beside it").

    python tests/tools/oracle_timing.py [--configs c1] [--sample c2,c3,c4,c5] [--seconds 20]

One JSON line per config: point-spans, seconds, point-spans/s, processes used.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def _eta_one(args):
    from oracle import egn
    link, kappa = args
    t0 = time.perf_counter()
    e, _ = egn.eta(link, coi=[kappa])
    return time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1")
    ap.add_argument("--sample", default="c2,c3,c4,c5")
    ap.add_argument("--seconds", type=float, default=20.0)
    a = ap.parse_args()
    import multiprocessing as mp
    from bench import oracle_sample
    from oracle import egn
    from workloads import bj_config
    cores = os.cpu_count() or 1
    for cfg in [c for c in a.configs.split(",") if c]:
        link = bj_config(cfg)
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(min(cores, link.n_ch)) as pool:
            pool.map(_eta_one, [(link, k) for k in range(link.n_ch)], chunksize=1)
        dt = time.perf_counter() - t0
        c = egn.canonicalize(link)
        pts = 0
        for k in range(link.n_ch):
            for k1 in range(link.n_ch):
                for k2 in range(link.n_ch):
                    if egn.has_support_bound(c, k, k1, k2):
                        pts += egn.region_partials(link, k, k1, k2, mu_mode="unit")[1]
        print(json.dumps({"config": cfg, "whole": True, "point_spans": pts * link.n_span, "seconds": dt,
                          "point_spans_per_s": pts * link.n_span / dt,
                          "processes": min(cores, link.n_ch)}), flush=True)
    for cfg in [c for c in a.sample.split(",") if c]:
        link = bj_config(cfg)
        rate, ps, dt, used, desc = oracle_sample(link, a.seconds)
        print(json.dumps({"config": cfg, "whole": False, "point_spans": ps, "seconds": dt,
                          "point_spans_per_s": rate, "processes": used, "sample": desc}), flush=True)


if __name__ == "__main__":
    main()
