"""Whole-eta parity of the CUDA path against the oracle for EVERY COI of a BASELINE config (the
GPU tests sample regions at full size; this runs the complete oracle, closed mode, on the host's
cores — c2 takes ~20 min on 16 cores).

    python tools/full_parity.py [--config c2] [--processes N]

Prints one JSON line: per-COI relative error, max, and the oracle wall time.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _oracle_coi(args):
    from oracle import egn
    link, kappa = args
    e, t = egn.eta(link, coi=[kappa])
    return kappa, float(e[0]), t[0].tolist()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--processes", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    import multiprocessing as mp
    import torch
    import paper_2412_11614_b200 as isrs
    from workloads import bj_config
    link = bj_config(a.config)
    with isrs.Engine(link) as e:
        eta_g, terms_g = e.nli(terms=True)
        torch.cuda.synchronize()
        eta_g = eta_g.cpu().numpy()
        terms_g = terms_g.cpu().numpy()
    t0 = time.perf_counter()
    # largest COIs (centre) first so the pool's tail is short
    order = sorted(range(link.n_ch), key=lambda k: abs(k - (link.n_ch - 1) / 2))
    with mp.get_context("fork").Pool(a.processes) as pool:
        res = pool.map(_oracle_coi, [(link, k) for k in order], chunksize=1)
    dt = time.perf_counter() - t0
    eta_o = np.zeros(link.n_ch)
    terms_o = np.zeros((link.n_ch, 5))
    for k, v, t in res:
        eta_o[k] = v
        terms_o[k] = t
    rel = np.abs(eta_g - eta_o) / eta_o
    trel = np.abs(terms_g - terms_o).max(axis=1) / np.abs(terms_o).sum(axis=1)
    print(json.dumps({"config": a.config, "n_coi": link.n_ch, "processes": a.processes,
                      "oracle_seconds": dt, "max_rel_eta": float(rel.max()),
                      "mean_rel_eta": float(rel.mean()), "max_rel_terms": float(trel.max()),
                      "tolerance": 1e-10, "pass": bool(rel.max() <= 1e-10 and trel.max() <= 1e-10),
                      "rel_eta": rel.tolist(), "eta_db_gpu": (10 * np.log10(eta_g)).tolist()}), flush=True)


if __name__ == "__main__":
    main()
