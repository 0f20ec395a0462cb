"""Whole-eta parity of the CUDA path against the oracle for EVERY COI of a BASELINE config (the
GPU tests sample regions at full size; this runs the complete oracle, closed mode, on the host's
cores — c2 takes ~20 min on 16 cores).

    python tests/tools/full_parity.py [--config c2] [--coi 0,50,99] [--processes N]

Prints one JSON line: per-COI relative error, max, and the oracle wall time.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def _canon(link):
    from oracle import egn
    return egn.canonicalize(link)


def _oracle_coi_k1(args):
    """The oracle's sum over the regions (kappa, k1, *) of one COI: egn.eta's loop body for one k1
    (same functions, same order within the k1 row), weighted per Eq. 15 / C2."""
    from oracle import egn
    link, kappa, k1 = args
    c = egn.canonicalize(link)
    acc = np.zeros(5)
    for k2 in range(c.f.size):
        if not egn.has_support_bound(c, kappa, k1, k2):
            continue
        for isl in egn.region_islands(c, kappa, k1, k2, "closed", egn._needed_terms(c, k1, k2)):
            acc = acc + egn.island_contributions(c, k1, k2, isl)
    return kappa, acc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--processes", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--coi", default=None, help="comma-separated COI subset (default: all channels)")
    a = ap.parse_args()
    import multiprocessing as mp
    import torch
    import paper_2412_11614_b200 as isrs
    from workloads import bj_config
    link = bj_config(a.config)
    cois = list(range(link.n_ch)) if a.coi is None else [int(x) for x in a.coi.split(",")]
    with isrs.Engine(link) as e:
        eta_g, terms_g = e.nli(coi=cois, terms=True)
        torch.cuda.synchronize()
        eta_g = eta_g.cpu().numpy()
        terms_g = terms_g.cpu().numpy()
    t0 = time.perf_counter()
    # one task per (COI, kappa1): the oracle's regions of a COI split over the pool
    tasks = [(link, k, k1) for k in cois for k1 in range(link.n_ch)]
    with mp.get_context("fork").Pool(a.processes) as pool:
        res = pool.map(_oracle_coi_k1, tasks, chunksize=1)
    dt = time.perf_counter() - t0
    acc = {k: np.zeros(5) for k in cois}
    for k, part in res:
        acc[k] = acc[k] + part
    c = _canon(link)
    eta_o = np.array([acc[k].sum() * c.R[k] / c.P[k] ** 3 for k in cois])
    terms_o = np.array([acc[k] * c.R[k] / c.P[k] ** 3 for k in cois])
    rel = np.abs(eta_g - eta_o) / eta_o
    trel = np.abs(terms_g - terms_o).max(axis=1) / np.abs(terms_o).sum(axis=1)
    print(json.dumps({"config": a.config, "coi": cois, "n_coi": len(cois), "processes": a.processes,
                      "oracle_seconds": dt, "max_rel_eta": float(rel.max()),
                      "mean_rel_eta": float(rel.mean()), "max_rel_terms": float(trel.max()),
                      "tolerance": 1e-10, "pass": bool(rel.max() <= 1e-10 and trel.max() <= 1e-10),
                      "rel_eta": rel.tolist(), "eta_db_gpu": (10 * np.log10(eta_g)).tolist()}), flush=True)


if __name__ == "__main__":
    main()
