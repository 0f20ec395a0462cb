"""Whole-eta parity of the CUDA path against every golden file (tests/golden/c*_eta_fastplain*.json,
written by make_golden.py from the fast-plain oracle): one JSON line per file with the observed
errors, for profiles/ (the -m gpu test asserts the same at 1e-10).

    python tests/tools/golden_parity.py
"""
import glob
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)


def main():
    import torch
    import paper_2412_11614_b200 as isrs
    from make_golden import link_hash
    from workloads import bj_config
    for fn in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "c*_eta_fastplain*.json"))):
        with open(fn) as fh:
            g = json.load(fh)
        link = bj_config(g["config"])
        ok_hash = link_hash(link) == g["link_sha256"]
        e_o, t_o = np.array(g["eta"]), np.array(g["terms"])
        with isrs.Engine(link) as e:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            eta, terms = e.nli(coi=g["coi"], terms=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            eta, terms = eta.cpu().numpy(), terms.cpu().numpy()
            pts = e.work()[0]
        rel = np.abs(eta - e_o) / e_o
        trel = np.abs(terms - t_o).max(axis=1) / np.abs(t_o).sum(axis=1)
        print(json.dumps({"golden": os.path.basename(fn), "config": g["config"], "n_coi": len(e_o),
                          "link_hash_ok": ok_hash, "points_equal": pts == int(sum(g["points"])),
                          "max_rel_eta": float(rel.max()), "mean_rel_eta": float(rel.mean()),
                          "argmax_coi": int(g["coi"][int(np.argmax(rel))]), "max_rel_terms": float(trel.max()),
                          "tolerance": 1e-10, "pass": bool(ok_hash and rel.max() <= 1e-10 and trel.max() <= 1e-10),
                          "gpu_seconds": dt, "oracle_seconds": g["oracle_seconds"],
                          "oracle_threads": g["threads"]}), flush=True)


if __name__ == "__main__":
    main()
