"""Time the NEXT-4a dedup mode (ISRS_EGN_FLAG_DEDUP, optionally | MIRROR) on one config with the library
ISRS_EGN_LIB points at; prints one JSON line (integrand-phase ms, eta of the first COI).

    ISRS_EGN_LIB=<lib> python tools/dedup_time.py --config c5 [--coi 0,100,199] [--mirror] [--reps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--coi", default=None)
    ap.add_argument("--mirror", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_2412_11614_b200 as isrs
    from workloads import bj_config
    link = bj_config(a.config)
    coi = [int(x) for x in a.coi.split(",")] if a.coi else None
    flags = isrs.FLAG_DEDUP | (isrs.FLAG_MIRROR if a.mirror else 0)
    with isrs.Engine(link, flags=flags) as e:
        e.nli(coi=coi)
        torch.cuda.synchronize()
        ms = []
        for _ in range(a.reps):
            eta = e.nli(coi=coi)
            torch.cuda.synchronize()
            ms.append(e.last_kernel_ms()[0][3])
        eta = eta.cpu().numpy()
    print(json.dumps({"lib": os.path.basename(os.environ.get("ISRS_EGN_LIB", "tree")), "config": a.config,
                      "coi": a.coi or "all", "mirror": a.mirror, "phase_ms": float(np.median(ms)),
                      "eta": [float(eta[0]), float(eta[-1])]}))


if __name__ == "__main__":
    main()
