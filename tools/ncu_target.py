"""Small ncu target: `reps` nli() calls over one BASELINE config (optionally a COI subset).

    python tools/ncu_target.py [--config c2] [--coi 0,19,39] [--reps 2]

Profile with e.g. `ncu --set full -k regex:integrand_kernel -s 2 -c 1 python tools/ncu_target.py`
(the first call's launches are warm-up).  Prints the kernel times of the last call.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--coi", default=None)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--precision", type=int, default=64)
    ap.add_argument("--f-samples", type=int, default=0)
    a = ap.parse_args()
    import torch
    import paper_2412_11614_b200 as isrs
    from workloads import bj_config
    link = bj_config(a.config)
    coi = [int(x) for x in a.coi.split(",")] if a.coi else None
    with isrs.Engine(link, precision=a.precision, f_samples=a.f_samples) as e:
        for _ in range(a.reps):
            eta = e.nli(coi=coi)
        torch.cuda.synchronize()
        ms, ps = e.last_kernel_ms()
        print(json.dumps({"config": a.config, "kernel_ms": ms, "point_spans": ps,
                          "eta0": float(eta[0].item())}))


if __name__ == "__main__":
    main()
