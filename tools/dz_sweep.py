"""Delta-z study on the GPU path (NEXT-3; paper Fig. 11): for each segment step dz,
the integrand kernel time and eta per COI, and the eta change against a fine-step reference.

    python tools/dz_sweep.py [--config c2] [--dz 500,1000,2000,...] [--ref 125] [--coi 0,19,39]

Prints one JSON line per dz: K per span, kernel ms (D-only, coherent), point-spans/s, and
max/mean |eta(dz) - eta(ref)| in dB over the COIs.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--dz", default="500,1000,2000,3000,4000,5000,6000,7000")
    ap.add_argument("--ref", type=float, default=125.0)
    ap.add_argument("--coi", default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--precision", type=int, default=64)
    a = ap.parse_args()
    import torch
    import paper_2412_11614_b200 as isrs
    from workloads import bj_config
    link = bj_config(a.config)
    coi = [int(x) for x in a.coi.split(",")] if a.coi else None

    def run(dz):
        with isrs.Engine(link, delta_z_m=dz, precision=a.precision) as e:
            e.nli(coi=coi)
            torch.cuda.synchronize()
            ms = []
            for _ in range(a.reps):
                eta = e.nli(coi=coi)
                ms.append(e.last_kernel_ms())
            eta = eta.cpu().numpy()
            k = e.span_chains()[1]
        kd = float(np.median([m[0][0] for m in ms]))
        kc = float(np.median([m[0][1] for m in ms]))
        kph = float(np.median([m[0][3] for m in ms]))
        ps = ms[-1][1][2]
        return eta, k, kd, kc, ps, kph

    ref = run(a.ref)[0]
    for dz in [float(x) for x in a.dz.split(",")]:
        eta, k, kd, kc, ps, kph = run(dz)
        d = np.abs(10 * np.log10(eta) - 10 * np.log10(ref))
        print(json.dumps({"config": a.config, "dz_m": dz, "K": int(k[0]), "integrand_D_ms": kd,
                          "integrand_coh_ms": kc, "integrand_phase_ms": kph, "point_spans_per_s": ps / (kph * 1e-3),
                          "ref_dz_m": a.ref, "max_abs_db_vs_ref": float(d.max()),
                          "mean_abs_db_vs_ref": float(d.mean()), "precision": a.precision}), flush=True)


if __name__ == "__main__":
    main()
