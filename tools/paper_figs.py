"""The paper's accuracy / time experiments (Figs. 8-11) on B200 with the GPU path.

For the Table-I link (PA-I: 101 x 10 GBd, 19 dBm, 100 km spans, QPSK) at C_r in {0.28, 1.12} and
1 or 10 spans, on COIs {0, 25, 50} (the paper's -50, -25, 0): eta from the integral form (Eq. 23,
NEXT-2, the reference), the segment closed form at dz = 1..7 km and the Maclaurin closed form (Eq. 4);
per method the per-COI error vs the integral form in dB, the MAE, and the integrand time.

    python tools/paper_figs.py [--spans 1,10] [--cr 0.28,1.12] [--dz 1,2,3,4,5,6,7] [--coi 0,25,50]

One JSON line per (C_r, spans, method, dz).
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
    ap.add_argument("--spans", default="1,10")
    ap.add_argument("--cr", default="0.28,1.12")
    ap.add_argument("--dz", default="1,2,3,4,5,6,7")
    ap.add_argument("--coi", default="0,25,50")
    ap.add_argument("--fmt", default="qpsk")
    a = ap.parse_args()
    import torch
    import paper_2412_11614_b200 as isrs
    from workloads import paper_analog
    coi = [int(x) for x in a.coi.split(",")]

    def run(link, mode, dz_m):
        with isrs.Engine(link, mu_mode=mode, delta_z_m=dz_m) as e:
            e.nli(coi=coi)
            torch.cuda.synchronize()
            eta = e.nli(coi=coi)
            torch.cuda.synchronize()
            kms, kps = e.last_kernel_ms()
            return eta.cpu().numpy(), kms[3], kps[2]

    for cr in [float(x) for x in a.cr.split(",")]:
        for ns in [int(x) for x in a.spans.split(",")]:
            link = paper_analog("I", n_span=ns, cr_w_km_thz=cr, fmt=a.fmt)
            ref, t_ref, ps = run(link, isrs.MU_INTEGRAL, 1000.0)
            base = {"config": "PA-I", "cr_w_km_thz": cr, "n_span": ns, "coi": coi, "point_spans": ps,
                    "eta_db_integral": (10 * np.log10(ref)).tolist(), "ms_integral": t_ref}
            cases = [("maclaurin", isrs.MU_MACLAURIN, 1000.0)] + \
                    [("segment", isrs.MU_SEGMENT, 1000.0 * float(d)) for d in a.dz.split(",")]
            for name, mode, dz in cases:
                eta, t, _ = run(link, mode, dz)
                err = 10 * np.log10(eta) - 10 * np.log10(ref)
                line = dict(base, method=name, dz_km=dz / 1000.0 if name == "segment" else None,
                            err_db=err.tolist(), mae_db=float(np.abs(err).mean()), ms=t,
                            time_reduction_pct=100.0 * (1.0 - t / t_ref))
                print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
