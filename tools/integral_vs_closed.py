"""NEXT-2 measurement: the paper's integral-form FWM factor (Eq. 23 by quadrature) against the
segment closed form (Eqs. 8-10) on the same B200, same grid and COIs (paper Figs. 8-10, P:181:
"computation time reduction ranging from 97.0% to 98.3%").

    python tools/integral_vs_closed.py [--config PA-I] [--coi 0,25,50] [--cr 1.12]

Prints one JSON line: per-COI eta (dB) of both forms, the segment error vs the integral form
(the paper's accuracy claim, MAE < 0.001 dB), and both kernel times and the time reduction.
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
    ap.add_argument("--config", default="PA-I")
    ap.add_argument("--coi", default="0,25,50")
    ap.add_argument("--cr", type=float, default=1.12)
    ap.add_argument("--fmt", default="qpsk")
    ap.add_argument("--spans", type=int, default=1)
    a = ap.parse_args()
    import torch
    import paper_2412_11614_b200 as isrs
    from workloads import bj_config, paper_analog
    if a.config.startswith("PA-"):
        link = paper_analog(a.config[3:], n_span=a.spans, cr_w_km_thz=a.cr, fmt=a.fmt)
    else:
        link = bj_config(a.config)
    coi = [int(x) for x in a.coi.split(",")]
    res = {"config": link.name, "n_ch": link.n_ch, "n_span": link.n_span, "grid_n": link.grid_n,
           "coi": coi, "cr_w_km_thz": a.cr}
    out = {}
    for name, mode in (("integral", isrs.MU_INTEGRAL), ("segment", isrs.MU_SEGMENT)):
        with isrs.Engine(link, mu_mode=mode) as e:
            e.nli(coi=coi)
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            eta = e.nli(coi=coi)
            ev1.record()
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1)
            kms, kps = e.last_kernel_ms()
            out[name] = (eta.cpu().numpy(), ms, kps[2])
    ei, ti, ps = out["integral"]
    es, ts, _ = out["segment"]
    err = 10 * np.log10(es) - 10 * np.log10(ei)
    res.update({"eta_db_integral": (10 * np.log10(ei)).tolist(), "eta_db_segment": (10 * np.log10(es)).tolist(),
                "segment_minus_integral_db": err.tolist(), "mae_db": float(np.abs(err).mean()),
                "ms_integral": ti, "ms_segment": ts, "speedup": ti / ts,
                "time_reduction_pct": 100.0 * (1.0 - ts / ti), "point_spans": ps,
                "paper": "97.0-98.3 % reduction, MAE < 0.001 dB (MATLAB, 16-worker CPU pool)"})
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
