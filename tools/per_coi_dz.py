"""Per-COI segment step (NEXT-3: "the value of dz may be adjusted flexibly depending on the
frequency of the COI ... a larger dz can be used for channels closer to the center frequency").

On the Table-I link (PA-I, C_r 1.12, QPSK, 1 span) with the GPU integral form as the reference:
for every COI pick the largest dz in {1..7} km whose segment-form error stays within a budget,
then time the whole link at uniform dz = 1 km against the per-COI plan (one handle per distinct
dz, each evaluating its COI subset — the C ABI takes a COI list per call).

    python tools/per_coi_dz.py [--budget-db 0.003] [--coi-stride 5]
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
    ap.add_argument("--budget-db", type=float, default=0.003)
    ap.add_argument("--coi-stride", type=int, default=5)
    ap.add_argument("--cr", type=float, default=1.12)
    a = ap.parse_args()
    import torch
    import paper_2412_11614_b200 as isrs
    from workloads import paper_analog
    link = paper_analog("I", n_span=1, cr_w_km_thz=a.cr, fmt="qpsk")
    coi = list(range(0, link.n_ch, a.coi_stride))

    def eta(mode, dz, c):
        with isrs.Engine(link, mu_mode=mode, delta_z_m=dz) as e:
            out = e.nli(coi=c)
            torch.cuda.synchronize()
            return out.cpu().numpy()

    def timed(dz, c):
        with isrs.Engine(link, delta_z_m=dz) as e:
            e.nli(coi=c)
            torch.cuda.synchronize()
            e.nli(coi=c)
            torch.cuda.synchronize()
            return e.last_kernel_ms()[0][3]

    ref = 10 * np.log10(eta(isrs.MU_INTEGRAL, 1000.0, coi))
    dzs = [1000.0 * k for k in range(1, 8)]
    err = {dz: 10 * np.log10(eta(isrs.MU_SEGMENT, dz, coi)) - ref for dz in dzs}
    best = []
    for i in range(len(coi)):
        ok = [dz for dz in dzs if abs(err[dz][i]) <= a.budget_db]
        best.append(max(ok) if ok else 1000.0)
    groups = {}
    for c, dz in zip(coi, best):
        groups.setdefault(dz, []).append(c)
    t_uniform = timed(1000.0, coi)
    t_plan = sum(timed(dz, cs) for dz, cs in groups.items())
    plan_err = np.array([err[dz][i] for i, dz in enumerate(best)])
    print(json.dumps({
        "config": "PA-I", "cr_w_km_thz": a.cr, "coi": coi, "budget_db": a.budget_db,
        "dz_km_per_coi": [d / 1000.0 for d in best],
        "err_db_uniform_1km": err[1000.0].tolist(), "err_db_plan": plan_err.tolist(),
        "max_abs_err_db_plan": float(np.abs(plan_err).max()),
        "ms_uniform_1km": t_uniform, "ms_per_coi_plan": t_plan,
        "time_saving_pct": 100.0 * (1.0 - t_plan / t_uniform),
        "note": "kernel time (integrand phase) per handle; each distinct dz is one handle / call"}))


if __name__ == "__main__":
    main()
