"""SCI / XCI / MCI parts of eta (ISRS_EGN_FLAG_SPLIT) for every channel of a BASELINE config.

    python tools/split_profile.py --config c5 > profiles/<tag>_split_c5.json

One JSON object: per channel eta [dB re 1/W^2] and the three shares, the integrand time of the split work
list, and the largest |eta_split - eta_unsplit| / eta when --check is given (a second, unsplit run).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_11614_b200 as isrs  # noqa: E402
from workloads import bj_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--check", action="store_true", help="also run the unsplit path and compare eta")
    a = ap.parse_args()
    link = bj_config(a.config)
    with isrs.Engine(link, flags=isrs.FLAG_SPLIT) as e:
        eta, parts = e.nli_split()
        torch.cuda.synchronize()
        ms = e.last_kernel_ms()[0][3]
        work = e.work()
    eta, parts = eta.cpu().numpy(), parts.cpu().numpy()
    out = {"config": a.config, "n_ch": int(link.n_ch), "integrand_ms": ms, "points": work[0], "point_spans": work[1],
           "regions": work[2], "parts_sum_max_rel": float(np.max(np.abs(parts.sum(axis=1) - eta) / eta)),
           "eta_db": np.round(10 * np.log10(eta), 4).tolist(),
           "share_sci": np.round(parts[:, 0] / eta, 5).tolist(),
           "share_xci": np.round(parts[:, 1] / eta, 5).tolist(),
           "share_mci": np.round(parts[:, 2] / eta, 6).tolist()}
    if a.check:
        with isrs.Engine(link) as e:
            ref = e.nli().cpu().numpy()
            out["unsplit_integrand_ms"] = e.last_kernel_ms()[0][3]
        out["eta_vs_unsplit_max_rel"] = float(np.max(np.abs(eta - ref) / ref))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
