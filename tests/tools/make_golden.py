"""Write whole-eta golden files of a BASELINE config with the fast-plain oracle (oracle/fastplain.c,
pinned to the literal closed mode by tests/test_oracle_fastplain.py).  Calls only oracle/ and
workloads/: no value here comes from the CUDA path.

    python tests/tools/make_golden.py --config c5 --coi 0,100,199 [--threads 8]
    python tests/tools/make_golden.py --config c5 --coi all --out tests/golden/c5_eta_fastplain_all.json

Writes tests/golden/<config>_eta_fastplain[_<tag>].json: eta (1/W^2), the D..H contributions, the
in-support point count per COI, the SHA-256 of the link's input arrays (so a drift of the seeded
workload is detected) and how long the oracle took on how many threads.  test_parity_gpu.py compares
the CUDA path's whole eta with these at 1e-10 (BASELINE.json north_star).
"""
import argparse
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

FIELDS = ("f_center_hz", "symbol_rate_hz", "launch_power_w", "phi", "psi", "length_m", "alpha_per_m",
          "beta2_s2_per_m", "beta3_s3_per_m", "gamma_per_w_m", "cr_per_w_m_hz")


def link_hash(link):
    h = hashlib.sha256()
    for f in FIELDS:
        h.update(np.ascontiguousarray(np.asarray(getattr(link, f), dtype=np.float64)).tobytes())
    h.update(np.array([link.grid_n, link.delta_z_m], dtype=np.float64).tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True)
    ap.add_argument("--coi", default="all")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from oracle import fastplain
    from workloads import bj_config
    link = bj_config(a.config)
    coi = list(range(link.n_ch)) if a.coi == "all" else [int(x) for x in a.coi.split(",")]
    t0 = time.time()
    eta, terms, npts = fastplain.eta(link, coi=coi, threads=a.threads, progress=True)
    dt = time.time() - t0
    out = a.out or os.path.join(ROOT, "tests", "golden", f"{a.config}_eta_fastplain.json")
    doc = {"what": f"whole eta of BASELINE config {a.config} (workloads.bj_config) for the listed COIs, "
                   "by the fast-plain oracle (oracle/fastplain.c: closed mode, Eqs. 5, 8-10, 14, 22 with "
                   "reading C3, 15-21 with C2/C7/C8/C10, 11), pinned to the literal closed mode at <= 1e-12 "
                   "by tests/test_oracle_fastplain.py; written by tests/tools/make_golden.py (oracle/ only)",
           "config": a.config, "seed": link.seed, "link_sha256": link_hash(link), "grid_n": link.grid_n,
           "delta_z_m": link.delta_z_m, "coi": coi, "eta": eta.tolist(), "terms": terms.tolist(),
           "points": [int(x) for x in npts], "oracle_seconds": dt,
           "threads": a.threads or os.cpu_count(), "host": platform.processor() or platform.machine()}
    with open(out, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps({"out": os.path.relpath(out, ROOT), "seconds": round(dt, 1), "n_coi": len(coi),
                      "points": int(npts.sum()),
                      "ns_per_point_core": dt * (a.threads or os.cpu_count()) / max(1, npts.sum()) * 1e9}))


if __name__ == "__main__":
    main()
