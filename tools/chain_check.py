"""max |eta_chained - eta_unchained| / eta for a library build (ISRS_EGN_LIB) on BASELINE configs.
usage: ISRS_EGN_LIB=build_variants/lib_x.so python tools/chain_check.py c2 c5:100"""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2412_11614_b200 as isrs
from workloads import bj_config
for arg in sys.argv[1:]:
    cfg, _, c = arg.partition(":")
    coi = [int(x) for x in c.split(",")] if c else None
    link = bj_config(cfg)
    out = []
    for fl in (0, isrs.FLAG_NO_CHAIN):
        with isrs.Engine(link, flags=fl) as e:
            out.append(e.nli(coi=coi).cpu().numpy())
            chains = e.span_chains()[0].tolist()
    rel = np.abs(out[0] - out[1]) / out[1]
    print(json.dumps({"lib": os.path.basename(isrs.library_path()), "cfg": cfg, "coi": coi,
                      "chains": chains, "max_rel": float(rel.max()), "mean_rel": float(rel.mean())}))
