"""Time the D-only integrand kernel of c2 (and optionally other configs) for each library variant.
usage: python tools/perf_variants.py build_variants/lib_*.so [--config c2] [--coi 0,19,39]"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_2412_11614_b200 as isrs
from workloads import bj_config
link = bj_config(CFG)
coi = COI
e = isrs.Engine(link, precision=PREC)
for _ in range(2): e.nli(coi=coi)
torch.cuda.synchronize()
ms = []
for _ in range(REPS):
    e.nli(coi=coi); torch.cuda.synchronize(); ms.append(e.last_kernel_ms())
eta = e.nli(coi=coi).cpu().numpy()
d = float(np.median([m[0][0] for m in ms])); c = float(np.median([m[0][1] for m in ms]))
ph = float(np.median([m[0][3] for m in ms])) if len(ms[0][0]) > 3 else d + c
ps = ms[-1][1]
print(json.dumps({"phase_ms": ph, "D_ms": d, "coh_ms": c, "ps_D": ps[0], "ps_all": ps[2], "rate_D": ps[0] / d * 1e3,
                  "eta0": float(eta[0])}))
'''
args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = "c2"; coi = None; reps = 3; prec = 64
for a in sys.argv[1:]:
    if a.startswith("--config="): cfg = a.split("=")[1]
    if a.startswith("--coi="): coi = [int(x) for x in a.split("=")[1].split(",")]
    if a.startswith("--reps="): reps = int(a.split("=")[1])
    if a.startswith("--precision="): prec = int(a.split("=")[1])
for lib in args:
    code = CHILD.replace("ROOT", repr(ROOT)).replace("CFG", repr(cfg)).replace("COI", repr(coi)).replace("REPS", str(reps)).replace("PREC", str(prec))
    env = dict(os.environ, ISRS_EGN_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    out = r.stdout.strip().splitlines()
    print(os.path.basename(lib), cfg, out[-1] if out else r.stderr[-500:], flush=True)
