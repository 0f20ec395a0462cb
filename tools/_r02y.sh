#!/bin/bash
OUT=gpurun_out/r02y; mkdir -p $OUT
python -m paper_2412_11614_b200.build > $OUT/build.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --backend gloo --steps 3 --warmup 3 --config c2 --coi all > $OUT/bench_2rank_gloo.json 2> $OUT/bench_2rank_gloo.err; echo "2rank rc=$?" >> $OUT/status
timeout 900 python - > $OUT/production_c5.json 2>&1 <<'PY'
import json, time, torch, numpy as np
import paper_2412_11614_b200 as isrs
from workloads import bj_config
link = bj_config("c5")
res = {}
for name, flags in (("dedup", isrs.FLAG_DEDUP), ("dedup+mirror", isrs.FLAG_DEDUP | isrs.FLAG_MIRROR)):
    with isrs.Engine(link, flags=flags) as e:
        e.nli(coi=[0]); torch.cuda.synchronize()
        t0 = time.perf_counter(); eta = e.nli(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
        res[name] = {"seconds_all_200_cois": dt, "channels_per_s": 200 / dt, "eta_db_0_100_199": [float(10*np.log10(eta[i].item())) for i in (0, 100, 199)]}
print(json.dumps({"config": "c5 all 200 COIs", "modes": res, "note": "production options (same eta as the headline path within 1e-10); the headline evaluates every span and region"}))
PY
echo "prod rc=$?" >> $OUT/status
