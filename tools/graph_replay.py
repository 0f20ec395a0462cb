"""Per-call time of isrs_egn_nli issued directly vs replayed from a CUDA graph (Engine.graph()):
host + device time per call over many back-to-back calls, for launch-bound small links.

    python tools/graph_replay.py [--configs c1,c2] [--calls 200]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2")
    ap.add_argument("--calls", type=int, default=200)
    a = ap.parse_args()
    import torch
    import paper_2412_11614_b200 as isrs
    from workloads import bj_config
    for cfg in a.configs.split(","):
        link = bj_config(cfg)
        calls = a.calls if cfg == "c1" else 10
        with isrs.Engine(link) as e:
            g = e.graph()
            s = g.stream
            eta = torch.empty_like(g.eta)

            def direct():
                e.nli_into(eta.data_ptr(), 0, None, s.cuda_stream)

            def timed(fn):
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                t = time.perf_counter()
                for _ in range(calls):
                    fn()
                torch.cuda.synchronize()
                return (time.perf_counter() - t) / calls * 1e6

            with torch.cuda.stream(s):
                us_direct = timed(direct)
            us_graph = timed(g.replay)
            same = bool(torch.equal(g.eta, eta))
        print(json.dumps({"config": cfg, "calls": calls, "us_per_call_direct": us_direct,
                          "us_per_call_graph": us_graph, "eta_bitwise_equal": same}), flush=True)


if __name__ == "__main__":
    main()
