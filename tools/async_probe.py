"""Does isrs_egn_nli return to the host before the GPU finishes -- also when the COI set changes?

Issues, on one stream with no host synchronisation in between, a long call (c3, COIs 0/50/99, ~70 ms of
kernels) and then calls with OTHER COI sets (each rebuilds the work list on the host and uploads it
stream-ordered); prints the host wall time of every call, the host planner's share (isrs_egn_work on
the same set: the planner alone, no device access) and the time the stream then still needed to drain.
A call whose host time is ~ the planner's time while the drain is long returned asynchronously.

    python tools/async_probe.py [--config c3]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2412_11614_b200 as isrs  # noqa: E402
from workloads import bj_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    a = ap.parse_args()
    link = bj_config(a.config)
    with isrs.Engine(link) as e:
        n = e.n_ch
        sets = [[0, n // 2, n - 1], [1, n // 2 + 1], [2, n // 3, n - 2], [0, n // 2, n - 1]]
        st = torch.cuda.Stream()
        # warm-up: module load, pool growth, side stream / events
        for s in sets:
            e.nli(coi=s, stream=st)
        st.synchronize()
        plan_ms = []
        for s in sets:
            t0 = time.perf_counter()
            e.planned_work(s)
            plan_ms.append(1e3 * (time.perf_counter() - t0))
        outs, host_ms = [], []
        t_start = time.perf_counter()
        for s in sets:
            t0 = time.perf_counter()
            outs.append(e.nli(coi=s, stream=st))
            host_ms.append(1e3 * (time.perf_counter() - t0))
        t_issued = time.perf_counter()
        st.synchronize()
        t_done = time.perf_counter()
        # the same calls one at a time, for their GPU durations and for the values
        gpu_ms, same = [], []
        for s, o in zip(sets, outs):
            t0 = time.perf_counter()
            r = e.nli(coi=s, stream=st)
            st.synchronize()
            gpu_ms.append(1e3 * (time.perf_counter() - t0))
            same.append(bool(torch.equal(r, o)))
        print(json.dumps({
            "config": a.config, "coi_sets": sets,
            "host_ms_per_call_back_to_back": [round(x, 3) for x in host_ms],
            "planner_only_ms": [round(x, 3) for x in plan_ms],
            "issue_all_ms": round(1e3 * (t_issued - t_start), 3),
            "drain_after_issue_ms": round(1e3 * (t_done - t_issued), 3),
            "each_call_alone_incl_sync_ms": [round(x, 3) for x in gpu_ms],
            "bitwise_equal_to_synchronised_calls": same,
        }))


if __name__ == "__main__":
    main()
