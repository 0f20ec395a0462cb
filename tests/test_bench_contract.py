"""bench.py contract on the CPU: the reference arm (the oracle, the only bench leg that runs without a
GPU) prints one JSON line with the driver's keys, and the product arm fails loudly (non-zero exit, no
JSON line) when no GPU is present instead of falling back to a CPU path."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout, env=env)


def test_reference_arm_prints_one_contract_line():
    r = _run(["--impl", "reference", "--config", "c1", "--coi", "0,2", "--steps", "1", "--warmup", "1",
              "--ref-seconds", "0.5"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"].startswith("c1") and "COIs 0,2" in d["config"]["workload"]
    assert d["config"]["coi"] == [0, 2] and "COIs [0, 2]" in d["cpu_baseline"]["sample"]


def test_product_arm_fails_loudly_without_gpu():
    pytest.importorskip("torch")
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = _run(["--steps", "1", "--warmup", "1", "--no-cpu", "--no-e2e", "--no-dedup"])
    assert r.returncode != 0
    assert not [l for l in r.stdout.splitlines() if l.strip().startswith("{")]


def test_roofline_unit_counts():
    # a chain of G spans with K segments (K_p = K rounded up to even) costs
    # 3 (G K_p - 1) + 40 flops and 2 (G K_p - 1) + 25 FP64 slots per point
    sys.path.insert(0, ROOT)
    import bench
    assert bench.algorithmic_work_per_point([10], [80] * 10) == (3 * 799 + 40, 2 * 799 + 25)
    # odd K pads to even; unchained spans count one chain each
    assert bench.algorithmic_work_per_point([1, 1], [73, 81]) == (3 * 73 + 40 + 3 * 81 + 40,
                                                                  2 * 73 + 25 + 2 * 81 + 25)
    # chain groups (c5: 5 chains of 10 spans, one group): one 40-flop epilogue + 4 Horner steps of 8
    assert bench.algorithmic_work_per_point([10] * 5, [80] * 50, [0, 5]) == (5 * 3 * 799 + 40 + 4 * 8,
                                                                             5 * 2 * 799 + 25 + 4 * 4)


@pytest.mark.parametrize("cfg", ["c2", "c5"])
def test_traffic_source_is_the_newest_capture_of_the_config(cfg):
    sys.path.insert(0, ROOT)
    import glob
    import bench
    traffic, src = bench.ncu_traffic(cfg)
    import re
    caps = [os.path.basename(f).split("_")[0] for f in glob.glob(os.path.join(ROOT, "profiles", f"*ncu_integrand*_{cfg}*.json"))
            if "fp32" not in f]

    def key(t):
        m = re.match(r"r(\d+)([a-z]+)$", t)
        return (int(m.group(1)), len(m.group(2)), m.group(2))
    newest = max(caps, key=key)
    assert src is not None and os.path.basename(src).startswith(newest + "_") and traffic > 0


def test_default_workload_is_the_north_star_subset():
    """The headline is c5 (the 20 THz / 50-span north-star link) on SURVEY 8(d)'s COI subset."""
    sys.path.insert(0, ROOT)
    import bench
    from workloads import bj_config
    assert bench.parse_coi("default", bj_config("c5")) == [0, 100, 199]
    assert bench.parse_coi("default", bj_config("c2")) is None
    assert bench.parse_coi("all", bj_config("c5")) is None
    assert bench.parse_coi("3,1", bj_config("c5")) == [3, 1]
