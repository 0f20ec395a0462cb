"""Summarise an ncu --set full capture (and optionally its launch list) for profiles/.

    python tools/ncu_summary.py gpurun_out/<tag>/prof.ncu-rep [--capture NAME] [--out profiles/x.json]

Prints / writes: kernel, duration, FP64 pipe utilisation, executed DP flop rate, issue activity,
occupancy, DRAM traffic (the roofline `traffic`), registers, the stall-reason mix and the
per-source-line sample shares of the top lines.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ms",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_inst_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_inst_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_inst_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__warps_eligible.avg.per_cycle_active": "eligible_warps_per_cycle",
    "launch__registers_per_thread": "registers",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__cycles_elapsed.avg": "sm_cycles",
    "smsp__cycles_elapsed.avg.per_second": "smsp_clock_hz",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed": "dfma_per_cycle",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed": "dadd_per_cycle",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed": "dmul_per_cycle",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
}


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    h, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
             "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    out = []
    for v in rows[2:]:
        d = dict(zip(h, v))
        rec = {"kernel": d.get("Kernel Name")}
        for k, name in KEYS.items():
            if k in d:
                try:
                    rec[name] = float(d[k].replace(",", "")) * scale.get(units.get(k, ""), 1.0)
                except ValueError:
                    rec[name] = d[k]
        stalls = {k.split("smsp__pcsamp_warps_issue_stalled_")[1]: float(d[k].replace(",", ""))
                  for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued") and d[k] not in ("", "n/a")}
        tot = sum(stalls.values()) or 1.0
        rec["stall_share"] = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])
                              if v / tot >= 0.005}
        if "dfma_per_cycle" in rec:
            # executed DP flop per SM cycle (sum over SMSPs -> per SM via /n_sm is not needed:
            # the .sum is over all SMSPs of the GPU)
            fl = 2 * rec["dfma_per_cycle"] + rec.get("dadd_per_cycle", 0) + rec.get("dmul_per_cycle", 0)
            rec["dp_flop_per_cycle_gpu"] = fl
            rec["dp_flop_frac_of_peak"] = fl / (148 * 64 * 2)
        if "dram_read_bytes" in rec:
            rec["dram_traffic_bytes"] = rec["dram_read_bytes"] + rec.get("dram_write_bytes", 0)
        out.append(rec)
    return out


def source_lines(rep, top=25):
    txt = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass")
    agg, src, fname, cur = {}, {}, None, None
    for r in csv.reader(io.StringIO(txt)):
        if len(r) == 2 and r[0] in ("File Path", "File Name"):
            fname = r[1].split("/")[-1]
            continue
        if len(r) < 8:
            continue
        if r[0]:
            try:
                cur = (fname, int(r[0]))
                src[cur] = r[1].strip()
            except ValueError:
                pass
            continue
        if r[2] == "...":
            continue
        try:
            s, i = int(r[6]), int(r[7])
        except ValueError:
            continue
        a = agg.setdefault(cur, [0, 0])
        a[0] += s
        a[1] += i
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    best = sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]
    return [{"line": f"{k[0]}:{k[1]}", "samples_pct": round(100 * v[0] / ts, 2),
             "instr_pct": round(100 * v[1] / ti, 2), "src": src.get(k, "")[:100]} for k, v in best]


def main():
    rep = sys.argv[1]
    cap = None
    out = None
    if "--capture" in sys.argv:
        cap = sys.argv[sys.argv.index("--capture") + 1]
    if "--out" in sys.argv:
        out = sys.argv[sys.argv.index("--out") + 1]
    res = {"capture": cap or rep, "kernels": raw(rep)}
    try:
        res["top_source_lines"] = source_lines(rep)
    except Exception as e:  # source page needs -lineinfo
        res["top_source_lines"] = str(e)
    js = json.dumps(res, indent=1)
    if out:
        with open(out, "w") as fh:
            fh.write(js + "\n")
    print(js)


if __name__ == "__main__":
    main()
