#!/usr/bin/env python
"""Benchmark of the ISRS EGN hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One step = one pass of the whole hot path (rows a2-a7: the nli() call: integrand kernels over
every region of every requested COI + per-COI assembly), inputs resident in HBM.  The default
workload is BASELINE.json configs[4] (c5: S+C+L 20 THz, 200 x 96 GBd, 50 x 80 km, N = 256 -- the
north-star link) on the COI subset {0, 100, 199} that SURVEY.md 8(d) prescribes for c3-c5
(lowest, centre, highest channel; ~2.5 s per step); `--config c2 --coi all` is round 1's
C-band headline, and c2 (all COIs) and c4 ({0, 40, 79}) are timed as extra keys.  At N GPUs
(torchrun, one process per GPU) the canonical region list is split into N cost-balanced
contiguous shards; each rank evaluates its shard, the per-COI sums (n_ch x 6 fp64) are
all-gathered over NCCL and combined in fixed rank order: strong scaling of one
link, the same eta on every rank.

Prints ONE JSON line (rank 0).  value = integrand point-spans/s over all ranks; the other parts
of the BASELINE metric (channels/s, % of FP64 peak) are extra keys and in `roofline`.
`--impl reference` times the oracle (oracle/, numpy fp64, the plain CPU reference) on a bounded
sample of the same workload on this host's cores.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "integrand point-spans/sec and NLI-eta channels/sec (fp64), % of FP64 peak"
UNIT = "point-spans/s"
# FP64 peak derived from unit counts and clocks (B200_PROFILING.md: 148 SMs, 1965 MHz max SM
# clock; 64 FP64 FMA lanes per SM): 148 * 64 * 2 * 1.965e9 = 37.2 TFLOP/s.
SMS, FP64_LANES, SM_MAX_MHZ = 148, 64, 1965.0


def fp64_peak_tflops(mhz=SM_MAX_MHZ):
    return SMS * FP64_LANES * 2 * mhz * 1e6 / 1e12


def algorithmic_work_per_point(chain_g, k_s, grp_c0=None):
    """Algorithmic FP64 work per grid point summed over the link, given the span
    chains (reading R9): a chain of G spans with K segments (K_p = K rounded up to even) runs
    one second-order recurrence over G*K_p segments, 1 DFMA + 1 DADD each = 3 flops / 2 FP64
    pipe slots (the first step is a bare add: -3 / -2); each chain GROUP (grp_c0: bounds of runs of
    chains of identical spans; default one chain per group) adds 40 flops / 25 slots of arithmetic
    (chi, 2cos, I_0, mu, Y accumulation, phase advance) and each chain after a group's first one 8
    flops / 4 slots (its complex Horner step); the sincospi and reciprocal seeds are not counted.
    Returns (flops, fp64 pipe slots)."""
    starts = [0]
    for g in chain_g:
        starts.append(starts[-1] + int(g))
    if grp_c0 is None:
        grp_c0 = list(range(len(chain_g) + 1))
    flops = slots = 0.0
    for gi in range(len(grp_c0) - 1):
        c0, c1 = int(grp_c0[gi]), int(grp_c0[gi + 1])
        flops += 40 + 8 * (c1 - c0 - 1)
        slots += 25 + 4 * (c1 - c0 - 1)
        for c in range(c0, c1):
            kp = 2 * ((int(k_s[starts[c]]) + 1) // 2)
            flops += 3 * (int(chain_g[c]) * kp - 1)
            slots += 2 * (int(chain_g[c]) * kp - 1)
    return flops, slots


DEFAULT_COI = {"c3": [0, 50, 99], "c4": [0, 40, 79], "c5": [0, 100, 199]}


def parse_coi(spec, link):
    """--coi: 'all' -> None (every channel), 'default' -> SURVEY 8(d)'s {0, n/2, n-1} subset for
    c3-c5 (all channels for c1, c2), else a comma-separated list."""
    if spec == "all":
        return None
    if spec == "default":
        return DEFAULT_COI.get(link.name)
    return [int(x) for x in spec.split(",")]


def ncu_traffic(config="c5"):
    """DRAM bytes (read + write) per launch of the D-only integrand kernel from the newest committed
    `ncu --set full` summary of `config` under profiles/ (tools/ncu_summary.py), or (None, None)."""
    import glob
    best = None
    def order(fn):            # r01a < ... < r01z < r01aa < ... < r02a < ...: by round, suffix length, suffix
        import re
        tag = os.path.basename(fn).split("_")[0]
        m = re.match(r"r(\d+)([a-z]+)$", tag)
        return (int(m.group(1)), len(m.group(2)), m.group(2)) if m else (0, len(tag), tag)

    for fn in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_integrand*.json")), key=order):
        if "fp32" in fn or f"_{config}" not in fn:   # the bench config's capture only
            continue
        try:
            with open(fn) as fh:
                d = json.load(fh)
            for k in (d.get("kernels", []) if isinstance(d, dict) else []):
                kn = k.get("kernel") or ""
                if ("integrand_kernel<0, 0>" in kn or "integrand_kernel<0, 7>" in kn) and "dram_traffic_bytes" in k:
                    best = (float(k["dram_traffic_bytes"]), os.path.relpath(fn, ROOT))
        except (OSError, ValueError):
            continue
    return best if best else (None, None)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = []
        pw = []
        reasons = set()
        smax = None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax = float(r[1])
            except (ValueError, IndexError):
                continue
            try:
                pw.append(float(r[2]))
            except (ValueError, IndexError):
                pass
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": float(np.median(pw)) if pw else None}


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours":
        import torch
        ndev = torch.cuda.device_count()
        if ndev and local >= ndev:
            # more ranks than GPUs (functional test of the multi-rank path only; the driver runs
            # one rank per GPU): ranks share devices round-robin
            local = local % ndev
        if ndev:
            torch.cuda.set_device(local)     # before NCCL init: barriers / comms bind to this GPU
    if ws > 1:
        import torch.distributed as dist
        backend = args.backend or ("nccl" if args.impl == "ours" else "gloo")
        if backend == "nccl":
            import torch
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return ws, rank, local


def _oracle_region(args):
    """One region of the oracle (closed mode, literal Eqs. 8-10): point-spans it covered."""
    from oracle import egn
    link, reg = args
    _, npts = egn.region_partials(link, *reg)
    return npts * link.n_span


def oracle_regions(link, coi=None):
    """Canonical (kappa, k1, k2) regions with support of the requested COIs (all channels when
    None), in canonical order (COI, k1, k2); the CPU sample is a stride through them so it covers
    short edge regions and long centre ones of every COI."""
    from oracle import egn
    c = egn.canonicalize(link)
    cois = list(range(link.n_ch)) if coi is None else list(coi)
    return [(k, k1, k2) for k in cois for k1 in range(link.n_ch) for k2 in range(link.n_ch)
            if egn.has_support_bound(c, k, k1, k2)]


def oracle_sample(link, seconds_target, coi=None, cores=None):
    """Time the oracle as it stands (numpy fp64, closed mode) on a bounded sample of the
    workload's regions, one process per host core.  Returns (point-spans/s, point-spans,
    seconds, cores, sample description)."""
    import multiprocessing as mp
    cores = cores or os.cpu_count() or 1
    regs = oracle_regions(link, coi)
    t0 = time.perf_counter()
    _oracle_region((link, regs[len(regs) // 2]))           # calibrate: one mid-list region
    t1 = max(time.perf_counter() - t0, 1e-3)
    m = int(min(len(regs), max(cores, round(seconds_target * cores / t1))))
    stride = max(1, len(regs) // m)
    sample = regs[::stride][:m]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        t0 = time.perf_counter()
        pspans = sum(pool.map(_oracle_region, [(link, r) for r in sample], chunksize=1))
        dt = time.perf_counter() - t0
    which = "every COI" if coi is None else f"COIs {list(coi)}"
    desc = (f"oracle closed mode (numpy fp64, {cores} processes) on {len(sample)} of the {len(regs)} "
            f"regions of {which} of {link.name} (every {stride}th, canonical order)")
    return pspans / dt, pspans, dt, cores, desc


def run_reference(args, link, coi, ws, rank):
    if rank != 0:
        return
    steps, warm = args.steps, args.warmup
    per_step = []
    pspans_tot = 0
    for i in range(warm + steps):
        rate, ps, dt, cores, desc = oracle_sample(link, args.ref_seconds, coi)
        if i >= warm:
            per_step.append(dt)
            pspans_tot += ps
    value = pspans_tot / sum(per_step)
    cfg = config_desc(link, coi, args)
    cfg["workload"] += "; each step a bounded region sample of it (see cpu_baseline.sample)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": steps, "warmup": warm, "ms_per_step": 1e3 * float(np.mean(per_step)),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": dict(cfg, l2="n/a (host CPU oracle)",
                           parallelism=f"{cores} host processes (oracle, closed mode)"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": desc + " per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def coi_text(link, coi):
    return "all channels as COI" if coi is None else f"COIs {','.join(str(c) for c in coi)}"


def config_desc(link, coi, args):
    return {"workload": f"{link.name}: {link.n_ch} ch x {int(link.symbol_rate_hz[0] / 1e9)} GBd, "
                        f"{link.n_span} spans, N={link.grid_n}, dz={link.delta_z_m:g} m, {coi_text(link, coi)}",
            "n_ch": link.n_ch, "n_span": link.n_span, "grid_n": link.grid_n,
            "n_coi": link.n_ch if coi is None else len(coi), "coi": "all" if coi is None else list(coi),
            "seed": link.seed,
            "l2": "flushed between timed steps (256 MiB write, outside the step events)",
            "parallelism": (f"region shards x{args.gpus} (cost-balanced contiguous shards of one link, "
                            f"{(args.backend or 'nccl').upper()} all-gather of per-COI sums, fixed-order combine; "
                            "strong scaling)"
                            if args.gpus > 1 else "1 GPU")}


def roofline_of(eng, link, kern_ms, precision):
    """Roofline of the dominant kernel: the integrand phase (D-only launch + the concurrent coherent
    launch on the library's side stream, fork to join; CUDA events inside the library, on the
    launching streams), algorithmic flops per point-span x point-spans / time."""
    ki_ms = float(np.mean([k[0][3] for k in kern_ms]))
    ps_i = kern_ms[-1][1][2]
    chain_g, k_s = eng.span_chains()
    grp_c0 = eng.chain_groups() if precision == 64 else None
    fpp, spp = (v / link.n_span for v in algorithmic_work_per_point(chain_g, k_s, grp_c0))  # per point-span
    ach = ps_i * fpp / (ki_ms * 1e-3) / 1e12
    # fp64: 64 FP64 FMA lanes per SM; the mixed fp32 variant (a8) runs its recurrence on the
    # 128 FP32 FMA lanes per SM, so its roofline takes the FP32 peak (2x)
    peak = fp64_peak_tflops() * (2.0 if precision == 32 else 1.0)
    slots_ach = ps_i * spp / (ki_ms * 1e-3) / 1e12
    slots_peak = SMS * FP64_LANES * SM_MAX_MHZ * 1e6 / 1e12
    return dict(ki_ms=ki_ms, ps_i=ps_i, chain_g=chain_g, k_s=k_s, grp_c0=grp_c0, fpp=fpp, spp=spp, ach=ach, peak=peak,
                slots_ach=slots_ach, slots_peak=slots_peak)


def time_steps(eng, step, stream, flush, steps, warmup, barrier=None, clocks=None):
    """W untimed warm-up steps, then `steps` steps each bracketed by CUDA events on `stream` (the
    L2 flush sits outside the events); returns (ms per step list, library kernel times list, clocks)."""
    import torch
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            flush.zero_()
            step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    kern_ms = []
    if barrier:
        barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
        time.sleep(0.3)
    with torch.cuda.stream(stream):
        for k in range(steps):
            flush.zero_()
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
            kern_ms.append(eng.last_kernel_ms())          # events inside the library, same stream
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    if barrier:
        barrier()
    return [a.elapsed_time(b) for a, b in ev], kern_ms, clk


def e2e_host(isrs, link, coi, device, precision, reps):
    """End to end through the public API with HOST buffers (isrs_egn_eta_host: validate + region
    plan + H2D + precompute + nli + D2H + free), wall clock, one warm-up call; returns seconds."""
    isrs.eta_host(link, coi=coi, device=device, precision=precision)
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        isrs.eta_host(link, coi=coi, device=device, precision=precision)
        t.append(time.perf_counter() - t0)
    return t


def extra_config(isrs, name, spec, args, local, stream, flush):
    """One more BASELINE config timed like the headline (fewer steps) and reported as an extra key."""
    import torch
    from workloads import bj_config
    link = bj_config(name)
    coi = parse_coi(spec, link)
    n = link.n_ch if coi is None else len(coi)
    dev = torch.device("cuda", local)
    eta = torch.empty(n, dtype=torch.float64, device=dev)
    with isrs.Engine(link, device=local, precision=args.precision) as eng:
        cp = coi

        def step():
            eng.nli_into(eta.data_ptr(), 0, cp, stream.cuda_stream)
        step_ms, kern_ms, _ = time_steps(eng, step, stream, flush, 5, 3)
        pts, pspans, nreg = eng.work()
        rf = roofline_of(eng, link, kern_ms, args.precision)
    ms = float(np.mean(step_ms))
    out = {"workload": f"{name}: {coi_text(link, coi)}", "value": pspans / (ms * 1e-3), "unit": UNIT,
           "ms_per_step": ms, "steps": 5, "warmup": 3, "point_spans_per_step": pspans,
           "channels_per_s": n / (ms * 1e-3), "roofline_frac": rf["ach"] / rf["peak"],
           "integrand_phase_ms": rf["ki_ms"]}
    if not args.no_e2e:
        t = e2e_host(isrs, link, coi, local, args.precision, 3)
        out["e2e"] = {"value": pspans / float(np.median(t)), "unit": UNIT,
                      "samples_ms": [round(1e3 * x, 2) for x in t]}
    return out


def run_ours(args, link, coi, ws, rank, local):
    import torch
    import paper_2412_11614_b200 as isrs
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    eng = isrs.Engine(link, device=local, precision=args.precision)
    n = link.n_ch if coi is None else len(coi)
    eta = torch.empty(n, dtype=torch.float64, device=dev)
    terms = torch.empty((n, 5), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    if ws > 1:
        # rank r evaluates shard r of the canonical region list (cost-balanced), the
        # per-COI sums [n, 6] are all-gathered over NCCL (NVLink/NVSwitch) and every rank combines
        # them in fixed rank order -> the same eta on every rank (strong scaling of one link).
        import torch.distributed as dist
        sums = torch.empty(n * 6, dtype=torch.float64, device=dev)          # flat: any backend
        gathered = torch.empty(ws * n * 6, dtype=torch.float64, device=dev)

        def step():
            eng.nli_shard_into(rank, ws, sums.data_ptr(), coi, stream.cuda_stream)
            dist.all_gather_into_tensor(gathered, sums)
            eng.combine_into(ws, gathered.data_ptr(), eta.data_ptr(), terms.data_ptr(), coi,
                             stream.cuda_stream)
        barrier = torch.distributed.barrier
    else:
        def step():
            eng.nli_into(eta.data_ptr(), terms.data_ptr(), coi, stream.cuda_stream)
        barrier = None

    # one untimed call so the work list exists, then the work counts of this rank's share
    with torch.cuda.stream(stream):
        step()
    torch.cuda.synchronize()
    pts, pspans, nreg = eng.work()
    launches_per_step = eng.last_launch_count() + (1 if ws > 1 else 0)
    if ws > 1:
        tot = torch.tensor([pts, pspans, nreg], dtype=torch.int64, device=dev)
        torch.distributed.all_reduce(tot)
        pts, pspans, nreg = (int(v) for v in tot.tolist())

    step_ms, kern_ms, clk = time_steps(eng, step, stream, flush, args.steps, args.warmup, barrier,
                                       ClockSampler(local))
    ms = float(np.mean(step_ms))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(t.item())
    eta_host = eta.cpu().numpy()
    same_eta = None
    if ws > 1:       # every rank combined the same gathered sums in the same order: bitwise equal
        ge = torch.empty(ws * n, dtype=torch.float64, device=dev)
        torch.distributed.all_gather_into_tensor(ge, eta)
        ge = ge.cpu().numpy().reshape(ws, n)
        same_eta = bool(all(np.array_equal(ge[0], ge[r]) for r in range(ws)))

    kd_ms = float(np.mean([k[0][0] for k in kern_ms]))
    kc_ms = float(np.mean([k[0][1] for k in kern_ms]))
    kr_ms = float(np.mean([k[0][2] for k in kern_ms]))
    rf = roofline_of(eng, link, kern_ms, args.precision)
    traffic, traffic_src = ncu_traffic(link.name)
    survey_fpp = float(np.mean(8 * np.asarray(rf["k_s"], dtype=float) + 100))     # 8 K_s + ~100

    # end to end through the public API with host buffers: create + nli + D2H + destroy
    e2e = None
    if not args.no_e2e:
        pa = isrs.ProblemArrays(link)
        h2d = pa.nbytes() + (0 if coi is None else 4 * len(coi))
        reps = max(1, min(5, args.steps))
        if ws == 1:
            t_e2e = e2e_host(isrs, link, coi, local, args.precision, reps)
        else:
            t_e2e = []
            for k in range(reps):
                torch.distributed.barrier()
                t0 = time.perf_counter()
                with isrs.Engine(link, device=local, precision=args.precision) as e2:
                    s2 = e2.nli_shard(rank, ws, coi=coi).reshape(-1)
                    g2 = torch.empty(ws * n * 6, dtype=torch.float64, device=dev)
                    torch.distributed.all_gather_into_tensor(g2, s2)
                    e2.combine(g2.reshape(ws, n, 6), coi=coi).cpu()
                dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
                torch.distributed.all_reduce(dt, op=torch.distributed.ReduceOp.MAX)
                t_e2e.append(float(dt.item()))
        e2e = {"value": pspans / float(np.median(t_e2e)), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 8 * n, "samples_ms": [round(1e3 * x, 2) for x in t_e2e],
               "note": ("isrs_egn_eta_host(): validate + region plan + H2D + precompute + nli + D2H + free"
                        if ws == 1 else f"per rank: create (H2D, precompute) + nli_shard + {(args.backend or 'nccl').upper()} all-gather "
                        "+ combine + D2H + destroy; max over ranks")}

    # NEXT-4a, reported separately (never the headline): span-class dedup evaluates each run of
    # identical spans' K-segment sum once per point; rate in LOGICAL point-spans/s
    dedup = None
    if ws == 1 and not args.no_dedup:
        with isrs.Engine(link, device=local, precision=64, flags=isrs.FLAG_DEDUP) as ed:
            dms, _, _ = time_steps(ed, lambda: ed.nli_into(eta.data_ptr(), 0, coi, stream.cuda_stream),
                                   stream, flush, 3, 2)
        dm = float(np.median(dms))
        dedup = {"value": pspans / (dm * 1e-3), "unit": UNIT + " (logical)", "ms_per_step": dm,
                 "note": "ISRS_EGN_FLAG_DEDUP: one K-segment sum per run of identical spans x the "
                         "phased-array factor; same eta (<= 1e-10), not the headline"}

    # f1 <-> f2 symmetry (ISRS_EGN_FLAG_MIRROR), reported separately like dedup: region (k, k1, k2),
    # k1 < k2, evaluated once for both orientations; rate in LOGICAL point-spans/s
    mirror = None
    if ws == 1 and not args.no_dedup:
        with isrs.Engine(link, device=local, precision=args.precision, flags=isrs.FLAG_MIRROR) as em:
            mms, _, _ = time_steps(em, lambda: em.nli_into(eta.data_ptr(), 0, coi, stream.cuda_stream),
                                   stream, flush, 3, 2)
            mpts = em.work()[0]
        mm = float(np.median(mms))
        mirror = {"value": pspans / (mm * 1e-3), "unit": UNIT + " (logical)", "ms_per_step": mm,
                  "evaluated_point_spans_per_step": mpts * link.n_span,
                  "note": "ISRS_EGN_FLAG_MIRROR: f1 <-> f2 symmetry (pin P2), each off-diagonal region pair "
                          "evaluated once; same eta (<= 1e-12 of the full evaluation), not the headline"}

    extras = {}
    if ws == 1 and not args.no_extra:
        for name, spec in (("c2", "all"), ("c4", "default")):
            if name != link.name:
                extras[name] = extra_config(isrs, name, spec, args, local, stream, flush)

    if rank == 0:
        value = pspans / (ms_max * 1e-3)          # the whole workload's point-spans over all ranks
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": "f64" if args.precision == 64 else "f32 (mixed, row a8)", "data": "synthetic",
                "config": config_desc(link, coi, args),
                "channels_per_s": n / (ms_max * 1e-3),
                "point_spans_per_step": pspans, "points_per_step": pts, "regions_per_step": nreg,
                "kernel_ms": {"integrand_D": kd_ms, "integrand_coherent": kc_ms, "reduce": kr_ms,
                              "integrand_phase": rf["ki_ms"],
                              "note": "coherent launch runs concurrently on a side stream"},
                "roofline": {"bound": "alu", "achieved": rf["ach"], "peak": rf["peak"], "unit": "TFLOP/s",
                             "frac": rf["ach"] / rf["peak"], "traffic": traffic, "traffic_source": traffic_src,
                             "kernel": "isrs::integrand_kernel<false,MODE> + <true,MODE> (D-only and coherent "
                                       "regions, concurrent; fork to join; MODE 7 = segment mode with chain "
                                       "groups when a group of identical spans holds > 1 chain, else 0)",
                             "flops_per_point_span": rf["fpp"],
                             "span_chains": [int(g) for g in rf["chain_g"]],
                             "chain_groups": [int(g) for g in rf["grp_c0"]] if rf["grp_c0"] is not None else None,
                             "peak_note": ("derived: 148 SM x 64 FP64 FMA/clk x 2 x 1965 MHz "
                                           "(tools/dmma_probe.cu: a DFMA stream reaches 128 flop/SM-cycle = this peak)"
                                           if args.precision == 64 else
                                           "derived FP32 peak: 148 SM x 128 FP32 FMA/clk x 2 x 1965 MHz (the "
                                           "variant's recurrence is fp32; chi h, phase and Y stay fp64)")},
                "survey_units": {"flops_per_point_span": survey_fpp,
                                 "achieved": rf["ps_i"] * survey_fpp / (rf["ki_ms"] * 1e-3) / 1e12,
                                 "unit": "TFLOP/s",
                                 "frac": rf["ps_i"] * survey_fpp / (rf["ki_ms"] * 1e-3) / 1e12 / rf["peak"],
                                 "note": "SURVEY.md 8(d) per-unit figure 8 K + 100 assumes a complex Horner "
                                         "step (8 flops per segment); this kernel's real second-order "
                                         "recurrence needs 3, so this ratio exceeds 1 and is not the "
                                         "roofline - `roofline` counts the flops the kernel's method needs"},
                "fp64_pipe_slots": {"achieved": rf["slots_ach"], "peak": rf["slots_peak"], "unit": "T slot/s",
                                    "frac": rf["slots_ach"] / rf["slots_peak"], "per_point_span": rf["spp"],
                                    "note": "same algorithmic count with DFMA and DADD one FP64 "
                                            "pipe issue slot each (the recurrence's real bound)"},
                "pct_fp64_peak": 100.0 * rf["ach"] / rf["peak"],
                "gpu_launches": launches_per_step * args.steps,
                "clocks": clk, "e2e": e2e,
                "eta_db": [float(10 * np.log10(x)) for x in (eta_host if n <= 8 else eta_host[[0, n // 2, n - 1]])]}
        if same_eta is not None:
            line["eta_bitwise_equal_across_ranks"] = same_eta
        if dedup is not None:
            line["dedup_effective"] = dedup
        if mirror is not None:
            line["mirror_effective"] = mirror
        if extras:
            line["other_configs"] = extras
        if not args.no_cpu and ws == 1:
            rate, ps, dt, cores, desc = oracle_sample(link, args.cpu_seconds, coi)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
                                    "sample": f"{desc}; {ps} point-spans in {dt:.1f} s"}
        print(json.dumps(line), flush=True)
    eng.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--coi", default="default",
                    help="'default' (c3-c5: SURVEY 8(d)'s {0, n/2, n-1}; c1, c2: all), 'all', or a list")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", type=int, default=64, choices=[64, 32],
                    help="64: the fp64 hot path (default); 32: the mixed fp32 variant (row a8)")
    ap.add_argument("--backend", default=None, help="torch.distributed backend (default nccl)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dedup", action="store_true", help="skip the separate NEXT-4a dedup timing")
    ap.add_argument("--no-extra", action="store_true", help="skip the extra c2 / c4 timings")
    ap.add_argument("--ref-seconds", type=float, default=8.0, help="CPU seconds per reference step")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU seconds of the cpu_baseline")
    args = ap.parse_args()
    from workloads import bj_config
    link = bj_config(args.config)
    coi = parse_coi(args.coi, link)
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, link, coi, ws, rank)
    else:
        run_ours(args, link, coi, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
