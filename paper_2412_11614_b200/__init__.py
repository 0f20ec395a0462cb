"""B200-native ISRS EGN hot path (arXiv 2412.11614): eta(f_COI) per channel with the segment
closed-form FWM efficiency factor, span phased-array sum and EGN corrections, in sm_100a
kernels behind the C ABI of include/isrs_egn.h.

Python here only marshals arguments; PyTorch is used only for device memory and streams.

    h = Engine(link)                 # isrs_egn_create
    eta = h.nli()                    # isrs_egn_nli -> torch.float64 CUDA tensor [n_coi] (1/W^2)
    h.close()                        # isrs_egn_destroy
"""
import ctypes

import numpy as np

from . import _abi
from ._abi import (FLAG_DEDUP, FLAG_LITERAL_GAIN, FLAG_MIRROR, FLAG_NO_CHAIN, FLAG_SPLIT, FLAG_UNIT_LINK, MU_INTEGRAL, MU_MACLAURIN, MU_SEGMENT,
                   IsrsEgnError, ProblemArrays,  # noqa: F401
                   numerics)

__all__ = ["Engine", "Problem", "NliGraph", "eta_host", "plan_shards", "IsrsEgnError", "MU_SEGMENT", "MU_MACLAURIN", "MU_INTEGRAL", "FLAG_UNIT_LINK", "FLAG_NO_CHAIN", "FLAG_DEDUP", "FLAG_LITERAL_GAIN", "FLAG_MIRROR", "FLAG_SPLIT",
           "library_path"]


def library_path():
    return _abi.LIB_PATH


def load():
    """Load libisrs_egn.so now (raises ImportError when it is missing: no CPU fallback)."""
    return _abi.get()


class Engine:
    """Handle over one link (isrs_egn_create / isrs_egn_nli / isrs_egn_destroy)."""

    def __init__(self, link, grid_n=None, delta_z_m=None, device=0, precision=64,
                 mu_mode=MU_SEGMENT, flags=0, f_samples=0):
        self._args = (link, dict(grid_n=grid_n, delta_z_m=delta_z_m, device=device, precision=precision,
                                 mu_mode=mu_mode, flags=flags, f_samples=f_samples))
        self._pa = ProblemArrays(link)
        n = numerics(grid_n if grid_n is not None else link.grid_n,
                     delta_z_m if delta_z_m is not None else getattr(link, "delta_z_m", 1000.0),
                     precision, mu_mode, flags, f_samples)
        self.n_ch = self._pa.struct.n_ch
        self.n_span = self._pa.struct.n_span
        self.device = device
        h = ctypes.c_void_p()
        _abi.check(_abi.get().isrs_egn_create(ctypes.byref(self._pa.struct), ctypes.byref(n), device,
                                            ctypes.byref(h)))
        self._h = h

    def nli_into(self, eta_ptr, terms_ptr=0, coi=None, stream=0):
        """Raw call: device pointers (ints) and a cudaStream_t handle (int)."""
        if coi is None:
            n, cp = self.n_ch, None
        else:
            c = np.ascontiguousarray(np.asarray(coi, dtype=np.int32))
            n, cp = len(c), c.ctypes.data_as(_abi._ip)
            self._coi_keep = c
        _abi.check(_abi.get().isrs_egn_nli(self._h, n, cp, ctypes.c_void_p(eta_ptr),
                                         ctypes.c_void_p(terms_ptr or None),
                                         ctypes.c_void_p(stream or None)))

    def nli(self, coi=None, terms=False, stream=None):
        """eta [n_coi] (and the D, E, F, G, H breakdown [n_coi, 5]) as float64 CUDA tensors."""
        import torch
        n = self.n_ch if coi is None else len(coi)
        dev = torch.device("cuda", self.device)
        eta = torch.empty(n, dtype=torch.float64, device=dev)
        tt = torch.empty((n, 5), dtype=torch.float64, device=dev) if terms else None
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        self.nli_into(eta.data_ptr(), tt.data_ptr() if terms else 0, coi, st.cuda_stream)
        return (eta, tt) if terms else eta

    def nli_split(self, coi=None, terms=False, stream=None):
        """isrs_egn_nli_split (an Engine created with flags=FLAG_SPLIT): eta [n_coi], its SCI / XCI / MCI
        parts [n_coi, 3] and, with terms=True, the D..H breakdown [n_coi, 5]."""
        import torch
        n, cp = self._coi(coi)
        dev = torch.device("cuda", self.device)
        eta = torch.empty(n, dtype=torch.float64, device=dev)
        parts = torch.empty((n, 3), dtype=torch.float64, device=dev)
        tt = torch.empty((n, 5), dtype=torch.float64, device=dev) if terms else None
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        _abi.check(_abi.get().isrs_egn_nli_split(self._h, n, cp, ctypes.c_void_p(eta.data_ptr()),
                                               ctypes.c_void_p(tt.data_ptr() if terms else None),
                                               ctypes.c_void_p(parts.data_ptr()),
                                               ctypes.c_void_p(st.cuda_stream or None)))
        return (eta, parts, tt) if terms else (eta, parts)

    def region_partials(self, regions):
        """[(kappa, k1, k2), ...] -> array [n, 6]: D_w, E_w, F_w, G_w, H_w, n_points (last call)."""
        r = np.asarray(regions, dtype=np.int32).reshape(-1, 3)
        k, a, b = (np.ascontiguousarray(r[:, i]) for i in range(3))
        out = np.zeros((len(r), 6))
        _abi.check(_abi.get().isrs_egn_region_partials(
            self._h, len(r), k.ctypes.data_as(_abi._ip), a.ctypes.data_as(_abi._ip),
            b.ctypes.data_as(_abi._ip), out.ctypes.data_as(_abi._dp)))
        return out

    def work(self):
        """(points, point_spans, regions) of the last nli call, as its kernels counted them."""
        p, ps, r = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _abi.check(_abi.get().isrs_egn_last_work(self._h, ctypes.byref(p), ctypes.byref(ps), ctypes.byref(r)))
        return p.value, ps.value, r.value

    def planned_work(self, coi=None):
        """(points, point_spans, regions) of nli(coi) from the host planner alone (no device work)."""
        n, cp = self._coi(coi)
        p, ps, r = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _abi.check(_abi.get().isrs_egn_work(self._h, n, cp, ctypes.byref(p), ctypes.byref(ps), ctypes.byref(r)))
        return p.value, ps.value, r.value

    def last_kernel_ms(self):
        """([ms_D_only, ms_coherent, ms_reduce, ms_integrand_phase],
        [point_spans_D_only, point_spans_coherent, total])."""
        ms = (ctypes.c_double * 4)()
        ps = (ctypes.c_double * 3)()
        _abi.check(_abi.get().isrs_egn_last_kernel_ms(self._h, ms, ps))
        return list(ms), list(ps)

    def _coi(self, coi):
        if coi is None:
            return self.n_ch, None
        c = np.ascontiguousarray(np.asarray(coi, dtype=np.int32))
        self._coi_keep = c
        return len(c), c.ctypes.data_as(_abi._ip)

    def nli_shard_into(self, rank, world, sums_ptr, coi=None, stream=0):
        """Multi-GPU shard (isrs_egn_nli_shard): per-COI sums [n_coi, 6] of shard `rank` of `world`."""
        n, cp = self._coi(coi)
        _abi.check(_abi.get().isrs_egn_nli_shard(self._h, n, cp, int(rank), int(world),
                                               ctypes.c_void_p(sums_ptr), ctypes.c_void_p(stream or None)))

    def combine_into(self, world, gathered_ptr, eta_ptr, terms_ptr=0, coi=None, stream=0):
        """eta from all-gathered shard sums [world, n_coi, 6] (isrs_egn_combine, fixed rank order)."""
        n, cp = self._coi(coi)
        _abi.check(_abi.get().isrs_egn_combine(self._h, n, cp, int(world), ctypes.c_void_p(gathered_ptr),
                                             ctypes.c_void_p(eta_ptr), ctypes.c_void_p(terms_ptr or None),
                                             ctypes.c_void_p(stream or None)))

    def nli_shard(self, rank, world, coi=None, stream=None):
        import torch
        n = self.n_ch if coi is None else len(coi)
        dev = torch.device("cuda", self.device)
        out = torch.empty((n, 6), dtype=torch.float64, device=dev)
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        self.nli_shard_into(rank, world, out.data_ptr(), coi, st.cuda_stream)
        return out

    def combine(self, gathered, coi=None, terms=False, stream=None):
        import torch
        world = gathered.shape[0]
        n = gathered.shape[1]
        g = gathered.contiguous()
        eta = torch.empty(n, dtype=torch.float64, device=g.device)
        tt = torch.empty((n, 5), dtype=torch.float64, device=g.device) if terms else None
        st = stream if stream is not None else torch.cuda.current_stream(g.device)
        self.combine_into(world, g.data_ptr(), eta.data_ptr(), tt.data_ptr() if terms else 0, coi,
                          st.cuda_stream)
        return (eta, tt) if terms else eta

    def span_chains(self):
        """(chain sizes G_c, K_s per span) of the handle's span chains (reading R9)."""
        n = ctypes.c_int32()
        g = np.zeros(self.n_span, dtype=np.int32)
        k = np.zeros(self.n_span, dtype=np.int32)
        _abi.check(_abi.get().isrs_egn_span_chains(self._h, ctypes.byref(n), g.ctypes.data_as(_abi._ip),
                                                 k.ctypes.data_as(_abi._ip)))
        return g[:n.value].copy(), k

    def chain_groups(self):
        """Bounds [n_grp + 1] of the chain groups (R9): group g covers chains grp_c0[g] .. grp_c0[g+1]-1."""
        n = ctypes.c_int32()
        g = np.zeros(self.n_span + 1, dtype=np.int32)
        _abi.check(_abi.get().isrs_egn_chain_groups(self._h, ctypes.byref(n), g.ctypes.data_as(_abi._ip)))
        return g[:n.value + 1].copy()

    def profile_tables(self, span=0):
        """(ln_a [K], zeta [K]) of span `span`: the precompute kernel's output (row a2, Eqs. 2, 10, 14)."""
        k = ctypes.c_int32()
        _abi.check(_abi.get().isrs_egn_profile_tables(self._h, int(span), ctypes.byref(k), None, None))
        la = np.zeros(k.value)
        ze = np.zeros(k.value)
        _abi.check(_abi.get().isrs_egn_profile_tables(self._h, int(span), ctypes.byref(k),
                                                    la.ctypes.data_as(_abi._dp), ze.ctypes.data_as(_abi._dp)))
        return la, ze

    def last_launch_count(self):
        return _abi.get().isrs_egn_last_launch_count(self._h)

    def graph(self, coi=None, terms=False):
        """A CUDA graph of one nli call (fixed COI set, fixed output tensors): NliGraph.replay()
        re-runs the whole hot path (fork, both integrand launches, join, reduce) as one graph
        launch -- for small links whose call is launch-bound (c1: 45 -> 31 us per call).  The graph
        owns a private handle on the same link, so this Engine stays free for other COI sets."""
        link, kw = self._args
        return NliGraph(Engine(link, **kw), coi, terms, own=True)

    def close(self):
        if getattr(self, "_h", None):
            _abi.get().isrs_egn_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NliGraph:
    """Captured isrs_egn_nli (torch.cuda.CUDAGraph).  The work list of the COI set is built and the
    handle is warmed up on the graph's own stream before capture (no host synchronisation or
    allocation happens inside it).  replay() writes the captured output tensors `eta` (and `terms`),
    ordered after the caller's current stream, which waits for it.  The graph bakes in its handle's
    device buffers, so it owns that handle (Engine.graph() passes a private one, own=True) and
    closes it with close()."""

    def __init__(self, engine, coi=None, terms=False, own=False):
        import torch
        dev = torch.device("cuda", engine.device)
        n = engine.n_ch if coi is None else len(coi)
        self.eta = torch.empty(n, dtype=torch.float64, device=dev)
        self.terms = torch.empty((n, 5), dtype=torch.float64, device=dev) if terms else None
        self.stream = torch.cuda.Stream(device=dev)
        self._engine = engine
        self._own = own
        tp = self.terms.data_ptr() if terms else 0
        with torch.cuda.stream(self.stream):
            for _ in range(2):
                engine.nli_into(self.eta.data_ptr(), tp, coi, self.stream.cuda_stream)
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            engine.nli_into(self.eta.data_ptr(), tp, coi, self.stream.cuda_stream)

    def replay(self):
        """One graph launch, ordered after the caller's current stream, which then waits for it."""
        import torch
        cur = torch.cuda.current_stream(self.eta.device)
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            self.graph.replay()
        cur.wait_stream(self.stream)
        return (self.eta, self.terms) if self.terms is not None else self.eta

    def close(self):
        if getattr(self, "graph", None) is not None:
            self.stream.synchronize()
            self.graph.reset()
            self.graph = None
        if self._own and self._engine is not None:
            self._engine.close()
            self._engine = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Problem:
    """A link description with the fields of `isrs_egn_problem` / `isrs_egn_numerics` (SI units, absolute
    frequencies in integer Hz; include/isrs_egn.h).  Pure marshalling: values are passed through as given.

        p = Problem.from_config("link.json")       # or a dict / a JSON string
        with Engine(p) as e: eta = e.nli()

    Config keys: the per-channel arrays f_center_hz, symbol_rate_hz, launch_power_w, excess_kurtosis
    (optional psi), the per-span entries length_m, alpha_per_m, beta2_s2_per_m, beta3_s3_per_m,
    gamma_per_w_m, cr_per_w_m_hz -- each a list of n_span values, or one number repeated for the
    config's "n_span" identical spans -- and grid_n (optional delta_z_m, default 1000 m)."""

    CHANNEL = ("f_center_hz", "symbol_rate_hz", "launch_power_w", "excess_kurtosis")
    SPAN = ("length_m", "alpha_per_m", "beta2_s2_per_m", "beta3_s3_per_m", "gamma_per_w_m", "cr_per_w_m_hz")

    def __init__(self, grid_n, delta_z_m=1000.0, psi=None, n_span=None, name="problem", **fields):
        missing = [k for k in self.CHANNEL + self.SPAN if k not in fields]
        unknown = [k for k in fields if k not in self.CHANNEL + self.SPAN]
        if missing or unknown:
            raise ValueError(f"Problem: missing {missing}, unknown {unknown}")
        for k in self.CHANNEL:
            setattr(self, k, np.ascontiguousarray(np.atleast_1d(np.asarray(fields[k], dtype=np.float64))))
        n_ch = self.f_center_hz.size
        if any(getattr(self, k).shape != (n_ch,) for k in self.CHANNEL):
            raise ValueError("Problem: the per-channel arrays must all have n_ch entries")
        self.psi = None if psi is None else np.ascontiguousarray(np.asarray(psi, dtype=np.float64))
        if self.psi is not None and self.psi.shape != (n_ch,):
            raise ValueError("Problem: psi must have n_ch entries")
        sizes = {np.size(fields[k]) for k in self.SPAN if np.ndim(fields[k]) > 0}
        if len(sizes) > 1 or (sizes and n_span is not None and sizes != {int(n_span)}):
            raise ValueError("Problem: the per-span arrays must all have n_span entries")
        ns = sizes.pop() if sizes else int(n_span if n_span is not None else 1)
        for k in self.SPAN:
            v = np.asarray(fields[k], dtype=np.float64)
            setattr(self, k, np.ascontiguousarray(np.full(ns, float(v)) if v.ndim == 0 else v.reshape(ns)))
        self.phi = self.excess_kurtosis          # the name Engine / ProblemArrays read
        self.grid_n = int(grid_n)
        self.delta_z_m = float(delta_z_m)
        self.name = name

    n_ch = property(lambda self: int(self.f_center_hz.size))
    n_span = property(lambda self: int(self.length_m.size))

    @classmethod
    def from_config(cls, cfg):
        """cfg: a dict, a JSON string, or the path of a JSON file."""
        import json
        import os
        if isinstance(cfg, (str, bytes, os.PathLike)):
            text = cfg.decode() if isinstance(cfg, bytes) else os.fspath(cfg)
            if text.lstrip().startswith("{"):
                cfg = json.loads(text)
            else:
                with open(text) as fh:
                    cfg = json.load(fh)
        if not isinstance(cfg, dict):
            raise TypeError("Problem.from_config: a dict, a JSON string or a JSON file path")
        return cls(**cfg)

    def to_config(self):
        """The dict `from_config` accepts (lists of Python floats: JSON-serialisable, exact round trip)."""
        d = {k: getattr(self, k).tolist() for k in self.CHANNEL + self.SPAN}
        if self.psi is not None:
            d["psi"] = self.psi.tolist()
        d.update(grid_n=self.grid_n, delta_z_m=self.delta_z_m, name=self.name)
        return d


def plan_shards(link, world, coi=None, grid_n=None, delta_z_m=None, f_samples=0):
    """Host-only shard plan (isrs_egn_plan_shards): (regions, points, first_region) arrays [world]."""
    pa = ProblemArrays(link)
    n = numerics(grid_n if grid_n is not None else link.grid_n,
                 delta_z_m if delta_z_m is not None else getattr(link, "delta_z_m", 1000.0),
                 64, MU_SEGMENT, 0, f_samples)
    if coi is None:
        nco, cp = pa.struct.n_ch, None
    else:
        c = np.ascontiguousarray(np.asarray(coi, dtype=np.int32))
        nco, cp = len(c), c.ctypes.data_as(_abi._ip)
    r = np.zeros(world, dtype=np.int64)
    p = np.zeros(world, dtype=np.int64)
    f = np.zeros(world, dtype=np.int64)
    _abi.check(_abi.get().isrs_egn_plan_shards(ctypes.byref(pa.struct), ctypes.byref(n), nco, cp, int(world),
                                             r.ctypes.data_as(_abi._lp), p.ctypes.data_as(_abi._lp),
                                             f.ctypes.data_as(_abi._lp)))
    return r, p, f


def eta_host(link, coi=None, grid_n=None, delta_z_m=None, device=0, precision=64, mu_mode=MU_SEGMENT,
             flags=0, terms=False, f_samples=0):
    """One-shot end-to-end call with host buffers (isrs_egn_eta_host)."""
    pa = ProblemArrays(link)
    n = numerics(grid_n if grid_n is not None else link.grid_n,
                 delta_z_m if delta_z_m is not None else getattr(link, "delta_z_m", 1000.0),
                 precision, mu_mode, flags, f_samples)
    if coi is None:
        nco, cp = pa.struct.n_ch, None
    else:
        c = np.ascontiguousarray(np.asarray(coi, dtype=np.int32))
        nco, cp = len(c), c.ctypes.data_as(_abi._ip)
    eta = np.zeros(nco)
    tt = np.zeros((nco, 5)) if terms else None
    _abi.check(_abi.get().isrs_egn_eta_host(ctypes.byref(pa.struct), ctypes.byref(n), device, nco, cp,
                                          eta.ctypes.data_as(_abi._dp),
                                          tt.ctypes.data_as(_abi._dp) if terms else _abi._dp()))
    return (eta, tt) if terms else eta
