"""Fast-plain oracle (test infrastructure only): ctypes wrapper of oracle/fastplain.c.

The same definition as egn.eta(mu_mode="closed") -- Eqs. 5, 8-10, 14, 22 (reading C3), 15-21
(C2, C7, C8, C10), 11 -- in plain C with the three savings SURVEY.md 8(d) lists for its
"fast-plain" variant (forward recurrence for e^{sigma k h}, SRS gain tabulated per f3 of a region,
mu once per distinct span parameter set); see the header of fastplain.c.  Pinned against the
literal closed mode by tests/test_oracle_fastplain.py (<= 1e-12).

    eta, terms, npts = fastplain.eta(link, coi=None, threads=0)
    part = fastplain.region_partials(link, kappa, k1, k2)    # = egn.region_partials(...)

The library is compiled on first use (gcc, -O3, no fast-math, no FMA contraction; OpenMP).
"""
import ctypes
import os
import subprocess
import threading
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "fastplain.c")
MARCH = os.environ.get("FASTPLAIN_MARCH", "x86-64-v3")
LIB = os.path.join(_HERE, f"libfastplain_{MARCH.replace('-', '_')}.so")
CFLAGS = ["-O3", f"-march={MARCH}", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC",
          "-shared"]

_dp = ctypes.POINTER(ctypes.c_double)


class _Link(ctypes.Structure):
    _fields_ = [("n_ch", ctypes.c_int32), ("f_center_hz", _dp), ("symbol_rate_hz", _dp),
                ("launch_power_w", _dp), ("phi", _dp), ("psi", _dp), ("n_span", ctypes.c_int32),
                ("length_m", _dp), ("alpha_per_m", _dp), ("beta2", _dp), ("beta3", _dp),
                ("gamma", _dp), ("cr", _dp), ("grid_n", ctypes.c_int32), ("delta_z_m", ctypes.c_double)]


def build(force=False):
    """Compile fastplain.c into an in-tree shared library (what __graft_entry__.build() calls)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc"] + CFLAGS + [SRC, "-o", LIB + ".tmp", "-lm"]
        subprocess.run(cmd, check=True, capture_output=True, text=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def _get():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.fp_eta.argtypes = [ctypes.POINTER(_Link), ctypes.c_int, ctypes.POINTER(ctypes.c_int32),
                               ctypes.c_int, _dp, _dp, ctypes.POINTER(ctypes.c_longlong),
                               ctypes.POINTER(ctypes.c_longlong)]
        lib.fp_eta.restype = ctypes.c_int
        lib.fp_region.argtypes = [ctypes.POINTER(_Link), ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]
        lib.fp_region.restype = ctypes.c_int
        _lib = lib
    return _lib


def _struct(link):
    keep = []

    def arr(x):
        a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        keep.append(a)
        return a.ctypes.data_as(_dp)

    s = _Link(int(link.n_ch), arr(link.f_center_hz), arr(link.symbol_rate_hz), arr(link.launch_power_w),
              arr(link.phi), arr(link.psi), int(link.n_span), arr(link.length_m), arr(link.alpha_per_m),
              arr(link.beta2_s2_per_m), arr(link.beta3_s3_per_m), arr(link.gamma_per_w_m),
              arr(link.cr_per_w_m_hz), int(link.grid_n), float(link.delta_z_m))
    return s, keep


def eta(link, coi=None, threads=0, progress=False):
    """(eta [n_coi] 1/W^2, terms [n_coi, 5] D..H contributions, in-support points [n_coi])."""
    s, keep = _struct(link)
    c = np.ascontiguousarray(np.arange(link.n_ch) if coi is None else np.asarray(coi), dtype=np.int32)
    e = np.zeros(len(c))
    t = np.zeros((len(c), 5))
    npts = np.zeros(len(c), dtype=np.int64)
    prog = ctypes.c_longlong(0)
    done = threading.Event()
    if progress:
        ntask = len(c) * link.n_ch
        t0 = time.time()

        def report():
            while not done.wait(60.0):
                v = prog.value
                el = time.time() - t0
                print(f"fastplain: {v}/{ntask} tasks, {el:.0f} s"
                      + (f", ~{el * (ntask - v) / v:.0f} s left" if v else ""), flush=True)
        th = threading.Thread(target=report, daemon=True)
        th.start()
    rc = _get().fp_eta(ctypes.byref(s), len(c), c.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                       int(threads), t.ctypes.data_as(_dp), e.ctypes.data_as(_dp),
                       npts.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), ctypes.byref(prog))
    done.set()
    if rc != 0:
        raise RuntimeError(f"fastplain.fp_eta failed ({rc}: -1 allocation, -2 inexact f3 lattice, "
                           "-3 bands not sorted/disjoint)")
    del keep
    return e, t, npts


def region_partials(link, kappa, k1, k2):
    """[D_w, E_w, F_w, G_w, H_w], n_points of region (kappa, k1, k2) -- egn.region_partials' quantities."""
    s, keep = _struct(link)
    out = np.zeros(6)
    rc = _get().fp_region(ctypes.byref(s), int(kappa), int(k1), int(k2), out.ctypes.data_as(_dp))
    if rc != 0:
        raise RuntimeError(f"fastplain.fp_region failed ({rc})")
    del keep
    return out[:5], int(out[5])
