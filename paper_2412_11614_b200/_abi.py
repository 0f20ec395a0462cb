"""ctypes binding of include/isrs_egn.h — argument marshalling only.

Every step of the hot path runs in libisrs_egn.so (sm_100a kernels).  There is no CPU
fallback: if the library is missing this module raises at import, and every call that
returns a non-zero status raises IsrsEgnError with the library's own message.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ISRS_EGN_LIB") or os.path.join(_HERE, "libisrs_egn.so")

OK, EINVAL, EOVERLAP, ERANGE, ENOMEM, ECUDA, EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
MU_SEGMENT, MU_MACLAURIN, MU_INTEGRAL = 0, 1, 2
FLAG_UNIT_LINK = 1
FLAG_NO_CHAIN = 2
FLAG_DEDUP = 4
FLAG_LITERAL_GAIN = 8
FLAG_MIRROR = 16
FLAG_SPLIT = 32

EXPORTED = ("isrs_egn_create", "isrs_egn_nli", "isrs_egn_nli_split", "isrs_egn_region_partials", "isrs_egn_work", "isrs_egn_last_work",
            "isrs_egn_eta_host", "isrs_egn_last_kernel_ms", "isrs_egn_last_launch_count",
            "isrs_egn_span_chains", "isrs_egn_chain_groups", "isrs_egn_profile_tables", "isrs_egn_nli_shard", "isrs_egn_combine", "isrs_egn_plan_shards",
            "isrs_egn_destroy",
            "isrs_egn_strerror", "isrs_egn_last_error")

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)
_lp = ctypes.POINTER(ctypes.c_int64)


class Problem(ctypes.Structure):
    _fields_ = [("n_ch", ctypes.c_int32), ("f_center_hz", _dp), ("symbol_rate_hz", _dp),
                ("launch_power_w", _dp), ("excess_kurtosis", _dp), ("psi", _dp),
                ("n_span", ctypes.c_int32), ("length_m", _dp), ("alpha_per_m", _dp),
                ("beta2_s2_per_m", _dp), ("beta3_s3_per_m", _dp), ("gamma_per_w_m", _dp),
                ("cr_per_w_m_hz", _dp)]


class Numerics(ctypes.Structure):
    _fields_ = [("grid_n", ctypes.c_int32), ("delta_z_m", ctypes.c_double),
                ("precision", ctypes.c_int32), ("mu_mode", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("f_samples", ctypes.c_int32)]


class IsrsEgnError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"isrs_egn error {code}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2412_11614_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    lib.isrs_egn_create.argtypes = [ctypes.POINTER(Problem), ctypes.POINTER(Numerics), ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_void_p)]
    lib.isrs_egn_create.restype = ctypes.c_int
    lib.isrs_egn_nli.argtypes = [ctypes.c_void_p, ctypes.c_int32, _ip, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p]
    lib.isrs_egn_nli.restype = ctypes.c_int
    lib.isrs_egn_nli_split.argtypes = [ctypes.c_void_p, ctypes.c_int32, _ip, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    lib.isrs_egn_nli_split.restype = ctypes.c_int
    lib.isrs_egn_region_partials.argtypes = [ctypes.c_void_p, ctypes.c_int32, _ip, _ip, _ip, _dp]
    lib.isrs_egn_region_partials.restype = ctypes.c_int
    lib.isrs_egn_chain_groups.argtypes = [ctypes.c_void_p, _ip, _ip]
    lib.isrs_egn_chain_groups.restype = ctypes.c_int
    lib.isrs_egn_profile_tables.argtypes = [ctypes.c_void_p, ctypes.c_int32, _ip, _dp, _dp]
    lib.isrs_egn_profile_tables.restype = ctypes.c_int
    lib.isrs_egn_work.argtypes = [ctypes.c_void_p, ctypes.c_int32, _ip, _lp, _lp, _lp]
    lib.isrs_egn_work.restype = ctypes.c_int
    lib.isrs_egn_last_work.argtypes = [ctypes.c_void_p, _lp, _lp, _lp]
    lib.isrs_egn_last_work.restype = ctypes.c_int
    lib.isrs_egn_eta_host.argtypes = [ctypes.POINTER(Problem), ctypes.POINTER(Numerics), ctypes.c_int,
                                      ctypes.c_int32, _ip, _dp, _dp]
    lib.isrs_egn_eta_host.restype = ctypes.c_int
    lib.isrs_egn_last_kernel_ms.argtypes = [ctypes.c_void_p, _dp, _dp]
    lib.isrs_egn_last_kernel_ms.restype = ctypes.c_int
    lib.isrs_egn_nli_shard.argtypes = [ctypes.c_void_p, ctypes.c_int32, _ip, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_void_p, ctypes.c_void_p]
    lib.isrs_egn_nli_shard.restype = ctypes.c_int
    lib.isrs_egn_combine.argtypes = [ctypes.c_void_p, ctypes.c_int32, _ip, ctypes.c_int32, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    lib.isrs_egn_combine.restype = ctypes.c_int
    lib.isrs_egn_plan_shards.argtypes = [ctypes.POINTER(Problem), ctypes.POINTER(Numerics), ctypes.c_int32, _ip,
                                         ctypes.c_int32, _lp, _lp, _lp]
    lib.isrs_egn_plan_shards.restype = ctypes.c_int
    lib.isrs_egn_span_chains.argtypes = [ctypes.c_void_p, _ip, _ip, _ip]
    lib.isrs_egn_span_chains.restype = ctypes.c_int
    lib.isrs_egn_last_launch_count.argtypes = [ctypes.c_void_p]
    lib.isrs_egn_last_launch_count.restype = ctypes.c_int
    lib.isrs_egn_destroy.argtypes = [ctypes.c_void_p]
    lib.isrs_egn_destroy.restype = None
    lib.isrs_egn_strerror.argtypes = [ctypes.c_int]
    lib.isrs_egn_strerror.restype = ctypes.c_char_p
    lib.isrs_egn_last_error.argtypes = []
    lib.isrs_egn_last_error.restype = ctypes.c_char_p
    return lib


_LIB = None


def get():
    """The loaded libisrs_egn.so (loaded on first use; raises ImportError if it is not built)."""
    global _LIB
    if _LIB is None:
        _LIB = _load()
    return _LIB


def check(rc):
    if rc != OK:
        raise IsrsEgnError(rc, get().isrs_egn_last_error().decode())
    return rc


def _arr(x):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return a, a.ctypes.data_as(_dp)


class ProblemArrays:
    """Keeps the numpy arrays alive while a Problem struct points at them."""

    FIELDS = ("f_center_hz", "symbol_rate_hz", "launch_power_w", "excess_kurtosis", "psi",
              "length_m", "alpha_per_m", "beta2_s2_per_m", "beta3_s3_per_m", "gamma_per_w_m",
              "cr_per_w_m_hz")

    def __init__(self, link):
        src = dict(f_center_hz=link.f_center_hz, symbol_rate_hz=link.symbol_rate_hz,
                   launch_power_w=link.launch_power_w, excess_kurtosis=link.phi,
                   psi=getattr(link, "psi", None), length_m=link.length_m,
                   alpha_per_m=link.alpha_per_m, beta2_s2_per_m=link.beta2_s2_per_m,
                   beta3_s3_per_m=link.beta3_s3_per_m, gamma_per_w_m=link.gamma_per_w_m,
                   cr_per_w_m_hz=link.cr_per_w_m_hz)
        self._keep = {}
        ptrs = {}
        for k in self.FIELDS:
            if src[k] is None:
                ptrs[k] = _dp()
                continue
            a, p = _arr(src[k])
            self._keep[k] = a
            ptrs[k] = p
        self.struct = Problem(n_ch=len(self._keep["f_center_hz"]), n_span=len(self._keep["length_m"]),
                              **ptrs)

    def nbytes(self):
        return sum(a.nbytes for a in self._keep.values())


def numerics(grid_n, delta_z_m=1000.0, precision=64, mu_mode=MU_SEGMENT, flags=0, f_samples=0):
    return Numerics(grid_n=int(grid_n), delta_z_m=float(delta_z_m), precision=int(precision),
                    mu_mode=int(mu_mode), flags=int(flags), f_samples=int(f_samples))
