"""C-ABI library checks that need no GPU: it loads, exports every symbol include/isrs_egn.h
declares, and rejects invalid input with the documented status before touching CUDA."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "isrs_egn.h")


@pytest.fixture(scope="module")
def abi():
    from paper_2412_11614_b200 import build
    build.build()
    from paper_2412_11614_b200 import _abi
    return _abi


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"ISRS_EGN_API\s+[\w\s\*]*?\b(isrs_egn_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("isrs_egn_create", "isrs_egn_nli", "isrs_egn_destroy"):
        assert s in syms
    assert "isrs_egn_nli_split" in syms and len(syms) == 18


def test_library_exports_every_declared_symbol(abi):
    lib = ctypes.CDLL(abi.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert sorted(abi.EXPORTED) == declared_symbols()


def test_library_is_sm100a_only(abi):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_strerror(abi):
    assert abi.get().isrs_egn_strerror(0) == b"ok"
    assert abi.get().isrs_egn_strerror(-2) == b"channel bands overlap"


def _create(abi, link, **kw):
    pa = abi.ProblemArrays(link)
    n = abi.numerics(kw.get("grid_n", link.grid_n), kw.get("dz", 1000.0), kw.get("precision", 64),
                     kw.get("mu_mode", 0), 0, kw.get("f_samples", 0))
    h = ctypes.c_void_p()
    rc = abi.get().isrs_egn_create(ctypes.byref(pa.struct), ctypes.byref(n), 0, ctypes.byref(h))
    return rc, abi.get().isrs_egn_last_error().decode(), h


def test_validation_errors_before_any_cuda(abi):
    from workloads import tiny_link
    l = tiny_link(n_ch=3, n_span=2, grid_n=8)
    rc, msg, h = _create(abi, l, grid_n=7)
    assert rc == abi.EINVAL and "even" in msg and not h.value
    rc, msg, _ = _create(abi, l, dz=0.0)
    assert rc == abi.EINVAL and "delta_z" in msg
    rc, msg, _ = _create(abi, l, precision=16)
    assert rc == abi.EUNSUPPORTED
    odd = l.with_(symbol_rate_hz=np.array([64e9, 64e9 + 256 * 8, 64e9]))   # ratio ~ 3.1e7 : 3.1e7+1
    rc, msg, _ = _create(abi, odd, grid_n=8)
    assert rc == abi.EUNSUPPORTED and "ratio" in msg
    rc, msg, _ = _create(abi, l, f_samples=-1)
    assert rc == abi.EINVAL and "f_samples" in msg
    rc, msg, _ = _create(abi, l, f_samples=3)          # 64 GBd / 6 is not an integer (R3)
    assert rc == abi.EINVAL and "f_samples" in msg
    rc, msg, _ = _create(abi, l, precision=32, mu_mode=abi.MU_MACLAURIN)
    assert rc == abi.EUNSUPPORTED and "segment" in msg
    bad = l.with_(f_center_hz=l.f_center_hz + 0.25)
    rc, msg, _ = _create(abi, bad)
    assert rc == abi.EINVAL and "integer" in msg
    over = l.with_(symbol_rate_hz=np.full(3, 128e9))
    rc, msg, _ = _create(abi, over, grid_n=8)
    assert rc == abi.EOVERLAP and "overlap" in msg
    neg = l.with_(alpha_per_m=np.array([4.6e-5, 0.0]))
    rc, msg, _ = _create(abi, neg)
    assert rc == abi.EINVAL and "alpha_per_m[1]" in msg
    unsorted = l.with_(f_center_hz=l.f_center_hz[::-1].copy())
    rc, msg, _ = _create(abi, unsorted)
    assert rc == abi.EINVAL and "increasing" in msg
    lat = l.with_(symbol_rate_hz=np.full(3, 64e9 + 2))
    rc, msg, _ = _create(abi, lat)
    assert rc == abi.EINVAL and "2 grid_n" in msg
    # empty inputs and non-finite values
    empty = l.with_(f_center_hz=np.zeros(0), symbol_rate_hz=np.zeros(0), launch_power_w=np.zeros(0),
                    phi=np.zeros(0), psi=np.zeros(0))
    rc, msg, _ = _create(abi, empty)
    assert rc == abi.EINVAL and "n_ch" in msg
    nospan = l.with_(length_m=np.zeros(0), alpha_per_m=np.zeros(0), beta2_s2_per_m=np.zeros(0),
                     beta3_s3_per_m=np.zeros(0), gamma_per_w_m=np.zeros(0), cr_per_w_m_hz=np.zeros(0))
    rc, msg, _ = _create(abi, nospan)
    assert rc == abi.EINVAL and "n_span" in msg
    nan = l.with_(launch_power_w=np.array([1e-3, np.nan, 1e-3]))
    rc, msg, _ = _create(abi, nan)
    assert rc == abi.EINVAL and "launch_power_w[1]" in msg
    neg_cr = l.with_(cr_per_w_m_hz=np.array([2.8e-17, -1e-18]))
    rc, msg, _ = _create(abi, neg_cr)
    assert rc == abi.EINVAL and "cr_per_w_m_hz[1]" in msg
    rc, msg, _ = _create(abi, l, grid_n=8192)
    assert rc == abi.EINVAL and "4096" in msg
    rc, msg, _ = _create(abi, l, dz=1e-3)               # K_s = 8e7 segments
    assert rc == abi.ERANGE and "K_s" in msg


def test_destroy_null_safe(abi):
    abi.get().isrs_egn_destroy(None)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2412_11614_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+(oracle|workloads)\b", txt, re.M), f
    for dp, _, fs in os.walk(os.path.join(ROOT, "oracle")):
        for f in fs:
            if f.endswith(".py"):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+paper_2412_11614_b200\b", txt, re.M), f


def test_c_example_compiles_against_the_header_and_library(abi, tmp_path):
    """The boundary is usable from plain C: the example builds against include/isrs_egn.h and links
    libisrs_egn.so (it runs in tests/test_parity_gpu.py::test_c_example_matches_oracle)."""
    from _helpers import compile_c_example
    compile_c_example(str(tmp_path / "eta_c_abi"))


def test_problem_from_config_marshals_the_same_struct(tmp_path):
    """SURVEY 8(b) Python layer: Problem.from_config (dict / JSON string / JSON file, scalars repeated for
    n_span identical spans) hands the C ABI exactly the arrays of the equivalent workloads Link, and the
    host planner (no device) returns the same shard plan for both."""
    import json

    import paper_2412_11614_b200 as isrs
    from paper_2412_11614_b200._abi import ProblemArrays
    from workloads import tiny_link

    link = tiny_link(n_ch=4, rates_gbd=(32, 64), guard_ghz=12.5, n_span=3, grid_n=8, fmts=("qpsk", "16qam"))
    cfg = dict(f_center_hz=link.f_center_hz.tolist(), symbol_rate_hz=link.symbol_rate_hz.tolist(),
               launch_power_w=link.launch_power_w.tolist(), excess_kurtosis=link.phi.tolist(),
               psi=link.psi.tolist(), n_span=3, length_m=float(link.length_m[0]),
               alpha_per_m=float(link.alpha_per_m[0]), beta2_s2_per_m=float(link.beta2_s2_per_m[0]),
               beta3_s3_per_m=float(link.beta3_s3_per_m[0]), gamma_per_w_m=link.gamma_per_w_m.tolist(),
               cr_per_w_m_hz=link.cr_per_w_m_hz.tolist(), grid_n=8, delta_z_m=link.delta_z_m)
    path = tmp_path / "link.json"
    path.write_text(json.dumps(cfg))
    for src in (cfg, json.dumps(cfg), path, str(path)):
        p = isrs.Problem.from_config(src)
        a, b = ProblemArrays(p), ProblemArrays(link)
        assert a.struct.n_ch == b.struct.n_ch == 4 and a.struct.n_span == b.struct.n_span == 3
        for k in ProblemArrays.FIELDS:
            assert np.array_equal(a._keep[k], b._keep[k]), k
        assert isrs.Problem.from_config(json.dumps(p.to_config())).to_config() == p.to_config()
    for x, y in zip(isrs.plan_shards(p, 2), isrs.plan_shards(link, 2)):
        assert np.array_equal(x, y)
    with pytest.raises(ValueError):
        isrs.Problem.from_config({k: v for k, v in cfg.items() if k != "length_m"})
    with pytest.raises(ValueError):
        isrs.Problem.from_config(dict(cfg, alpha_db_km=0.2))
    with pytest.raises(ValueError):
        isrs.Problem.from_config(dict(cfg, length_m=[80e3, 80e3]))
