"""Parity of the CUDA path (through the C ABI) against the oracle, on the same seeded inputs.

Bar (BASELINE.json north_star): |eta_gpu - eta_oracle| / eta <= 1e-10 for every COI.
At full BASELINE sizes the oracle cannot finish whole configs, so the per-region partial
integrals written by the very nli() launch bench.py times are sampled and recomputed one by
one by the oracle.  Their tolerance is max(1e-10, 4 eps Theta_max): Theta_max is the largest
accumulated dispersion phase sum_s |chi_s| L_s in the region; a 1-ulp change of any input moves
Y there by ~eps Theta_max (SURVEY [X5b]), so no fp64 evaluation of Eqs. 8-22 is more
determined than that.  Whole-eta parity stays at 1e-10 on every config the
oracle finishes in seconds.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import egn, fwm  # noqa: E402
from workloads import bj_config, paper_analog, tiny_link  # noqa: E402

EPS = np.finfo(np.float64).eps
TOL_ETA = 1e-10


@pytest.fixture(scope="module")
def isrs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_11614_b200 import build
    build.build()
    import paper_2412_11614_b200 as m
    return m


def gpu_eta(isrs, link, coi=None, **kw):
    with isrs.Engine(link, **kw) as e:
        eta, terms = e.nli(coi=coi, terms=True)
        torch.cuda.synchronize()
        return eta.cpu().numpy(), terms.cpu().numpy()


TINY = {
    "uniform_64gbd_2span": dict(n_ch=3, rates_gbd=(64,), n_span=2, grid_n=8, fmts=("16qam",)),
    "three_islands_96gbd": dict(n_ch=4, rates_gbd=(96,), n_span=3, grid_n=8, fmts=("qpsk", "64qam")),
    "mixed_rates_guard": dict(n_ch=5, rates_gbd=(32, 64, 96), guard_ghz=12.5, n_span=2, grid_n=8,
                              fmts=("qpsk", "16qam", "64qam")),
    "touching_bands": dict(n_ch=4, rates_gbd=(32,), guard_ghz=0.0, n_span=2, grid_n=8,
                           fmts=("qpsk",)),
    "random_spans_multiclass": dict(n_ch=3, rates_gbd=(64, 32), guard_ghz=20.0, n_span=4, grid_n=8,
                                    random_spans=True, fmts=("16qam", "gauss")),
    "ragged_chunks_N34": dict(n_ch=2, rates_gbd=(68,), spacing_ghz=100.0, n_span=2, grid_n=34,
                              fmts=("64qam",), tilt_db=2.0),
    "single_channel_N64": dict(n_ch=1, rates_gbd=(64,), n_span=3, grid_n=64, fmts=("qpsk",)),
    "long_link_chained": dict(n_ch=3, rates_gbd=(96,), spacing_ghz=100.0, n_span=23, grid_n=8,
                              fmts=("16qam", "qpsk"), power_dbm=4.0),
    "strong_isrs": dict(n_ch=3, rates_gbd=(96,), spacing_ghz=100.0, n_span=2, grid_n=8,
                        cr_w_km_thz=5.0, power_dbm=12.0, fmts=("16qam",)),
}


def two_chain_groups_link():
    """Two runs of identical spans, each longer than one 800-segment chain: 12 x 80 km (chains of 10 + 2)
    then 14 x 60 km (13 + 1), so MODE_SEGGRP has two groups of two chains each (R13)."""
    link = tiny_link(n_ch=3, rates_gbd=(64,), n_span=26, grid_n=8, fmts=("16qam", "qpsk"))
    L = np.r_[np.full(12, 80e3), np.full(14, 60e3)]
    return link.with_(length_m=L)


def test_eta_parity_two_chain_groups(isrs):
    link = two_chain_groups_link()
    with isrs.Engine(link) as e:
        g = e.chain_groups()
        chains, _ = e.span_chains()
    assert list(chains) == [10, 2, 13, 1] and list(g) == [0, 2, 4]
    e_o, t_o = egn.eta(link)
    e_g, t_g = gpu_eta(isrs, link)
    assert np.all(np.abs(e_g - e_o) / e_o <= TOL_ETA), np.abs(e_g - e_o) / e_o
    scale = np.abs(t_o).sum(axis=1, keepdims=True)
    assert np.all(np.abs(t_g - t_o) <= TOL_ETA * scale)


@pytest.mark.parametrize("name", sorted(TINY))
def test_eta_parity_tiny(isrs, name):
    link = tiny_link(**TINY[name])
    e_o, t_o = egn.eta(link)
    e_g, t_g = gpu_eta(isrs, link)
    rel = np.abs(e_g - e_o) / e_o
    assert np.all(rel <= TOL_ETA), (name, rel)
    scale = np.abs(t_o).sum(axis=1, keepdims=True)
    assert np.all(np.abs(t_g - t_o) <= TOL_ETA * scale), (name, t_g, t_o)


EDGE = {
    # N = 2 (the smallest even grid), one channel
    "min_grid_N2": (dict(n_ch=1, rates_gbd=(64,), n_span=2, grid_n=2, fmts=("qpsk",)), {}),
    # N = 1024 single channel: the largest grid the oracle finishes in seconds (1 M points)
    "big_grid_N1024": (dict(n_ch=1, rates_gbd=(64,), n_span=1, grid_n=1024, fmts=("16qam",)), {}),
    # J = 2N - 1 = 519 lattice lines > LINE_CAP = 512: two line segments per region
    "two_line_segments_N260": (dict(n_ch=2, rates_gbd=(65,), spacing_ghz=100.0, n_span=1, grid_n=260,
                                    fmts=("qpsk",)), {}),
    # odd K (dz = 1100 m -> K = 73): no chains, odd-length recurrence
    "odd_K73": (dict(n_ch=3, rates_gbd=(64,), n_span=3, grid_n=8, fmts=("16qam",)), {"delta_z_m": 1100.0}),
    # K = 800 (dz = 100 m): only 3 table rows fit the envelope table, frequent rebuilds
    "large_K800": (dict(n_ch=2, rates_gbd=(64,), n_span=2, grid_n=8, fmts=("64qam",)), {"delta_z_m": 100.0}),
}


@pytest.mark.parametrize("name", sorted(EDGE))
def test_eta_parity_edge_cases(isrs, name):
    kw, num = EDGE[name]
    link = tiny_link(**kw)
    if "delta_z_m" in num:
        link = link.with_(delta_z_m=num["delta_z_m"])
    e_o, t_o = egn.eta(link)
    e_g, t_g = gpu_eta(isrs, link)
    assert np.all(np.abs(e_g - e_o) / e_o <= TOL_ETA), (name, np.abs(e_g - e_o) / e_o)
    scale = np.abs(t_o).sum(axis=1, keepdims=True)
    assert np.all(np.abs(t_g - t_o) <= TOL_ETA * scale), name


def random_tiny_kwargs(seed):
    """Seeded random small link: 1-5 channels with rates drawn from {16..96} GBd (lattice ratios up
    to 6:1), guard-packed (incl. touching bands) or on a uniform plan, 1-5 spans (identical or
    drawn), N in {8, 10, 16, 20}, dz in {1, 2.5, 5} km, C_r in {0, 0.028, 0.28} /W/km/THz, tilted
    powers, mixed formats."""
    rng = np.random.default_rng(1000 + seed)
    n_ch = int(rng.integers(1, 6))
    rates = tuple(int(x) for x in rng.choice([16, 32, 48, 64, 96], size=int(rng.integers(1, 4))))
    kw = dict(n_ch=n_ch, rates_gbd=rates, n_span=int(rng.integers(1, 6)),
              grid_n=int(rng.choice([8, 10, 16, 20])), random_spans=bool(rng.integers(0, 2)),
              cr_w_km_thz=float(rng.choice([0.0, 0.028, 0.28])), power_dbm=float(rng.uniform(-2, 4)),
              tilt_db=float(rng.uniform(-3, 3)), seed=seed,
              fmts=tuple(rng.choice(["gauss", "qpsk", "16qam", "64qam"], size=3)))
    if rng.integers(0, 2):
        kw["guard_ghz"] = float(rng.choice([0.0, 12.5, 25.0, 50.0]))
    else:
        kw["spacing_ghz"] = float(max(rates) + rng.choice([0, 4, 36]))
    return kw, float(rng.choice([1000.0, 2500.0, 5000.0]))


@pytest.mark.parametrize("seed", range(24))
def test_eta_parity_random_links(isrs, seed):
    kw, dz = random_tiny_kwargs(seed)
    link = tiny_link(**kw).with_(delta_z_m=dz)
    e_o, t_o = egn.eta(link)
    e_g, t_g = gpu_eta(isrs, link)
    rel = np.abs(e_g - e_o) / e_o
    assert np.all(rel <= TOL_ETA), (seed, kw, rel)
    scale = np.abs(t_o).sum(axis=1, keepdims=True)
    assert np.all(np.abs(t_g - t_o) <= TOL_ETA * scale), (seed, kw)


RANDOM_MODES = {
    # mode: (oracle kwargs, Engine kwargs builder, tolerance kind)
    "dedup": ({}, lambda m: {"flags": m.FLAG_DEDUP}, "rel"),
    "literal_gain": ({"gain": "literal"}, lambda m: {"flags": m.FLAG_LITERAL_GAIN}, "rel"),
    "maclaurin": ({"mu_mode": "maclaurin"}, lambda m: {"mu_mode": m.MU_MACLAURIN}, "rel"),
    "no_chain": ({}, lambda m: {"flags": m.FLAG_NO_CHAIN}, "rel"),
    "fp32": ({}, lambda m: {"precision": 32}, "db"),
    "3d_f2": ({"f_samples": 2}, lambda m: {"f_samples": 2}, "rel"),
    "mirror": ({}, lambda m: {"flags": m.FLAG_MIRROR}, "rel"),
    "mirror_3d": ({"f_samples": 2}, lambda m: {"flags": m.FLAG_MIRROR, "f_samples": 2}, "rel"),
}


@pytest.mark.parametrize("mode", sorted(RANDOM_MODES))
@pytest.mark.parametrize("seed", range(8))
def test_modes_parity_random_links(isrs, seed, mode):
    """Every option of the ABI on the seeded random links: the same oracle bar as its fixed tests."""
    kw, dz = random_tiny_kwargs(seed)
    link = tiny_link(**kw).with_(delta_z_m=dz)
    okw, ekw, kind = RANDOM_MODES[mode]
    e_o, _ = egn.eta(link, **okw)
    e_g, _ = gpu_eta(isrs, link, **ekw(isrs))
    if kind == "rel":
        assert np.all(np.abs(e_g - e_o) / e_o <= TOL_ETA), (seed, mode, np.abs(e_g - e_o) / e_o)
    else:
        assert np.all(np.abs(10 * np.log10(e_g / e_o)) <= 1e-3), (seed, mode, 10 * np.log10(e_g / e_o))


def test_degenerate_zero_gamma_and_empty_coi(isrs):
    """gamma = 0 in every span: Y = 0, eta = 0 exactly; an empty COI list is rejected."""
    link = tiny_link(n_ch=3, rates_gbd=(64,), n_span=2, grid_n=8, fmts=("16qam",))
    link = link.with_(gamma_per_w_m=np.zeros(2))
    e_g, t_g = gpu_eta(isrs, link)
    assert np.all(e_g == 0.0) and np.all(t_g == 0.0)
    with isrs.Engine(link) as e:
        with pytest.raises(isrs.IsrsEgnError):
            e.nli(coi=[])


def test_c_example_matches_oracle(isrs, tmp_path):
    """examples/eta_c_abi.c (plain C, no Python/PyTorch) through the C ABI against the oracle on the
    same 9-channel link it builds (16QAM, 3 x 80 km, N = 64)."""
    import subprocess
    from _helpers import compile_c_example
    exe = compile_c_example(str(tmp_path / "eta_c_abi"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = np.array([float(l.split()[3]) for l in r.stdout.splitlines() if l.startswith("channel")])
    link = tiny_link(n_ch=9, rates_gbd=(64,), spacing_ghz=100.0, n_span=3, grid_n=64, fmts=("16qam",))
    e_o, _ = egn.eta(link)
    assert got.shape == e_o.shape
    assert np.all(np.abs(got - e_o) / e_o <= TOL_ETA), np.abs(got - e_o) / e_o


def test_eta_parity_c1_full(isrs):
    link = bj_config("c1")
    e_o, t_o = egn.eta(link)
    e_g, t_g = gpu_eta(isrs, link)
    assert np.all(np.abs(e_g - e_o) / e_o <= TOL_ETA), (e_g, e_o)


def test_eta_parity_coi_subset_and_order(isrs):
    link = tiny_link(**TINY["mixed_rates_guard"])
    coi = [4, 0, 2]
    e_o, _ = egn.eta(link, coi=coi)
    e_g, _ = gpu_eta(isrs, link, coi=coi)
    assert np.all(np.abs(e_g - e_o) / e_o <= TOL_ETA)


def test_unit_link_hook_matches_closed_form(isrs):
    # pin P6 through the CUDA path: Y := 1, single channel
    for fmt, (phi, psi) in (("qpsk", (-1.0, 4.0)), ("16qam", (-0.68, 2.08))):
        link = tiny_link(n_ch=1, rates_gbd=(48,), n_span=1, grid_n=64, fmts=(fmt,))
        e_g, t_g = gpu_eta(isrs, link, flags=isrs.FLAG_UNIT_LINK)
        e_o, _ = egn.eta(link, mu_mode="unit")
        assert abs(e_g[0] - e_o[0]) <= 1e-13
        assert abs(e_g[0] - egn.unit_link_eta(phi, psi)) < 2e-5


def test_unit_link_maximum_grid_N4096(isrs):
    """Maximum grid (grid_n = 4096: 16.7 M points, 8191 lattice lines in 16 line segments, the
    coherent kernel's 64 KB row/column accumulators): with Y := 1 the D and H integrals are exact at
    every even N (pin P6), so the CUDA path must return 4/9 and Psi/9 to rounding."""
    link = tiny_link(n_ch=1, rates_gbd=(64,), n_span=1, grid_n=4096, fmts=("qpsk",))
    e_g, t_g = gpu_eta(isrs, link, flags=isrs.FLAG_UNIT_LINK)
    assert abs(t_g[0, 0] - 4.0 / 9.0) < 1e-12
    assert abs(t_g[0, 4] - 4.0 / 9.0) < 1e-12                   # Psi(QPSK) / 9 = 4/9
    assert abs(e_g[0] - egn.unit_link_eta(-1.0, 4.0)) < 1e-6    # E, F, G at O(h^2), h = R/4096


def test_maclaurin_mode_parity(isrs):
    link = tiny_link(**TINY["three_islands_96gbd"])
    e_o, _ = egn.eta(link, mu_mode="maclaurin")
    e_g, _ = gpu_eta(isrs, link, mu_mode=isrs.MU_MACLAURIN)
    assert np.all(np.abs(e_g - e_o) / e_o <= TOL_ETA)


def test_gn_reduction_bitwise_and_determinism(isrs):
    link = tiny_link(n_ch=3, rates_gbd=(64,), n_span=2, grid_n=16, fmts=("gauss",))
    e1, t1 = gpu_eta(isrs, link)
    e2, t2 = gpu_eta(isrs, link)
    assert np.array_equal(e1, e2) and np.array_equal(t1, t2)
    assert np.array_equal(e1, t1[:, 0]) and np.all(t1[:, 1:] == 0.0)
    lq = link.with_(phi=np.full(3, -0.68), psi=np.full(3, 2.08))
    _, tq = gpu_eta(isrs, lq)
    assert np.array_equal(tq[:, 0], t1[:, 0])


def test_errors_surface_from_nli(isrs):
    link = tiny_link(n_ch=3, n_span=1, grid_n=8)
    with isrs.Engine(link) as e:
        with pytest.raises(isrs.IsrsEgnError):
            e.nli(coi=[3])
    # K_s = 8000 segments (dz = 10 m) leaves no room for two envelope-table rows in shared memory
    with pytest.raises(isrs.IsrsEgnError, match="shared-memory"):
        isrs.Engine(link, delta_z_m=10.0)


# ------------------------------------------------------------------ full BASELINE sizes

def _golden_files():
    import glob
    import os
    here = os.path.dirname(os.path.abspath(__file__))
    return sorted(os.path.basename(f) for f in glob.glob(os.path.join(here, "golden", "c*_eta_fastplain*.json")))


@pytest.mark.parametrize("fname", _golden_files())
def test_whole_eta_full_size_matches_golden(isrs, fname):
    """North-star acceptance: whole eta (every requested COI, every region) of a BASELINE config at
    full size through the C ABI against the fast-plain oracle's values (tests/golden/, written by
    tests/tools/make_golden.py from oracle/ only; the fast-plain oracle is pinned to the literal
    closed mode at <= 1e-12).  Bar: |eta_gpu - eta_oracle| / eta <= 1e-10 for every COI, the D..H
    contributions within 1e-10 of the COI's total, exact in-support point counts."""
    import json
    import os
    sys_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tools")
    import sys
    sys.path.insert(0, sys_path)
    from make_golden import link_hash
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", fname)) as fh:
        g = json.load(fh)
    link = bj_config(g["config"])
    assert link_hash(link) == g["link_sha256"], "seeded workload drifted from the golden file"
    e_o, t_o, n_o = np.array(g["eta"]), np.array(g["terms"]), np.array(g["points"])
    with isrs.Engine(link) as e:
        eta, terms = e.nli(coi=g["coi"], terms=True)
        torch.cuda.synchronize()
        eta, terms = eta.cpu().numpy(), terms.cpu().numpy()
        pts = e.work()[0]
    rel = np.abs(eta - e_o) / e_o
    trel = np.abs(terms - t_o).max(axis=1) / np.abs(t_o).sum(axis=1)
    print(f"{fname}: {len(e_o)} COIs, max rel eta {rel.max():.3e}, mean {rel.mean():.3e}, "
          f"max rel terms {trel.max():.3e}")
    assert pts == int(n_o.sum())
    assert np.all(rel <= TOL_ETA), (fname, rel.max(), int(np.argmax(rel)))
    assert np.all(trel <= TOL_ETA), (fname, trel.max())

def theta_max(link, kappa, k1, k2):
    c = egn.canonicalize(link)
    F1, F2, _ = egn.region_points(c, kappa, k1, k2)
    th = 0.0
    for sp in c.spans:
        th = th + np.abs(fwm.chi(F1, F2, c.f[kappa], sp["beta2"], sp["beta3"])) * sp["L"]
    return float(np.max(th))


def sampled_regions(n, kappas):
    out = []
    for k in kappas:
        out += [(k, k, k), (k, min(k + 1, n - 1), k), (k, k, max(k - 1, 0)),
                (k, min(k + 3, n - 1), max(k - 2, 0)), (k, max(k - 5, 0), max(k - 5, 0))]
    return out


FULL = {
    "c2": (None, sampled_regions(40, (0, 19))),
    "c3": (None, sampled_regions(100, (50,))),
    "c4": (None, sampled_regions(80, (7, 41))),
    "c5": ([0, 100, 199], [(100, 100, 100), (100, 103, 98), (199, 199, 198), (0, 40, 0)]),
}


@pytest.mark.parametrize("cfg", sorted(FULL))
def test_full_size_region_parity(isrs, cfg):
    """Sampled per-region partial integrals at full size, written by the very nli() launch bench.py
    times, against egn.region_partials (the literal oracle) one region at a time.  Whole-eta parity
    at 1e-10 on every config is test_whole_eta_full_size_matches_golden; this test pins the per-region
    terms.  Tolerance per term: max(1e-10, 4 eps Theta_max) relative (reading R1: a region whose
    accumulated dispersion phase reaches Theta_max = max sum_s |chi_s| L_s is determined only to
    ~eps Theta_max -- the literal oracle forms theta in radians -- so no fp64 evaluation agrees better
    there), no absolute escape.  The observed errors are printed (pytest -s)."""
    link = bj_config(cfg)
    coi, regs = FULL[cfg]
    with isrs.Engine(link) as e:
        eta = e.nli(coi=coi)
        torch.cuda.synchronize()
        eta = eta.cpu().numpy()
        assert np.all(np.isfinite(eta)) and np.all(eta > 0)
        got = e.region_partials(regs)
        pts, pspans, nreg = e.work()
    assert pspans == pts * link.n_span and nreg > 0
    worst = 0.0
    for (kappa, k1, k2), g in zip(regs, got):
        want, npts = egn.region_partials(link, kappa, k1, k2)
        if npts == 0:      # empty region: either not listed (-1) or listed with no support
            assert g[5] in (0, -1) and np.all(g[:5] == 0.0) and np.all(want == 0.0)
            continue
        assert g[5] == npts, (cfg, kappa, k1, k2)
        th = theta_max(link, kappa, k1, k2)
        tol = max(TOL_ETA, 4 * EPS * th)
        rel = [abs(g[t] - want[t]) / abs(want[t]) if want[t] != 0.0 else abs(g[t]) for t in range(5)]
        print(f"{cfg} region {(kappa, k1, k2)}: Theta_max {th:.3g} rad, tol {tol:.2g}, "
              f"rel err D..H {['%.1e' % r for r in rel]}")
        worst = max(worst, max(rel) / tol)
        for t in range(5):
            if want[t] == 0.0:
                assert g[t] == 0.0, (cfg, (kappa, k1, k2), t, g[t])
            else:
                assert rel[t] <= tol, (cfg, (kappa, k1, k2), t, g[t], want[t], tol)
    print(f"{cfg}: worst error / tolerance {worst:.3g}")


@pytest.mark.parametrize("cfg,coi", [("c2", [0, 19, 39]), ("c5", [100])])
def test_span_chaining_matches_unchained(isrs, cfg, coi):
    """R9: chaining identical consecutive spans into one recurrence is the same sum (Eqs. 8, 22);
    it must agree with the per-span evaluation to the parity bar at full BASELINE sizes."""
    link = bj_config(cfg)
    a, ta = gpu_eta(isrs, link, coi=coi)
    b, tb = gpu_eta(isrs, link, coi=coi, flags=isrs.FLAG_NO_CHAIN)
    assert np.all(np.abs(a - b) / b <= TOL_ETA), (a, b, np.abs(a - b) / b)
    assert np.all(np.abs(ta - tb) <= TOL_ETA * np.abs(tb).sum(axis=1, keepdims=True))


@pytest.mark.parametrize("name", ["uniform_64gbd_2span", "three_islands_96gbd", "mixed_rates_guard",
                                  "touching_bands", "random_spans_multiclass"])
def test_eta_parity_3d_tiny(isrs, name):
    """NEXT-3: the 3-D form (f over the COI band, 4 midpoint samples) against the oracle."""
    link = tiny_link(**TINY[name])
    e_o, t_o = egn.eta(link, f_samples=4)
    e_g, t_g = gpu_eta(isrs, link, f_samples=4)
    assert np.all(np.abs(e_g - e_o) / e_o <= TOL_ETA), (name, np.abs(e_g - e_o) / e_o)
    scale = np.abs(t_o).sum(axis=1, keepdims=True)
    assert np.all(np.abs(t_g - t_o) <= TOL_ETA * scale)


def test_eta_parity_3d_c1(isrs):
    link = bj_config("c1")
    e_o, _ = egn.eta(link, coi=[0, 2], f_samples=4)
    e_g, _ = gpu_eta(isrs, link, coi=[0, 2], f_samples=4)
    assert np.all(np.abs(e_g - e_o) / e_o <= TOL_ETA), (e_g, e_o)


def test_unit_link_3d_through_cuda(isrs):
    # pin P14 through the CUDA path: D exact (2/3 R^2 (1 + 1/(2N^2))), eta -> 32/81 + 48/81 Phi + 4/45 Psi
    link = tiny_link(n_ch=1, rates_gbd=(48,), n_span=1, grid_n=32, fmts=("qpsk",))
    e_g, t_g = gpu_eta(isrs, link, flags=isrs.FLAG_UNIT_LINK, f_samples=32)
    e_o, t_o = egn.eta(link, mu_mode="unit", f_samples=32)
    assert abs(e_g[0] - e_o[0]) <= 1e-13 and np.all(np.abs(t_g - t_o) <= 1e-13)
    assert abs(t_g[0, 0] - 16.0 / 27.0 * 2.0 / 3.0 * (1.0 + 0.5 / 32 ** 2)) < 1e-13
    assert abs(e_g[0] - egn.unit_link_eta_3d(-1.0, 4.0)) < 2e-3


@pytest.mark.parametrize("cfg,coi,world", [("c1", None, 3), ("c2", None, 2), ("c2", [0, 19, 39], 4),
                                            ("c4", [7, 41], 3)])
def test_shards_combine_to_the_single_gpu_eta(isrs, cfg, coi, world):
    """shard r of `world` + all-gather + combine == the one-GPU eta (<= 1e-12; only the
    summation order differs), bitwise reproducible, and the shards' work adds up."""
    link = bj_config(cfg)
    with isrs.Engine(link) as e:
        full, tfull = e.nli(coi=coi, terms=True)
        pts_full = e.work()[0]
        sums, pts = [], 0
        for r in range(world):
            sums.append(e.nli_shard(r, world, coi=coi))
            pts += e.work()[0]
        g = torch.stack(sums)
        eta, terms = e.combine(g, coi=coi, terms=True)
        eta2 = e.combine(g.clone(), coi=coi)
        torch.cuda.synchronize()
        full, eta, eta2 = full.cpu().numpy(), eta.cpu().numpy(), eta2.cpu().numpy()
    assert pts == pts_full
    assert np.all(np.abs(eta - full) / full <= 1e-12), np.abs(eta - full) / full
    assert np.array_equal(eta, eta2)
    assert np.allclose(terms.cpu().numpy(), tfull.cpu().numpy(), rtol=1e-12, atol=1e-12 * np.abs(full).max())


@pytest.mark.parametrize("name", ["long_link_chained", "uniform_64gbd_2span", "random_spans_multiclass"])
def test_dedup_mode_parity_tiny(isrs, name):
    """NEXT-4a: span-class dedup (one K-segment sum x the phased-array factor) is the same Y."""
    link = tiny_link(**TINY[name])
    e_o, _ = egn.eta(link)
    e_g, _ = gpu_eta(isrs, link, flags=isrs.FLAG_DEDUP)
    assert np.all(np.abs(e_g - e_o) / e_o <= TOL_ETA), (name, np.abs(e_g - e_o) / e_o)


def test_dedup_closed_form_long_run_parity(isrs):
    """NEXT-4a on a run of 40 identical spans (> 32: the closed-form phased-array factor
    e^{i(G-1)chi L/2} sin(G chi L/2)/sin(chi L/2), with the product loop near rho = 1) against the
    oracle's span-by-span Eq. 22 sum and against the full GPU evaluation."""
    link = tiny_link(n_ch=3, rates_gbd=(96,), spacing_ghz=100.0, n_span=40, grid_n=8,
                     fmts=("16qam", "qpsk"), power_dbm=4.0)
    e_o, _ = egn.eta(link)
    e_d, _ = gpu_eta(isrs, link, flags=isrs.FLAG_DEDUP)
    e_f, _ = gpu_eta(isrs, link)
    assert np.all(np.abs(e_d - e_o) / e_o <= TOL_ETA), np.abs(e_d - e_o) / e_o
    assert np.all(np.abs(e_d - e_f) / e_f <= TOL_ETA), np.abs(e_d - e_f) / e_f


@pytest.mark.parametrize("cfg,coi", [("c2", None), ("c5", [100])])
def test_dedup_mode_matches_full_evaluation(isrs, cfg, coi):
    link = bj_config(cfg)
    a, _ = gpu_eta(isrs, link, coi=coi, flags=isrs.FLAG_DEDUP)
    b, _ = gpu_eta(isrs, link, coi=coi)
    assert np.all(np.abs(a - b) / b <= TOL_ETA), np.abs(a - b) / b


@pytest.mark.parametrize("name", ["long_link_chained", "random_spans_multiclass", "strong_isrs",
                                  "mixed_rates_guard"])
def test_literal_gain_parity_tiny(isrs, name):
    """NEXT-4b: Eq. 22's gain / sqrt(rho) products as printed (R11), against the oracle written
    literally from the products."""
    link = tiny_link(**TINY[name])
    e_o, t_o = egn.eta(link, gain="literal")
    e_g, t_g = gpu_eta(isrs, link, flags=isrs.FLAG_LITERAL_GAIN)
    assert np.all(np.abs(e_g - e_o) / e_o <= TOL_ETA), (name, np.abs(e_g - e_o) / e_o)
    e_i, _ = egn.eta(link)
    if name in ("strong_isrs", "long_link_chained"):
        assert np.max(np.abs(e_o - e_i) / e_i) > 1e-4      # the persistent tilt is visible


def test_literal_gain_chained_matches_unchained_c2(isrs):
    link = bj_config("c2")
    a, _ = gpu_eta(isrs, link, coi=[0, 19, 39], flags=isrs.FLAG_LITERAL_GAIN)
    b, _ = gpu_eta(isrs, link, coi=[0, 19, 39], flags=isrs.FLAG_LITERAL_GAIN | isrs.FLAG_NO_CHAIN)
    assert np.all(np.abs(a - b) / b <= TOL_ETA), np.abs(a - b) / b


@pytest.mark.parametrize("name", ["uniform_64gbd_2span", "strong_isrs", "mixed_rates_guard"])
def test_integral_form_parity_tiny(isrs, name):
    """NEXT-2: GPU Eq. 23 by the oracle's quadrature rule (C12) against oracle quad mode."""
    link = tiny_link(**TINY[name])
    e_o, _ = egn.eta(link, mu_mode="quad")
    e_g, _ = gpu_eta(isrs, link, mu_mode=isrs.MU_INTEGRAL)
    assert np.all(np.abs(e_g - e_o) / e_o <= TOL_ETA), (name, np.abs(e_g - e_o) / e_o)


def test_integral_form_vs_segment_c1_all_cois(isrs):
    """Pin P4 on BASELINE configs[0]: the segment closed form (dz = 1 km) within 0.001 dB MAE of the
    integral form (Eq. 23) for every COI of c1."""
    link = bj_config("c1")
    quad, _ = gpu_eta(isrs, link, mu_mode=isrs.MU_INTEGRAL)
    seg, _ = gpu_eta(isrs, link)
    err = np.abs(10 * np.log10(seg) - 10 * np.log10(quad))
    assert err.mean() < 1e-3 and err.max() < 2.7e-3, err


def test_integral_form_vs_segment_pa_ir(isrs):
    """P4 on the GPU at the paper's reduced Table-I analog (Delta-rho ~ 8.2 dB): the segment closed
    form (dz = 1 km) stays within the paper's MAE < 0.001 dB of the integral form, and the
    GPU integral form matches the oracle's quad mode on the sampled COIs."""
    link = paper_analog("Ir", fmt="qpsk")
    coi = [0, 7, 14]
    quad, _ = gpu_eta(isrs, link, coi=coi, mu_mode=isrs.MU_INTEGRAL)
    seg, _ = gpu_eta(isrs, link, coi=coi)
    err = np.abs(10 * np.log10(seg) - 10 * np.log10(quad))
    assert err.mean() < 1e-3 and err.max() < 2.7e-3, err
    e_o, _ = egn.eta(link, coi=[7], mu_mode="quad")
    assert abs(quad[1] - e_o[0]) / e_o[0] <= TOL_ETA


DB_TOL_FP32 = 1e-3     # north star: optional fp32 path within 0.001 dB


def _db(x):
    return 10.0 * np.log10(x)


@pytest.mark.parametrize("name", ["uniform_64gbd_2span", "three_islands_96gbd", "mixed_rates_guard",
                                  "strong_isrs", "long_link_chained", "single_channel_N64"])
def test_fp32_variant_vs_oracle_tiny(isrs, name):
    """Row a8: the mixed fp32 variant stays within 0.001 dB of the fp64 oracle."""
    link = tiny_link(**TINY[name])
    e_o, _ = egn.eta(link)
    e_g, _ = gpu_eta(isrs, link, precision=32)
    assert np.all(np.abs(_db(e_g) - _db(e_o)) <= DB_TOL_FP32), (name, _db(e_g) - _db(e_o))


@pytest.mark.parametrize("cfg,coi", [("c1", None), ("c2", None), ("c3", [0, 50, 99]), ("c4", [0, 40, 79]),
                                     ("c5", [0, 100, 199])])
def test_fp32_variant_vs_fp64_full_size(isrs, cfg, coi):
    """Row a8 at BASELINE sizes: |eta_fp32 - eta_fp64| <= 0.001 dB for every requested COI."""
    link = bj_config(cfg)
    a, _ = gpu_eta(isrs, link, coi=coi, precision=32)
    b, _ = gpu_eta(isrs, link, coi=coi)
    d = np.abs(_db(a) - _db(b))
    assert np.all(d <= DB_TOL_FP32), (cfg, d.max())


def test_streams_one_handle_and_two_handles(isrs):
    """Successive calls on one handle issued on different streams stay ordered on the device, and
    two handles run concurrently on two streams: every result equals its single-stream eta bitwise."""
    l1 = bj_config("c1")
    l2 = tiny_link(**TINY["mixed_rates_guard"])
    ref1, _ = gpu_eta(isrs, l1)
    ref2, _ = gpu_eta(isrs, l2)
    s = [torch.cuda.Stream() for _ in range(3)]
    with isrs.Engine(l1) as e1, isrs.Engine(l2) as e2:
        outs = []
        for i in range(6):
            outs.append((e1.nli(stream=s[i % 3]), e2.nli(stream=s[(i + 1) % 3]), e1.nli(coi=[0, 4], stream=s[(i + 2) % 3])))
        torch.cuda.synchronize()
        for a, b, c in outs:
            assert np.array_equal(a.cpu().numpy(), ref1)
            assert np.array_equal(b.cpu().numpy(), ref2)
            assert np.array_equal(c.cpu().numpy(), ref1[[0, 4]])


def test_graph_replay_equals_nli(isrs):
    """Engine.graph(): the captured call (fork, both integrand launches, join, reduce) replays to the
    same eta and D..H bitwise, repeatedly, for c1 and a multi-class tiny link with a COI subset."""
    for link, coi in ((bj_config("c1"), None), (tiny_link(**TINY["random_spans_multiclass"]), [2, 0])):
        ref, tref = gpu_eta(isrs, link, coi=coi)
        with isrs.Engine(link) as e:
            g = e.graph(coi=coi, terms=True)
            for _ in range(3):
                g.eta.zero_()
                eta, terms = g.replay()
                torch.cuda.synchronize()
                assert np.array_equal(eta.cpu().numpy(), ref)
                assert np.array_equal(terms.cpu().numpy(), tref)


def test_full_size_determinism_c2(isrs):
    link = bj_config("c2")
    with isrs.Engine(link) as e:
        a = e.nli().cpu().numpy()
        b = e.nli().cpu().numpy()
    assert np.array_equal(a, b)


def test_graph_then_direct_calls_on_other_streams(isrs):
    """after Engine.graph() the engine keeps working on any stream, last_kernel_ms()
    describes the last direct call, and calling the engine with another COI set does not disturb the
    graph (it owns a private handle)."""
    link = tiny_link(**TINY["mixed_rates_guard"])
    ref, _ = gpu_eta(isrs, link)
    with isrs.Engine(link) as e:
        g = e.graph(coi=[0, 2, 4])
        s = torch.cuda.Stream()
        a = e.nli(stream=s)                         # all COIs: a different set than the graph's
        b = e.nli(coi=[1, 3])                       # and another, on the default stream
        ms, ps = e.last_kernel_ms()
        assert ms[3] > 0 and ps[2] > 0
        for _ in range(2):
            eta = g.replay()
            torch.cuda.synchronize()
            assert np.array_equal(eta.cpu().numpy(), ref[[0, 2, 4]])
        torch.cuda.synchronize()
        assert np.array_equal(a.cpu().numpy(), ref)
        assert np.array_equal(b.cpu().numpy(), ref[[1, 3]])
        g.close()


def test_coi_set_changes_back_to_back_without_host_sync(isrs):
    """nli with a new COI set rebuilds its work list stream-ordered (no host or
    device synchronisation); several different sets issued back to back on one stream, and then on a
    second stream, each give the bitwise eta of a fresh call."""
    link = bj_config("c1")
    ref, tref = gpu_eta(isrs, link)
    sets = [[0, 1, 2, 3, 4], [3], [4, 0], [2, 1, 0], [1], [0, 1, 2, 3, 4]]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with isrs.Engine(link) as e:
        outs = [(c, e.nli(coi=c, terms=True, stream=s1 if i % 3 else s2)) for i, c in enumerate(sets * 2)]
        torch.cuda.synchronize()
        for c, (eta, terms) in outs:
            assert np.array_equal(eta.cpu().numpy(), ref[c])
            assert np.array_equal(terms.cpu().numpy(), tref[c])


def test_coi_set_changes_return_before_the_gpu_finishes(isrs):
    """Row b, "nli enqueues and returns": four calls with different COI sets (each rebuilds and uploads
    its work list) issued back to back on one busy stream come back to the host long before the GPU is
    done -- the uploads behind in-flight kernels are staged in pinned memory (a pageable source blocked
    the third call for the first one's whole duration, profiles/r02zt_async_probe.jsonl) -- and each
    gives the bitwise eta of a synchronised call."""
    import time
    link = bj_config("c3")
    sets = [[0, 50, 99], [1, 51], [2, 33, 98], [0, 50, 99], [3, 52]]
    st = torch.cuda.Stream()
    with isrs.Engine(link) as e:
        ref = []
        for c in sets:                               # warm-up + the synchronised values
            ref.append(e.nli(coi=c, stream=st))
            st.synchronize()
        t0 = time.perf_counter()
        outs = [e.nli(coi=c, stream=st) for c in sets]
        t_issue = time.perf_counter() - t0
        st.synchronize()
        t_all = time.perf_counter() - t0
        for a, b in zip(outs, ref):
            assert torch.equal(a, b)
    print(f"\nasync COI-set changes (c3, 5 calls): issued in {1e3 * t_issue:.1f} ms, finished after {1e3 * t_all:.1f} ms")
    assert t_issue < 0.15 * t_all, (t_issue, t_all)


def test_problem_from_config_runs_the_same_eta(isrs):
    """The binding's Problem.from_config (SURVEY 8(b) Python layer) drives the same hot path: eta is
    bitwise the Link's, through a JSON round trip."""
    import json
    link = tiny_link(**TINY["mixed_rates_guard"])
    ref, tref = gpu_eta(isrs, link)
    p = isrs.Problem.from_config(json.dumps(dict(
        f_center_hz=link.f_center_hz.tolist(), symbol_rate_hz=link.symbol_rate_hz.tolist(),
        launch_power_w=link.launch_power_w.tolist(), excess_kurtosis=link.phi.tolist(), psi=link.psi.tolist(),
        length_m=link.length_m.tolist(), alpha_per_m=link.alpha_per_m.tolist(),
        beta2_s2_per_m=link.beta2_s2_per_m.tolist(), beta3_s3_per_m=link.beta3_s3_per_m.tolist(),
        gamma_per_w_m=link.gamma_per_w_m.tolist(), cr_per_w_m_hz=link.cr_per_w_m_hz.tolist(),
        grid_n=link.grid_n, delta_z_m=link.delta_z_m)))
    eta, terms = gpu_eta(isrs, p)
    assert np.array_equal(eta, ref) and np.array_equal(terms, tref)
    assert np.array_equal(isrs.eta_host(p), ref)


def test_planned_work_equals_the_kernels_count(isrs):
    """isrs_egn_work (host planner, no device) = isrs_egn_last_work (the kernels' own count)."""
    for link, coi in ((bj_config("c1"), None), (tiny_link(**TINY["touching_bands"]), [1, 2]),
                      (tiny_link(**TINY["mixed_rates_guard"]), None)):
        with isrs.Engine(link) as e:
            plan = e.planned_work(coi)
            e.nli(coi=coi)
            assert e.work() == plan, (plan, e.work())


def test_capture_requires_an_existing_work_list(isrs):
    """A call that would have to allocate (new COI set) inside a stream capture fails cleanly with
    EINVAL instead of allocating in the graph; the handle stays usable."""
    link = bj_config("c1")
    ref, _ = gpu_eta(isrs, link)
    with isrs.Engine(link) as e:
        e.nli(coi=[0, 1])
        s = torch.cuda.Stream()
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        g = torch.cuda.CUDAGraph()
        with pytest.raises(Exception):
            with torch.cuda.graph(g, stream=s):
                e.nli_into(out.data_ptr(), 0, [3], s.cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(e.nli(coi=[3]).cpu().numpy(), ref[[3]])


@pytest.mark.parametrize("cfg", ["c2", "c4", "c5"])
def test_precompute_tables_match_the_oracle_profile(isrs, cfg):
    """Row a2 on its own: the create-time precompute kernel's zeta_k (Eq. 2 at z_k, Eq. 10) and
    ln c_k - alpha h k (Eq. 14's normalisation with the attenuation folded in) for every span class,
    against oracle.isrs.zeta / srs_gain at the same midpoints: <= 1e-14 relative."""
    from oracle import isrs as oisrs
    link = bj_config(cfg)
    c = egn.canonicalize(link)
    with isrs.Engine(link) as e:
        for s in range(link.n_span):
            la, ze = e.profile_tables(s)
            sp = c.spans[s]
            K = fwm.segment_count(sp["L"], c.dz)
            assert la.size == K
            h = sp["L"] / K
            zk = (np.arange(K) + 0.5) / K * sp["L"]
            z_o = oisrs.zeta(zk, sp["alpha"], c.p_tot, sp["cr"])
            # c_k = SRS_G(z_k, f3 = 0) (Eq. 14 at f3 = 0 is exactly the normalisation factor)
            c_o = oisrs.srs_gain(zk, 0.0, sp["alpha"], c.p_tot, sp["cr"], c.b_tot)
            assert np.all(np.abs(ze - z_o) <= 1e-14 * np.abs(z_o)), (cfg, s)
            lna_o = np.log(c_o) - sp["alpha"] * h * np.arange(K)
            assert np.all(np.abs(la - lna_o) <= 1e-14 * np.maximum(1.0, np.abs(lna_o))), (cfg, s)


@pytest.mark.parametrize("name", sorted(TINY))
def test_mirror_mode_parity_tiny(isrs, name):
    """ISRS_EGN_FLAG_MIRROR (f1 <-> f2 symmetry, pin P2): half the off-diagonal regions evaluated, the
    oracle's eta and D..H to the same bar."""
    link = tiny_link(**TINY[name])
    e_o, t_o = egn.eta(link)
    e_g, t_g = gpu_eta(isrs, link, flags=isrs.FLAG_MIRROR)
    assert np.all(np.abs(e_g - e_o) / e_o <= TOL_ETA), (name, np.abs(e_g - e_o) / e_o)
    scale = np.abs(t_o).sum(axis=1, keepdims=True)
    assert np.all(np.abs(t_g - t_o) <= TOL_ETA * scale), name


@pytest.mark.parametrize("cfg,coi", [("c2", None), ("c4", [0, 40, 79]), ("c5", [100])])
def test_mirror_mode_equals_full_evaluation(isrs, cfg, coi):
    link = bj_config(cfg)
    a, ta = gpu_eta(isrs, link, coi=coi, flags=isrs.FLAG_MIRROR)
    b, tb = gpu_eta(isrs, link, coi=coi)
    assert np.all(np.abs(a - b) / b <= 1e-12), np.abs(a - b) / b
    assert np.all(np.abs(ta - tb) <= 1e-12 * np.abs(tb).sum(axis=1, keepdims=True))
    with isrs.Engine(link, flags=isrs.FLAG_MIRROR) as e:
        e.nli(coi=coi)
        pts_eval = e.work()[0]
        pts_logical = e.planned_work(coi)[0]
        with pytest.raises(isrs.IsrsEgnError):
            e.nli_shard(0, 2, coi=coi)
    assert pts_eval < 0.6 * pts_logical          # about half the points evaluated


def test_mirror_mode_fp32(isrs):
    link = tiny_link(**TINY["mixed_rates_guard"])
    e_o, _ = egn.eta(link)
    e_g, _ = gpu_eta(isrs, link, precision=32, flags=isrs.FLAG_MIRROR)
    assert np.all(np.abs(10 * np.log10(e_g / e_o)) <= 1e-3)


# ---------------------------------------------------------------- SCI / XCI / MCI split (ISRS_EGN_FLAG_SPLIT)

def _split_links():
    d = {k: tiny_link(**TINY[k]) for k in ("uniform_64gbd_2span", "three_islands_96gbd", "mixed_rates_guard",
                                           "touching_bands", "random_spans_multiclass", "single_channel_N64",
                                           "long_link_chained", "ragged_chunks_N34")}
    d["two_chain_groups"] = two_chain_groups_link()          # MODE_SEGGRPSPL
    for seed in range(8):
        kw, dz = random_tiny_kwargs(seed)
        d[f"random{seed}"] = tiny_link(**kw).with_(delta_z_m=dz)
    return d


SPLIT_LINKS = _split_links()


def _check_split(isrs, link, f_samples=0):
    e_o, t_o, s_o = egn.eta(link, split=True, f_samples=f_samples)
    with isrs.Engine(link, flags=isrs.FLAG_SPLIT, f_samples=f_samples) as e:
        eta, parts, terms = e.nli_split(terms=True)
        torch.cuda.synchronize()
        assert e.work() == e.planned_work()
        assert e.last_launch_count() <= 4
    eta, parts, terms = eta.cpu().numpy(), parts.cpu().numpy(), terms.cpu().numpy()
    assert np.all(np.abs(eta - e_o) <= TOL_ETA * e_o), np.abs(eta - e_o) / e_o
    assert np.all(np.abs(parts - s_o) <= TOL_ETA * e_o[:, None]), (parts, s_o)
    assert np.all(np.abs(parts.sum(axis=1) - eta) <= 1e-13 * eta)
    assert np.all(np.abs(terms - t_o) <= TOL_ETA * np.abs(t_o).sum(axis=1, keepdims=True))
    if link.n_ch == 1:
        assert np.all(parts[:, 1:] == 0.0)
    if link.n_ch == 2:
        assert np.all(parts[:, 2] == 0.0)
    e_n, _ = gpu_eta(isrs, link, f_samples=f_samples)         # the unsplit work list: same eta
    assert np.all(np.abs(eta - e_n) <= 1e-12 * e_n)


@pytest.mark.parametrize("name", sorted(SPLIT_LINKS))
def test_sci_xci_mci_split_parity(isrs, name):
    """eta's SCI / XCI / MCI parts against the oracle's island-by-island classification (pin P17),
    <= 1e-10 of eta; parts sum to eta; eta equals the unsplit evaluation; the planner's point count of the
    split work list equals the kernels'."""
    _check_split(isrs, SPLIT_LINKS[name])


def test_sci_xci_mci_split_3d_and_errors(isrs):
    link = tiny_link(**TINY["three_islands_96gbd"])
    _check_split(isrs, link, f_samples=2)
    with isrs.Engine(link) as e:                               # not created with FLAG_SPLIT
        with pytest.raises(isrs.IsrsEgnError):
            e.nli_split()
    for bad in (isrs.FLAG_DEDUP, isrs.FLAG_MIRROR, isrs.FLAG_LITERAL_GAIN, isrs.FLAG_UNIT_LINK):
        with pytest.raises(isrs.IsrsEgnError):
            isrs.Engine(link, flags=isrs.FLAG_SPLIT | bad)
    with pytest.raises(isrs.IsrsEgnError):
        isrs.Engine(link, flags=isrs.FLAG_SPLIT, precision=32)
    with isrs.Engine(link, flags=isrs.FLAG_SPLIT) as e:
        with pytest.raises(isrs.IsrsEgnError):
            e.nli_shard(0, 2)
        ref, _ = gpu_eta(isrs, link)
        assert np.all(np.abs(e.nli().cpu().numpy() - ref) <= 1e-12 * ref)     # plain nli on a split handle
        e.nli(coi=[1])
        torch.cuda.synchronize()
        with isrs.Engine(link) as e0:
            e0.nli(coi=[1])
            torch.cuda.synchronize()
            q = [(1, 1, 1), (1, 0, 1), (1, 0, 2), (1, 2, 2)]
            a, b = e.region_partials(q), e0.region_partials(q)   # a region's two entries are summed
            assert np.allclose(a[:, :5], b[:, :5], rtol=1e-12, atol=0)


@pytest.mark.parametrize("cfg,coi", [("c2", [0, 19, 39]), ("c3", [0, 50, 99]), ("c4", [0, 40, 79]), ("c5", [100])])
def test_sci_xci_mci_split_full_size(isrs, cfg, coi):
    """At full size: eta of the split work list = eta of the headline path (<= 1e-12), the parts sum to it,
    and every class is populated (MCI dominates the count of regions, SCI is one island)."""
    link = bj_config(cfg)
    with isrs.Engine(link) as e:
        ref = e.nli(coi=coi).cpu().numpy()
        ms0 = e.last_kernel_ms()[0][3]
    with isrs.Engine(link, flags=isrs.FLAG_SPLIT) as e:
        eta, parts = e.nli_split(coi=coi)
        eta, parts = eta.cpu().numpy(), parts.cpu().numpy()
        ms1 = e.last_kernel_ms()[0][3]
    print(f"\n{cfg} split: integrand {ms1:.1f} ms vs {ms0:.1f} ms unsplit; SCI/XCI/MCI shares "
          f"{np.round(parts / eta[:, None], 4).tolist()}")
    assert np.all(np.abs(eta - ref) <= 1e-12 * ref)
    assert np.all(np.abs(parts.sum(axis=1) - eta) <= 1e-13 * eta)
    assert np.all(parts > 0)


@pytest.mark.parametrize("cfg,kappa", [("c2", 20), ("c3", 50), ("c4", 40), ("c5", 100)])
def test_sci_part_full_size_matches_the_oracle_island(isrs, cfg, kappa):
    """The split's values (not only their sum) at full size: the SCI part of a COI is the single island
    (kappa, kappa, kappa), which the literal oracle evaluates on its own in seconds -- at 96 GBd on
    100 GHz (c3, c5) the same region also holds the kappa3 = kappa +- 1 islands, which must NOT be in it."""
    link = bj_config(cfg)
    c = egn.canonicalize(link)
    isls = egn.region_islands(c, kappa, kappa, kappa, "closed", egn._needed_terms(c, kappa, kappa))
    own = [i for i in isls if i["k3"] == kappa]
    assert len(own) == 1 and (cfg in ("c2", "c4") or len(isls) == 3)
    scale = c.R[kappa] / c.P[kappa] ** 3
    sci = egn.island_contributions(c, kappa, kappa, own[0]).sum() * scale
    others = sum(egn.island_contributions(c, kappa, kappa, i).sum() for i in isls if i["k3"] != kappa) * scale
    with isrs.Engine(link, flags=isrs.FLAG_SPLIT) as e:
        eta, parts = e.nli_split(coi=[kappa])
        eta, parts = eta.cpu().numpy(), parts.cpu().numpy()
    rel = abs(parts[0, 0] - sci) / sci
    print(f"\n{cfg} COI {kappa}: SCI oracle {sci:.6e} gpu {parts[0, 0]:.6e} rel {rel:.1e}; the region's other "
          f"islands (XCI) are {others / sci:.3%} of it")
    assert rel <= TOL_ETA
