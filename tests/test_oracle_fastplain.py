"""Pins of the fast-plain oracle (oracle/fastplain.c) against the literal closed mode (oracle/egn.py).

The fast-plain variant is the same definition evaluated with a forward recurrence for e^{sigma k h},
the SRS gain tabulated per f3 of a region and mu computed once per distinct span parameter set
(SURVEY.md 8(d)).  It is what certifies whole-eta parity at the BASELINE configs' full sizes
(tests/golden/*_eta_fastplain.json), so it must agree with the literal path to <= 1e-12 (SURVEY 8(d):
"the two oracle variants must agree to <= 1e-12").
"""
import numpy as np
import pytest

from oracle import egn, fastplain, fwm
from workloads import bj_config, tiny_link

TOL = 1e-12
EPS = np.finfo(np.float64).eps

LINKS = {
    "uniform_64gbd_2span": dict(n_ch=3, rates_gbd=(64,), n_span=2, grid_n=8, fmts=("16qam",)),
    "three_islands_96gbd": dict(n_ch=4, rates_gbd=(96,), n_span=3, grid_n=8, fmts=("qpsk", "64qam")),
    "mixed_rates_guard": dict(n_ch=5, rates_gbd=(32, 64, 96), guard_ghz=12.5, n_span=2, grid_n=8,
                              fmts=("qpsk", "16qam", "64qam")),
    "touching_bands": dict(n_ch=4, rates_gbd=(32,), guard_ghz=0.0, n_span=2, grid_n=8, fmts=("qpsk",)),
    "random_spans_multiclass": dict(n_ch=3, rates_gbd=(64, 32), guard_ghz=20.0, n_span=4, grid_n=8,
                                    random_spans=True, fmts=("16qam", "gauss")),
    "ragged_N34_tilt": dict(n_ch=2, rates_gbd=(68,), spacing_ghz=100.0, n_span=2, grid_n=34,
                            fmts=("64qam",), tilt_db=2.0),
    "long_link_23_spans": dict(n_ch=3, rates_gbd=(96,), spacing_ghz=100.0, n_span=23, grid_n=8,
                               fmts=("16qam", "qpsk"), power_dbm=4.0),
    "strong_isrs": dict(n_ch=3, rates_gbd=(96,), spacing_ghz=100.0, n_span=2, grid_n=8,
                        cr_w_km_thz=5.0, power_dbm=12.0, fmts=("16qam",)),
    # C-band-like: 10 x 64 GBd at 100 GHz, 10 identical spans, 16QAM (c2's link at reduced size)
    "cband_10ch_10span": dict(n_ch=10, rates_gbd=(64,), spacing_ghz=100.0, n_span=10, grid_n=16,
                              fmts=("16qam",), power_dbm=1.0),
}


def _check(e_o, t_o, e_f, t_f, name):
    rel = np.abs(e_f - e_o) / e_o
    assert np.all(rel <= TOL), (name, rel)
    scale = np.abs(t_o).sum(axis=1, keepdims=True)
    assert np.all(np.abs(t_f - t_o) <= TOL * scale), (name, np.abs(t_f - t_o) / scale)


@pytest.mark.parametrize("name", sorted(LINKS))
def test_fastplain_equals_literal_closed_mode(name):
    link = tiny_link(**LINKS[name])
    e_o, t_o = egn.eta(link)
    e_f, t_f, npts = fastplain.eta(link)
    _check(e_o, t_o, e_f, t_f, name)
    assert np.all(npts > 0)


@pytest.mark.parametrize("seed", range(12))
def test_fastplain_equals_literal_on_random_links(seed):
    from test_parity_gpu import random_tiny_kwargs
    kw, dz = random_tiny_kwargs(seed)
    link = tiny_link(**kw).with_(delta_z_m=dz)
    e_o, t_o = egn.eta(link)
    e_f, t_f, _ = fastplain.eta(link)
    _check(e_o, t_o, e_f, t_f, seed)


def test_fastplain_equals_literal_c1_all_cois():
    link = bj_config("c1")
    e_o, t_o = egn.eta(link)
    e_f, t_f, npts = fastplain.eta(link)
    _check(e_o, t_o, e_f, t_f, "c1")


def test_fastplain_thread_count_does_not_change_eta():
    """Per-(COI, kappa1) task sums are combined in a fixed order: bitwise independent of threads."""
    link = tiny_link(**LINKS["cband_10ch_10span"])
    a = fastplain.eta(link, threads=1)
    b = fastplain.eta(link, threads=3)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def _theta_max(link, kappa, k1, k2):
    c = egn.canonicalize(link)
    F1, F2, _ = egn.region_points(c, kappa, k1, k2)
    th = 0.0
    for sp in c.spans:
        th = th + np.abs(fwm.chi(F1, F2, c.f[kappa], sp["beta2"], sp["beta3"])) * sp["L"]
    return float(np.max(th))


C2_REGIONS = [(19, 19, 19), (0, 0, 0), (39, 39, 39), (0, 39, 0), (19, 0, 39), (19, 39, 0), (19, 5, 33),
              (0, 20, 20)]


def test_fastplain_region_partials_c2_sampled():
    """Sampled regions of c2 (configs[1], full size) against egn.region_partials.  Regions near the
    COI's phase-matched axes (|chi| small, where eta lives) agree to 1e-12 per term.  Corner regions
    carry accumulated dispersion phase Theta up to 2.7e6 rad, which the literal path forms as a sum of
    chi_s L_s in radians (absolute phase error ~ eps Theta per point, reading R1) and the fast-plain
    path as a product of phasors: there the per-term agreement is bounded by 8 eps Theta_max, and their
    D_w is still within 1e-12 of the COI-centre region's D_w (the scale that reaches eta)."""
    link = bj_config("c2")
    ref_scale = None
    for reg in C2_REGIONS:
        w, n = egn.region_partials(link, *reg)
        f, m = fastplain.region_partials(link, *reg)
        assert n == m, reg
        if n == 0:
            assert np.all(w == 0.0) and np.all(f == 0.0)
            continue
        if ref_scale is None:
            ref_scale = w[0]            # the first listed region is the COI-centre one
        th = _theta_max(link, *reg)
        tol = TOL if th < 1e4 else max(TOL, 8 * EPS * th)
        for t in range(5):
            assert abs(f[t] - w[t]) <= tol * abs(w[t]), (reg, t, f[t], w[t], tol)
        assert abs(f[0] - w[0]) <= TOL * ref_scale, reg


def test_fastplain_rejects_an_inexact_lattice():
    """f3 must be exact on the integer-Hz lattice (C10); the library refuses otherwise."""
    link = tiny_link(n_ch=3, rates_gbd=(64,), n_span=1, grid_n=8)
    bad = link.with_(symbol_rate_hz=link.symbol_rate_hz + np.array([0.1, 0.2, 0.3]),
                     f_center_hz=link.f_center_hz + np.array([0.1, 0.37, 0.11]))
    with pytest.raises(RuntimeError):
        fastplain.eta(bad)
