"""Pins of the oracle against what the paper and the mathematics fix (no GPU).

Each test names the pin (this build's P14-P16) and the passage it follows.  A plausible
mistake in the oracle (dropped term, wrong sign or index, transposed operand) must fail
at least one of these.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import egn, formats, fwm, isrs, link as link_mod, units
from workloads import bj_config, paper_analog, tiny_link
from workloads import configs as wl

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_anchors.json")))

SPAN = dict(L=80e3, alpha=units.alpha_db_km_to_np_m(0.2), beta2=-2.168587e-26,
            beta3=1.447181e-40, gamma=1.3e-3, cr=2.8e-17)


def _rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.maximum(np.abs(b), 1e-300))


# ---------------------------------------------------------------- units, formats (C9, C15)

def test_units_cross_pin_with_workloads():
    b2, b3 = units.beta_from_dispersion(17.0, 0.067, 193.4e12)
    wb2, wb3 = wl.dispersion_to_beta(17.0, 0.067)
    assert abs(b2 - wb2) <= 1e-15 * abs(b2) and abs(b3 - wb3) <= 1e-15 * abs(b3)
    # SURVEY [X8]: -21.6859 ps^2/km, 0.14472 ps^3/km at lambda = c / 193.4 THz
    assert abs(b2 / 1e-27 - (-21.6859)) < 1e-3      # ps^2/km = 1e-24 s^2 / 1e3 m
    assert abs(b3 / 1e-39 - 0.14472) < 1e-4
    assert abs(units.alpha_db_km_to_np_m(0.2) - float(wl.db_per_km_to_per_m(0.2))) < 1e-20
    assert abs(units.dbm_to_watt(19.0) - 0.0794328) < 1e-6   # SPEC S:61 example


def test_phi_psi_from_constellations_match_inputs():
    # C9: Phi = E|a|^4/(E|a|^2)^2 - 2; BASELINE.json's kurtosis values -1, -0.68, -0.619
    qpsk = np.array([1 + 1j, 1 - 1j, -1 + 1j, -1 - 1j])
    p, s = formats.phi_psi(qpsk)
    assert abs(p + 1.0) < 1e-15 and abs(s - 4.0) < 1e-14
    p, s = formats.phi_psi(formats.square_qam(16))
    assert abs(p + 0.68) < 1e-14 and abs(s - 2.08) < 1e-13
    p, s = formats.phi_psi(formats.square_qam(64))
    assert abs(p - (-13.0 / 21.0)) < 1e-14 and abs(p - wl.FORMATS["64qam"][0]) < 1e-3
    assert abs(s - wl.FORMATS["64qam"][1]) < 1e-4
    assert formats.gaussian_moments_phi_psi() == (0.0, 0.0)
    # Monte-Carlo circular Gaussian -> Phi, Psi ~ 0
    rng = np.random.default_rng(0)
    g = rng.standard_normal(400000) + 1j * rng.standard_normal(400000)
    p, s = formats.phi_psi(g)
    assert abs(p) < 0.02 and abs(s) < 0.1


# ---------------------------------------------------------------- ISRS profile (P8)

@pytest.mark.parametrize("row", GOLDEN["delta_rho_db"])
def test_P8_delta_rho_printed_values(row):
    a = units.alpha_db_km_to_np_m(row["alpha_db_km"])
    v = isrs.delta_rho_db(row["z_km"] * 1e3, a, units.dbm_to_watt(row["p_tot_dbm"]),
                          units.cr_per_w_km_thz_to_si(row["cr_w_km_thz"]), row["b_tot_hz"])
    assert abs(v - row["value"]) <= GOLDEN["delta_rho_tolerance_db"], (v, row["cite"])


def test_P8_canonical_totals_of_table_I():
    # reading C5 on the paper's Table I link: P_tot is the SUM of the launch powers
    # (19 dBm total over 101 channels) and B_tot the edge-to-edge occupied band, which the paper
    # rounds to "B_tot = 1 THz"; with those totals Eq. 12 gives the printed 8.2 dB up to
    # that rounding
    link = paper_analog("I", cr_w_km_thz=1.12)
    c = egn.canonicalize(link)
    assert abs(10.0 * math.log10(c.p_tot / 1e-3) - 19.0) < 1e-9
    assert abs(c.b_tot - (100 * 10.1e9 + 10e9)) < 1.0 and abs(c.b_tot / 1e12 - 1.0) < 0.025
    v = isrs.delta_rho_db(100e3, c.spans[0]["alpha"], c.p_tot, c.spans[0]["cr"], c.b_tot)
    assert abs(v - 8.2) < 0.25, v


def test_P8_power_conservation_and_tilt():
    # (1/B) int_{-B/2}^{B/2} rho(z,f) df = e^{-alpha z} (sinh normalisation of Eq. 13/25)
    a, p, cr, B = units.alpha_db_km_to_np_m(0.2), 0.316, 2.8e-17, 20e12
    x, w = np.polynomial.legendre.leggauss(60)
    f = x * B / 2
    for z in (0.0, 1e3, 3e4, 8e4):
        avg = np.sum(w * isrs.rho(z, f, a, p, cr, B)) / 2
        assert abs(avg - math.exp(-a * z)) < 1e-13
    # the tilt between band edges equals zeta B nepers: ln(g(-B/2)/g(B/2)) = zeta B  (Eq. 14)
    z = 1e5
    g_lo = isrs.srs_gain(z, -B / 2, a, p, cr, B)
    g_hi = isrs.srs_gain(z, B / 2, a, p, cr, B)
    assert abs(math.log(g_lo / g_hi) - float(isrs.zeta(z, a, p, cr)) * B) < 1e-12
    # rho decreases in f when C_r > 0, is e^{-alpha z} flat when C_r = 0, rho(0, f) = 1
    r = isrs.rho(z, np.linspace(-B / 2, B / 2, 11), a, p, cr, B)
    assert np.all(np.diff(r) < 0)
    assert np.all(isrs.rho(z, np.linspace(-B / 2, B / 2, 11), a, p, 0.0, B) == math.exp(-a * z))
    assert np.all(isrs.rho(0.0, np.linspace(-B / 2, B / 2, 5), a, p, cr, B) == 1.0)


# ---------------------------------------------------------------- FWM factor (P1, P3, Eq. 9, Eq. 4)

def _points(n=200, B=4e12, seed=3):
    rng = np.random.default_rng(seed)
    return rng.uniform(-B / 2, B / 2, n), rng.uniform(-B / 2, B / 2, n), float(rng.uniform(-B / 4, B / 4))


def test_P1_segment_with_cr0_is_gn_closed_form():
    # BASELINE north_star / Eq. 6: with C_r = 0, sum_k I_k telescopes to (e^{(i chi - a)L} - 1)/(i chi - a)
    f1, f2, f = _points()
    sp = dict(SPAN, cr=0.0)
    mu = fwm.mu_segment(f1, f2, f, sp, 0.1, 4e12, 1000.0)
    ch = fwm.chi(f1, f2, f, sp["beta2"], sp["beta3"])
    gn = fwm.eta_gn(ch, sp["alpha"], sp["L"])
    assert _rel(mu, gn) < 1e-12
    # |mu|^2 = |(1 - e^{-aL + i chi L}) / (a - i chi)|^2 exactly as the north star states it
    ref = np.abs((1 - np.exp(-sp["alpha"] * sp["L"] + 1j * ch * sp["L"])) / (sp["alpha"] - 1j * ch)) ** 2
    assert _rel(np.abs(mu) ** 2, ref) < 1e-12
    # Maclaurin (Eq. 4) and quad (Eq. 23) reduce to the same closed form
    assert _rel(fwm.mu_maclaurin(f1, f2, f, sp, 0.1, 4e12), gn) < 1e-15
    assert _rel(fwm.mu_quad(f1[:20], f2[:20], f, sp, 0.1, 4e12), gn[:20]) < 1e-11


def test_P16_chi_is_the_taylor_phase_mismatch():
    # Eq. 5 abbreviates the FWM phase mismatch of the Taylor-expanded propagation
    # constant beta(w) = beta2 w^2/2 + beta3 w^3/6 (w = 2 pi f, offsets from f_c, reading C5):
    # chi = -(beta(w1) + beta(w2) - beta(w) - beta(w1 + w2 - w)) (sign as printed, reading C4).
    # Built here from beta itself, not from Eq. 5's factored form.
    f1, f2, f = _points(n=500, B=10e12, seed=11)
    b2, b3 = SPAN["beta2"], SPAN["beta3"]

    def beta(fr):
        w = 2.0 * math.pi * fr
        return b2 * w ** 2 / 2.0 + b3 * w ** 3 / 6.0
    mismatch = beta(f1) + beta(f2) - beta(f) - beta(f1 + f2 - f)
    scale = abs(b2) * (2.0 * math.pi * 10e12) ** 2
    ch = fwm.chi(f1, f2, f, b2, b3)
    assert np.allclose(ch, -mismatch, rtol=1e-9, atol=1e-12 * scale)
    # the beta3 part on its own (beta2 = 0): (w1 - w)(w2 - w)(w1 + w2) beta3 / 2
    ch3 = fwm.chi(f1, f2, f, 0.0, b3)
    w1, w2, w = 2 * math.pi * f1, 2 * math.pi * f2, 2 * math.pi * f
    assert np.allclose(ch3, (w1 - w) * (w2 - w) * (w1 + w2) * b3 / 2.0, rtol=1e-12, atol=0.0)


def test_P3_peak_efficiency_is_one():
    # P:65 Fig. 3: |mu| / L_eff = 1 at f1 = f2 = f (chi = 0), C_r = 0
    sp = dict(SPAN, cr=0.0, L=100e3)
    mu = fwm.mu_segment(np.array([0.3e12]), np.array([0.3e12]), 0.3e12, sp, 0.1, 1e12, 1000.0)
    leff = isrs.effective_length(sp["L"], sp["alpha"])
    assert abs(abs(mu[0]) / leff - GOLDEN["fwm_efficiency_peak"]["value"]) < 1e-13


def test_segment_terms_are_exact_piecewise_integrals():
    # Eq. 7 -> Eq. 8/9: with the envelope frozen at z_k on each sub-interval, the segment sum equals
    # the numerical integral of the piecewise-constant-envelope integrand (independent GL quadrature).
    f1, f2, f = _points(n=5)
    sp = dict(SPAN, L=10e3)
    p, B = 0.2, 4e12
    K = fwm.segment_count(sp["L"], 1000.0)
    ch = fwm.chi(f1, f2, f, sp["beta2"], sp["beta3"])
    x, w = np.polynomial.legendre.leggauss(20)
    h = sp["L"] / K
    nsub = 2048                                   # sub-panels per segment: < 1/4 period each
    hs = h / nsub
    acc = np.zeros(5, dtype=complex)
    for k in range(K):
        zk = (k + 0.5) * h
        z = (k * h + np.arange(nsub)[:, None] * hs + (x[None, :] + 1) * hs / 2).ravel()
        ww = np.tile(w * hs / 2, nsub)
        g = isrs.srs_gain(zk, f1 + f2 - f, sp["alpha"], p, sp["cr"], B)
        acc += g * (np.exp((1j * ch[:, None] - sp["alpha"]) * z[None, :]) @ ww)
    assert _rel(fwm.mu_segment(f1, f2, f, sp, p, B, 1000.0), acc) < 5e-11   # reference rounding ~ phase 3e4 rad
    assert K == 10 and fwm.segment_count(80e3, 1000.0) == 80 and fwm.segment_count(63457.0, 1000.0) == 64


def test_segment_converges_to_integral_form_as_dz_shrinks():
    # P:125 "The smaller the sampling step dz, the more accurate the approximation";
    # once chi dz << 2 pi the midpoint-envelope error falls as dz^2.
    sp = dict(SPAN, L=20e3, cr=1.12e-15)
    p, B = 0.0794, 1e12
    f1, f2, f = np.array([0.05e12]), np.array([-0.03e12]), 0.0
    q = fwm.mu_quad(f1, f2, f, sp, p, B)
    errs = [abs(fwm.mu_segment(f1, f2, f, sp, p, B, dz) - q)[0] for dz in (2000.0, 1000.0, 500.0, 250.0)]
    assert errs[0] > errs[1] > errs[2] > errs[3]
    assert 3.7 < errs[1] / errs[2] < 4.4 and 3.8 < errs[2] / errs[3] < 4.2
    assert errs[1] / abs(q[0]) < 2e-4


def test_maclaurin_is_exact_integral_of_first_order_profile():
    # Eq. 3 -> Eq. 4: mu_M = int_0^L (1 - zeta(z) f3) e^{-a z} e^{i chi z} dz (independent GL quadrature)
    f1, f2, f = _points(n=4, B=1e12)
    sp = dict(SPAN, L=30e3, cr=1.12e-15)
    p = 0.0794
    ch = fwm.chi(f1, f2, f, sp["beta2"], sp["beta3"])
    x, w = np.polynomial.legendre.leggauss(64)
    npan = 400
    h = sp["L"] / npan
    z = (np.arange(npan)[:, None] * h + (x[None, :] + 1) * h / 2).ravel()
    ww = np.tile(w * h / 2, npan)
    f3 = f1 + f2 - f
    integrand = (1 - isrs.zeta(z[None, :], sp["alpha"], p, sp["cr"]) * f3[:, None]) * \
        np.exp((1j * ch[:, None] - sp["alpha"]) * z[None, :])
    assert _rel(fwm.mu_maclaurin(f1, f2, f, sp, p, 1e12), integrand @ ww) < 1e-10


def test_quad_matches_scipy_qawo_on_sampled_points():
    # C12: cross-validate the composite GL quadrature of Eq. 23 against QUADPACK QAWO
    from scipy.integrate import quad
    sp = dict(SPAN, L=100e3, cr=1.12e-15, beta3=0.0)
    p, B = 0.0794, 1e12
    rng = np.random.default_rng(11)
    f1, f2 = rng.uniform(-B / 2, B / 2, 4), rng.uniform(-B / 2, B / 2, 4)
    f = 0.0
    ours = fwm.mu_quad(f1, f2, f, sp, p, B)
    ch = fwm.chi(f1, f2, f, sp["beta2"], sp["beta3"])
    for i in range(4):
        g = lambda z: float(isrs.rho(z, f1[i] + f2[i] - f, sp["alpha"], p, sp["cr"], B))
        re = quad(g, 0, sp["L"], weight="cos", wvar=ch[i], epsabs=0, epsrel=1e-13, limit=2000)[0]
        im = quad(g, 0, sp["L"], weight="sin", wvar=ch[i], epsabs=0, epsrel=1e-13, limit=2000)[0]
        assert abs(ours[i] - (re + 1j * im)) <= 1e-9 * abs(re + 1j * im)


def test_P2_f1_f2_symmetry():
    f1, f2, f = _points(n=50)
    mu_a = fwm.mu_segment(f1, f2, f, SPAN, 0.2, 4e12, 1000.0)
    mu_b = fwm.mu_segment(f2, f1, f, SPAN, 0.2, 4e12, 1000.0)
    # exact up to the rounding of chi's product order, amplified by the phase chi L (~1e4 rad here)
    assert _rel(mu_a, mu_b) < 1e-11
    spans = [SPAN, dict(SPAN, L=60e3, beta2=-2.0e-26)]
    ya = link_mod.link_function(f1, f2, f, spans, 0.2, 4e12, 1000.0)
    yb = link_mod.link_function(f2, f1, f, spans, 0.2, 4e12, 1000.0)
    # |Y| can be much smaller than the span terms it sums (phased array), so compare on their scale
    scale = sum(sp["gamma"] * np.abs(fwm.mu_segment(f1, f2, f, sp, 0.2, 4e12, 1000.0)) for sp in spans)
    assert np.max(np.abs(ya - yb) / scale) < 1e-10


# ---------------------------------------------------------------- link function (P7, C3)

def test_P7_phased_array_identity():
    # C3 (preceding-span phase): identical spans, C_r = 0 ->
    # |Y|^2 = gamma^2 |mu|^2 sin^2(Ns chi L/2) / sin^2(chi L/2);  chi = 0 -> Y = Ns gamma mu
    f1, f2, f = _points(n=64, B=1e12)
    sp = dict(SPAN, cr=0.0)
    for ns in (1, 2, 5):
        Y = link_mod.link_function(f1, f2, f, [sp] * ns, 0.1, 1e12, 1000.0)
        mu = fwm.mu_segment(f1, f2, f, sp, 0.1, 1e12, 1000.0)
        ch = fwm.chi(f1, f2, f, sp["beta2"], sp["beta3"])
        x = ch * sp["L"] / 2
        af = np.sin(ns * x) ** 2 / np.sin(x) ** 2
        assert _rel(np.abs(Y) ** 2, sp["gamma"] ** 2 * np.abs(mu) ** 2 * af) < 1e-9
    Y0 = link_mod.link_function(np.array([0.1e12]), np.array([0.1e12]), 0.1e12, [sp] * 4, 0.1, 1e12, 1000.0)
    mu0 = fwm.mu_segment(np.array([0.1e12]), np.array([0.1e12]), 0.1e12, sp, 0.1, 1e12, 1000.0)
    assert abs(Y0[0] - 4 * sp["gamma"] * mu0[0]) < 1e-13 * abs(Y0[0])


def test_link_phase_uses_preceding_spans_only():
    # two different spans: Y = g1 mu1 + g2 mu2 e^{i chi1 L1} (not e^{i(chi1 L1 + chi2 L2)})
    f1, f2, f = _points(n=8, B=1e12)
    s1, s2 = SPAN, dict(SPAN, beta2=-1.5e-26, L=50e3, gamma=1.1e-3)
    Y = link_mod.link_function(f1, f2, f, [s1, s2], 0.1, 1e12, 1000.0)
    m1 = fwm.mu_segment(f1, f2, f, s1, 0.1, 1e12, 1000.0)
    m2 = fwm.mu_segment(f1, f2, f, s2, 0.1, 1e12, 1000.0)
    c1 = fwm.chi(f1, f2, f, s1["beta2"], s1["beta3"])
    assert _rel(Y, s1["gamma"] * m1 + s2["gamma"] * m2 * np.exp(1j * c1 * s1["L"])) < 1e-14


# ---------------------------------------------------------------- geometry (P9), Eq. 16

@pytest.mark.parametrize("row", GOLDEN["eq16_island_counts"])
def test_P9_eq16_counts(row):
    assert len(egn.island_set_eq16(row["M"], row["kappa"])) == row["count"]


def test_generalised_islands_reduce_to_eq16_when_spacing_equals_R():
    # uniform plan with spacing = R (the paper's B_tot = (2M+1) R): our islands are Eq. 16's
    for M, kappa in ((1, 0), (1, 1), (2, -1)):
        l = tiny_link(n_ch=2 * M + 1, rates_gbd=(32,), guard_ghz=0.0, n_span=1, grid_n=8)
        got = sorted(set(egn.island_set_generalised(l, kappa + M)))
        want = sorted((k1 + M, k2 + M, k1 + k2 - kappa + ll + M)
                      for k1, k2, ll in egn.island_set_eq16(M, kappa))
        assert got == want
        # and the islands region_islands integrates are those same (k1, k2, k3)
        c = egn.canonicalize(l)
        integrated = sorted((k1, k2, isl["k3"]) for k1 in range(2 * M + 1) for k2 in range(2 * M + 1)
                            for isl in egn.region_islands(c, kappa + M, k1, k2, "unit"))
        assert integrated == want


def test_P9_only_l0_islands_when_R_below_two_thirds_spacing():
    # P:51 'B_ch <= 2/3 Delta f': every region then holds a single island (k3 = k1 + k2 - kappa)
    l = tiny_link(n_ch=5, rates_gbd=(64,), spacing_ghz=100.0, n_span=1, grid_n=8)
    for kappa in range(5):
        for k1, k2, k3 in egn.island_set_generalised(l, kappa):
            assert k3 == k1 + k2 - kappa
    # and l = +-1 islands do appear once R > 2/3 spacing (96 GBd at 100 GHz)
    l = tiny_link(n_ch=5, rates_gbd=(96,), spacing_ghz=100.0, n_span=1, grid_n=8)
    assert any(k3 != k1 + k2 - 2 for k1, k2, k3 in egn.island_set_generalised(l, 2))


def test_P9_max_phase_mismatch_geometry():
    # max |(f1 - f)(f2 - f)| over the domain = B^2/4 (centre, edge COI), 3 B^2/16 (quarter COI)
    n = 41
    l = tiny_link(n_ch=n, rates_gbd=(10,), guard_ghz=0.0, n_span=1, grid_n=8)
    c = egn.canonicalize(l)
    want = GOLDEN["max_abs_uv_over_btot2"]
    for kappa, key in ((n // 2, "coi_center"), (n // 4, "coi_quarter"), (0, "coi_edge")):
        best = 0.0
        for k1 in range(n):
            for k2 in range(n):
                F1, F2, f3 = egn.region_points(c, kappa, k1, k2)
                sup = (f3 >= c.lo.min()) & (f3 <= c.hi.max())
                if sup.any():
                    best = max(best, np.max(np.abs((F1 - c.f[kappa]) * (F2 - c.f[kappa]))[sup]))
        assert abs(best / c.b_tot ** 2 - want[key]) < 0.01, key


# ---------------------------------------------------------------- EGN assembly (P6, P10-P13)

@pytest.mark.parametrize("fmt", ["gauss", "qpsk", "16qam"])
def test_P6_unit_link_closed_form(fmt):
    # Appendix A of SURVEY (C2, C7, C10): single channel, Y := 1: eta = 4/9 + 56/81 Phi + Psi/9;
    # D and H exact at every even N (1/2 tie rule), E, F, G O(h^2).
    phi, psi = wl.FORMATS[fmt]
    errs = []
    for N in (16, 32, 64):
        l = tiny_link(n_ch=1, rates_gbd=(48,), n_span=1, grid_n=N, fmts=(fmt,))
        e, t = egn.eta(l, mu_mode="unit")
        errs.append(abs(e[0] - egn.unit_link_eta(phi, psi)))
        assert abs(t[0, 0] - 4.0 / 9.0) < 1e-14                    # D exact
        assert abs(t[0, 4] - psi / 9.0) < 1e-14                    # H exact
    assert errs[-1] < 2e-5
    if fmt != "gauss":
        assert 3.5 < errs[0] / errs[1] < 4.5 and 3.5 < errs[1] / errs[2] < 4.5


def test_P6_unit_link_raw_integrals():
    # D = 3/4 R^2, E = F = G = 7/12 R^3, H = 9/16 R^4 on the SCI hexagon
    R = 32e9
    l = tiny_link(n_ch=1, rates_gbd=(32,), n_span=1, grid_n=256, fmts=("qpsk",))
    c = egn.canonicalize(l)
    isl = egn.region_islands(c, 0, 0, 0, "unit")[0]
    assert abs(isl["D"] / R ** 2 - 0.75) < 1e-14
    assert abs(isl["H"] / R ** 4 - 9.0 / 16.0) < 1e-13
    for k in "EFG":
        assert abs(isl[k] / R ** 3 - 7.0 / 12.0) < 1e-5


def test_P6_two_rate_unit_link_coherent_axes():
    # C7 on a two-rate link with Y := 1 (geometry only): COI = the 32 GBd channel (R1), the other
    # channel 64 GBd (R0).  Region (kappa=1, k1=0, k2=1): f3 = f1 + (f2 - f) stays in band 0, so
    # the island is k3 = k1 (E gate); E is coherent over f1 at fixed f2:
    #   E = int_{-R1/2}^{R1/2} (R0 - |u|)^2 du = 2/3 (R0^3 - (R0 - R1/2)^3),  D = R0 R1 - R1^2/4.
    # Region (kappa=1, k1=1, k2=0) mirrors it with k3 = k2 (F gate), F coherent over f2 at fixed
    # f1 takes the same value.  Summing over the other axis would give (R0 - R1) R1^2 + 2/3 R1^3.
    R0, R1 = 64e9, 32e9
    l = tiny_link(n_ch=2, rates_gbd=(64, 32), spacing_ghz=100.0, n_span=1, grid_n=64, fmts=("qpsk",))
    c = egn.canonicalize(l)
    coh = 2.0 / 3.0 * (R0 ** 3 - (R0 - R1 / 2) ** 3)
    area = R0 * R1 - R1 ** 2 / 4
    (isl_e,) = egn.region_islands(c, 1, 0, 1, "unit")
    assert isl_e["k3"] == 0 and abs(isl_e["D"] / area - 1) < 1e-14
    assert abs(isl_e["E"] / coh - 1) < 1e-4 and isl_e["F"] == 0.0
    (isl_f,) = egn.region_islands(c, 1, 1, 0, "unit")
    assert isl_f["k3"] == 0 and abs(isl_f["D"] / area - 1) < 1e-14
    assert abs(isl_f["F"] / coh - 1) < 1e-4 and isl_f["E"] == 0.0


def test_P14_unit_link_3d_D_exact_discrete():
    # NEXT-3 (3-D form, Eqs. 17-21 integrate f over the COI band): single channel, Y := 1, n = N
    # f samples.  With f_m on the same bin-centre lattice, f3 = f1 + f2 - f_m is a bin centre (no
    # ties) and the island of f_m holds #{m1 + m2 - m in [0, N-1]} points; summing over m counts
    # every anti-diagonal s with weight n(s) = min(s, 2N-2-s) + 1 twice, so
    # mean_m D(f_m) = delta^2 sum_s n(s)^2 / N = (2/3) R^2 (1 + 1/(2 N^2))   (combinatorics, exact).
    R = 48e9
    for N in (8, 16, 32):
        l = tiny_link(n_ch=1, rates_gbd=(48,), n_span=1, grid_n=N, fmts=("qpsk",))
        c = egn.canonicalize(l)
        fs = egn.coi_frequencies(c, 0, N)
        D = np.mean([egn.region_islands(c, 0, 0, 0, "unit", f=f)[0]["D"] for f in fs])
        assert abs(D / R ** 2 - 2.0 / 3.0 * (1.0 + 0.5 / N ** 2)) < 1e-14


@pytest.mark.parametrize("fmt", ["qpsk", "16qam"])
def test_P14_unit_link_3d_closed_form(fmt):
    # continuous limit over the band (derivation in DESIGN.md P14): D(f) = 3/4 R^2 - f^2,
    # E(f) = F(f) = G(f) = 7/12 R^3 - R f^2, H(f) = (3/4 R^2 - f^2)^2; averaged over f:
    # 2/3 R^2, R^3/2, 9/20 R^4  ->  eta = 32/81 + 48/81 Phi + 4/45 Psi, reached at O(h^2).
    phi, psi = wl.FORMATS[fmt]
    errs = []
    for N in (8, 16, 32):
        l = tiny_link(n_ch=1, rates_gbd=(48,), n_span=1, grid_n=N, fmts=(fmt,))
        e, _ = egn.eta(l, mu_mode="unit", f_samples=N)
        errs.append(abs(e[0] - egn.unit_link_eta_3d(phi, psi)))
    assert errs[-1] < 1e-3
    assert 3.5 < errs[0] / errs[1] < 4.5 and 3.5 < errs[1] / errs[2] < 4.5, errs


# ---------------------------------------------------------------- NEXT-4b literal gain (R11)

def _pts(c, kappa=1, k1=0, k2=2, n=6):
    F1, F2, f3 = egn.region_points(c, kappa, k1, k2)
    return F1.ravel()[:n * 7:7], F2.ravel()[:n * 7:7], c.f[kappa]


def test_P15_literal_gain_reduces_to_ideal_at_cr0_and_one_span():
    # Eq. 22 as printed with g = e^{alpha L}: at C_r = 0, g rho = 1 (Eq. 25), so every product is 1;
    # with one span both products are empty.
    l0 = tiny_link(n_ch=3, rates_gbd=(64,), n_span=3, grid_n=8, cr_w_km_thz=0.0, random_spans=True)
    c0 = egn.canonicalize(l0)
    f1, f2, f = _pts(c0)
    a = link_mod.link_function(f1, f2, f, c0.spans, c0.p_tot, c0.b_tot, c0.dz, "closed", "literal")
    b = link_mod.link_function(f1, f2, f, c0.spans, c0.p_tot, c0.b_tot, c0.dz, "closed", "ideal")
    assert _rel(a, b) < 1e-13
    l1 = tiny_link(n_ch=3, rates_gbd=(64,), n_span=1, grid_n=8, cr_w_km_thz=1.0, power_dbm=10.0)
    c1 = egn.canonicalize(l1)
    f1, f2, f = _pts(c1)
    a = link_mod.link_function(f1, f2, f, c1.spans, c1.p_tot, c1.b_tot, c1.dz, "closed", "literal")
    b = link_mod.link_function(f1, f2, f, c1.spans, c1.p_tot, c1.b_tot, c1.dz, "closed", "ideal")
    assert np.array_equal(a, b)


def test_P15_literal_gain_span_ratio_is_the_srs_gain_at_f3():
    # identical spans: Lambda_{s+1} / Lambda_s = g^{3/2} sqrt(rho(f1) rho(f3) rho(f2)) / (g^{1/2} sqrt(rho(f)))
    # = c e^{-zeta (f1 + f2 + f3 - f) / 2} = c e^{-zeta f3} (f1 + f2 = f3 + f): the SRS gain at the
    # end of a span, Eq. 14 at z = L and frequency f1 + f2 - f.  Evaluated here from Eq. 14 directly.
    l = tiny_link(n_ch=3, rates_gbd=(96,), n_span=3, grid_n=8, cr_w_km_thz=1.0, power_dbm=12.0)
    c = egn.canonicalize(l)
    f1, f2, f = _pts(c)
    lam = link_mod._gain_products(f1, f2, f, c.spans, c.p_tot, c.b_tot)
    sp = c.spans[0]
    zeta = c.p_tot * sp["cr"] * (1.0 - math.exp(-sp["alpha"] * sp["L"])) / sp["alpha"]
    x = c.b_tot * zeta
    want = x / (2.0 * math.sinh(x / 2.0)) * np.exp(-zeta * (f1 + f2 - f))
    assert _rel(lam[1] / lam[0], want) < 1e-12 and _rel(lam[2] / lam[1], want) < 1e-12
    assert np.any(np.abs(want - 1.0) > 1e-3)      # the tilt is not negligible here


def test_P10_grid_convergence_order_two():
    # single 10 GBd channel, 1 span: successive differences fall ~4x per halving of delta (midpoint rule)
    vals = []
    for N in (8, 16, 32, 64):
        l = tiny_link(n_ch=1, rates_gbd=(10,), n_span=1, grid_n=N, fmts=("gauss",), length_km=30.0)
        vals.append(egn.eta(l)[0][0])
    d = np.abs(np.diff(vals))
    p = np.log2(d[:-1] / d[1:])
    assert np.all(np.abs(p - 2.0) < 0.3), p


def test_P11_mirror_symmetry():
    # C_r = 0, beta3 = 0, uniform plan and power -> eta_k = eta_{-k} (needs the 1/2 tie rule, C10)
    l = tiny_link(n_ch=5, rates_gbd=(96,), spacing_ghz=100.0, n_span=2, grid_n=8, cr_w_km_thz=0.0,
                  s=0.0, d=17.0, fmts=("16qam",))
    l = l.with_(beta3_s3_per_m=np.zeros(2))
    e, _ = egn.eta(l)
    assert _rel(e, e[::-1]) < 1e-12
    # touching bands exercise the shared-edge split
    l2 = tiny_link(n_ch=3, rates_gbd=(32,), guard_ghz=0.0, n_span=1, grid_n=8, cr_w_km_thz=0.0,
                   fmts=("qpsk",)).with_(beta3_s3_per_m=np.zeros(1))
    e2, _ = egn.eta(l2)
    assert _rel(e2, e2[::-1]) < 1e-12


def test_P12_gn_reduction_bitwise():
    # Phi = Psi = 0 -> only D is evaluated; the D part does not depend on the format
    base = tiny_link(n_ch=3, rates_gbd=(64,), n_span=2, grid_n=8, fmts=("gauss",))
    e_g, t_g = egn.eta(base)
    assert np.array_equal(e_g, t_g[:, 0]) and np.all(t_g[:, 1:] == 0.0)
    e_q, t_q = egn.eta(base.with_(phi=np.full(3, -0.68), psi=np.full(3, 2.08)))
    assert np.array_equal(t_q[:, 0], t_g[:, 0])


def test_P13_modulation_correction_sign():
    # eta_QPSK < eta_Gauss at equal power (Phi < 0 corrections dominate)
    base = tiny_link(n_ch=3, rates_gbd=(64,), n_span=3, grid_n=8, fmts=("gauss",))
    e_g, _ = egn.eta(base)
    e_q, t_q = egn.eta(base.with_(phi=np.full(3, -1.0), psi=np.full(3, 4.0)))
    assert np.all(e_q < e_g)
    assert np.all(t_q[:, 1] <= 0) and np.all(t_q[:, 2] <= 0) and np.all(t_q[:, 3] <= 0)


def test_region_partials_consistent_with_eta():
    # the per-region weighted partials (what the CUDA path writes) re-assemble to eta
    l = tiny_link(n_ch=3, rates_gbd=(64, 96), spacing_ghz=100.0, n_span=2, grid_n=8,
                  fmts=("qpsk", "16qam", "gauss"))
    c = egn.canonicalize(l)
    e, t, regs = egn.eta(l, return_regions=True)
    for ci, kappa in enumerate(range(3)):
        acc = 0.0
        for (kk, k1, k2) in regs:
            if kk != kappa:
                continue
            (Dw, Ew, Fw, Gw, Hw), _ = egn.region_partials(l, kappa, k1, k2)
            G1, G2, R1, R2 = c.G[k1], c.G[k2], c.R[k1], c.R[k2]
            acc += (16 / 27 * G1 * G2 * Dw + 16 / 27 * c.phi[k1] * G1 ** 2 * G2 * Ew / R1
                    + 32 / 81 * c.phi[k2] * G2 ** 2 * G1 * Fw / R2 + 16 / 81 * c.phi[k1] * G1 ** 2 * Gw / R1
                    + 16 / 81 * c.psi[k1] * G1 ** 3 * Hw / R1 ** 2)
        acc *= c.R[kappa] / c.P[kappa] ** 3
        assert abs(acc - e[ci]) < 1e-12 * e[ci]


def test_c1_config_shape_and_values_finite():
    l = bj_config("c1")
    assert l.n_ch == 5 and l.grid_n == 64 and l.n_span == 1
    c = egn.canonicalize(l)
    assert abs(c.b_tot - 464e9) < 1 and abs(c.f_c - 193.4e12) < 1


SUPPORT_LINKS = {
    # touching bands: regions whose f3 range ends exactly on a band edge (tie points, t = 1/2)
    "touching_32": dict(n_ch=4, rates_gbd=(32,), guard_ghz=0.0, n_span=1, grid_n=8, fmts=("qpsk",)),
    "touching_mixed": dict(n_ch=5, rates_gbd=(48, 16, 96), guard_ghz=0.0, n_span=1, grid_n=4,
                           fmts=("16qam",)),
    # mixed rates with guards: a:b lattices, regions clipped at a band by one bin
    "mixed_guard": dict(n_ch=5, rates_gbd=(32, 64, 96), guard_ghz=12.5, n_span=1, grid_n=8,
                        fmts=("qpsk", "64qam")),
    "uniform_spacing_eq_R": dict(n_ch=5, rates_gbd=(50,), spacing_ghz=50.0, n_span=1, grid_n=2,
                                 fmts=("qpsk",)),
}


@pytest.mark.parametrize("name", sorted(SUPPORT_LINKS))
def test_support_bound_filter_drops_only_empty_regions(name, monkeypatch):
    """egn.has_support_bound (a cheap necessary condition for a region to hold an island, Eq. 16
    generalised) must never drop a region with support: eta and every D..H term with the
    filter equal, bitwise, the brute force over every (kappa1, kappa2) pair; and the filter keeps
    exactly the regions that have a point with f3 in some closed band (C10)."""
    link = tiny_link(**SUPPORT_LINKS[name])
    e1, t1 = egn.eta(link)
    c = egn.canonicalize(link)
    kept = {(k, a, b) for k in range(link.n_ch) for a in range(link.n_ch) for b in range(link.n_ch)
            if egn.has_support_bound(c, k, a, b)}
    monkeypatch.setattr(egn, "has_support_bound", lambda *a, **kw: True)
    e2, t2 = egn.eta(link)
    assert np.array_equal(e1, e2) and np.array_equal(t1, t2), (name, e1, e2)
    for k in range(link.n_ch):
        for a in range(link.n_ch):
            for b in range(link.n_ch):
                _, _, f3 = egn.region_points(c, k, a, b)
                has = any(np.any((f3 >= c.lo[i]) & (f3 <= c.hi[i])) for i in range(link.n_ch))
                assert has == ((k, a, b) in kept), (name, k, a, b, has)


# ---------------------------------------------------------------- SCI / XCI / MCI split

def test_P17_sci_xci_mci_split():
    """SCI = the COI alone, XCI = one interfering channel, MCI = two or three.  Pins: the three
    parts sum to eta; a single channel has only SCI; two channels have no MCI (only one interferer
    exists) but do have XCI; with C_r = 0 the SCI of the middle channel of a symmetric 3-channel link
    (same band centre f_c, no ISRS coupling to the neighbours) IS the eta of that channel alone --
    although at 96 GBd on 100 GHz its (kappa, kappa) region also holds kappa3 = kappa +- 1 islands,
    which are XCI; and the split of Eq. 16's island set for M = 1, kappa = 0 counted by hand."""
    kw = dict(rates_gbd=(96,), spacing_ghz=100.0, n_span=2, grid_n=8, fmts=("16qam",))
    l3 = tiny_link(n_ch=3, **kw)
    e, t, s = egn.eta(l3, split=True)
    assert np.allclose(s.sum(axis=1), e, rtol=1e-13, atol=0)
    assert np.all(s > 0)
    e1, _, s1 = egn.eta(tiny_link(n_ch=1, **kw), split=True)
    assert s1[0, 1] == 0.0 and s1[0, 2] == 0.0 and s1[0, 0] == e1[0]
    e2, _, s2 = egn.eta(tiny_link(n_ch=2, **kw), split=True)
    assert np.all(s2[:, 2] == 0.0) and np.all(s2[:, 1] > 0)
    # C_r = 0: SCI of the middle channel = eta of that channel alone (same f_c)
    l3n = l3.with_(cr_per_w_m_hz=np.zeros(2))
    mid = l3n.with_(f_center_hz=l3n.f_center_hz[1:2], symbol_rate_hz=l3n.symbol_rate_hz[1:2],
                    launch_power_w=l3n.launch_power_w[1:2], phi=l3n.phi[1:2], psi=l3n.psi[1:2])
    _, _, s3 = egn.eta(l3n, coi=[1], split=True)
    e_mid, _ = egn.eta(mid)
    assert abs(s3[0, 0] - e_mid[0]) <= 1e-13 * e_mid[0]
    isl = egn.island_set_generalised(l3n, 1)                   # the (1, 1) region holds three islands
    assert sorted(k3 for k1, k2, k3 in isl if k1 == k2 == 1) == [0, 1, 2]
    # Eq. 16 with M = 1, kappa = 0 (channels -1, 0, 1), by hand: of its 19 islands (k1, k2, k3 = k1+k2+l)
    # 1 is SCI (0,0,0); XCI are the islands over {0, j} with j = +-1 present: (0,0,j), (0,j,0), (j,0,0),
    # (0,j,j), (j,0,j), (j,j,0)*, (j,j,j) -- (j,j,0) needs l = -2j, not in {-1,0,1} -- so 6 per j = 12
    cnt = [0, 0, 0]
    for k1, k2, ll in egn.island_set_eq16(1, 0):
        cnt[egn.nli_class(0, k1, k2, k1 + k2 - 0 + ll)] += 1
    assert cnt == [1, 12, 6]
