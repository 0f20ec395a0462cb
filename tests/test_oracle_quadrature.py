"""The oracle's quadrature of Eq. 23 (the integral form mu = int_0^L rho_s(z, f3) e^{i chi z} dz)
against two independent integrators, on the paper's Table-I and Table-II links and on c5's span
(reading R12 in DESIGN.md: the `quad` mode -- and the GPU's MU_INTEGRAL -- use a fixed composite
12-node Gauss-Legendre rule on quarter-period panels; SURVEY reading C12's adaptive Gauss-Kronrod 7/15
and Filon-type rules serve as the checks here):

  * fwm.mu_quad_adaptive -- adaptive Gauss-Kronrod 7/15 (C12), for |chi| L up to ~3e4 rad;
  * QUADPACK QAWO (scipy quad with a cos / sin weight) -- Clenshaw-Curtis with modified Chebyshev
    moments of the oscillatory weight, i.e. a Filon-type rule, which C12 asks for at |chi| L > 1e4 and
    which reaches c5's corner phases (|chi| L ~ 1e6 .. 1e7 rad per span).

Tolerance: every evaluation of e^{i chi z} rounds the phase chi z, an absolute error ~ eps |chi| z, so no
fp64 quadrature of Eq. 23 is better determined than ~eps |chi| L relative (the cancellation of the
oscillating integrand, |mu| ~ int rho / (|chi| / alpha), turns these absolute errors into relative ones);
the bar is max(2e-12, 8 eps |chi| L) (the largest ratio seen over these 107 points is ~5).
"""
import math

import numpy as np
import pytest

from oracle import egn, fwm, isrs
from workloads import bj_config, paper_analog

EPS = np.finfo(np.float64).eps


def _tol(ch, L):
    return max(2e-12, 8 * EPS * abs(ch) * L)


def _points(link, n, chil_max, seed, chil_min=0.0, span=0):
    c = egn.canonicalize(link)
    sp = c.spans[span]
    rng = np.random.default_rng(seed)
    pts = []
    while len(pts) < n:
        f1, f2 = rng.uniform(-c.b_tot / 2, c.b_tot / 2, 2)
        f = c.f[rng.integers(0, c.f.size)]
        chl = abs(fwm.chi(f1, f2, f, sp["beta2"], sp["beta3"])) * sp["L"]
        if chil_min <= chl <= chil_max:
            pts.append((f1, f2, f))
    return c, sp, pts


REGIMES = {
    # name: (link, points, max |chi| L)
    "PA-I_Cr1.12": (lambda: paper_analog("I", cr_w_km_thz=1.12), 28, 3e4),
    "PA-I_Cr0.28": (lambda: paper_analog("I", cr_w_km_thz=0.28), 20, 3e4),
    "PA-II_beta3": (lambda: paper_analog("II"), 28, 3e4),
    "c5_span_beta3": (lambda: bj_config("c5"), 28, 3e4),
}


def test_gk15_rule_exactness():
    """The Kronrod constants: K15 integrates x^d exactly up to d = 22, its Gauss subset G7 up to 13."""
    x, wk, wg = fwm._gk15_nodes()
    for d in range(23):
        assert abs((x ** d) @ wk - (1 + (-1) ** d) / (d + 1)) < 4e-16, d
    for d in range(14):
        assert abs((x ** d) @ wg - (1 + (-1) ** d) / (d + 1)) < 4e-16, d
    assert abs((x ** 14) @ wg - 2 / 15) > 1e-6         # and not beyond


@pytest.mark.parametrize("regime", sorted(REGIMES))
def test_fixed_rule_equals_adaptive_gk_and_qawo(regime):
    """104 points over the four regimes: fixed GL12 panels == adaptive GK 7/15 == QAWO."""
    from scipy.integrate import quad
    mk, n, chil_max = REGIMES[regime]
    c, sp, pts = _points(mk(), n, chil_max, seed=17 + sorted(REGIMES).index(regime))
    for f1, f2, f in pts:
        a1, a2 = np.array([f1]), np.array([f2])
        ch = fwm.chi(f1, f2, f, sp["beta2"], sp["beta3"])
        fixed = fwm.mu_quad(a1, a2, f, sp, c.p_tot, c.b_tot)[0]
        adapt = fwm.mu_quad_adaptive(a1, a2, f, sp, c.p_tot, c.b_tot)[0]

        def g(z):
            return float(isrs.rho(z, f1 + f2 - f, sp["alpha"], c.p_tot, sp["cr"], c.b_tot))
        with np.errstate(all="ignore"):
            import warnings
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                re = quad(g, 0, sp["L"], weight="cos", wvar=ch, epsabs=0, epsrel=1e-13, limit=2000)[0]
                im = quad(g, 0, sp["L"], weight="sin", wvar=ch, epsabs=0, epsrel=1e-13, limit=2000)[0]
        qawo = re + 1j * im
        tol = _tol(ch, sp["L"])
        assert abs(fixed - adapt) <= tol * abs(adapt), (regime, ch * sp["L"], abs(fixed - adapt) / abs(adapt))
        assert abs(fixed - qawo) <= tol * abs(qawo), (regime, ch * sp["L"], abs(fixed - qawo) / abs(qawo))


def test_fixed_rule_at_c5_corner_phases_equals_qawo():
    """c5's largest phases (|chi| L ~ 1e6 rad per span, 20 THz band): the fixed rule (>= 4 panels per
    period, ~1e6 panels) against QAWO's moment-based Filon-type rule."""
    from scipy.integrate import quad
    c, sp, pts = _points(bj_config("c5"), 3, 2.0e6, seed=5, chil_min=1.0e6)
    for f1, f2, f in pts:
        ch = fwm.chi(f1, f2, f, sp["beta2"], sp["beta3"])
        fixed = fwm.mu_quad(np.array([f1]), np.array([f2]), f, sp, c.p_tot, c.b_tot)[0]

        def g(z):
            return float(isrs.rho(z, f1 + f2 - f, sp["alpha"], c.p_tot, sp["cr"], c.b_tot))
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            re = quad(g, 0, sp["L"], weight="cos", wvar=ch, epsabs=0, epsrel=1e-13, limit=2000)[0]
            im = quad(g, 0, sp["L"], weight="sin", wvar=ch, epsabs=0, epsrel=1e-13, limit=2000)[0]
        qawo = re + 1j * im
        assert abs(fixed - qawo) <= _tol(ch, sp["L"]) * abs(qawo), (ch * sp["L"], abs(fixed - qawo) / abs(qawo))
        assert math.isfinite(abs(fixed))
