"""FWM efficiency factor mu_s(f1, f2, f) (oracle; test infrastructure only).

PAPER.md §II.C and Appendix B:
  Eq. 5  chi = 4 pi^2 (f1 - f)(f2 - f) [beta2 + pi beta3 (f1 + f2)]
  Eq. 6  eta = (e^{(i chi - alpha) L} - 1) / (i chi - alpha)          (GN, C_r = 0)
  Eq. 4  Maclaurin:  mu ~ eta - P C (f1+f2-f)/alpha (eta - (e^{(i chi - 2 alpha)L} - 1)/(i chi - 2 alpha))
  Eq. 7-10 segment:  mu ~ sum_k SRS_G(z_k, f1+f2-f) I_k,
          I_k = (e^{(i chi - alpha)(k+1)L/K} - e^{(i chi - alpha) k L/K}) / (i chi - alpha),  z_k = (k+0.5)L/K
  Eq. 23/24 integral form: mu = int_0^L rho_s(z, f1+f2-f) e^{i phi_s} dz, phi_s = chi z
K = ceil(L/dz).  All frequencies are offsets from f_c (reading C5); the sign of chi
follows Eq. 5 (reading C4: eta is invariant under chi -> -chi).
All functions are vectorised over point arrays f1, f2 (same shape); f is a scalar.
"""
import math

import numpy as np

from . import isrs


def chi(f1, f2, f, beta2, beta3):
    """Eq. 5 / Eq. 24: phase-mismatch rate [rad/m]."""
    return 4.0 * math.pi ** 2 * (f1 - f) * (f2 - f) * (beta2 + math.pi * beta3 * (f1 + f2))


def eta_gn(ch, alpha, L):
    """Eq. 6: (e^{(i chi - alpha) L} - 1) / (i chi - alpha)."""
    sig = 1j * ch - alpha
    return (np.exp(sig * L) - 1.0) / sig


def segment_count(L, dz):
    """K = ceil(L_s / dz)."""
    return int(math.ceil(L / dz))


def mu_segment(f1, f2, f, span, p_tot, b_tot, dz):
    """Eqs. 8-10, evaluated literally term by term (no recurrence, no tables)."""
    L, alpha = span["L"], span["alpha"]
    K = segment_count(L, dz)
    ch = chi(f1, f2, f, span["beta2"], span["beta3"])
    f3 = f1 + f2 - f
    sig = 1j * ch - alpha
    mu = np.zeros(np.shape(ch), dtype=np.complex128)
    for k in range(K):
        z_k = (k + 0.5) / K * L                                                   # Eq. 10
        g_k = isrs.srs_gain(z_k, f3, alpha, p_tot, span["cr"], b_tot)               # Eq. 8 factor
        I_k = (np.exp(sig * ((k + 1) / K * L)) - np.exp(sig * (k / K * L))) / sig   # Eq. 9
        mu = mu + g_k * I_k                                                        # Eq. 8
    return mu


def mu_maclaurin(f1, f2, f, span, p_tot, b_tot, dz=None):
    """Eq. 4, with eta from Eq. 6 and chi from Eq. 5."""
    L, alpha = span["L"], span["alpha"]
    ch = chi(f1, f2, f, span["beta2"], span["beta3"])
    eta = eta_gn(ch, alpha, L)
    sig2 = 1j * ch - 2.0 * alpha
    return eta - p_tot * span["cr"] * (f1 + f2 - f) / alpha * (eta - (np.exp(sig2 * L) - 1.0) / sig2)


_GL_NODES, _GL_WEIGHTS = np.polynomial.legendre.leggauss(12)


def mu_quad(f1, f2, f, span, p_tot, b_tot, dz=None, panels_per_period=4, min_panels=64):
    """Eq. 23 by composite 12-node Gauss-Legendre on equal panels.

    Reading C12: the paper only says the oscillation needs "a larger number of samples"
    (P:71).  Panels: max(min_panels, panels_per_period * |chi| L / (2 pi)), so every panel
    spans at most a quarter period of e^{i chi z} and at most L/64 of the smooth envelope
    rho_s (Eq. 25); 12-node GL is then exact to rounding for both.
    """
    L, alpha = span["L"], span["alpha"]
    f1 = np.atleast_1d(np.asarray(f1, dtype=np.float64))
    f2 = np.atleast_1d(np.asarray(f2, dtype=np.float64))
    ch = chi(f1, f2, f, span["beta2"], span["beta3"])
    f3 = f1 + f2 - f
    n_pan = np.maximum(min_panels, np.ceil(panels_per_period * np.abs(ch) * L / (2 * math.pi)))
    n_pan = (2 ** np.ceil(np.log2(n_pan))).astype(np.int64)     # bucket by power of two
    out = np.zeros(f1.shape, dtype=np.complex128)
    for npn in np.unique(n_pan):
        sel = np.nonzero(n_pan == npn)[0]
        h = L / npn
        # z nodes: panel j, node q -> j h + (x_q + 1) h/2
        z = (np.arange(npn)[:, None] * h + (_GL_NODES[None, :] + 1.0) * (h / 2.0)).ravel()
        w = np.tile(_GL_WEIGHTS * (h / 2.0), npn)
        for chunk in np.array_split(sel, max(1, (sel.size * z.size) // 4_000_000 + 1)):
            r = isrs.rho(z[None, :], f3[chunk, None], alpha, p_tot, span["cr"], b_tot)
            ph = np.exp(1j * ch[chunk, None] * z[None, :])                     # Eq. 24: phi = chi z
            out[chunk] = (r * ph) @ w
    return out


# Gauss-Kronrod 7/15 on [-1, 1] (the standard QUADPACK QK15 abscissae and weights, written from the
# Kronrod extension of the 7-point Gauss-Legendre rule; the 7 Gauss nodes are xgk[1::2]).
_GK15_X = np.array([0.991455371120812639206854697526329, 0.949107912342758524526189684047851,
                    0.864864423359769072789712788640926, 0.741531185599394439863864773280788,
                    0.586087235467691130294144845693013, 0.405845151377397166906606412076961,
                    0.207784955007898467600689403773245, 0.0])
_GK15_WK = np.array([0.022935322010529224963732008058970, 0.063092092629978553290700663189204,
                     0.104790010322250183839876322541518, 0.140653259715525918745189590510238,
                     0.169004726639267902826583426598550, 0.190350578064785409913256402421014,
                     0.204432940075298892414161999234649, 0.209482141084727828012999174891714])
_GK15_WG = np.array([0.129484966168869693270611432679082, 0.279705391489276667901467771423780,
                     0.381830050505118944950369775488975, 0.417959183673469387755102040816327])


def _gk15_nodes():
    x = np.concatenate([-_GK15_X[:-1], _GK15_X[::-1]])               # 15 ascending nodes
    wk = np.concatenate([_GK15_WK[:-1], _GK15_WK[::-1]])
    wg = np.zeros(15)
    gi = [1, 3, 5, 7, 9, 11, 13]                                       # Gauss nodes among the 15
    wg[gi] = np.concatenate([_GK15_WG[:-1], _GK15_WG[::-1]])
    return x, wk, wg


def mu_quad_adaptive(f1, f2, f, span, p_tot, b_tot, dz=None, rtol=1e-13, max_panels=2_000_000):
    """Eq. 23 by adaptive Gauss-Kronrod 7/15 (SURVEY reading C12): initial panels of at most a
    quarter period pi/(2|chi|) of e^{i chi z} and at least 8 per span; every panel whose |K15 - G7|
    exceeds rtol |mu| / n_panels, and is above the panel's rounding floor
    50 eps (1 + |chi| z) int|integrand| (the phase chi z is rounded at every node), is
    bisected until all pass.  One point at a time (pins only: an independent check of the
    fixed-panel rule mu_quad, for |chi| L up to ~1e5 rad)."""
    L, alpha = span["L"], span["alpha"]
    f1 = np.atleast_1d(np.asarray(f1, dtype=np.float64))
    f2 = np.atleast_1d(np.asarray(f2, dtype=np.float64))
    ch = chi(f1, f2, f, span["beta2"], span["beta3"])
    x, wk, wg = _gk15_nodes()
    out = np.zeros(f1.shape, dtype=np.complex128)
    for i in range(f1.size):
        f3 = f1[i] + f2[i] - f
        n0 = int(max(8, math.ceil(abs(ch[i]) * L / (math.pi / 2))))
        a = np.linspace(0.0, L, n0 + 1)
        lo, hi = a[:-1], a[1:]
        total = 0.0 + 0.0j
        while True:
            mid, half = (lo + hi) / 2, (hi - lo) / 2
            z = mid[:, None] + half[:, None] * x[None, :]
            g = isrs.rho(z, f3, alpha, p_tot, span["cr"], b_tot) * np.exp(1j * ch[i] * z)
            k15 = (g @ wk) * half
            g7 = (g @ wg) * half
            err = np.abs(k15 - g7)
            # rounding floor: the phase chi z of every node carries ~eps |chi| z absolute error
            floor = 50 * np.finfo(np.float64).eps * (1.0 + abs(ch[i]) * hi) * (np.abs(g) @ wk) * half
            est = total + k15.sum()
            bad = (err > rtol * abs(est) / max(1, lo.size)) & (err > floor)
            total = total + k15[~bad].sum()
            if not bad.any():
                break
            if lo.size > max_panels:
                raise RuntimeError("mu_quad_adaptive: panel budget exceeded")
            lo, hi = lo[bad], hi[bad]
            m = (lo + hi) / 2
            lo, hi = np.concatenate([lo, m]), np.concatenate([m, hi])
        out[i] = total
    return out


MU_MODES = {"closed": mu_segment, "segment": mu_segment, "maclaurin": mu_maclaurin,
            "quad": mu_quad, "quad_adaptive": mu_quad_adaptive}
