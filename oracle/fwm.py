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


MU_MODES = {"closed": mu_segment, "segment": mu_segment, "maclaurin": mu_maclaurin,
            "quad": mu_quad}
