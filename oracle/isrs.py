"""ISRS power profile (oracle; test infrastructure only).

PAPER.md Appendix A and B:
  Eq. 2   zeta = P_tot C_r L_eff;  rho(z,f) = zeta B e^{-zeta f} / (e^{zeta B/2} - e^{-zeta B/2}) e^{-alpha z}
  Eq. 12     Delta-rho(z)[dB] = 4.3 P_tot C_r L_eff B_tot
  Eq. 13/25  rho_s(z,f) = B P C L_eff(z) e^{-alpha z - P C L_eff(z) f} / (2 sinh(P B C L_eff(z)/2))
  Eq. 14     SRS_G(z,f) = rho(z,f) without the attenuation factor
Frequencies f are offsets from the band centre f_c (reading C5).
L_eff(z) = (1 - e^{-alpha z}) / alpha is the standard effective length (P:223 symbol), evaluated
with expm1 (reading C11).
"""
import numpy as np


def effective_length(z, alpha):
    """L_eff(z) = (1 - e^{-alpha z}) / alpha."""
    return -np.expm1(-alpha * z) / alpha


def zeta(z, alpha, p_tot, cr):
    """Eq. 2: zeta = P_tot C_r L_eff(z)."""
    return p_tot * cr * effective_length(z, alpha)


def srs_gain(z, f, alpha, p_tot, cr, b_tot):
    """Eq. 14: B P C L_eff e^{-P C L_eff f} / (2 sinh(P B C L_eff / 2)).

    At P C L_eff = 0 (z = 0 or C_r = 0) the factor is the limit 1 (reading C11, C_r = 0 pin P1).
    """
    ze = zeta(z, alpha, p_tot, cr)
    x = b_tot * ze
    x = np.asarray(x, dtype=np.float64)
    f = np.asarray(f, dtype=np.float64)
    safe_x = np.where(x == 0.0, 1.0, x)
    g = safe_x * np.exp(-ze * f) / (2.0 * np.sinh(safe_x / 2.0))
    return np.where(x == 0.0, 1.0, g)


def rho(z, f, alpha, p_tot, cr, b_tot):
    """Eq. 13 / Eq. 25: normalised power profile rho_s(z, f) = SRS_G(z,f) e^{-alpha z}."""
    return srs_gain(z, f, alpha, p_tot, cr, b_tot) * np.exp(-alpha * z)


def delta_rho_db(z, alpha, p_tot, cr, b_tot, factor=4.3):
    """Eq. 12: Delta-rho(z) [dB] = 4.3 P_tot C_r L_eff B_tot."""
    return factor * p_tot * cr * effective_length(z, alpha) * b_tot
