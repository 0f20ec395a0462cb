"""Datasheet unit conversions (oracle copy; test infrastructure only).

These are not equations of the paper; the paper quotes its parameters in datasheet units
(Table I; Table II) and the model (Eqs. 22-25) needs SI.
Reading C15: beta2, beta3 at lambda_ref = c / f_c.
"""
import math

C_LIGHT = 299792458.0


def alpha_db_km_to_np_m(a_db_km):
    """Power attenuation: dB/km -> 1/m (natural units). a[1/m] = a[dB/km] * ln(10)/10 / 1000."""
    return a_db_km / (10.0 * math.log10(math.e)) / 1000.0


def dbm_to_watt(p_dbm):
    return 1e-3 * 10.0 ** (p_dbm / 10.0)


def watt_to_dbm(p_w):
    return 10.0 * math.log10(p_w / 1e-3)


def beta_from_dispersion(d_ps_nm_km, s_ps_nm2_km, f_ref_hz):
    """beta2 = -D lambda^2 / (2 pi c); beta3 = (lambda^2 / (2 pi c))^2 (S + 2 D / lambda)   (C15).

    D in ps/nm/km -> s/m^2 (x 1e-12 / 1e-9 / 1e3), S in ps/nm^2/km -> s/m^3 (x 1e-12/1e-18/1e3).
    """
    lam = C_LIGHT / f_ref_hz
    D = d_ps_nm_km * 1e-12 / 1e-9 / 1e3
    S = s_ps_nm2_km * 1e-12 / 1e-18 / 1e3
    beta2 = -D * lam ** 2 / (2.0 * math.pi * C_LIGHT)
    beta3 = (lam ** 2 / (2.0 * math.pi * C_LIGHT)) ** 2 * (S + 2.0 * D / lam)
    return beta2, beta3


def cr_per_w_km_thz_to_si(cr):
    """Raman gain slope 1/W/km/THz -> 1/W/m/Hz."""
    return cr / 1e3 / 1e12
