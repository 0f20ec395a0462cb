"""Seeded synthetic link descriptions (BASELINE.json `configs`).

Every array is in SI units and every frequency is an integer number of Hz, with
R_i/(2N) also an integer, so that all grid frequencies f = lo + (m + 1/2) R/N and
all f1 + f2 - f sums are exact in fp64 (ambiguity reading C10 in DESIGN.md).

Unit conversions here are the standard datasheet ones (dB/km -> 1/m, ps/nm/km ->
beta2 at lambda_ref = c/f_ref, dBm -> W, 1/W/km/THz -> 1/W/m/Hz); they prepare inputs
and are not part of the ISRS-EGN method.  The oracle carries its own independent copy
of the conversions (oracle/units.py) and tests/ pins one against the other.

Generator: numpy.random.default_rng(241211614 + c) for BJ config c; draw order
formats -> symbol rates -> powers -> span lengths -> span alpha.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

C_LIGHT = 299792458.0
F_REF = 193.4e12

# Modulation formats: (Phi = excess kurtosis, Psi = normalised sixth-order cumulant).
# Phi values are BASELINE.json's; Psi values are SURVEY.md C9 ([X8]); both are inputs.
FORMATS = {
    "gauss": (0.0, 0.0),
    "qpsk": (-1.0, 4.0),
    "16qam": (-0.68, 2.08),
    "64qam": (-0.619, 1.7972),
}
MIXED = ("qpsk", "16qam", "64qam")


@dataclasses.dataclass
class Link:
    """One WDM link: channels, spans and numerics (SI units, absolute frequencies)."""

    name: str
    f_center_hz: np.ndarray
    symbol_rate_hz: np.ndarray
    launch_power_w: np.ndarray
    phi: np.ndarray
    psi: np.ndarray
    length_m: np.ndarray
    alpha_per_m: np.ndarray
    beta2_s2_per_m: np.ndarray
    beta3_s3_per_m: np.ndarray
    gamma_per_w_m: np.ndarray
    cr_per_w_m_hz: np.ndarray
    grid_n: int
    delta_z_m: float = 1000.0
    seed: int | None = None
    formats: tuple = ()

    @property
    def n_ch(self) -> int:
        return int(self.f_center_hz.size)

    @property
    def n_span(self) -> int:
        return int(self.length_m.size)

    def with_(self, **kw) -> "Link":
        d = dataclasses.asdict(self)
        d.update(kw)
        for k in ("f_center_hz", "symbol_rate_hz", "launch_power_w", "phi", "psi", "length_m",
                  "alpha_per_m", "beta2_s2_per_m", "beta3_s3_per_m", "gamma_per_w_m",
                  "cr_per_w_m_hz"):
            d[k] = np.ascontiguousarray(np.asarray(d[k], dtype=np.float64))
        return Link(**d)

    def check_lattice(self) -> None:
        """Inputs must sit on the exact integer-Hz lattice (C10)."""
        for a in (self.f_center_hz, self.symbol_rate_hz):
            assert np.all(a == np.round(a)), "frequencies must be integer Hz"
        half = self.symbol_rate_hz / (2 * self.grid_n)
        assert np.all(half == np.round(half)), "R/(2N) must be an integer number of Hz"


def db_per_km_to_per_m(a_db_km):
    return np.asarray(a_db_km, dtype=np.float64) * math.log(10.0) / 10.0 / 1000.0


def dbm_to_w(p_dbm):
    return 10.0 ** (np.asarray(p_dbm, dtype=np.float64) / 10.0) / 1000.0


def dispersion_to_beta(d_ps_nm_km, s_ps_nm2_km, f_ref=F_REF):
    """beta2 = -D l^2/(2 pi c); beta3 = (l^2/(2 pi c))^2 (S + 2D/l), l = c/f_ref (C15)."""
    lam = C_LIGHT / f_ref
    d = d_ps_nm_km * 1e-6      # s/m^2
    s = s_ps_nm2_km * 1e3      # s/m^3
    k = lam * lam / (2.0 * math.pi * C_LIGHT)
    return -d * k, k * k * (s + 2.0 * d / lam)


def _spans(n, length_km=80.0, alpha_db_km=0.2, d=17.0, s=0.067, gamma_w_km=1.3,
           cr_w_km_thz=0.028, f_ref=F_REF):
    b2, b3 = dispersion_to_beta(d, s, f_ref)
    ones = np.ones(n)
    return dict(
        length_m=np.asarray(length_km, dtype=np.float64) * 1000.0 * ones,
        alpha_per_m=db_per_km_to_per_m(alpha_db_km) * ones,
        beta2_s2_per_m=b2 * ones,
        beta3_s3_per_m=b3 * ones,
        gamma_per_w_m=gamma_w_km * 1e-3 * ones,
        cr_per_w_m_hz=cr_w_km_thz * 1e-3 * 1e-12 * ones,
    )


def _fmt_arrays(names):
    phi = np.array([FORMATS[n][0] for n in names], dtype=np.float64)
    psi = np.array([FORMATS[n][1] for n in names], dtype=np.float64)
    return phi, psi


def _uniform_plan(n, spacing_hz, f0=F_REF):
    """Centres f0 + (i - (n-1)/2) spacing, integer Hz."""
    i = np.arange(n, dtype=np.float64)
    f = f0 + (i - (n - 1) / 2.0) * spacing_hz
    return np.round(f)


CONFIG_NAMES = ("c1", "c2", "c3", "c4", "c5")


def bj_config(name: str) -> Link:
    """BASELINE.json configs[0..4] as concrete seeded inputs."""
    c = CONFIG_NAMES.index(name) + 1
    seed = 241211614 + c
    rng = np.random.default_rng(seed)
    if c == 1:
        n = 5
        fmts = ("gauss",) * n
        f = _uniform_plan(n, 100e9)
        r = np.full(n, 64e9)
        p = dbm_to_w(np.zeros(n))
        sp = _spans(1)
        N = 64
    elif c == 2:
        n = 40
        fmts = ("16qam",) * n
        f = _uniform_plan(n, 100e9)
        r = np.full(n, 64e9)
        p = dbm_to_w(np.ones(n))
        sp = _spans(10)
        N = 128
    elif c == 3:
        n = 100
        fmts = tuple(MIXED[k] for k in rng.integers(0, 3, n))
        f = _uniform_plan(n, 100e9)
        r = np.full(n, 96e9)
        p = dbm_to_w(-2.0 + 4.0 * np.arange(n) / (n - 1))
        sp = _spans(20)
        N = 128
    elif c == 4:
        n = 80
        fmts = tuple(MIXED[k] for k in rng.integers(0, 3, n))
        r = np.array([32e9, 64e9, 96e9])[rng.integers(0, 3, n)]
        p = dbm_to_w(rng.uniform(-2.0, 3.0, n))
        lengths_km = np.round(rng.uniform(60.0, 100.0, 30) * 1000.0) / 1000.0
        alpha_db = rng.uniform(0.16, 0.22, 30)
        guard = 12.5e9
        f = np.zeros(n)
        for i in range(1, n):
            f[i] = f[i - 1] + r[i - 1] / 2 + guard + r[i] / 2
        lo = f[0] - r[0] / 2
        hi = f[-1] + r[-1] / 2
        f = f + np.round((F_REF - (lo + hi) / 2) / 1e9) * 1e9  # centre on 193.4 THz, 1 GHz grid
        sp = _spans(30)
        sp["length_m"] = lengths_km * 1000.0
        sp["alpha_per_m"] = db_per_km_to_per_m(alpha_db)
        N = 128
    elif c == 5:
        n = 200
        fmts = tuple(MIXED[k] for k in rng.integers(0, 3, n))
        f = _uniform_plan(n, 100e9)
        r = np.full(n, 96e9)
        p = dbm_to_w(-3.0 + 6.0 * np.arange(n) / (n - 1))
        sp = _spans(50)
        N = 256
    phi, psi = _fmt_arrays(fmts)
    link = Link(name=name, f_center_hz=f.astype(np.float64), symbol_rate_hz=r.astype(np.float64),
                launch_power_w=p, phi=phi, psi=psi, grid_n=N, delta_z_m=1000.0, seed=seed,
                formats=fmts, **sp)
    link.check_lattice()
    return link


def paper_analog(which: str, n_span: int = 1, cr_w_km_thz: float | None = None,
                 fmt: str = "gauss", n_ch: int | None = None, grid_n: int | None = None) -> Link:
    """Paper parameter tables as inputs.

    "I"  : Table I - 101 x 10 GBd at 10.1 GHz, P_tot 19 dBm uniform,
           C_r 0.28 or 1.12 /W/km/THz, D 17, S 0 (beta3 = 0, C15), gamma 1.2, 100 km spans,
           1 GHz resolution (N = 10).
    "Ir" : Table I reduced to n_ch channels (default 15) with C_r scaled by 1 THz / B_tot so
           that P_tot C_r B_tot (hence Delta-rho, Eq. 12) matches the 1 THz case - the paper's
           own trick.
    "II" : Table II - 101 x 100 GBd at 101 GHz, 25 dBm, C_r 0.028,
           S 0.067, 1 x 100 km, N = 100.
    """
    if which in ("I", "Ir"):
        n = 101 if which == "I" else (n_ch or 15)
        spacing, R = 10.1e9, 10e9
        p_tot_dbm = 19.0
        cr = 1.12 if cr_w_km_thz is None else cr_w_km_thz
        if which == "Ir":
            b_tot = (n - 1) * spacing + R
            cr = cr * 1e12 / b_tot
        N = grid_n or 10
        sp = _spans(n_span, length_km=100.0, alpha_db_km=0.2, d=17.0, s=0.0, gamma_w_km=1.2,
                    cr_w_km_thz=cr)
        sp["beta3_s3_per_m"] = np.zeros(n_span)
    elif which == "II":
        n = n_ch or 101
        spacing, R = 101e9, 100e9
        p_tot_dbm = 25.0
        cr = 0.028 if cr_w_km_thz is None else cr_w_km_thz
        N = grid_n or 100
        sp = _spans(n_span, length_km=100.0, alpha_db_km=0.2, d=17.0, s=0.067, gamma_w_km=1.2,
                    cr_w_km_thz=cr)
    else:
        raise ValueError(which)
    f = _uniform_plan(n, spacing)
    r = np.full(n, R)
    p = np.full(n, float(dbm_to_w(p_tot_dbm)) / n)
    phi, psi = _fmt_arrays((fmt,) * n)
    link = Link(name=f"PA-{which}", f_center_hz=f, symbol_rate_hz=r, launch_power_w=p, phi=phi,
                psi=psi, grid_n=N, delta_z_m=1000.0, formats=(fmt,) * n, **sp)
    link.check_lattice()
    return link


def tiny_link(n_ch=3, rates_gbd=(64,), spacing_ghz=100.0, guard_ghz=None, n_span=2, grid_n=8,
              length_km=80.0, alpha_db_km=0.2, cr_w_km_thz=0.028, d=17.0, s=0.067,
              gamma_w_km=1.3, power_dbm=0.0, fmts=("gauss",), delta_z_m=1000.0, seed=7,
              random_spans=False, tilt_db=0.0) -> Link:
    """Small links for parity at sizes the oracle finishes in seconds.

    rates cycle over `rates_gbd`; with guard_ghz the channels are packed edge-to-guard-to-edge
    (touching bands when guard_ghz == 0), else placed on a uniform `spacing_ghz` plan.
    """
    rng = np.random.default_rng(seed)
    r = np.array([rates_gbd[i % len(rates_gbd)] * 1e9 for i in range(n_ch)])
    if guard_ghz is None:
        f = _uniform_plan(n_ch, spacing_ghz * 1e9)
    else:
        f = np.zeros(n_ch)
        for i in range(1, n_ch):
            f[i] = f[i - 1] + r[i - 1] / 2 + guard_ghz * 1e9 + r[i] / 2
        f = f + F_REF - np.round(((f[0] - r[0] / 2) + (f[-1] + r[-1] / 2)) / 2 / 1e9) * 1e9
    p_dbm = power_dbm + tilt_db * (np.arange(n_ch) / max(n_ch - 1, 1) - 0.5)
    names = tuple(fmts[i % len(fmts)] for i in range(n_ch))
    phi, psi = _fmt_arrays(names)
    sp = _spans(n_span, length_km=length_km, alpha_db_km=alpha_db_km, d=d, s=s,
                gamma_w_km=gamma_w_km, cr_w_km_thz=cr_w_km_thz)
    if random_spans:
        sp["length_m"] = np.round(rng.uniform(0.6, 1.0, n_span) * length_km * 1000.0)
        sp["alpha_per_m"] = db_per_km_to_per_m(rng.uniform(0.16, 0.22, n_span))
        b2, b3 = dispersion_to_beta(rng.uniform(15.0, 20.0, n_span), s)
        sp["beta2_s2_per_m"] = b2
        sp["beta3_s3_per_m"] = b3
        sp["gamma_per_w_m"] = rng.uniform(1.0, 1.5, n_span) * 1e-3
    link = Link(name="tiny", f_center_hz=f, symbol_rate_hz=r, launch_power_w=dbm_to_w(p_dbm),
                phi=phi, psi=psi, grid_n=grid_n, delta_z_m=delta_z_m, seed=seed, formats=names,
                **sp)
    link.check_lattice()
    return link
