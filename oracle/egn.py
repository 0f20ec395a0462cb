"""ISRS EGN assembly: eta(f_COI) per channel (oracle; test infrastructure only).

PAPER.md Appendix B:
  Eq. 15      sigma^2_NLI,kappa = sum over islands (kappa1,kappa2,l) of P P P (D + Phi E delta + Phi F delta
                      + Phi G delta + delta delta Psi H)
  Eq. 16  island set T_kappa
  Eqs. 17-21  D, E, F, G, H
  Eq. 11      eta_kappa = sigma^2_NLI,kappa / P^3
Readings (restated in DESIGN.md):
  C1  2-D: f is fixed at the COI centre; P_NLI = R_kappa G_NLI(f_kappa) (locally white).
  C2  PSD normalisation: each cumulant-tied channel i contributes one coherent integral and 1/R_i:
      eta = (R_k / P_k^3) sum_islands [ 16/27 G1 G2 G3 D + 16/27 Phi1 G1^2 G2 E / R1
            + 32/81 Phi2 G2^2 G1 F / R2 + 16/81 Phi1 G1^2 G3 G / R1 + 16/81 Psi1 G1^3 H / R1^2 ],  G_i = P_i / R_i.
  C5  offsets from f_c = midpoint of the occupied band; B_tot = edge-to-edge occupied bandwidth;
      P_tot = sum P_i.
  C6  region = (kappa, kappa1, kappa2) rectangle, N x N bin-centre grid, weight delta1 delta2;
      islands = the kappa3-partition of the region's points.
  C7  E coherent over f1 at fixed f2; F coherent over f2 at fixed f1; G coherent along
      f1 + f2 = const with |S(f3)|^2 outside the modulus; H coherent over the island.
  C8  gates: E <- Phi_k1 [k3 == k1]; F <- Phi_k2 [k3 == k2]; G <- Phi_k1 [k1 == k2];
      H <- Psi_k1 [k1 == k2 == k3]; a term whose gate or weight is 0 is not evaluated.
  C10 f3 on a band edge takes the average of the one-sided limits: |S|^2 -> 1/2 (D, G),
      S -> 1/2 (E, F, H); touching bands split 1/2 / 1/2 between the two islands.
  C16 rectangular spectra, G_i = P_i / R_i.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import link as link_mod


@dataclasses.dataclass
class Canon:
    f: np.ndarray        # channel centres, offsets from f_c [Hz]
    R: np.ndarray
    P: np.ndarray
    G: np.ndarray        # PSD P/R  (C16)
    phi: np.ndarray
    psi: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    delta: np.ndarray    # R/N (C6)
    N: int
    f_c: float
    b_tot: float
    p_tot: float
    dz: float
    spans: list


def canonicalize(link) -> Canon:
    """Reading C5: offsets from the occupied-band midpoint; B_tot edge-to-edge; P_tot = sum P."""
    F = np.asarray(link.f_center_hz, dtype=np.float64)
    R = np.asarray(link.symbol_rate_hz, dtype=np.float64)
    lo_abs, hi_abs = F - R / 2, F + R / 2
    f_c = (lo_abs.min() + hi_abs.max()) / 2
    b_tot = hi_abs.max() - lo_abs.min()
    f = F - f_c
    P = np.asarray(link.launch_power_w, dtype=np.float64)
    spans = [dict(L=float(link.length_m[s]), alpha=float(link.alpha_per_m[s]),
                  beta2=float(link.beta2_s2_per_m[s]), beta3=float(link.beta3_s3_per_m[s]),
                  gamma=float(link.gamma_per_w_m[s]), cr=float(link.cr_per_w_m_hz[s]))
             for s in range(len(link.length_m))]
    N = int(link.grid_n)
    return Canon(f=f, R=R, P=P, G=P / R, phi=np.asarray(link.phi, dtype=np.float64),
                 psi=np.asarray(link.psi, dtype=np.float64), lo=f - R / 2, hi=f + R / 2,
                 delta=R / N, N=N, f_c=f_c, b_tot=b_tot, p_tot=float(P.sum()),
                 dz=float(link.delta_z_m), spans=spans)


def grid(c: Canon, i: int) -> np.ndarray:
    """C6: bin centres f = lo_i + (m + 1/2) delta_i, m = 0..N-1."""
    return c.lo[i] + (np.arange(c.N) + 0.5) * c.delta[i]


def region_points(c: Canon, kappa: int, k1: int, k2: int, f=None):
    """Point arrays of region (kappa, k1, k2), indexed [m2, m1]; f = the NLI frequency (the COI
    centre c.f[kappa] unless given: 3-D mode, NEXT-3)."""
    f = c.f[kappa] if f is None else f
    F1 = grid(c, k1)[None, :] * np.ones((c.N, 1))
    F2 = grid(c, k2)[:, None] * np.ones((1, c.N))
    f3 = F1 + F2 - f
    return F1, F2, f3


def coi_frequencies(c: Canon, kappa: int, f_samples: int = 0):
    """Frequencies f at which G_NLI is evaluated for COI kappa.
    f_samples = 0: the COI centre only (reading C1, locally white: P_NLI = R_kappa G_NLI(f_kappa)).
    f_samples = n > 0 (NEXT-3, the 3-D form): Eqs. 17-21 integrate f over the COI band
    [-R/2, R/2] about kappa R; midpoint rule f_m = lo_kappa + (m + 1/2) R_kappa / n,
    m = 0..n-1, so P_NLI = sum_m G_NLI(f_m) R_kappa / n."""
    if f_samples <= 0:
        return np.array([c.f[kappa]])
    return c.lo[kappa] + (np.arange(f_samples) + 0.5) * (c.R[kappa] / f_samples)


def island_gates(c: Canon, f3: np.ndarray):
    """C10 / Eq. 17 gate |S(f1+f2-f)|^2: for every channel k3 whose closed band [lo, hi]
    holds some f3, the per-point factor t = 1 strictly inside, 1/2 on an edge, 0 outside."""
    out = []
    for k3 in range(c.f.size):
        inside = (f3 >= c.lo[k3]) & (f3 <= c.hi[k3])
        if not inside.any():
            continue
        t = np.where((f3 > c.lo[k3]) & (f3 < c.hi[k3]), 1.0, 0.5) * inside
        out.append((k3, t))
    return out


def region_islands(c: Canon, kappa: int, k1: int, k2: int, mu_mode: str = "closed",
                   need=("D", "E", "F", "G", "H"), f=None, gain: str = "ideal"):
    """Per-island raw integrals D, E, F, G, H of region (kappa, k1, k2) (Eqs. 17-21, C6, C7, C10)
    at NLI frequency f (default: the COI centre)."""
    f = c.f[kappa] if f is None else f
    F1, F2, f3 = region_points(c, kappa, k1, k2, f)
    gates = island_gates(c, f3)
    if not gates:
        return []
    support = np.zeros(f3.shape, dtype=bool)
    for _, t in gates:
        support |= t > 0
    Y = np.zeros(f3.shape, dtype=np.complex128)
    if mu_mode == "unit":                           # test hook P6: Y := 1
        Y[support] = 1.0
    else:
        Y[support] = link_mod.link_function(F1[support], F2[support], f, c.spans,
                                            c.p_tot, c.b_tot, c.dz, mu_mode, gain)
    d1, d2 = c.delta[k1], c.delta[k2]
    N = c.N
    m1 = np.arange(N)[None, :] * np.ones((N, 1), dtype=np.int64)
    m2 = np.arange(N)[:, None] * np.ones((1, N), dtype=np.int64)
    diag = (m1 + m2).astype(np.int64)
    res = []
    for k3, t in gates:
        isl = dict(k3=k3, npts=int((t > 0).sum()), D=0.0, E=0.0, F=0.0, G=0.0, H=0.0)
        # D, Eq. 17: |S(f1)|^2 |S(f2)|^2 |S(f3)|^2 |Y|^2 over the island
        isl["D"] = float(np.sum(t * np.abs(Y) ** 2) * d1 * d2)
        if k3 == k1 and "E" in need:
            # E, Eq. 18 (C7): coherent over f1 at fixed f2, S*(f3) inside the modulus
            r = np.sum(t * Y, axis=1) * d1               # [m2]
            isl["E"] = float(np.sum(np.abs(r) ** 2) * d2)
        if k3 == k2 and "F" in need:
            # F, Eq. 19 (C7): coherent over f2 at fixed f1
            col = np.sum(t * Y, axis=0) * d2             # [m1]
            isl["F"] = float(np.sum(np.abs(col) ** 2) * d1)
        if k1 == k2 and "G" in need:
            # G, Eq. 20 (C7): coherent along f1 + f2 = s, |S(f3)|^2 outside the modulus
            G = 0.0
            for d in range(2 * N - 1):
                on = (diag == d) & (t > 0)
                if not on.any():
                    continue
                t_d = t[on][0]                       # f3 (hence t) is constant on the anti-diagonal
                a_d = np.sum(Y[on]) * d1
                G += t_d * abs(a_d) ** 2 * d1
            isl["G"] = float(G)
        if k1 == k2 == k3 and "H" in need:
            # H, Eq. 21 (C7): coherent over the whole island
            isl["H"] = float(abs(np.sum(t * Y) * d1 * d2) ** 2)
        res.append(isl)
    return res


def has_support_bound(c: Canon, kappa: int, k1: int, k2: int, f=None) -> bool:
    """Cheap necessary condition for a non-empty region: the f3 range of the bin centres
    overlaps some band."""
    f = c.f[kappa] if f is None else f
    lo3 = c.lo[k1] + c.lo[k2] - f + (c.delta[k1] + c.delta[k2]) / 2
    hi3 = c.hi[k1] + c.hi[k2] - f - (c.delta[k1] + c.delta[k2]) / 2
    return bool(np.any((c.hi >= lo3) & (c.lo <= hi3)))


def _needed_terms(c: Canon, k1: int, k2: int):
    """C8: a term whose gate or weight is zero is not evaluated."""
    need = ["D"]
    if c.phi[k1] != 0.0:
        need += ["E", "G"]
    if c.phi[k2] != 0.0:
        need += ["F"]
    if c.psi[k1] != 0.0:
        need += ["H"]
    return tuple(need)


def island_contributions(c: Canon, k1: int, k2: int, isl: dict):
    """Eq. 15 with reading C2: the five weighted contributions of one island (1/W^2 * W/Hz...)."""
    G1, G2, G3 = c.G[k1], c.G[k2], c.G[isl["k3"]]
    R1, R2 = c.R[k1], c.R[k2]
    k3 = isl["k3"]
    tD = 16.0 / 27.0 * G1 * G2 * G3 * isl["D"]
    tE = 16.0 / 27.0 * c.phi[k1] * G1 ** 2 * G2 * isl["E"] / R1 if k3 == k1 else 0.0
    tF = 32.0 / 81.0 * c.phi[k2] * G2 ** 2 * G1 * isl["F"] / R2 if k3 == k2 else 0.0
    tG = 16.0 / 81.0 * c.phi[k1] * G1 ** 2 * G3 * isl["G"] / R1 if k1 == k2 else 0.0
    tH = 16.0 / 81.0 * c.psi[k1] * G1 ** 3 * isl["H"] / R1 ** 2 if k1 == k2 == k3 else 0.0
    return np.array([tD, tE, tF, tG, tH])


def nli_class(kappa: int, k1: int, k2: int, k3: int) -> int:
    """an island is SCI (0) when it involves the COI alone, XCI (1) when it involves ONE
    interfering channel, MCI (2) when it involves two or three: the number of distinct channels of
    (k1, k2, k3) other than the COI."""
    return min(2, len({k1, k2, k3} - {kappa}))


def eta(link, coi=None, mu_mode: str = "closed", return_regions: bool = False, f_samples: int = 0,
        gain: str = "ideal", split: bool = False):
    """eta_kappa (1/W^2, Eq. 11 with P = P_kappa, reading C13) and the D/E/F/G/H breakdown.

    Brute force over every (kappa1, kappa2) pair and every grid point (Eq. 16 generalised to
    arbitrary channel plans: an island exists wherever f3 lands in a band).  f_samples > 0: the
    3-D form (NEXT-3), G_NLI averaged over f_samples midpoints of the COI band (coi_frequencies).
    split=True also returns [n_coi, 3]: eta's SCI / XCI / MCI parts (nli_class), island by island.
    """
    c = canonicalize(link)
    n = c.f.size
    coi = list(range(n)) if coi is None else list(coi)
    etas = np.zeros(len(coi))
    terms = np.zeros((len(coi), 5))
    regions = {}
    parts = np.zeros((len(coi), 3))
    for ci, kappa in enumerate(coi):
        acc = np.zeros(5)
        cls = np.zeros(3)
        fs = coi_frequencies(c, kappa, f_samples)
        for f in fs:
            for k1 in range(n):
                for k2 in range(n):
                    if not has_support_bound(c, kappa, k1, k2, f):
                        continue
                    isls = region_islands(c, kappa, k1, k2, mu_mode, _needed_terms(c, k1, k2), f, gain)
                    if not isls:
                        continue
                    if return_regions:
                        regions[(kappa, k1, k2) if f_samples <= 0 else (kappa, float(f), k1, k2)] = isls
                    for isl in isls:
                        contrib = island_contributions(c, k1, k2, isl)
                        acc = acc + contrib
                        cls[nli_class(kappa, k1, k2, isl["k3"])] += contrib.sum()
        # P_NLI = R G_NLI(f_kappa) (C1) or sum_m G_NLI(f_m) R / n (3-D); Eq. 11
        scale = c.R[kappa] / c.P[kappa] ** 3 / len(fs)
        terms[ci] = acc * scale
        etas[ci] = acc.sum() * scale
        parts[ci] = cls * scale
    if return_regions:
        return etas, terms, regions
    if split:
        return etas, terms, parts
    return etas, terms


def region_partials(link, kappa: int, k1: int, k2: int, mu_mode: str = "closed"):
    """Per-region weighted partial integrals, the quantities the CUDA path writes per region:
        D_w = sum_islands G_k3 D,  E_w = E[k3 == k1],  F_w = F[k3 == k2],
        G_w = sum_islands G_k3 G (k1 == k2),  H_w = H[k1 == k2 == k3],  npts.
    Terms not needed under C8 are returned as 0.0.
    """
    c = canonicalize(link)
    out = np.zeros(5)
    npts = 0
    isls = region_islands(c, kappa, k1, k2, mu_mode, _needed_terms(c, k1, k2))
    for isl in isls:
        k3 = isl["k3"]
        out[0] += c.G[k3] * isl["D"]
        if k3 == k1:
            out[1] += isl["E"]
        if k3 == k2:
            out[2] += isl["F"]
        if k1 == k2:
            out[3] += c.G[k3] * isl["G"]
        if k1 == k2 == k3:
            out[4] += isl["H"]
    # a point sitting on a shared edge of two touching bands belongs to two islands
    F1, F2, f3 = region_points(c, kappa, k1, k2)
    sup = np.zeros(f3.shape, dtype=bool)
    for _, t in island_gates(c, f3):
        sup |= t > 0
    npts = int(sup.sum())
    return out, npts


def island_set_eq16(M: int, kappa: int):
    """Eq. 16 literally: {(k1,k2,l) in {-M..M}^2 x {-1,0,1} : -M <= k1+k2-kappa+l <= M}."""
    return [(k1, k2, l) for k1 in range(-M, M + 1) for k2 in range(-M, M + 1) for l in (-1, 0, 1)
            if -M <= k1 + k2 - kappa + l <= M]


def island_set_generalised(link, kappa: int):
    """The islands this implementation integrates for COI `kappa`: every (k1, k2, k3) with at
    least one grid point of region (kappa, k1, k2) whose f3 lies in band k3 (C6, C10).  For a
    uniform plan with spacing = R this is Eq. 16's T_kappa with k3 = k1 + k2 - kappa + l."""
    c = canonicalize(link)
    out = []
    for k1 in range(c.f.size):
        for k2 in range(c.f.size):
            _, _, f3 = region_points(c, kappa, k1, k2)
            for k3, t in island_gates(c, f3):
                out.append((k1, k2, k3))
    return out


def eta_db(eta_val):
    """C13: dB re 1 W^-2."""
    return 10.0 * np.log10(eta_val)


def unit_link_eta_3d(phi, psi):
    """Continuous limit of the 3-D unit-link pin (P14): single channel, Y := 1, f
    averaged over the band: D = 2/3 R^2, E = F = G = R^3/2, H = 9/20 R^4
    ->  eta = 32/81 + 48/81 Phi + 4/45 Psi."""
    return 32.0 / 81.0 + 48.0 / 81.0 * phi + 4.0 / 45.0 * psi


def unit_link_eta(phi, psi):
    """Closed form of pin P6: single channel, Y := 1, f at the centre:
    D = 3/4 R^2, E = F = G = 7/12 R^3, H = 9/16 R^4  ->  eta = 4/9 + 56/81 Phi + Psi/9 (1/W^2 units
    with |Y| = 1 /W)."""
    return 4.0 / 9.0 + 56.0 / 81.0 * phi + psi / 9.0


__all__ = ["Canon", "canonicalize", "grid", "region_points", "island_gates", "region_islands",
           "island_contributions", "nli_class", "eta", "region_partials", "eta_db", "unit_link_eta",
           "unit_link_eta_3d", "coi_frequencies",
           "has_support_bound", "math"]
