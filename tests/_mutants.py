"""Plausible mistakes planted in the oracle, one at a time, to check that the pins of
tests/test_oracle_pins.py catch them (tests/test_oracle_mutants.py).  Each mutant replaces one
oracle function by a copy with ONE slip: a dropped factor, a wrong sign or index, a swapped
coefficient or operand.  Applied by tests/conftest.py when ISRS_ORACLE_MUTANT names one.
"""
import math

import numpy as np


def _apply_chi_beta3_no_pi(fwm, isrs, link, egn):
    def chi(f1, f2, f, beta2, beta3):
        return 4.0 * math.pi ** 2 * (f1 - f) * (f2 - f) * (beta2 + beta3 * (f1 + f2))
    fwm.chi = chi


def _apply_chi_sum_minus(fwm, isrs, link, egn):
    def chi(f1, f2, f, beta2, beta3):
        return 4.0 * math.pi ** 2 * (f1 - f) * (f2 + f) * (beta2 + math.pi * beta3 * (f1 + f2))
    fwm.chi = chi


def _apply_segment_left_endpoint(fwm, isrs, link, egn):
    def mu_segment(f1, f2, f, span, p_tot, b_tot, dz):
        L, alpha = span["L"], span["alpha"]
        K = fwm.segment_count(L, dz)
        ch = fwm.chi(f1, f2, f, span["beta2"], span["beta3"])
        f3 = f1 + f2 - f
        sig = 1j * ch - alpha
        mu = np.zeros(np.shape(ch), dtype=np.complex128)
        for k in range(K):
            z_k = k / K * L                                       # slip: left end, not midpoint
            g_k = isrs.srs_gain(z_k, f3, alpha, p_tot, span["cr"], b_tot)
            I_k = (np.exp(sig * ((k + 1) / K * L)) - np.exp(sig * (k / K * L))) / sig
            mu = mu + g_k * I_k
        return mu
    fwm.mu_segment = mu_segment
    fwm.MU_MODES.update(closed=mu_segment, segment=mu_segment)


def _apply_segment_no_attenuation(fwm, isrs, link, egn):
    def mu_segment(f1, f2, f, span, p_tot, b_tot, dz):
        L, alpha = span["L"], span["alpha"]
        K = fwm.segment_count(L, dz)
        ch = fwm.chi(f1, f2, f, span["beta2"], span["beta3"])
        f3 = f1 + f2 - f
        sig = 1j * ch                                             # slip: dropped -alpha
        mu = np.zeros(np.shape(ch), dtype=np.complex128)
        for k in range(K):
            z_k = (k + 0.5) / K * L
            g_k = isrs.srs_gain(z_k, f3, alpha, p_tot, span["cr"], b_tot)
            I_k = (np.exp(sig * ((k + 1) / K * L)) - np.exp(sig * (k / K * L))) / sig
            mu = mu + g_k * I_k
        return mu
    fwm.mu_segment = mu_segment
    fwm.MU_MODES.update(closed=mu_segment, segment=mu_segment)


def _apply_srs_gain_sign(fwm, isrs, link, egn):
    orig = isrs.srs_gain

    def srs_gain(z, f, alpha, p_tot, cr, b_tot):
        return orig(z, -np.asarray(f, dtype=np.float64), alpha, p_tot, cr, b_tot)   # slip: e^{+zeta f}
    isrs.srs_gain = srs_gain


def _apply_leff_linear(fwm, isrs, link, egn):
    def effective_length(z, alpha):
        return np.asarray(z, dtype=np.float64) * 1.0                # slip: L_eff(z) = z
    isrs.effective_length = effective_length


def _apply_phase_includes_current_span(fwm, isrs, link, egn):
    def link_function(f1, f2, f, spans, p_tot, b_tot, dz, mu_mode="closed", gain="ideal"):
        mu_fn = fwm.MU_MODES[mu_mode]
        f1 = np.asarray(f1, dtype=np.float64)
        f2 = np.asarray(f2, dtype=np.float64)
        Y = np.zeros(np.broadcast(f1, f2).shape, dtype=np.complex128)
        theta = np.zeros(Y.shape)
        for sp in spans:
            theta = theta + fwm.chi(f1, f2, f, sp["beta2"], sp["beta3"]) * sp["L"]   # slip: before
            Y = Y + sp["gamma"] * mu_fn(f1, f2, f, sp, p_tot, b_tot, dz) * np.exp(1j * theta)
        return Y
    link.link_function = link_function


def _contrib(coef, norm_e="R1"):
    def island_contributions(c, k1, k2, isl):
        G1, G2, G3 = c.G[k1], c.G[k2], c.G[isl["k3"]]
        R1, R2 = c.R[k1], c.R[k2]
        k3 = isl["k3"]
        RE = R1 if norm_e == "R1" else R2
        tD = coef[0] * G1 * G2 * G3 * isl["D"]
        tE = coef[1] * c.phi[k1] * G1 ** 2 * G2 * isl["E"] / RE if k3 == k1 else 0.0
        tF = coef[2] * c.phi[k2] * G2 ** 2 * G1 * isl["F"] / R2 if k3 == k2 else 0.0
        tG = coef[3] * c.phi[k1] * G1 ** 2 * G3 * isl["G"] / R1 if k1 == k2 else 0.0
        tH = coef[4] * c.psi[k1] * G1 ** 3 * isl["H"] / R1 ** 2 if k1 == k2 == k3 else 0.0
        return np.array([tD, tE, tF, tG, tH])
    return island_contributions


_C = [16 / 27, 16 / 27, 32 / 81, 16 / 81, 16 / 81]


def _apply_coef_E_swapped(fwm, isrs, link, egn):
    egn.island_contributions = _contrib([_C[0], _C[2], _C[2], _C[3], _C[4]])


def _apply_coef_H_doubled(fwm, isrs, link, egn):
    egn.island_contributions = _contrib([_C[0], _C[1], _C[2], _C[3], 2 * _C[4]])


def _apply_E_normalised_by_R2(fwm, isrs, link, egn):
    egn.island_contributions = _contrib(_C, norm_e="R2")


def _apply_grid_bin_edges(fwm, isrs, link, egn):
    def grid(c, i):
        return c.lo[i] + np.arange(c.N) * c.delta[i]                # slip: left edges
    egn.grid = grid


def _apply_gate_edge_full_weight(fwm, isrs, link, egn):
    def island_gates(c, f3):
        out = []
        for k3 in range(c.f.size):
            inside = (f3 >= c.lo[k3]) & (f3 <= c.hi[k3])
            if not inside.any():
                continue
            out.append((k3, inside.astype(np.float64)))              # slip: edges weigh 1, not 1/2
        return out
    egn.island_gates = island_gates


def _apply_literal_gain_pre_exponent(fwm, isrs, link, egn):
    def _gain_products(f1, f2, f, spans, p_tot, b_tot):
        f3 = f1 + f2 - f
        out = []
        for s in range(len(spans)):
            lam = np.ones(np.broadcast(f1, f2).shape)
            for sp in spans[:s]:
                g = np.exp(sp["alpha"] * sp["L"])
                r = lambda x: isrs.rho(sp["L"], x, sp["alpha"], p_tot, sp["cr"], b_tot)  # noqa: E731
                lam = lam * g ** 0.5 * np.sqrt(r(f1) * r(f3) * r(f2))      # slip: g^{1/2}
            for sp in spans[s + 1:]:
                g = np.exp(sp["alpha"] * sp["L"])
                lam = lam * g ** 0.5 * np.sqrt(isrs.rho(sp["L"], f, sp["alpha"], p_tot, sp["cr"], b_tot))
            out.append(lam)
        return out
    link._gain_products = _gain_products


MUTANTS = {
    "chi_beta3_no_pi": _apply_chi_beta3_no_pi,
    "chi_sum_minus": _apply_chi_sum_minus,
    "segment_left_endpoint": _apply_segment_left_endpoint,
    "segment_no_attenuation": _apply_segment_no_attenuation,
    "srs_gain_sign": _apply_srs_gain_sign,
    "leff_linear": _apply_leff_linear,
    "phase_includes_current_span": _apply_phase_includes_current_span,
    "coef_E_swapped": _apply_coef_E_swapped,
    "coef_H_doubled": _apply_coef_H_doubled,
    "E_normalised_by_R2": _apply_E_normalised_by_R2,
    "grid_bin_edges": _apply_grid_bin_edges,
    "gate_edge_full_weight": _apply_gate_edge_full_weight,
    "literal_gain_pre_exponent": _apply_literal_gain_pre_exponent,
}


def _apply_segment_count_floor(fwm, isrs, link, egn):
    fwm.segment_count = lambda L, dz: max(1, int(math.floor(L / dz)))   # slip: floor, not ceil


def _apply_gain_sinh_full_argument(fwm, isrs, link, egn):
    def srs_gain(z, f, alpha, p_tot, cr, b_tot):
        ze = isrs.zeta(z, alpha, p_tot, cr)
        x = np.asarray(b_tot * ze, dtype=np.float64)
        f = np.asarray(f, dtype=np.float64)
        safe_x = np.where(x == 0.0, 1.0, x)
        g = safe_x * np.exp(-ze * f) / (2.0 * np.sinh(safe_x))     # slip: sinh(x), not sinh(x/2)
        return np.where(x == 0.0, 1.0, g)
    isrs.srs_gain = srs_gain


def _apply_rho_no_attenuation(fwm, isrs, link, egn):
    isrs.rho = lambda z, f, alpha, p_tot, cr, b_tot: isrs.srs_gain(z, f, alpha, p_tot, cr, b_tot)


def _apply_maclaurin_single_alpha(fwm, isrs, link, egn):
    def mu_maclaurin(f1, f2, f, span, p_tot, b_tot, dz=None):
        L, alpha = span["L"], span["alpha"]
        ch = fwm.chi(f1, f2, f, span["beta2"], span["beta3"])
        eta = fwm.eta_gn(ch, alpha, L)
        sig2 = 1j * ch - 1.0 * alpha                                   # slip: alpha, not 2 alpha
        return eta - p_tot * span["cr"] * (f1 + f2 - f) / alpha * (eta - (np.exp(sig2 * L) - 1.0) / sig2)
    fwm.mu_maclaurin = mu_maclaurin
    fwm.MU_MODES.update(maclaurin=mu_maclaurin)


def _apply_quad_conjugate_phase(fwm, isrs, link, egn):
    orig = fwm.mu_quad
    fwm.mu_quad = lambda *a, **k: np.conj(orig(*a, **k))               # slip: e^{-i chi z}
    fwm.MU_MODES.update(quad=fwm.mu_quad)


def _apply_phi_minus_three(fwm, isrs, link, egn):
    from oracle import formats
    orig = formats.phi_psi

    def phi_psi(points):
        phi, psi = orig(points)
        return phi - 1.0, psi                                          # slip: E|a|^4/(E|a|^2)^2 - 3
    formats.phi_psi = phi_psi


def _apply_btot_sum_of_rates(fwm, isrs, link, egn):
    orig = egn.canonicalize

    def canonicalize(lk):
        c = orig(lk)
        return c._replace(b_tot=float(np.sum(c.R))) if hasattr(c, "_replace") else _set(c, "b_tot",
                                                                                          float(np.sum(c.R)))
    egn.canonicalize = canonicalize


def _apply_ptot_mean(fwm, isrs, link, egn):
    orig = egn.canonicalize

    def canonicalize(lk):
        c = orig(lk)
        return _set(c, "p_tot", float(np.mean(c.P)))
    egn.canonicalize = canonicalize


def _set(c, name, value):
    import dataclasses
    if dataclasses.is_dataclass(c):
        return dataclasses.replace(c, **{name: value})
    return c._replace(**{name: value})


def _apply_H_over_R1(fwm, isrs, link, egn):
    def island_contributions(c, k1, k2, isl):
        out = _contrib(_C)(c, k1, k2, isl)
        if k1 == k2 == isl["k3"]:
            out[4] = out[4] * c.R[k1]                                  # slip: H / R1, not / R1^2
        return out
    egn.island_contributions = island_contributions


MUTANTS.update({
    "segment_count_floor": _apply_segment_count_floor,
    "gain_sinh_full_argument": _apply_gain_sinh_full_argument,
    "rho_no_attenuation": _apply_rho_no_attenuation,
    "maclaurin_single_alpha": _apply_maclaurin_single_alpha,
    "quad_conjugate_phase": _apply_quad_conjugate_phase,
    "phi_minus_three": _apply_phi_minus_three,
    "btot_sum_of_rates": _apply_btot_sum_of_rates,
    "ptot_mean": _apply_ptot_mean,
    "H_over_R1": _apply_H_over_R1,
})


def _region_islands_with(slip):
    """egn.region_islands (Eqs. 17-21, C6, C7, C10) with one slip in the island sums."""
    def region_islands(c, kappa, k1, k2, mu_mode="closed", need=("D", "E", "F", "G", "H"), f=None,
                       gain="ideal"):
        from oracle import egn, link as link_mod
        f = c.f[kappa] if f is None else f
        F1, F2, f3 = egn.region_points(c, kappa, k1, k2, f)
        if slip == "f3_plus_f":
            f3 = F1 + F2 + f
        gates = egn.island_gates(c, f3)
        if not gates:
            return []
        support = np.zeros(f3.shape, dtype=bool)
        for _, t in gates:
            support |= t > 0
        Y = np.zeros(f3.shape, dtype=np.complex128)
        if mu_mode == "unit":
            Y[support] = 1.0
        else:
            Y[support] = link_mod.link_function(F1[support], F2[support], f, c.spans, c.p_tot, c.b_tot, c.dz,
                                                mu_mode, gain)
        d1, d2 = c.delta[k1], c.delta[k2]
        N = c.N
        m1 = np.arange(N)[None, :] * np.ones((N, 1), dtype=np.int64)
        m2 = np.arange(N)[:, None] * np.ones((1, N), dtype=np.int64)
        diag = (m1 - m2 + N - 1) if slip == "G_diagonal_difference" else (m1 + m2)
        ax_e, ax_f = (0, 1) if slip == "E_F_axes_swapped" else (1, 0)
        res = []
        for k3, t in gates:
            isl = dict(k3=k3, npts=int((t > 0).sum()), D=0.0, E=0.0, F=0.0, G=0.0, H=0.0)
            tD = (t > 0).astype(np.float64) if slip == "D_without_edge_weight" else t
            isl["D"] = float(np.sum(tD * np.abs(Y) ** 2) * d1 * d2)
            if k3 == k1 and "E" in need:
                r = np.sum(t * Y, axis=ax_e) * d1
                isl["E"] = float(np.sum(np.abs(r) ** 2) * d2)
            if k3 == k2 and "F" in need:
                col = np.sum(t * Y, axis=ax_f) * d2
                isl["F"] = float(np.sum(np.abs(col) ** 2) * d1)
            if k1 == k2 and "G" in need:
                G = 0.0
                for d in range(2 * N - 1):
                    on = (diag == d) & (t > 0)
                    if not on.any():
                        continue
                    G += t[on][0] * abs(np.sum(Y[on]) * d1) ** 2 * d1
                isl["G"] = float(G)
            if k1 == k2 == k3 and "H" in need:
                tH = 1.0 if slip == "H_without_gate" else t
                isl["H"] = float(abs(np.sum(tH * Y) * d1 * d2) ** 2)
            res.append(isl)
        return res
    return region_islands


def _islands(slip):
    def apply(fwm, isrs, link, egn):
        egn.region_islands = _region_islands_with(slip)
    return apply


def _apply_eta_over_p_squared(fwm, isrs, link, egn):
    orig = egn.eta

    def eta(lk, coi=None, **kw):
        e, t = orig(lk, coi=coi, **kw)[:2]
        c = egn.canonicalize(lk)
        idx = list(range(c.f.size)) if coi is None else list(coi)
        s = c.P[idx]                                                 # slip: / P^2, not / P^3
        return e * s, t * s[:, None]
    egn.eta = eta


def _apply_support_bound_strict(fwm, isrs, link, egn):
    def has_support_bound(c, kappa, k1, k2, f=None):
        f = c.f[kappa] if f is None else f
        lo3 = c.lo[k1] + c.lo[k2] - f + (c.delta[k1] + c.delta[k2]) / 2
        hi3 = c.hi[k1] + c.hi[k2] - f - (c.delta[k1] + c.delta[k2]) / 2
        return bool(np.any((c.hi > lo3) & (c.lo < hi3)))            # slip: open intervals
    egn.has_support_bound = has_support_bound


def _apply_support_bound_bin_edges(fwm, isrs, link, egn):
    def has_support_bound(c, kappa, k1, k2, f=None):
        f = c.f[kappa] if f is None else f
        lo3 = c.lo[k1] + c.lo[k2] - f + (c.delta[k1] + c.delta[k2])   # slip: a full bin, not half
        hi3 = c.hi[k1] + c.hi[k2] - f - (c.delta[k1] + c.delta[k2])
        return bool(np.any((c.hi >= lo3) & (c.lo <= hi3)))
    egn.has_support_bound = has_support_bound


MUTANTS.update({
    "support_bound_strict": _apply_support_bound_strict,
    "support_bound_bin_edges": _apply_support_bound_bin_edges,
    "E_F_axes_swapped": _islands("E_F_axes_swapped"),
    "G_diagonal_difference": _islands("G_diagonal_difference"),
    "H_without_gate": _islands("H_without_gate"),
    "D_without_edge_weight": _islands("D_without_edge_weight"),
    "f3_plus_f": _islands("f3_plus_f"),
    "eta_over_p_squared": _apply_eta_over_p_squared,
})


def _apply_class_ignores_k3(fwm, isrs, link, egn):
    def nli_class(kappa, k1, k2, k3):
        return min(2, len({k1, k2} - {kappa}))                  # slip: k3 not counted
    egn.nli_class = nli_class


def _apply_class_counts_slots(fwm, isrs, link, egn):
    def nli_class(kappa, k1, k2, k3):
        return min(2, sum(k != kappa for k in (k1, k2, k3)) - 1 + (k1 == k2 == k3 == kappa))   # slip: slots, not channels
    egn.nli_class = nli_class


MUTANTS.update({
    "nli_class_ignores_k3": _apply_class_ignores_k3,
    "nli_class_counts_slots": _apply_class_counts_slots,
})


def apply(name):
    from oracle import egn, fwm, isrs, link
    MUTANTS[name](fwm, isrs, link, egn)
