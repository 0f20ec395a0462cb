"""Link function Y (oracle; test infrastructure only).

Two readings of the gain / sqrt(rho) products of Eq. 22:
  gain="ideal" (reading C3, the hot path): the products are identically 1.
  gain="literal" (NEXT-4b, R11): Eq. 22 as printed with a transparent scalar gain
      g_s = e^{alpha_s L_s} that restores the mean span loss only, so the SRS tilt persists:
      Lambda_s = prod_{s'<s} g_{s'}^{3/2} sqrt(rho_{s'}(L, f1) rho_{s'}(L, f1+f2-f) rho_{s'}(L, f2))
               * prod_{s'>s} g_{s'}^{1/2} sqrt(rho_{s'}(L, f)),   rho from Eq. 25 (isrs.rho).

Eq. 22:  Y(f1,f2,f) = sum_s gamma_s mu_s(f1,f2,f) e^{i 4 pi^2 (f1-f)(f2-f) sum(beta2 L + pi (f1+f2) beta3 L)} x (gain products)
Reading C3: the phase sum runs over the spans PRECEDING s,
    theta_1 = 0,  theta_{s+1} = theta_s + chi_s L_s   (chi_s from Eq. 5 with span s's beta2, beta3),
and the gain / sqrt(rho) products are identically 1 (ideal per-span gain equalisation
restores the launch spectrum; the ABI carries no gain input).
"""
import numpy as np

from . import fwm, isrs


def _gain_products(f1, f2, f, spans, p_tot, b_tot):
    """Lambda_s of the literal reading of Eq. 22, one array per span, written out as
    printed: preceding spans contribute g^{3/2} sqrt(rho rho rho) at f1, f1+f2-f, f2; succeeding
    spans g^{1/2} sqrt(rho) at f."""
    f3 = f1 + f2 - f
    out = []
    for s in range(len(spans)):
        lam = np.ones(np.broadcast(f1, f2).shape)
        for sp in spans[:s]:
            g = np.exp(sp["alpha"] * sp["L"])
            r = lambda x: isrs.rho(sp["L"], x, sp["alpha"], p_tot, sp["cr"], b_tot)  # noqa: E731
            lam = lam * g ** 1.5 * np.sqrt(r(f1) * r(f3) * r(f2))
        for sp in spans[s + 1:]:
            g = np.exp(sp["alpha"] * sp["L"])
            lam = lam * g ** 0.5 * np.sqrt(isrs.rho(sp["L"], f, sp["alpha"], p_tot, sp["cr"], b_tot))
        out.append(lam)
    return out


def link_function(f1, f2, f, spans, p_tot, b_tot, dz, mu_mode="closed", gain="ideal"):
    mu_fn = fwm.MU_MODES[mu_mode]
    f1 = np.asarray(f1, dtype=np.float64)
    f2 = np.asarray(f2, dtype=np.float64)
    Y = np.zeros(np.broadcast(f1, f2).shape, dtype=np.complex128)
    theta = np.zeros(Y.shape)
    lam = _gain_products(f1, f2, f, spans, p_tot, b_tot) if gain == "literal" else None
    for s, sp in enumerate(spans):
        mu = mu_fn(f1, f2, f, sp, p_tot, b_tot, dz)
        term = sp["gamma"] * mu * np.exp(1j * theta)
        Y = Y + (term * lam[s] if lam is not None else term)
        theta = theta + fwm.chi(f1, f2, f, sp["beta2"], sp["beta3"]) * sp["L"]
    return Y
