"""Link function Y (oracle; test infrastructure only).

Eq. 22:  Y(f1,f2,f) = sum_s gamma_s mu_s(f1,f2,f) e^{i 4 pi^2 (f1-f)(f2-f) sum(beta2 L + pi (f1+f2) beta3 L)} x (gain products)
Reading C3: the phase sum runs over the spans PRECEDING s,
    theta_1 = 0,  theta_{s+1} = theta_s + chi_s L_s   (chi_s from Eq. 5 with span s's beta2, beta3),
and the gain / sqrt(rho) products are identically 1 (ideal per-span gain equalisation
restores the launch spectrum; the ABI carries no gain input).
"""
import numpy as np

from . import fwm


def link_function(f1, f2, f, spans, p_tot, b_tot, dz, mu_mode="closed"):
    mu_fn = fwm.MU_MODES[mu_mode]
    f1 = np.asarray(f1, dtype=np.float64)
    f2 = np.asarray(f2, dtype=np.float64)
    Y = np.zeros(np.broadcast(f1, f2).shape, dtype=np.complex128)
    theta = np.zeros(Y.shape)
    for sp in spans:
        mu = mu_fn(f1, f2, f, sp, p_tot, b_tot, dz)
        Y = Y + sp["gamma"] * mu * np.exp(1j * theta)
        theta = theta + fwm.chi(f1, f2, f, sp["beta2"], sp["beta3"]) * sp["L"]
    return Y
