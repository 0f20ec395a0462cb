"""Modulation-format constants Phi, Psi from constellation moments (oracle; test infra only).

The paper uses Phi_kappa, Psi_kappa in Eq. 15 but never defines them (reading C9).
Reading C9: for unit-average-energy i.i.d. symbols a,
    Phi = E|a|^4 / (E|a|^2)^2 - 2                         (excess kurtosis; Gaussian 0)
    Psi = E|a|^6 / (E|a|^2)^3 - 9 E|a|^4/(E|a|^2)^2 + 12  (sixth-order circular cumulant; Gaussian 0)
The values BASELINE.json quotes (QPSK -1, 16QAM -0.68, 64QAM -0.619) follow from the first line.
"""
import numpy as np


def square_qam(m):
    """Points of a square M-QAM constellation (odd integer levels per quadrature)."""
    k = int(round(np.sqrt(m)))
    assert k * k == m
    lv = np.arange(-(k - 1), k, 2, dtype=np.float64)
    x, y = np.meshgrid(lv, lv)
    return (x + 1j * y).ravel()


def phi_psi(points):
    a = np.asarray(points, dtype=np.complex128)
    m2 = np.mean(np.abs(a) ** 2)
    m4 = np.mean(np.abs(a) ** 4)
    m6 = np.mean(np.abs(a) ** 6)
    phi = m4 / m2 ** 2 - 2.0
    psi = m6 / m2 ** 3 - 9.0 * m4 / m2 ** 2 + 12.0
    return phi, psi


def gaussian_moments_phi_psi():
    """Circular complex Gaussian: E|a|^4 = 2 s^2, E|a|^6 = 6 s^3 -> Phi = Psi = 0."""
    return 2.0 - 2.0, 6.0 - 18.0 + 12.0
