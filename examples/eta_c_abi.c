/* Standalone use of the C ABI (include/isrs_egn.h) without Python or PyTorch.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/eta_c_abi.c -L paper_2412_11614_b200 -lisrs_egn \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2412_11614_b200 -o eta_c_abi
 *   ./eta_c_abi            # prints eta [dB re 1/W^2] for every channel of a 9-channel C-band link
 *
 * The link: 9 channels x 64 GBd on a 100 GHz grid at 193.4 THz, 1 mW each, 16QAM (Phi = -0.68,
 * Psi = 2.08), 3 x 80 km SSMF spans (0.2 dB/km, D 17 ps/nm/km, S 0.067 ps/nm^2/km, gamma 1.3 /W/km,
 * C_r 0.028 /W/km/THz), N = 64, dz = 1 km.  Exit status 0 on success.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "isrs_egn.h"

#define NCH 9
#define NSP 3

int main(void) {
  double f[NCH], r[NCH], p[NCH], phi[NCH], psi[NCH];
  for (int i = 0; i < NCH; ++i) {
    f[i] = 193.4e12 + (i - NCH / 2) * 100e9;   /* integer Hz (reading C10) */
    r[i] = 64e9;
    p[i] = 1e-3;
    phi[i] = -0.68;
    psi[i] = 2.08;
  }
  const double c = 299792458.0, lam = c / 193.4e12;
  const double D = 17e-6, S = 0.067e3;                      /* s/m^2 and s/m^3 */
  const double b2 = -D * lam * lam / (2 * M_PI * c);
  const double b3 = (lam * lam / (2 * M_PI * c)) * (lam * lam / (2 * M_PI * c)) * (S + 2 * D / lam);
  double L[NSP], a[NSP], B2[NSP], B3[NSP], g[NSP], cr[NSP];
  for (int s = 0; s < NSP; ++s) {
    L[s] = 80e3;
    a[s] = 0.2 / (10 * log10(exp(1.0))) * 1e-3;            /* 0.2 dB/km -> 1/m */
    B2[s] = b2;
    B3[s] = b3;
    g[s] = 1.3e-3;
    cr[s] = 2.8e-17;
  }
  isrs_egn_problem prob = {NCH, f, r, p, phi, psi, NSP, L, a, B2, B3, g, cr};
  isrs_egn_numerics num = {64, 1000.0, 64, ISRS_EGN_MU_SEGMENT, 0u, 0};
  isrs_egn_t *h = NULL;
  int rc = isrs_egn_create(&prob, &num, 0, &h);
  if (rc) {
    fprintf(stderr, "create: %s (%s)\n", isrs_egn_strerror(rc), isrs_egn_last_error());
    return 1;
  }
  double *eta_dev = NULL;
  if (cudaMalloc((void **)&eta_dev, NCH * sizeof(double)) != cudaSuccess) return 1;
  rc = isrs_egn_nli(h, NCH, NULL, eta_dev, NULL, NULL);
  if (rc) {
    fprintf(stderr, "nli: %s (%s)\n", isrs_egn_strerror(rc), isrs_egn_last_error());
    return 1;
  }
  double eta[NCH];
  if (cudaMemcpy(eta, eta_dev, sizeof(eta), cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  int64_t pts = 0, ps = 0, nreg = 0;
  isrs_egn_last_work(h, &pts, &ps, &nreg);
  for (int i = 0; i < NCH; ++i) printf("channel %d  eta %.17e 1/W^2  %.6f dB\n", i, eta[i], 10 * log10(eta[i]));
  printf("regions %lld  points %lld  point-spans %lld\n", (long long)nreg, (long long)pts, (long long)ps);
  cudaFree(eta_dev);
  isrs_egn_destroy(h);
  for (int i = 0; i < NCH; ++i)
    if (!(eta[i] > 0) || !isfinite(eta[i])) return 2;
  return 0;
}
