/* ORACLE — test infrastructure only (see oracle/__init__.py).  Only tests/ (and the scripts under
 * tests/tools/ that write golden files) load this library; the product path never does, and this
 * file shares no code with paper_2412_11614_b200/ (no headers, helpers or tables).
 *
 * "Fast-plain" variant of the oracle's `closed` mode (oracle cost table): the same
 * definition as oracle/egn.py + fwm.py + link.py + isrs.py, evaluated in plain C (fp64, OpenMP over
 * (COI, kappa1) tasks, no fast-math, no FMA contraction) with three savings that do not change the
 * mathematics:
 *   (i)   the segment terms I_k of Eq. 9 come from the FORWARD recurrence
 *         e^{sigma (k+1) h} = e^{sigma k h} e^{sigma h}  (sigma = i chi - alpha, h = L/K),
 *         I_k = (e^{sigma (k+1) h} - e^{sigma k h}) / sigma;
 *   (ii)  the SRS-gain factors SRS_G(z_k, f3) of Eq. 8 (Eq. 14) are tabulated once per
 *         distinct f3 of a region (f3 = f1 + f2 - f is exact in fp64 on the integer-Hz lattice,
 *         reading C10; every point's f3 is checked bitwise against its table row's);
 *   (iii) mu_s (Eq. 8) is computed once per point for each DISTINCT span parameter set (L, alpha,
 *         beta2, beta3, C_r) and reused for every span of that set (the values are identical), and
 *         the span phase e^{i theta_s} of Eq. 22 (reading C3: theta_1 = 0,
 *         theta_{s+1} = theta_s + chi_s L_s) is advanced as e^{i theta_{s+1}} = e^{i theta_s} e^{i chi_s L_s}.
 * Everything else follows egn.py step by step: reading C5 canonicalisation, C6 bin-centre grid, C10
 * gates (1 inside, 1/2 on a band edge), islands = the kappa3 partition of a region's points, Eqs. 17-21
 * with C7 (E coherent over f1 at fixed f2, F over f2 at fixed f1, G along anti-diagonals with
 * |S(f3)|^2 outside the modulus, H over the island), C8 gating, Eq. 15 weights with C2, Eq. 11.
 * Pinned to the literal closed mode (egn.eta, fwm.mu_segment) at <= 1e-12 by
 * tests/test_oracle_fastplain.py.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#ifndef FP_BLK
#define FP_BLK 16
#endif

typedef struct {
  int32_t n_ch;
  const double *f_center_hz, *symbol_rate_hz, *launch_power_w, *phi, *psi;
  int32_t n_span;
  const double *length_m, *alpha_per_m, *beta2, *beta3, *gamma, *cr;
  int32_t grid_n;
  double delta_z_m;
} fp_link;

typedef struct {
  int n, N, ns, nset;
  double fc, btot, ptot, dz;
  double *f, *R, *P, *G, *phi, *psi, *lo, *hi, *d;
  long long *rate;
  int *set_of;      /* [ns] distinct span parameter set of span s                     */
  int *rep;         /* [nset] first span of each set                                  */
  int *K;           /* [nset] K = ceil(L / dz)                                        */
  double **zeta;    /* [nset][K] zeta_k = P_tot C_r L_eff(z_k)       (Eq. 2, Eq. 10)   */
  double **pref;    /* [nset][K] x / (2 sinh(x/2)), x = B_tot zeta_k (Eq. 14; 1 at x=0) */
} canon;

static void canon_free(canon *c) {
  free(c->f); free(c->R); free(c->P); free(c->G); free(c->phi); free(c->psi);
  free(c->lo); free(c->hi); free(c->d); free(c->rate); free(c->set_of); free(c->rep); free(c->K);
  if (c->zeta) for (int i = 0; i < c->nset; ++i) free(c->zeta[i]);
  if (c->pref) for (int i = 0; i < c->nset; ++i) free(c->pref[i]);
  free(c->zeta); free(c->pref);
}

/* Reading C5: offsets from the occupied-band midpoint, B_tot edge-to-edge, P_tot = sum P_i;
 * C16: G_i = P_i / R_i; C6: delta_i = R_i / N.  Spans: distinct parameter sets. */
static int canon_build(const fp_link *L, canon *c) {
  memset(c, 0, sizeof(*c));
  const int n = L->n_ch, ns = L->n_span;
  c->n = n; c->N = L->grid_n; c->ns = ns; c->dz = L->delta_z_m;
  double lo_min = 1e300, hi_max = -1e300;
  for (int i = 0; i < n; ++i) {
    const double lo = L->f_center_hz[i] - L->symbol_rate_hz[i] / 2, hi = L->f_center_hz[i] + L->symbol_rate_hz[i] / 2;
    if (lo < lo_min) lo_min = lo;
    if (hi > hi_max) hi_max = hi;
  }
  c->fc = (lo_min + hi_max) / 2;
  c->btot = hi_max - lo_min;
#define ALLOC(p, cnt) p = calloc((size_t)(cnt) > 0 ? (size_t)(cnt) : 1, sizeof(*p))
  ALLOC(c->f, n); ALLOC(c->R, n); ALLOC(c->P, n); ALLOC(c->G, n); ALLOC(c->phi, n); ALLOC(c->psi, n);
  ALLOC(c->lo, n); ALLOC(c->hi, n); ALLOC(c->d, n); ALLOC(c->rate, n);
  ALLOC(c->set_of, ns); ALLOC(c->rep, ns); ALLOC(c->K, ns); ALLOC(c->zeta, ns); ALLOC(c->pref, ns);
  c->ptot = 0;
  for (int i = 0; i < n; ++i) {
    c->f[i] = L->f_center_hz[i] - c->fc;
    c->R[i] = L->symbol_rate_hz[i];
    c->P[i] = L->launch_power_w[i];
    c->G[i] = c->P[i] / c->R[i];
    c->phi[i] = L->phi[i];
    c->psi[i] = L->psi ? L->psi[i] : 0.0;
    c->lo[i] = c->f[i] - c->R[i] / 2;
    c->hi[i] = c->f[i] + c->R[i] / 2;
    c->d[i] = c->R[i] / c->N;
    c->rate[i] = (long long)c->R[i];
    c->ptot += c->P[i];
  }
  for (int i = 1; i < n; ++i)
    if (!(c->lo[i] >= c->hi[i - 1])) return -1;   /* bands must be sorted and disjoint (touching allowed) */
  for (int s = 0; s < ns; ++s) {
    int found = -1;
    for (int t = 0; t < c->nset && found < 0; ++t) {
      const int r = c->rep[t];
      if (L->length_m[r] == L->length_m[s] && L->alpha_per_m[r] == L->alpha_per_m[s] &&
          L->beta2[r] == L->beta2[s] && L->beta3[r] == L->beta3[s] && L->cr[r] == L->cr[s])
        found = t;
    }
    if (found < 0) {
      found = c->nset++;
      c->rep[found] = s;
      const double Ls = L->length_m[s], a = L->alpha_per_m[s];
      const int K = (int)ceil(Ls / c->dz);
      c->K[found] = K;
      c->zeta[found] = calloc(K, sizeof(double));
      c->pref[found] = calloc(K, sizeof(double));
      for (int k = 0; k < K; ++k) {
        const double zk = (k + 0.5) / K * Ls;                 /* Eq. 10 */
        const double leff = -expm1(-a * zk) / a;              /* L_eff(z) = (1 - e^{-alpha z}) / alpha */
        const double ze = c->ptot * L->cr[s] * leff;          /* Eq. 2 */
        const double x = c->btot * ze;
        c->zeta[found][k] = ze;
        c->pref[found][k] = (x == 0.0) ? 1.0 : x / (2.0 * sinh(x / 2.0));   /* Eq. 14 */
      }
    }
    c->set_of[s] = found;
  }
  return 0;
}

static long long gcdll(long long a, long long b) {
  while (b) { const long long t = a % b; a = b; b = t; }
  return a;
}

/* per-thread scratch */
typedef struct {
  int cap_pts, cap_lines, lp;
  double *Yr, *Yi;           /* [N*N] link function Y at (m2, m1); 0 outside support */
  int *line_of;              /* [N*N] line index of the point (-1: no support)        */
  double *lf3;               /* [lines] f3 of the line                               */
  int *lset;                 /* [lines] 1 once lf3 is set                            */
  int *gk[2];                /* [lines] up to two bands containing f3 (-1: none)      */
  double *gt[2];             /* [lines] their C10 factors t                          */
  int *start, *cnt, *pts;    /* counting sort of points by line                      */
  /* vector scratch over one line's points */
  double *chi, *Er, *Ei, *wr, *wi, *ar, *ai, *yr, *yi, *pr, *pim, *sr, *si;
  double *mur, *mui;         /* [nset * N] mu of each span set at the line's points      */
  double *stepr, *stepi;     /* [nset * N] e^{i chi L} of each span set                */
  double *g;                 /* [Kmax] SRS gain row                                  */
} scratch;

static void scratch_free(scratch *w) {
  free(w->Yr); free(w->Yi); free(w->line_of); free(w->lf3); free(w->lset);
  free(w->gk[0]); free(w->gk[1]); free(w->gt[0]); free(w->gt[1]); free(w->start); free(w->cnt);
  free(w->pts); free(w->chi); free(w->Er); free(w->Ei); free(w->wr); free(w->wi); free(w->ar);
  free(w->ai); free(w->yr); free(w->yi); free(w->pr); free(w->pim); free(w->sr); free(w->si);
  free(w->mur); free(w->mui); free(w->stepr); free(w->stepi); free(w->g);
}

static int scratch_init(scratch *w, const canon *c, int max_ratio_sum) {
  memset(w, 0, sizeof(*w));
  const int N = c->N;
  /* <= N points per line; padded to whole blocks */
  const int np = N * N, nl = max_ratio_sum * (N - 1) + 1, lp = N + FP_BLK;
  int kmax = 1;
  for (int t = 0; t < c->nset; ++t) if (c->K[t] > kmax) kmax = c->K[t];
  w->cap_pts = np;
  w->lp = lp;
  w->cap_lines = nl;
  w->Yr = malloc(sizeof(double) * np); w->Yi = malloc(sizeof(double) * np);
  w->line_of = malloc(sizeof(int) * np); w->pts = malloc(sizeof(int) * np);
  w->lf3 = malloc(sizeof(double) * nl); w->lset = malloc(sizeof(int) * nl);
  for (int q = 0; q < 2; ++q) { w->gk[q] = malloc(sizeof(int) * nl); w->gt[q] = malloc(sizeof(double) * nl); }
  w->start = malloc(sizeof(int) * (nl + 1)); w->cnt = malloc(sizeof(int) * nl);
  double **v[] = {&w->chi, &w->Er, &w->Ei, &w->wr, &w->wi, &w->ar, &w->ai, &w->yr, &w->yi, &w->pr,
                  &w->pim, &w->sr, &w->si};
  for (size_t q = 0; q < sizeof(v) / sizeof(v[0]); ++q) *v[q] = calloc(lp, sizeof(double));
  w->mur = calloc((size_t)lp * c->nset, sizeof(double)); w->mui = calloc((size_t)lp * c->nset, sizeof(double));
  w->stepr = calloc((size_t)lp * c->nset, sizeof(double)); w->stepi = calloc((size_t)lp * c->nset, sizeof(double));
  w->g = malloc(sizeof(double) * kmax);
  return (w->Yr && w->Yi && w->line_of && w->pts && w->lf3 && w->mur && w->mui && w->g) ? 0 : -1;
}

/* C10 gate of f3: every band [lo, hi] containing f3, t = 1 strictly inside, 1/2 on an edge.  The
 * bands are disjoint and sorted (canonicalize checks it), so only the last band starting at or below
 * f3 and the one before it (touching bands) can hold it. */
static void gates(const canon *c, double f3, int *k, double *t) {
  k[0] = k[1] = -1;
  t[0] = t[1] = 0.0;
  int lo = 0, hi = c->n - 1;
  if (f3 < c->lo[0]) return;
  while (lo < hi) {                       /* largest i with lo[i] <= f3 */
    const int mid = (lo + hi + 1) / 2;
    if (c->lo[mid] <= f3) lo = mid; else hi = mid - 1;
  }
  int q = 0;
  for (int i = (lo > 0 ? lo - 1 : 0); i <= lo; ++i) {
    if (f3 >= c->lo[i] && f3 <= c->hi[i]) {
      k[q] = i;
      t[q] = (f3 > c->lo[i] && f3 < c->hi[i]) ? 1.0 : 0.5;
      ++q;
    }
  }
}

/* One region (kappa, k1, k2) at NLI frequency f.  Writes, per island k3 of the region, the Eq. 15
 * (reading C2) contributions into contrib[5] (summed over islands) and the raw partials
 * part[6] = {sum G_k3 D, E[k3==k1], F[k3==k2], sum G_k3 G [k1==k2], H[k1==k2==k3], n_points}.
 * Returns -1 if a point's f3 differs from its line's (lattice not exact), else 0. */
static int region(const fp_link *Lk, const canon *c, scratch *w, double f, int k1, int k2,
                  double contrib[5], double part[6]) {
  const int N = c->N;
  for (int q = 0; q < 5; ++q) contrib[q] = 0.0;
  for (int q = 0; q < 6; ++q) part[q] = 0.0;
  /* cheap necessary condition: the f3 range of the bin centres meets some band */
  const double lo3 = c->lo[k1] + c->lo[k2] - f + (c->d[k1] + c->d[k2]) / 2;
  const double hi3 = c->hi[k1] + c->hi[k2] - f - (c->d[k1] + c->d[k2]) / 2;
  int any = 0;
  for (int i = 0; i < c->n && !any; ++i) any = (c->hi[i] >= lo3 && c->lo[i] <= hi3);
  if (!any) return 0;
  const long long gg = gcdll(c->rate[k1], c->rate[k2]);
  const int a = (int)(c->rate[k1] / gg), b = (int)(c->rate[k2] / gg);
  const int nl = (a + b) * (N - 1) + 1;
  const double d1 = c->d[k1], d2 = c->d[k2];
  /* C6 bin centres; points bucketed by the lattice line j = a m1 + b m2 on which f3 is constant */
  for (int j = 0; j < nl; ++j) { w->lset[j] = 0; w->cnt[j] = 0; }
  for (int m2 = 0; m2 < N; ++m2) {
    const double f2 = c->lo[k2] + (m2 + 0.5) * d2;
    for (int m1 = 0; m1 < N; ++m1) {
      const double f1 = c->lo[k1] + (m1 + 0.5) * d1;
      const double f3 = f1 + f2 - f;
      const int j = a * m1 + b * m2;
      if (!w->lset[j]) {
        w->lset[j] = 1;
        w->lf3[j] = f3;
        int kk[2];
        double tt[2];
        gates(c, f3, kk, tt);
        w->gk[0][j] = kk[0]; w->gk[1][j] = kk[1]; w->gt[0][j] = tt[0]; w->gt[1][j] = tt[1];
      } else if (w->lf3[j] != f3) {
        return -1;
      }
      const int idx = m2 * N + m1;
      w->Yr[idx] = 0.0;
      w->Yi[idx] = 0.0;
      if (w->gk[0][j] >= 0) {
        w->line_of[idx] = j;
        w->cnt[j] += 1;
      } else {
        w->line_of[idx] = -1;
      }
    }
  }
  w->start[0] = 0;
  for (int j = 0; j < nl; ++j) w->start[j + 1] = w->start[j] + w->cnt[j];
  for (int j = 0; j < nl; ++j) w->cnt[j] = 0;
  for (int idx = 0; idx < N * N; ++idx) {
    const int j = w->line_of[idx];
    if (j >= 0) w->pts[w->start[j] + w->cnt[j]++] = idx;
  }
  /* the link function Y (Eq. 22, C3) at every supported point, one line at a time */
  for (int j = 0; j < nl; ++j) {
    const int np = w->cnt[j];
    if (np == 0) continue;
    const int *pp = w->pts + w->start[j];
    const double f3 = w->lf3[j];
    double *restrict uv = w->chi, *restrict sf = w->yr;
    for (int p = 0; p < np; ++p) {
      const int m1 = pp[p] % N, m2 = pp[p] / N;
      const double f1 = c->lo[k1] + (m1 + 0.5) * d1, f2 = c->lo[k2] + (m2 + 0.5) * d2;
      uv[p] = (f1 - f) * (f2 - f);       /* the span-independent factors of Eq. 5 */
      sf[p] = f1 + f2;
    }
    for (int t = 0; t < c->nset; ++t) {
      const int s = c->rep[t], K = c->K[t];
      const double Ls = Lk->length_m[s], al = Lk->alpha_per_m[s], h = Ls / K;
      const double b2 = Lk->beta2[s], b3 = Lk->beta3[s];
      double *restrict g = w->g;
      /* Eq. 8 factor SRS_G(z_k, f3) (Eq. 14) for this line */
      for (int k = 0; k < K; ++k) g[k] = c->pref[t][k] * exp(-c->zeta[t][k] * f3);
      double *restrict mr = w->mur + (size_t)t * w->lp, *restrict mi = w->mui + (size_t)t * w->lp;
      double *restrict str = w->stepr + (size_t)t * w->lp, *restrict sti = w->stepi + (size_t)t * w->lp;
      double *restrict Er = w->Er, *restrict Ei = w->Ei, *restrict wr = w->wr, *restrict wi = w->wi;
      double *restrict ar = w->ar, *restrict ai = w->ai, *restrict chi = w->pr;
      const double e = exp(-al * h);
      for (int p = 0; p < np; ++p) {
        /* Eq. 5: chi = 4 pi^2 (f1 - f)(f2 - f) [beta2 + pi beta3 (f1 + f2)] */
        const double ch = 4.0 * M_PI * M_PI * uv[p] * (b2 + M_PI * b3 * sf[p]);
        chi[p] = ch;
        double sn, cs;
        sincos(ch * h, &sn, &cs);
        wr[p] = e * cs;                          /* e^{sigma h} = e^{-alpha h} e^{i chi h} */
        wi[p] = e * sn;
        Er[p] = 1.0;                             /* e^{sigma k h} at k = 0 */
        Ei[p] = 0.0;
        ar[p] = 0.0;
        ai[p] = 0.0;
        sincos(ch * Ls, &sti[p], &str[p]);      /* e^{i chi L}: the phase step of Eq. 22 (C3) */
      }
      /* the K-term sum of Eq. 8, FP_BLK points at a time (their recurrence state in registers) */
      for (int p0 = 0; p0 < np; p0 += FP_BLK) {
        double er[FP_BLK], ei[FP_BLK], xr[FP_BLK], xi[FP_BLK], sr[FP_BLK], si[FP_BLK];
        for (int q = 0; q < FP_BLK; ++q) {
          const int p = (p0 + q < np) ? p0 + q : np - 1;
          er[q] = Er[p]; ei[q] = Ei[p]; xr[q] = wr[p]; xi[q] = wi[p]; sr[q] = 0.0; si[q] = 0.0;
        }
        for (int k = 0; k < K; ++k) {
          const double gk = g[k];
          for (int q = 0; q < FP_BLK; ++q) {
            const double nr = er[q] * xr[q] - ei[q] * xi[q];   /* e^{sigma (k+1) h} */
            const double ni = er[q] * xi[q] + ei[q] * xr[q];
            sr[q] += gk * (nr - er[q]);                         /* SRS_G(z_k) sigma I_k (Eq. 9) */
            si[q] += gk * (ni - ei[q]);
            er[q] = nr;
            ei[q] = ni;
          }
        }
        for (int q = 0; q < FP_BLK && p0 + q < np; ++q) {
          ar[p0 + q] = sr[q];
          ai[p0 + q] = si[q];
        }
      }
      for (int p = 0; p < np; ++p) {
        /* Eq. 8: mu = sum_k SRS_G(z_k) I_k = [sum_k SRS_G(z_k) (e^{sigma(k+1)h} - e^{sigma k h})] / sigma */
        const double sr = -al, si = chi[p];
        const double den = sr * sr + si * si;
        mr[p] = (ar[p] * sr + ai[p] * si) / den;
        mi[p] = (ai[p] * sr - ar[p] * si) / den;
      }
    }
    /* Eq. 22 (C3): Y = sum_s gamma_s mu_s e^{i theta_s}, theta_1 = 0,
     * e^{i theta_{s+1}} = e^{i theta_s} e^{i chi_s L_s} */
    double *restrict yr = w->ar, *restrict yi = w->ai, *restrict pr = w->pr, *restrict pim = w->pim;
    for (int p = 0; p < np; ++p) { yr[p] = 0.0; yi[p] = 0.0; pr[p] = 1.0; pim[p] = 0.0; }
    for (int s = 0; s < c->ns; ++s) {
      const int t = c->set_of[s];
      const double gam = Lk->gamma[s];
      const double *restrict mr = w->mur + (size_t)t * w->lp, *restrict mi = w->mui + (size_t)t * w->lp;
      const double *restrict str = w->stepr + (size_t)t * w->lp, *restrict sti = w->stepi + (size_t)t * w->lp;
      for (int p = 0; p < np; ++p) {
        const double tr = gam * mr[p], ti = gam * mi[p];
        yr[p] += tr * pr[p] - ti * pim[p];
        yi[p] += tr * pim[p] + ti * pr[p];
        const double nr = pr[p] * str[p] - pim[p] * sti[p];
        pim[p] = pr[p] * sti[p] + pim[p] * str[p];
        pr[p] = nr;
      }
    }
    for (int p = 0; p < np; ++p) {
      w->Yr[pp[p]] = yr[p];
      w->Yi[pp[p]] = yi[p];
    }
  }
  /* islands: every band k3 holding some supported point (ascending k3) */
  long long npts = 0;
  for (int j = 0; j < nl; ++j) npts += w->cnt[j];
  part[5] = (double)npts;
  int k3lo = c->n, k3hi = -1;
  for (int j = 0; j < nl; ++j) {
    if (!w->cnt[j]) continue;
    for (int q = 0; q < 2; ++q) {
      const int k = w->gk[q][j];
      if (k < 0) continue;
      if (k < k3lo) k3lo = k;
      if (k > k3hi) k3hi = k;
    }
  }
  const int needE = c->phi[k1] != 0.0, needF = c->phi[k2] != 0.0, needG = c->phi[k1] != 0.0,
            needH = c->psi[k1] != 0.0;   /* C8 */
  for (int k3 = k3lo; k3 <= k3hi; ++k3) {
    /* t of point idx in island k3 */
#define TAT(idx) (w->line_of[idx] < 0 ? 0.0 : (w->gk[0][w->line_of[idx]] == k3 ? w->gt[0][w->line_of[idx]] : (w->gk[1][w->line_of[idx]] == k3 ? w->gt[1][w->line_of[idx]] : 0.0)))
    int present = 0;
    double D = 0.0;
    for (int idx = 0; idx < N * N; ++idx) {
      const double t = TAT(idx);
      if (t > 0.0) {
        present = 1;
        D += t * (w->Yr[idx] * w->Yr[idx] + w->Yi[idx] * w->Yi[idx]);   /* Eq. 17 */
      }
    }
    if (!present) continue;
    D *= d1 * d2;
    double E = 0.0, F = 0.0, Gv = 0.0, H = 0.0;
    if (k3 == k1 && needE) {       /* Eq. 18, C7: coherent over f1 at fixed f2 */
      for (int m2 = 0; m2 < N; ++m2) {
        double rr = 0.0, ri = 0.0;
        for (int m1 = 0; m1 < N; ++m1) {
          const int idx = m2 * N + m1;
          const double t = TAT(idx);
          rr += t * w->Yr[idx];
          ri += t * w->Yi[idx];
        }
        rr *= d1; ri *= d1;
        E += rr * rr + ri * ri;
      }
      E *= d2;
    }
    if (k3 == k2 && needF) {       /* Eq. 19, C7: coherent over f2 at fixed f1 */
      for (int m1 = 0; m1 < N; ++m1) {
        double cr_ = 0.0, ci_ = 0.0;
        for (int m2 = 0; m2 < N; ++m2) {
          const int idx = m2 * N + m1;
          const double t = TAT(idx);
          cr_ += t * w->Yr[idx];
          ci_ += t * w->Yi[idx];
        }
        cr_ *= d2; ci_ *= d2;
        F += cr_ * cr_ + ci_ * ci_;
      }
      F *= d1;
    }
    if (k1 == k2 && needG) {       /* Eq. 20, C7: coherent along f1 + f2 = const, |S(f3)|^2 outside */
      for (int dd = 0; dd <= 2 * (N - 1); ++dd) {
        double sr = 0.0, si = 0.0, td = 0.0;
        int on = 0;
        for (int m1 = (dd < N ? 0 : dd - N + 1); m1 <= (dd < N ? dd : N - 1); ++m1) {
          const int idx = (dd - m1) * N + m1;
          const double t = TAT(idx);
          if (t > 0.0) {
            if (!on) td = t;
            on = 1;
            sr += w->Yr[idx];
            si += w->Yi[idx];
          }
        }
        if (!on) continue;
        sr *= d1; si *= d1;
        Gv += td * (sr * sr + si * si) * d1;
      }
    }
    if (k1 == k2 && k2 == k3 && needH) {   /* Eq. 21, C7: coherent over the island */
      double hr = 0.0, hi = 0.0;
      for (int idx = 0; idx < N * N; ++idx) {
        const double t = TAT(idx);
        hr += t * w->Yr[idx];
        hi += t * w->Yi[idx];
      }
      hr *= d1 * d2; hi *= d1 * d2;
      H = hr * hr + hi * hi;
    }
#undef TAT
    /* Eq. 15 with reading C2 */
    const double G1 = c->G[k1], G2 = c->G[k2], G3 = c->G[k3], R1 = c->R[k1], R2 = c->R[k2];
    contrib[0] += 16.0 / 27.0 * G1 * G2 * G3 * D;
    if (k3 == k1) contrib[1] += 16.0 / 27.0 * c->phi[k1] * G1 * G1 * G2 * E / R1;
    if (k3 == k2) contrib[2] += 32.0 / 81.0 * c->phi[k2] * G2 * G2 * G1 * F / R2;
    if (k1 == k2) contrib[3] += 16.0 / 81.0 * c->phi[k1] * G1 * G1 * G3 * Gv / R1;
    if (k1 == k2 && k2 == k3) contrib[4] += 16.0 / 81.0 * c->psi[k1] * G1 * G1 * G1 * H / (R1 * R1);
    part[0] += G3 * D;
    if (k3 == k1) part[1] += E;
    if (k3 == k2) part[2] += F;
    if (k1 == k2) part[3] += G3 * Gv;
    if (k1 == k2 && k2 == k3) part[4] += H;
  }
  return 0;
}

static int max_ratio_sum(const canon *c) {
  int m = 2;
  for (int i = 0; i < c->n; ++i)
    for (int j = 0; j < c->n; ++j) {
      const long long g = gcdll(c->rate[i], c->rate[j]);
      const int s = (int)((c->rate[i] + c->rate[j]) / g);
      if (s > m) m = s;
    }
  return m;
}

/* eta for n_coi COIs (Eq. 11, reading C13: P = P_kappa): terms_out[n_coi][5] (D..H contributions
 * after the Eq. 11 scale), eta_out[n_coi], npts_out[n_coi].  Tasks = (COI, kappa1), dynamic
 * schedule; per-task sums are combined in fixed order, so the result does not depend on the thread
 * count.  progress (or NULL) is incremented once per finished task.  Returns 0, -1 (allocation), -2
 * (inexact lattice). */
int fp_eta(const fp_link *Lk, int n_coi, const int32_t *coi, int nthreads, double *terms_out,
           double *eta_out, long long *npts_out, volatile long long *progress) {
  canon c;
  if (canon_build(Lk, &c) != 0) { canon_free(&c); return -3; }
  const int n = c.n;
  const long long ntask = (long long)n_coi * n;
  double *tsum = calloc((size_t)ntask * 5, sizeof(double));
  long long *tpts = calloc((size_t)ntask, sizeof(long long));
  int err = 0;
  const int mrs = max_ratio_sum(&c);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel
  {
    scratch w;
    if (scratch_init(&w, &c, mrs) != 0) {
#pragma omp atomic write
      err = -1;
    }
#pragma omp for schedule(dynamic, 1)
    for (long long task = 0; task < ntask; ++task) {
      if (err) continue;
      const int ci = (int)(task / n), k1 = (int)(task % n);
      const int kappa = coi[ci];
      double con[5], part[6];
      for (int k2 = 0; k2 < n; ++k2) {
        if (region(Lk, &c, &w, c.f[kappa], k1, k2, con, part) != 0) {
#pragma omp atomic write
          err = -2;
          break;
        }
        for (int q = 0; q < 5; ++q) tsum[task * 5 + q] += con[q];
        tpts[task] += (long long)part[5];
      }
      if (progress) {
#pragma omp atomic
        *progress += 1;
      }
    }
    scratch_free(&w);
  }
  if (!err) {
    for (int ci = 0; ci < n_coi; ++ci) {
      const int kappa = coi[ci];
      double acc[5] = {0, 0, 0, 0, 0};
      long long np = 0;
      for (int k1 = 0; k1 < n; ++k1) {
        for (int q = 0; q < 5; ++q) acc[q] += tsum[((long long)ci * n + k1) * 5 + q];
        np += tpts[(long long)ci * n + k1];
      }
      /* P_NLI = R_kappa G_NLI(f_kappa) (C1); Eq. 11 */
      const double scale = c.R[kappa] / (c.P[kappa] * c.P[kappa] * c.P[kappa]);
      double e = 0.0;
      for (int q = 0; q < 5; ++q) {
        terms_out[ci * 5 + q] = acc[q] * scale;
        e += acc[q] * scale;
      }
      eta_out[ci] = e;
      if (npts_out) npts_out[ci] = np;
    }
  }
  free(tsum);
  free(tpts);
  canon_free(&c);
  return err;
}

/* Raw partials of one region at the COI centre: out[6] = {sum G_k3 D, E, F, sum G_k3 G, H, n_points}
 * (the quantities oracle/egn.py region_partials returns).  Returns 0, -1, -2 as fp_eta. */
int fp_region(const fp_link *Lk, int kappa, int k1, int k2, double *out) {
  canon c;
  if (canon_build(Lk, &c) != 0) { canon_free(&c); return -3; }
  scratch w;
  int rc = scratch_init(&w, &c, max_ratio_sum(&c));
  double con[5];
  if (rc == 0) rc = region(Lk, &c, &w, c.f[kappa], k1, k2, con, out) ? -2 : 0;
  scratch_free(&w);
  canon_free(&c);
  return rc;
}
