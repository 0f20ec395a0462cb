/*
 * isrs_egn.h — C ABI of the B200-native ISRS EGN hot path (paper arXiv 2412.11614).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, P:n = line n):
 *   eta_kappa = sigma^2_NLI,kappa / P_kappa^3                     Eq. 11
 * for every requested channel of interest (COI) kappa, with sigma^2 assembled from the
 * ISRS EGN island integrals D, E, F, G, H (Eqs. 15-21) over the 2-D (f1, f2)
 * domain at f = f_kappa (reading C1 of DESIGN.md), the link function Y (Eq. 22, P:267,
 * reading C3: phase of the preceding spans, gain products = 1), and the FWM efficiency
 * factor mu_s in the paper's segment closed form (Eqs. 7-10).
 * Readings C1-C17 fix everything the paper leaves open; the oracle in
 * oracle/ implements the same definition independently.
 *
 * Units: SI throughout (Hz, W, m, s^2/m, s^3/m, 1/(W m), 1/(W m Hz)); frequencies absolute.
 * Exactness requirement (reading C10): every f_center_hz and symbol_rate_hz is an integer
 * number of Hz, and symbol_rate_hz / (2 * grid_n) is an integer, so that every grid frequency
 * and every f1 + f2 - f is exact in fp64 and band-edge ties are decided exactly.
 *
 * Threading: a handle is not thread-safe; distinct handles are independent.  Successive calls on
 * one handle are ordered on the device even when issued on different streams (a call on a new
 * stream waits for the previous call's end on the device, not on the host).
 * Devices: every call makes the handle's device current for its duration and restores the
 * caller's current device before returning.
 * Asynchrony: isrs_egn_nli / _nli_shard / _combine only enqueue.  A new COI set (or shard) makes
 * nli rebuild its work list on the host and allocate, upload and free the device copy stream-ordered
 * on the caller's stream (cudaMallocAsync / cudaMemcpyAsync / cudaFreeAsync), after that stream has
 * been ordered behind the handle's previous call: no call synchronises the host or the device except
 * create (synchronous), destroy (synchronises the device) and the inspection calls that say so.
 * An upload issued while that stream still has work in flight is staged in pinned host memory owned
 * by the handle (a pageable source would hold the call until the stream reaches the copy), so such a
 * call returns after the host planner's time; on an idle stream the source is pageable.
 * Errors: every call returns a status and isrs_egn_last_error() (thread-local) names the offending
 * field / index.  Validation, work-list limits, allocation and kernel attributes are checked before
 * the first kernel is enqueued, so on those errors no kernel runs and outputs are untouched (a work
 * list already rebuilt for the new COI set stays valid for the next call); a CUDA launch failure after
 * that point (ECUDA) may leave a partial enqueue whose outputs are undefined.
 * CUDA graphs: once a handle has run a COI set (and shard) on a non-capturing stream, a further call
 * for the same set neither allocates nor synchronises, so it can be captured (cudaStreamBeginCapture)
 * and replayed; inside a capture the call records no timing or ordering events and leaves
 * isrs_egn_last_kernel_ms / the cross-stream ordering describing the last direct call (a call that
 * would have to rebuild its work list inside a capture fails with EINVAL).  A graph bakes in the
 * handle's work-list buffers: calling that handle with another COI set frees them, so a graph should
 * own its handle (the Python Engine.graph() creates a private one).
 * Memory: a handle's device buffers come from the device's default stream-ordered memory pool
 * (cudaMallocAsync), whose release threshold the library raises so that repeated create / destroy
 * reuse pool memory; memory a destroyed handle frees stays reserved in that pool for the process.
 * Tracing: create, nli, nli_shard and eta_host are NVTX ranges of the same names.
 */
#ifndef ISRS_EGN_H
#define ISRS_EGN_H

#include <stdint.h>

#if defined(__GNUC__)
#define ISRS_EGN_API __attribute__((visibility("default")))
#else
#define ISRS_EGN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct isrs_egn isrs_egn_t; /* opaque handle; owns all device memory */

enum {
  ISRS_EGN_OK = 0,
  ISRS_EGN_EINVAL = -1,      /* bad argument: non-finite, out of range, not on the Hz lattice */
  ISRS_EGN_EOVERLAP = -2,    /* channel bands [f - R/2, f + R/2] overlap (touching is allowed) */
  ISRS_EGN_ERANGE = -3,      /* B_tot * zeta overflows sinh, or K_s / table too large           */
  ISRS_EGN_ENOMEM = -4,      /* device or host allocation failed                                */
  ISRS_EGN_ECUDA = -5,       /* any CUDA error (asynchronous ones surface at the next call)     */
  ISRS_EGN_EUNSUPPORTED = -6 /* precision / mu_mode not available                               */
};

/* Link description.  create() deep-copies every array; the caller may free them on return. */
typedef struct {
  int32_t n_ch;                    /* >= 1                                                    */
  const double *f_center_hz;       /* [n_ch] strictly increasing, integer Hz                  */
  const double *symbol_rate_hz;    /* [n_ch] R_i > 0, integer Hz; band = [f - R/2, f + R/2]   */
  const double *launch_power_w;    /* [n_ch] P_i > 0                                          */
  const double *excess_kurtosis;   /* [n_ch] Phi_i (Gaussian 0, QPSK -1), Eq. 15 (reading C9) */
  const double *psi;               /* [n_ch] Psi_i sixth-order factor, or NULL (=> 0)         */
  int32_t n_span;                  /* >= 1                                                    */
  const double *length_m;          /* [n_span] L_s > 0                                        */
  const double *alpha_per_m;       /* [n_span] power attenuation alpha_s > 0 (Eq. 9 divides by i chi - alpha) */
  const double *beta2_s2_per_m;    /* [n_span] at the band centre f_c (readings C5, C15)      */
  const double *beta3_s3_per_m;    /* [n_span]                                                */
  const double *gamma_per_w_m;     /* [n_span] >= 0                                           */
  const double *cr_per_w_m_hz;     /* [n_span] Raman gain slope C_r >= 0 (0.028/W/km/THz = 2.8e-17) */
} isrs_egn_problem;

enum { ISRS_EGN_MU_SEGMENT = 0,    /* Eqs. 8-10 (default, the hot path)                       */
       ISRS_EGN_MU_MACLAURIN = 1,  /* Eq. 4 (NEXT-1)                                          */
       ISRS_EGN_MU_INTEGRAL = 2    /* Eq. 23 by quadrature (NEXT-2, the paper's slow integral
                                      form; reading C12: composite 12-node Gauss-Legendre on
                                      max(64, 4|chi|L/2pi) equal panels rounded up to 2^k)       */ };

enum { ISRS_EGN_FLAG_UNIT_LINK = 1u, /* test hook: Y := 1 (oracle pin P6)                    */
       ISRS_EGN_FLAG_NO_CHAIN = 2u,  /* evaluate every span's segment sum (Eq. 8) on its own
                                        instead of chaining runs of identical consecutive spans
                                        into one recurrence (R9); same sum, A/B hook */
       ISRS_EGN_FLAG_DEDUP = 4u,     /* span-class dedup (SURVEY §8(f) NEXT-4a): for G identical
                                        consecutive spans evaluate the K-segment sum ONCE per point
                                        and multiply by the phased-array factor sum_g e^{i g chi L};
                                        same Y (Eq. 22), ~G x less work.  Its rate is reported
                                        separately, never as the headline point-spans/s */
       ISRS_EGN_FLAG_LITERAL_GAIN = 8u, /* NEXT-4b (R11): Eq. 22's gain / sqrt(rho) products
                                        as printed with a transparent scalar gain g_s = e^{alpha_s L_s}
                                        (mean loss restored, SRS tilt persists) instead of reading C3's
                                        ideal per-frequency equalisation (products = 1); fp64 segment
                                        mode only */
       ISRS_EGN_FLAG_MIRROR = 16u,   /* f1 <-> f2 symmetry (Eqs. 5, 8, 22 and the gates are symmetric in
                                        f1, f2; pin P2): region (kappa, k1, k2), k1 < k2, is evaluated once
                                        and also yields (kappa, k2, k1) with E and F exchanged -- about half
                                        the point-spans evaluated, the same eta.  Like DEDUP its rate is
                                        reported separately (logical point-spans), never as the headline.
                                        Not with isrs_egn_nli_shard (EUNSUPPORTED). */
       ISRS_EGN_FLAG_SPLIT = 32u     /* SCI / XCI / MCI parts of eta (interference from the COI alone,
                                        from one interfering channel, from two or three), returned by
                                        isrs_egn_nli_split.  An island (k1, k2, k3) belongs to the class given
                                        by the number of distinct channels among k1, k2, k3 other than the COI;
                                        a region whose islands fall into two classes is evaluated as two work-list
                                        entries, each over the lattice lines of one class (same points, same
                                        eta up to summation order).  fp64 segment mode only, not with DEDUP,
                                        LITERAL_GAIN, MIRROR, UNIT_LINK or shards (EUNSUPPORTED);
                                        isrs_egn_region_partials then sums a region's two entries, and a point on
                                        an edge shared by bands of both classes is counted in both entries. */ };

typedef struct {
  int32_t grid_n;      /* N: N x N bin-centre grid per (kappa1, kappa2) region; even, >= 2 (C6) */
  double delta_z_m;    /* segment step; K_s = ceil(L_s / delta_z_m); paper default 1000 */
  int32_t precision;   /* 64 (fp64, default) | 32 (mixed fp32 variant, row a8)                  */
  int32_t mu_mode;     /* ISRS_EGN_MU_*                                                          */
  uint32_t flags;      /* ISRS_EGN_FLAG_*                                                        */
  int32_t f_samples;   /* 0 (default): G_NLI at the COI centre, P_NLI = R G_NLI(f_kappa) (reading
                          C1, the 2-D path).  n > 0: the 3-D form of Eqs. 17-21 (NEXT-3):
                          f integrated over the COI band by the midpoint rule with n samples
                          f_m = f_kappa - R/2 + (m + 1/2) R/n, P_NLI = sum_m G_NLI(f_m) R/n; requires
                          every R_i / (2n) to be an integer (exact lattice, reading R3).  n x work. */
} isrs_egn_numerics;

/* Validate, canonicalise (f_c, B_tot, P_tot, K_s; reading C5), enumerate the regions of every
 * channel and run the per-span ISRS profile precompute on `device` (synchronous). */
ISRS_EGN_API int isrs_egn_create(const isrs_egn_problem *p, const isrs_egn_numerics *n, int device,
                    isrs_egn_t **out);

/* eta for n_coi COIs (coi: HOST array of channel indices, NULL = all channels 0..n_ch-1 with
 * n_coi = n_ch).  eta_dev: DEVICE [n_coi] (1/W^2).  terms_dev: DEVICE [n_coi * 5] contributions
 * of D, E, F, G, H to eta (row-major) or NULL.  Enqueued on cuda_stream (cudaStream_t; NULL =
 * legacy default stream); results are valid after the stream synchronises.  Deterministic:
 * bitwise-identical results across calls. */
ISRS_EGN_API int isrs_egn_nli(isrs_egn_t *h, int32_t n_coi, const int32_t *coi, double *eta_dev,
                 double *terms_dev, void *cuda_stream);

/* isrs_egn_nli plus the SCI / XCI / MCI parts of eta (the handle must have been created with
 * ISRS_EGN_FLAG_SPLIT, else EINVAL): split_dev DEVICE [n_coi * 3], row-major {SCI, XCI, MCI} in 1/W^2,
 * eta = SCI + XCI + MCI up to rounding.  Same asynchrony and determinism as isrs_egn_nli. */
ISRS_EGN_API int isrs_egn_nli_split(isrs_egn_t *h, int32_t n_coi, const int32_t *coi, double *eta_dev,
                 double *terms_dev, double *split_dev, void *cuda_stream);

/* ---- Multi-GPU: one process and one handle per GPU.  The canonical region list of
 * the COI set (COI, f sample, k1, k2 order) is split into `world` contiguous shards of near-equal cost
 * (in-support points); shard `rank` is evaluated and the per-COI sums of its regions, BEFORE the
 * Eq. 11 scale, are written to coi_sums_dev (DEVICE [n_coi * 6]: Eq. 15-weighted D, E, F, G, H sums and
 * the point count).  The caller all-gathers them into [world][n_coi][6] (e.g. ncclAllGather) and calls
 * isrs_egn_combine, which adds them in fixed rank order and scales: the same eta on every rank, bitwise.
 * Asynchronous on cuda_stream like isrs_egn_nli. */
ISRS_EGN_API int isrs_egn_nli_shard(isrs_egn_t *h, int32_t n_coi, const int32_t *coi, int32_t rank,
                                    int32_t world, double *coi_sums_dev, void *cuda_stream);
/* eta_dev [n_coi] (and terms_dev [n_coi * 5] or NULL) from gathered_dev [world][n_coi][6] (DEVICE).
 * coi must be the COI set of the preceding isrs_egn_nli_shard call on this handle. */
ISRS_EGN_API int isrs_egn_combine(isrs_egn_t *h, int32_t n_coi, const int32_t *coi, int32_t world,
                                  const double *gathered_dev, double *eta_dev, double *terms_dev,
                                  void *cuda_stream);
/* Host-only planner query (touches no device): for each rank r < world, the number of regions,
 * in-support points and first canonical region index of its shard (each array [world] or NULL). */
ISRS_EGN_API int isrs_egn_plan_shards(const isrs_egn_problem *p, const isrs_egn_numerics *n, int32_t n_coi,
                                      const int32_t *coi, int32_t world, int64_t *regions_out,
                                      int64_t *points_out, int64_t *first_region_out);

/* Per-region partial integrals written by the most recent isrs_egn_nli() call (synchronises
 * the handle's last stream).  For each query q: region (kappa[q], k1[q], k2[q]) ->
 * out_host[6q .. 6q+5] = { D_w, E_w, F_w, G_w, H_w, n_points } with
 *   D_w = sum_islands G_k3 D,  E_w = E[k3 == k1],  F_w = F[k3 == k2],
 *   G_w = sum_islands G_k3 G [k1 == k2],  H_w = H[k1 == k2 == k3]
 * (raw integrals of Eqs. 17-21 in the PSD normalisation of reading C2; a term whose gate or
 * Phi/Psi weight is zero is not evaluated and reads 0).  A region outside the last call's
 * work list reads as all zeros with n_points = -1. */
ISRS_EGN_API int isrs_egn_region_partials(isrs_egn_t *h, int32_t n, const int32_t *kappa, const int32_t *k1,
                             const int32_t *k2, double *out_host);

/* Work of isrs_egn_nli for a COI set (coi: HOST, NULL = all with n_coi = n_ch), from the host
 * planner alone (no device access, no synchronisation): exact in-support grid points summed over its
 * regions (f3 in some closed band, reading C10; a point on a shared edge of touching bands counts
 * once), point-spans = points * n_span (the work metric, R7), and the number of regions
 * listed (Eq. 16 generalised). */
ISRS_EGN_API int isrs_egn_work(const isrs_egn_t *h, int32_t n_coi, const int32_t *coi, int64_t *points,
                               int64_t *point_spans, int64_t *regions);

/* The same counts for the most recent isrs_egn_nli() / isrs_egn_nli_shard() call, as the kernels
 * wrote them (synchronises that call): points of the regions it launched (one shard at world > 1). */
ISRS_EGN_API int isrs_egn_last_work(isrs_egn_t *h, int64_t *points, int64_t *point_spans, int64_t *regions);

/* One-shot end-to-end call with HOST buffers: create + nli (all given COIs) + copy back +
 * destroy.  eta_host [n_coi], terms_host [n_coi * 5] or NULL. */
ISRS_EGN_API int isrs_egn_eta_host(const isrs_egn_problem *p, const isrs_egn_numerics *n, int device,
                      int32_t n_coi, const int32_t *coi, double *eta_host, double *terms_host);

/* Device time of each kernel of the most recent isrs_egn_nli() (CUDA events; synchronises).
 * The coherent-region integrand runs on an internal side stream concurrently with the D-only one
 * (fork/join with events around the caller's stream).  ms_out[4]: [0] = D-only integrand (on the
 * caller's stream), [1] = coherent (E/F/G/H) integrand (side stream, overlapping [0]), [2] =
 * per-COI reduction, [3] = the whole integrand phase (both launches, fork to join); a kernel that
 * was not launched reads 0.  point_spans_out (or NULL): the point-spans each integrand launch
 * processed ([0], [1]) and their sum ([2]). */
ISRS_EGN_API int isrs_egn_last_kernel_ms(isrs_egn_t *h, double *ms_out, double *point_spans_out);

/* Span chains of the handle (reading R9): *n_chain chains; chain_g (or NULL, capacity n_span)
 * receives the number of spans G_c of each chain, k_s (or NULL, capacity n_span) the segment
 * count K_s of every span.  Spans of a chain are consecutive; sum_c G_c = n_span. */
ISRS_EGN_API int isrs_egn_span_chains(const isrs_egn_t *h, int32_t *n_chain, int32_t *chain_g, int32_t *k_s);

/* The per-span ISRS profile tables the create-time precompute kernel wrote (row a2; synchronous
 * copy): *k_out = K_s of span `span`; ln_a_out[K] (or NULL) = ln c_k - alpha h k with
 * c_k = x_k / (2 sinh(x_k / 2)), x_k = B_tot zeta_k, the SRS-gain normalisation of Eq. 14;
 * zeta_out[K] (or NULL) = zeta_k = P_tot C_r L_eff(z_k) (Eq. 2) at the segment midpoints
 * z_k = (k + 1/2) h, h = L_s / K_s (Eq. 10).  So SRS_G(z_k, f3) e^{-alpha h k} =
 * exp(ln_a_k - zeta_k f3), the envelope the integrand kernel tabulates. */
ISRS_EGN_API int isrs_egn_profile_tables(isrs_egn_t *h, int32_t span, int32_t *k_out, double *ln_a_out,
                                         double *zeta_out);

/* Chain groups of the handle (reading R9, fp64 segment mode): runs of consecutive chains of identical
 * spans whose z = e^{i chi h} and I_0 the integrand forms once; group g covers chains
 * [grp_c0[g], grp_c0[g + 1]).  *n_grp receives the count; grp_c0 (or NULL, capacity n_span + 1) the
 * bounds.  Other modes: one chain per group.  (For the bench's algorithmic flop count.) */
ISRS_EGN_API int isrs_egn_chain_groups(const isrs_egn_t *h, int32_t *n_grp, int32_t *grp_c0);

/* Number of kernel launches the most recent isrs_egn_nli() enqueued (for bench accounting). */
ISRS_EGN_API int isrs_egn_last_launch_count(const isrs_egn_t *h);

ISRS_EGN_API void isrs_egn_destroy(isrs_egn_t *h); /* NULL-safe; synchronises the device */
ISRS_EGN_API const char *isrs_egn_strerror(int code);
ISRS_EGN_API const char *isrs_egn_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* ISRS_EGN_H */
