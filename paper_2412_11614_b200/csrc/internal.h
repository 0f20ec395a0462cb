// Internal device-side data layout shared by the host planner (abi.cu) and the kernels
// (kernels.cu).  Not part of the public ABI (include/isrs_egn.h is).
#pragma once
#include <cstdint>

namespace isrs {

#ifndef ISRS_BLOCK
#define ISRS_BLOCK 128
#endif
#ifndef ISRS_PPT
#define ISRS_PPT 4
#endif
#ifndef ISRS_MINB
#define ISRS_MINB 3
#endif
constexpr int BLOCK = ISRS_BLOCK;   // threads per CTA (4 warps; 3 CTAs per SM, up to 168 registers)
constexpr int PPT = ISRS_PPT;       // grid points per thread in flight (independent Goertzel chains)
constexpr int MIN_BLOCKS = ISRS_MINB;  // __launch_bounds__ min CTAs per SM
constexpr int CP = BLOCK * PPT;     // points per chunk
#ifndef ISRS_LINE_CAP
#define ISRS_LINE_CAP 512
#endif
constexpr int LINE_CAP = ISRS_LINE_CAP;  // f3-lines compacted per segment (2N-1 <= 511 at N = 256)
#ifndef ISRS_TW
#define ISRS_TW 64
#endif
#ifndef ISRS_TBYTES
#define ISRS_TBYTES (32 * 1024)
#endif
constexpr int TW_MAX = ISRS_TW;     // envelope-table rows (f3-lines) resident in smem
constexpr int T_BYTES = ISRS_TBYTES;  // smem budget of the envelope table
constexpr int LPT = LINE_CAP / BLOCK;  // lattice lines scanned per thread
#ifndef ISRS_WALK
#define ISRS_WALK 4
#endif
// -DISRS_CHECK: device-side bounds checks on every shared-memory index family (debug builds; the
// pool has no compute-sanitizer), a violation prints the site and traps
#ifdef ISRS_CHECK
#define ISRS_BOUND(i, n)                                                                        \
  do {                                                                                          \
    if (!((unsigned)(i) < (unsigned)(n))) {                                                     \
      printf("ISRS_CHECK %s:%d %s = %d not in [0, %d)\n", __FILE__, __LINE__, #i, (int)(i), (int)(n)); \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define ISRS_BOUND(i, n) \
  do {                   \
  } while (0)
#endif
#ifndef ISRS_CHAIN_MAX
#define ISRS_CHAIN_MAX 800
#endif
// longest chained recurrence (segments): the phase of the implicit z^n drifts by <= n^2 eps
// (fl(2 cos(chi h)) is exact to eps), 800^2 * 1.1e-16 = 7e-11 relative per point (DESIGN R9)
constexpr int CHAIN_MAX = ISRS_CHAIN_MAX;
// largest a + b of a channel-pair rate ratio a:b (lowest terms) the lattice line scan accepts
constexpr long long RATIO_MAX = 64;
static_assert(LINE_CAP % BLOCK == 0, "LINE_CAP must be a multiple of BLOCK");
static_assert(BLOCK % 32 == 0 && (BLOCK & (BLOCK - 1)) == 0 && BLOCK <= 1024,
              "BLOCK must be a power-of-two number of whole warps (fixed-tree block_sum)");

// region flags (reading C8: a term whose gate or weight is zero is not evaluated); bits >= 8
// hold the index of the region's NLI frequency f in KParams::fv (COI centre, or one of the
// f samples of the 3-D form)
enum : int { NEED_E = 1, NEED_F = 2, NEED_G = 4, NEED_H = 8, FV_SHIFT = 8 };
// ISRS_EGN_FLAG_SPLIT (SCI / XCI / MCI parts of eta): a region (kappa, k1, k2) whose islands can
// fall into two classes is listed twice, once restricted to the lattice lines whose k3 is one of
// {kappa, k1, k2} (K3_IN) and once to the others (K3_OUT); MODE_SEGSPL / MODE_SEGGRPSPL apply the filter
enum : int { K3_IN = 16, K3_OUT = 32 };

// MODE_SEG32: row a8, the mixed fp32 variant of the segment form (fp32 recurrence, mu, phase
// factor; fp64 chi h and its exact reduction, the phase advance and every accumulation)
// MODE_SEGDD: the segment form with span-class dedup (NEXT-4a, ISRS_EGN_FLAG_DEDUP)
// MODE_SEGLG: the segment form with the literal gain products of Eq. 22 (NEXT-4b)
// MODE_SEGGRP: MODE_SEGMENT with chain groups (some group of identical spans holds > 1 chain, R9)
enum : int { MODE_SEGMENT = 0, MODE_MACLAURIN = 1, MODE_UNIT = 2, MODE_SEG32 = 3, MODE_SEGDD = 4,
             MODE_SEGLG = 5, MODE_QUAD = 6, MODE_SEGGRP = 7, MODE_SEGDDL = 8, MODE_SEGSPL = 9,
             MODE_SEGGRPSPL = 10 };
// MODE_SEGSPL / MODE_SEGGRPSPL: MODE_SEGMENT / MODE_SEGGRP with the k3 line filter of the SCI / XCI / MCI
// split; their own instantiations so that the headline kernels' code (and schedule) is unchanged
constexpr bool mode_grouped(int mode) { return mode == MODE_SEGGRP || mode == MODE_SEGGRPSPL; }
// MODE_SEGDDL: MODE_SEGDD on links with a run of > 32 identical spans (closed-form phased-array factor);
// its own instantiation so that the MODE_SEGDD kernel's code (and schedule) is unchanged

struct RegionDesc {
  int kappa, k1, k2, flags;
};

// Everything a kernel needs, passed by value (all pointers are device pointers).
struct KParams {
  // channels (offset frequencies from f_c, exact multiples of 1/2 Hz)
  const double* lo;
  const double* hi;
  const double* f;
  const double* G;      // PSD P/R
  const double* R;
  const double* P;
  const double* phi;
  const double* psi;
  const double* delta;  // R/N
  const long long* rate;  // R as integer Hz (for the lattice ratio a:b)
  int n_ch;
  // spans
  const double* A2;     // 4 pi beta2 h        (chi h / pi = u v (A2 + A3 (f1+f2)))
  const double* A3;     // 4 pi^2 beta3 h
  const double* Eh;     // e^{-alpha h}
  const double* ah;     // alpha h
  const double* gh;     // gamma h
  const double* mac_c;  // Maclaurin: P_tot C_r / alpha
  const double* aL;     // alpha L
  const int* K;         // segments K_s = ceil(L/dz)
  const int* cls;       // span class (spans sharing L, alpha, C_r share envelope tables)
  int n_span;
  // span chains (reading R9): runs of identical consecutive spans whose segment sums are
  // evaluated as ONE recurrence over G*K segments; chain c covers spans [s0[c], s0[c] + g[c])
  const int* chain_s0;
  const int* chain_g;
  int n_chain;
  // chain groups (MODE_SEGMENT): runs of consecutive chains of identical spans (a chain split only by
  // the CHAIN_MAX cap); group g covers chains [grp_c0[g], grp_c0[g + 1]).  Their z = e^{i chi h} and
  // I_0 are formed once per group and the chains' segment sums are combined with their span phases
  // before the single mu = I_0 S multiply (reading R9).  Other modes: one chain per group.
  const int* grp_c0;
  int n_grp;
  // literal gain (NEXT-4b): ln S_s(x) = lnc_L[s] - zeta_L[s] x is the SRS gain at the end of span s;
  // ln Lambda_s = (lgA - lgB (f1+f2+f3)) / 2 + (lgC - lgD f) / 2 with prefix (A, B) / suffix (C, D) sums
  const double* lnc_L;
  const double* zeta_L;
  const double* lgA;
  const double* lgB;
  const double* lgC;
  const double* lgD;
  // integral form (NEXT-2): per span L, alpha, gamma, P_tot C_r; B_tot; Gauss-Legendre rule
  const double* Ls;
  const double* alpha;
  const double* gamma;
  const double* pcr;
  double b_tot;
  double gl_x[12];
  double gl_w[12];
  // span classes: envelope a'_k(f3) = exp(lnA[c][k] - zeta[c][k] f3)
  const double* lnA;    // [n_cls][kstride]  ln(c_k) - alpha h k
  const double* zeta;   // [n_cls][kstride]
  const int* Kc;        // [n_cls]
  int n_cls;
  int kstride;          // row length of lnA/zeta
  int tstride;          // smem table row stride (even, = Kpad + 2)
  int tw;               // table rows resident (<= TW_MAX)
  int N;                // grid points per channel axis
  // regions
  const double* fv;     // NLI frequencies (offsets) indexed by flags >> FV_SHIFT
  const RegionDesc* desc;
  double* partials;     // [n_regions][6]: D_w, E_w, F_w, G_w, H_w, n_points
  const int* mirror;    // ISRS_EGN_FLAG_MIRROR: [n_regions] canonical id of region (kappa, k2, k1) whose
                        // partials this region's launch also writes (E and F swapped), or -1; NULL = off
  int mode;
  unsigned long long* prof;   // ISRS_PROF builds only: per-phase warp-cycle counters [8]
};

struct RParams {
  const RegionDesc* desc;
  const double* partials;
  const long long* coi_off;  // [n_coi + 1] region ranges per COI (canonical order)
  const int* coi;            // [n_coi]
  const double* G;
  const double* R;
  const double* P;
  const double* phi;
  const double* psi;
  int n_coi;
  double inv_fs;             // 1 / (number of f samples per COI): 1 in the 2-D path
  double* eta;
  double* terms;             // may be null
  double* npts;              // [n_coi]
  long long r_lo, r_hi;      // canonical region range summed (a shard; [0, inf) = all)
  double* part_out;          // shard mode: raw per-COI sums [n_coi][6] instead of eta/terms/npts
};

struct CParams {             // combine gathered shard sums [world][n_coi][6] in rank order
  const double* gathered;
  int world;
  const int* coi;
  const double* R;
  const double* P;
  int n_coi;
  double inv_fs;
  double* eta;
  double* terms;             // may be null
  double* npts;              // may be null
};

struct PParams {  // precompute
  const double* cls_L;
  const double* cls_alpha;
  const double* cls_cr;
  const int* Kc;
  int n_cls;
  int kstride;
  double p_tot;
  double b_tot;
  double* lnA;
  double* zeta;
};

size_t integrand_smem_bytes(int tstride, int tw, int N, bool coherent, bool grouped);
int launch_precompute(const PParams& p, void* stream);
int integrand_prepare(int mode, int tstride, int tw, int N);
int launch_integrand(const KParams& p, const int* list, long long n_list, bool coherent,
                     void* stream, int* n_launches);
int launch_reduce(const RParams& p, void* stream);
int launch_reduce_split(const RParams& p, double* split_out, void* stream);
int launch_combine(const CParams& p, void* stream);

}  // namespace isrs
