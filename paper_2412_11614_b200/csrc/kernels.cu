// sm_100a kernels of the ISRS EGN hot path (paper arXiv 2412.11614).
//
//   precompute_kernel  (row a2)  per span class c and segment k: zeta_k = P_tot C_r L_eff(z_k)
//                                 (Eq. 2; z_k Eq. 10) and the SRS-gain normalisation
//                                 c_k = x / (2 sinh(x/2)), x = B_tot zeta_k (Eq. 14), stored
//                                 as lnA = ln c_k - alpha h k  (the attenuation factor folded in).
//   integrand_kernel   (rows a3-a6) one CTA per region (kappa, kappa1, kappa2): f3-gate per line
//                                 (Eq. 17 gate, reading C10), the segment closed form mu_s (Eqs. 8-9,
//                                 P:119-121) for every point and span, the span phased-array sum Y
//                                 (Eq. 22, reading C3) in registers, and the D, E, F, G, H
//                                 region reductions (Eqs. 17-21, reading C7), fixed order.
//   reduce_kernel      (row a7)  per COI: Eq. 15 coefficients (reading C2) and Eq. 11; in
//                                 shard mode the raw per-COI sums of one rank's regions.
//   combine_kernel     (§8(e))   gathered shard sums added in fixed rank order, Eq. 11 scale.
//
// integrand_kernel<COH, MODE>: COH = the region needs the coherent E/F/G/H sums (reading C8);
// MODE = MODE_SEGMENT (the hot path, fp64, span chains R9), MODE_SEG32 (row a8, mixed fp32),
// MODE_SEGDD (NEXT-4a span-class dedup), MODE_SEGLG (NEXT-4b literal Eq. 22 gain products),
// MODE_MACLAURIN (NEXT-1, Eq. 4), MODE_QUAD (NEXT-2, Eq. 23 by quadrature), MODE_UNIT (Y := 1,
// test hook for pin P6/P14).  Optional -DISRS_PROF adds per-phase warp-cycle timers.
//
// FP64 CUDA-core work (no tensor cores: the path is not a dense contraction).  The segment sum
//   mu_s = I_0 * sum_k a_k w^k,  w = e^{(i chi - alpha) h},  I_0 = (w - 1)/(i chi - alpha)
// (Eq. 9 gives I_k = I_0 w^k) has REAL coefficients a_k = c_k e^{-zeta_k f3}; with the attenuation
// folded in (a'_k = a_k e^{-alpha h k}, z = e^{i chi h}, |z| = 1) it is evaluated by the
// second-order real recurrence b_k = a'_k + 2 cos(chi h) b_{k+1} - b_{k+2} (Goertzel), i.e.
// ONE DFMA + ONE DADD per segment instead of a complex Horner step (4 DP instructions).
// Envelope values a'_k(f3) depend on the point only through f3, which is constant along the
// lattice lines j = a m1 + b m2 of a region (a:b = R1:R2), so they are tabulated per line in
// shared memory and read with 16-byte loads that a warp mostly broadcasts.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "internal.h"
#include "cis_table.h"

#ifndef ISRS_CISTAB
#define ISRS_CISTAB 1
#endif
#ifndef ISRS_UNROLL
#define ISRS_UNROLL 4
#endif
#ifdef ISRS_PROF
// phase timers (debug builds only, -DISRS_PROF): per-warp clock64 deltas summed into p.prof
#define PROF_DECL unsigned long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long prof_t = clock64();
#define PROF_MARK(i) { const long long t_ = clock64(); prof_acc[i] += (unsigned long long)(t_ - prof_t); prof_t = t_; }
#define PROF_COUNT(i, v) { if (threadIdx.x == 0 && p.prof) atomicAdd(p.prof + (i), (unsigned long long)(v)); }
#define PROF_FLUSH if ((threadIdx.x & 31) == 0 && p.prof) { for (int i_ = 0; i_ < 8; ++i_) atomicAdd(p.prof + i_, prof_acc[i_]); }
#else
#define PROF_DECL
#define PROF_MARK(i)
#define PROF_COUNT(i, v)
#define PROF_FLUSH
#endif
#define ISRS_STR(x) #x
#define ISRS_UNROLL_PRAGMA(n) _Pragma(ISRS_STR(unroll n))

namespace isrs {

// ------------------------------------------------------------------------------------------
// precompute (row a2)

__global__ void precompute_kernel(const PParams p) {
  const int c = blockIdx.y;
  const int K = p.Kc[c];
  const double L = p.cls_L[c], alpha = p.cls_alpha[c], cr = p.cls_cr[c];
  const double h = L / K;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < p.kstride; k += gridDim.x * blockDim.x) {
    double lnA = 0.0, ze = 0.0;
    if (k < K) {
      const double zk = (k + 0.5) * h;                    // Eq. 10
      const double leff = -expm1(-alpha * zk) / alpha;     // L_eff(z_k)
      ze = p.p_tot * cr * leff;                            // Eq. 2: zeta = P_tot C_r L_eff
      const double x = p.b_tot * ze;
      const double ck = (x == 0.0) ? 1.0 : x / (2.0 * sinh(0.5 * x));  // Eq. 14 normalisation
      lnA = log(ck) - alpha * h * k;                       // attenuation |w|^k folded in
    }
    p.lnA[(size_t)c * p.kstride + k] = lnA;
    p.zeta[(size_t)c * p.kstride + k] = ze;
  }
}

int launch_precompute(const PParams& p, void* stream) {
  dim3 grid((p.kstride + 127) / 128, p.n_cls);
  precompute_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ------------------------------------------------------------------------------------------
// integrand helpers

struct Smem {
  double* T;         // [tw][tstride] reversed envelope rows: T[row][i] = a'_{Kp-1-i}(f3_row)
  int* sl_j;         // [LINE_CAP] compacted supported line index j
  int* sl_first;     // [LINE_CAP] first m1 on the line
  int* sl_start;     // [LINE_CAP+1] exclusive prefix of point counts padded to multiples of PPT
  int* sl_cnt;       // [LINE_CAP] points on the line (unpadded)
  double* wD;        // [LINE_CAP] sum_t t G_k3         (D, G weights)
  double* wE;        // [LINE_CAP] sum_t t [k3 == k1]   (E, H weights)
  int* scan;         // [BLOCK] scan scratch (int2)
  double* red;       // [BLOCK] reduction scratch
  double2* ybuf;     // [CP] chunk Y values (coherent only)
  double2* rowacc;   // [N]
  double2* colacc;   // [N]
  double2* lineacc;  // [LINE_CAP]
  double* wF;        // [LINE_CAP] sum_t t [k3 == k2]
  double* gst;       // [5 PPT][BLOCK] per-thread chain-group state: (f1-f)(f2-f), f1+f2, chi h / pi,
                     // e^{i G chi L} (re, im)
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline size_t smem_layout(int tstride, int tw, int N, bool coh, bool grp, char* base,
                                              Smem* s) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align16(off + bytes);
    return o;
  };
  size_t oT = take(sizeof(double) * (size_t)tw * tstride);
  size_t oJ = take(sizeof(int) * LINE_CAP);
  size_t oF = take(sizeof(int) * LINE_CAP);
  size_t oS = take(sizeof(int) * (LINE_CAP + 1));
  size_t oN = take(sizeof(int) * LINE_CAP);
  size_t oD = take(sizeof(double) * LINE_CAP);
  size_t oE = take(sizeof(double) * LINE_CAP);
  size_t oW = take(sizeof(double) * LINE_CAP);
  size_t oG = grp ? take(sizeof(double) * 5 * PPT * BLOCK) : 0;
  size_t oC = take(sizeof(int4) * (BLOCK / 32 + 1));
  size_t oR = take(sizeof(double) * BLOCK);
  size_t oY = 0, oRow = 0, oCol = 0, oLine = 0;
  if (coh) {
    oY = take(sizeof(double2) * CP);
    oRow = take(sizeof(double2) * N);
    oCol = take(sizeof(double2) * N);
    oLine = take(sizeof(double2) * LINE_CAP);
  }
  if (s) {
    s->T = (double*)(base + oT);
    s->sl_j = (int*)(base + oJ);
    s->sl_first = (int*)(base + oF);
    s->sl_start = (int*)(base + oS);
    s->sl_cnt = (int*)(base + oN);
    s->wD = (double*)(base + oD);
    s->wE = (double*)(base + oE);
    s->wF = (double*)(base + oW);
    s->gst = grp ? (double*)(base + oG) : nullptr;
    s->scan = (int*)(base + oC);
    s->red = (double*)(base + oR);
    s->ybuf = coh ? (double2*)(base + oY) : nullptr;
    s->rowacc = coh ? (double2*)(base + oRow) : nullptr;
    s->colacc = coh ? (double2*)(base + oCol) : nullptr;
    s->lineacc = coh ? (double2*)(base + oLine) : nullptr;
  }
  return off;
}

size_t integrand_smem_bytes(int tstride, int tw, int N, bool coherent, bool grouped) {
  return smem_layout(tstride, tw, N, coherent, grouped, nullptr, nullptr);
}

// Block-wide exclusive scan of an int triple (w unused); returns totals.  All threads must call.
__device__ inline int4 block_scan3(int4 v, int* scratch, int4* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int4 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, x.x, o);
    const int b = __shfl_up_sync(0xffffffffu, x.y, o);
    const int c = __shfl_up_sync(0xffffffffu, x.z, o);
    if (lane >= o) { x.x += a; x.y += b; x.z += c; }
  }
  int4* ws = (int4*)scratch;
  __syncthreads();
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int4 w = (lane < BLOCK / 32) ? ws[lane] : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, w.x, o);
      const int b = __shfl_up_sync(0xffffffffu, w.y, o);
      const int c = __shfl_up_sync(0xffffffffu, w.z, o);
      if (lane >= o) { w.x += a; w.y += b; w.z += c; }
    }
    if (lane < BLOCK / 32) ws[lane] = w;   // inclusive warp prefix
  }
  __syncthreads();
  const int4 base = (warp > 0) ? ws[warp - 1] : make_int4(0, 0, 0, 0);
  *total = ws[BLOCK / 32 - 1];
  __syncthreads();
  return make_int4(base.x + x.x - v.x, base.y + x.y - v.y, base.z + x.z - v.z, 0);
}

// Fixed-tree block sum (deterministic) through shared memory; the D-only kernel's once-per-region
// sum (its register allocation, hence the recurrence's schedule, is tuned with this form).  All
// threads must call.
__device__ inline double block_sum(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
#pragma unroll
  for (int s = BLOCK / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  double r = red[0];
  __syncthreads();
  return r;
}

// Deterministic block sums of NV values (all threads must call; every thread gets the totals): a
// butterfly of warp shuffles (xor 16, 8, 4, 2, 1 -- a fixed tree, so bitwise reproducible) inside each
// warp, then the BLOCK/32 warp partials added in warp order from shared memory.
template <int NV>
__device__ inline void block_sum_n(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) red[NV * warp + k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double t = red[k];
#pragma unroll
    for (int w = 1; w < BLOCK / 32; ++w) t += red[NV * w + k];
    v[k] = t;
  }
  __syncthreads();
}

// index i with sl_start[i] <= p < sl_start[i+1], searched in [lo, hi]
__device__ inline int line_of(const int* sl_start, int hi, int p, int lo = 0) {
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (sl_start[mid] <= p) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// f3-gate of one lattice line (reading C10): every band [lo, hi] containing f3 contributes
// t = 1 strictly inside, 1/2 on an edge (touching bands split 1/2 / 1/2).
// SPLIT (MODE_SEGSPL / MODE_SEGGRPSPL): only the bands c of the region entry's class count -- K3_IN:
// c one of {kappa, k1, k2}, K3_OUT: the others (the SCI / XCI / MCI split).
template <bool SPLIT>
__device__ inline void line_gate(const KParams& p, double f3, int kappa, int k1, int k2, int flags, double* wD,
                                 double* wE, double* wF) {
  double d = 0.0, e = 0.0, ff = 0.0;
  int lo = 0, hi = p.n_ch - 1;       // largest i with lo[i] <= f3
  if (f3 >= __ldg(p.lo)) {
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (__ldg(p.lo + mid) <= f3) lo = mid; else hi = mid - 1;
    }
    for (int c = lo; c >= lo - 1 && c >= 0; --c) {
      const double l = __ldg(p.lo + c), h = __ldg(p.hi + c);
      if (f3 >= l && f3 <= h) {
        if (SPLIT) {
          const bool in = (c == kappa || c == k1 || c == k2);
          if (((flags & K3_IN) && !in) || ((flags & K3_OUT) && in)) continue;
        }
        const double t = (f3 > l && f3 < h) ? 1.0 : 0.5;
        d += t * __ldg(p.G + c);
        if (c == k1) e += t;
        if (c == k2) ff += t;
      }
    }
  }
  *wD = d;
  *wE = e;
  *wF = ff;
}


// sin(pi x), cos(pi x): exact reduction to r = x - q/2 in [-1/4, 1/4] (q = rint(2x)), Taylor
// polynomials in r^2 accurate to ~1 ulp on that interval, quadrant fix-up by selects and
// sign-bit flips.  Branch-free so the PPT independent evaluations interleave (the library
// sincospi() is ~2x the issue slots here because of its special-case branches).
__device__ __forceinline__ void sincospi_d(double x, double* sp, double* cp) {
#if ISRS_CISTAB
  // table-driven (round 2): j = rint(128 x) by the 1.5*2^52 rounding constant (its low word is j
  // mod 2^32), r = x - j/128 in [-1/256, 1/256] (exact: a multiple of ulp(x) below 2^-8), and
  // e^{i pi x} = kCisTab[j mod 256] * (1 + (cos(pi r) - 1) + i sin(pi r)), degree-6 polynomials
  // in r (truncation < 1.4e-20); |error| <= 1.65e-16 over 2e7 samples of |x| <= 3e4 against
  // x87 sinl/cosl.  15 FP64 instructions instead of 23 plus the quadrant selects.
  const double M = 6755399441055744.0;
  const double t = fma(x, 128.0, M);
  const double r = fma(t - M, -0.0078125, x);
  const double2 e = __ldg(&kCisTab[__double2loint(t) & 255]);
  const double r2 = r * r;
  double ps = fma(r2, -0.5992645293207921, 2.5501640398773455);
  ps = fma(ps, r2, -5.16771278004997);
  ps = fma(ps, r2, 3.141592653589793);
  const double s = r * ps;
  double pc = fma(r2, -1.3352627688545895, 4.0587121264167685);
  pc = fma(pc, r2, -4.934802200544679);
  const double cm1 = pc * r2;
  *cp = fma(e.x, cm1, fma(-e.y, s, e.x));
  *sp = fma(e.y, cm1, fma(e.x, s, e.y));
#else
  const double q = rint(x + x);
  const double r = fma(q, -0.5, x);
  const double r2 = r * r;
  double ps = 7.952054001475508e-07;
  ps = fma(ps, r2, -2.1915353447830204e-05);
  ps = fma(ps, r2, 0.00046630280576761234);
  ps = fma(ps, r2, -0.007370430945714348);
  ps = fma(ps, r2, 0.08214588661112819);
  ps = fma(ps, r2, -0.5992645293207919);
  ps = fma(ps, r2, 2.550164039877345);
  ps = fma(ps, r2, -5.167712780049969);
  ps = fma(ps, r2, 3.141592653589793);
  double pc = -1.387895246221376e-07;
  pc = fma(pc, r2, 4.303069587032944e-06);
  pc = fma(pc, r2, -0.00010463810492484565);
  pc = fma(pc, r2, 0.001929574309403922);
  pc = fma(pc, r2, -0.02580689139001405);
  pc = fma(pc, r2, 0.23533063035889312);
  pc = fma(pc, r2, -1.3352627688545893);
  pc = fma(pc, r2, 4.058712126416768);
  pc = fma(pc, r2, -4.934802200544679);
  pc = fma(pc, r2, 1.0);
  const double sr = r * ps;
  const int n = (int)(__double2ll_rn(q) & 3);
  double so = (n & 1) ? pc : sr;
  double co = (n & 1) ? sr : pc;
  const int sgn_s = (n & 2) ? (int)0x80000000 : 0;
  const int sgn_c = ((n + 1) & 2) ? (int)0x80000000 : 0;
  *sp = __hiloint2double(__double2hiint(so) ^ sgn_s, __double2loint(so));
  *cp = __hiloint2double(__double2hiint(co) ^ sgn_c, __double2loint(co));
#endif
}

// 1/d for d > 0 normal: hardware approximation + two Newton steps (full double precision).
__device__ __forceinline__ double rcp_d(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

__device__ inline long long gcd_ll(long long a, long long b) {
  while (b) {
    long long t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// Line scan of lines [seg0, seg0 + nl) of a region (rows a3 of SURVEY §8): on each lattice line
// j = a m1 + b m2 the f3 = C + g j is constant (exact), so the point count, the first m1 and the
// C10 gate weights (line_gate) are per line; supported lines are compacted in order into sm.sl_*
// with their slot offsets (each line padded to whole PPT-groups).  Returns (lines, slots, points).
// All threads must call (block scan).
template <bool SPLIT>
__device__ __forceinline__ int4 scan_lines(const KParams& p, const Smem& sm, int seg0, int nl, int N, int a,
                                           int b, int inv_a, int kappa, int k1, int k2, int flags, double C,
                                           double g) {
  const int tid = threadIdx.x;
  // ---- line scan: each thread owns LPT consecutive lines (order-preserving compaction)
  int cnt[LPT], first[LPT];
  double lwD[LPT], lwE[LPT], lwF[LPT];
  int4 v = make_int4(0, 0, 0, 0);
#pragma unroll
  for (int q = 0; q < LPT; ++q) {
    const int jl = LPT * tid + q;
    cnt[q] = 0;
    first[q] = 0;
    lwD[q] = lwE[q] = lwF[q] = 0.0;
    if (jl < nl) {
      const int j = seg0 + jl;
      // points on the line: a m1 + b m2 = j, 0 <= m1, m2 < N
      int lowb = j - b * (N - 1);
      lowb = (lowb <= 0) ? 0 : (lowb + a - 1) / a;
      const int upb = min(N - 1, j / a);
      int fm = lowb;
      if (b > 1) {
        const int r = (int)(((long long)(j % b) * inv_a) % b);
        fm = lowb + (((r - lowb) % b) + b) % b;
      }
      const int n = (fm <= upb) ? (upb - fm) / b + 1 : 0;
      if (n > 0) {
        const double f3 = __dadd_rn(C, g * (double)j);
        line_gate<SPLIT>(p, f3, kappa, k1, k2, flags, &lwD[q], &lwE[q], &lwF[q]);
        if (lwD[q] > 0.0) {
          cnt[q] = n;
          first[q] = fm;
          v.x += 1;
          v.y += (n + PPT - 1) / PPT * PPT;   // slots: each line padded to whole PPT-groups
          v.z += n;
        }
      }
    }
  }
  int4 tot;
  int4 pos = block_scan3(v, sm.scan, &tot);
#pragma unroll
  for (int q = 0; q < LPT; ++q) {
    if (cnt[q] > 0) {
      ISRS_BOUND(pos.x, LINE_CAP);
      sm.sl_j[pos.x] = seg0 + LPT * tid + q;
      sm.sl_first[pos.x] = first[q];
      sm.sl_start[pos.x] = pos.y;
      sm.sl_cnt[pos.x] = cnt[q];
      sm.wD[pos.x] = lwD[q];
      sm.wE[pos.x] = lwE[q];
      sm.wF[pos.x] = lwF[q];
      pos.x += 1;
      pos.y += (cnt[q] + PPT - 1) / PPT * PPT;
    }
  }
  return tot;
}

// Envelope table (row a2 values at this region's lines): rows [tb, tb + tn) of the compacted
// lines, row r holding a'_k(f3(j_r)) = c_k e^{-zeta_k f3} e^{-alpha h k} for k = Kp-1 .. 0 (reversed
// for the recurrence), fp64 with the first pair repeated at the end (chain wrap, R9) or fp32 (a8).
template <bool F32>
__device__ __forceinline__ void build_table(const KParams& p, const Smem& sm, int cls, int tb, int tn, double C,
                                            double g) {
  const int tid = threadIdx.x;
  const int Kc = __ldg(p.Kc + cls);
  // fp64 rows: K rounded up to even (16-byte pair loads); fp32 rows (a8): to a
  // multiple of 4 (float4 loads), row stride 2 tstride floats
  const int Kp = F32 ? ((Kc + 3) & ~3) : ((Kc + 1) & ~1);
  float* T32 = reinterpret_cast<float*>(sm.T);
  ISRS_BOUND(tn - 1, p.tw);
  ISRS_BOUND(tb + tn - 1, LINE_CAP);
  if (F32) ISRS_BOUND(Kp - 1, 2 * p.tstride); else ISRS_BOUND(Kp + 1, p.tstride);
  const double* lnA = p.lnA + (size_t)cls * p.kstride;
  const double* zt = p.zeta + (size_t)cls * p.kstride;
  // one thread per coefficient k walks the rows: a'_k(f3 + g) = a'_k(f3) e^{-zeta_k g}.
  // A run of WALK consecutive lines takes every entry from the run's predecessor with one DMUL
  // by step^m (m = 1..WALK), so the dependent chain is one DMUL per WALK rows; rows whose line
  // index jumps restart from exp (relative error <= 2 tw eps).
  constexpr int WALK = ISRS_WALK;
  static_assert(TW_MAX <= 64, "the restart mask holds one bit per table row");
  // restart mask (per warp, by ballot): bit r set when row r does not continue its predecessor's
  // line (j_r != j_{r-1} + 1; row 0 always), so the walk's control flow reads no shared memory
  unsigned long long rmask;
  {
    const int lane = tid & 31;
    const int r0 = lane, r1 = lane + 32;
    const bool b0 = (r0 >= tn) || r0 == 0 || sm.sl_j[tb + r0] != sm.sl_j[tb + r0 - 1] + 1;
    const bool b1 = (r1 >= tn) || sm.sl_j[tb + r1] != sm.sl_j[tb + r1 - 1] + 1;
    rmask = (unsigned long long)__ballot_sync(0xffffffffu, b0) |
            ((unsigned long long)__ballot_sync(0xffffffffu, b1) << 32);
  }
  for (int ii = tid; ii < Kp; ii += BLOCK) {
    const int k = Kp - 1 - ii;
    const bool live = k < Kc;
    const double la = live ? __ldg(lnA + k) : 0.0, ze = live ? __ldg(zt + k) : 0.0;
    double sp[WALK];
    sp[0] = exp(-ze * g);
#pragma unroll
    for (int m = 1; m < WALK; ++m) sp[m] = sp[m - 1] * sp[0];
    double v = 0.0;
    int row = 0;
    auto put = [&](int r, double x) {
      if (F32) {
        T32[r * 2 * p.tstride + ii] = (float)x;
      } else {
        sm.T[r * p.tstride + ii] = x;
        if (ii < 2) sm.T[r * p.tstride + Kp + ii] = x;   // wrap pair for span chains (R9)
      }
    };
    while (row < tn) {
      const unsigned long long rest = rmask >> row;
      if (WALK > 1 && row + WALK <= tn && (rest & ((1ull << WALK) - 1ull)) == 0ull) {   // block-uniform
        double vr[WALK];
#pragma unroll
        for (int m = 0; m < WALK; ++m) vr[m] = v * sp[m];
#pragma unroll
        for (int m = 0; m < WALK; ++m) put(row + m, vr[m]);
        v = vr[WALK - 1];
        row += WALK;
        continue;
      }
      if (rest & 1ull) {
        const int j = sm.sl_j[tb + row];
        if (live) v = exp(la - ze * __dadd_rn(C, g * (double)j));
      } else {
        v *= sp[0];
      }
      put(row, v);
      ++row;
    }
  }
}

// Coherent sums of one chunk (reading C7; Eqs. 18-21), the chunk's Y values staged in sm.ybuf:
// line sums (G, H) by one thread per line, row sums r[m2] (E) and column sums c[m1] (F) by one
// thread per row / column, each accumulated over the chunk's lines in line order (deterministic).
__device__ __forceinline__ void coherent_chunk(const Smem& sm, int flags, int N, int a, int b, int i_first,
                                               int i_last, int p0, int p_end) {
  const int tid = threadIdx.x;
  // lines (G, H): one thread per line in the chunk, points in order
  if (flags & (NEED_G | NEED_H)) {
    for (int i = i_first + tid; i <= i_last; i += BLOCK) {
      const int s0 = max(sm.sl_start[i], p0), s1 = min(sm.sl_start[i] + sm.sl_cnt[i], p_end);
      double2 acc = sm.lineacc[i];
      for (int t = s0; t < s1; ++t) {
        ISRS_BOUND(t - p0, CP);
        const double2 y = sm.ybuf[t - p0];
        acc.x += y.x;
        acc.y += y.y;
      }
      sm.lineacc[i] = acc;
    }
  }
  // rows (E): r[m2] += sum over the chunk's lines of wE Y(m1, m2), line order
  if (flags & NEED_E) {
    for (int m2 = tid; m2 < N; m2 += BLOCK) {
      double2 acc = sm.rowacc[m2];
      for (int i = i_first; i <= i_last; ++i) {
        const double w = sm.wE[i];
        if (w == 0.0) continue;
        const int num = sm.sl_j[i] - b * m2;
        if (num < 0) continue;
        if (a > 1 && num % a) continue;                 // equal rates (a = b = 1): no division
        const int m1 = (a == 1) ? num : num / a;
        if (m1 >= N) continue;
        const int idx = sm.sl_start[i] + ((b == 1) ? m1 - sm.sl_first[i] : (m1 - sm.sl_first[i]) / b);
        if (m1 < sm.sl_first[i] || idx < p0 || idx >= p_end) continue;
        ISRS_BOUND(idx - p0, CP);
        const double2 y = sm.ybuf[idx - p0];
        acc.x = fma(w, y.x, acc.x);
        acc.y = fma(w, y.y, acc.y);
      }
      sm.rowacc[m2] = acc;
    }
  }
  // columns (F): c[m1] += sum over the chunk's lines of wF Y(m1, m2)
  if (flags & NEED_F) {
    for (int m1 = tid; m1 < N; m1 += BLOCK) {
      double2 acc = sm.colacc[m1];
      for (int i = i_first; i <= i_last; ++i) {
        const double w = sm.wF[i];
        if (w == 0.0) continue;
        const int num = sm.sl_j[i] - a * m1;
        if (num < 0) continue;
        if (b > 1 && num % b) continue;
        const int m2 = (b == 1) ? num : num / b;
        if (m2 >= N || m1 < sm.sl_first[i]) continue;
        const int idx = sm.sl_start[i] + ((b == 1) ? m1 - sm.sl_first[i] : (m1 - sm.sl_first[i]) / b);
        if (idx < p0 || idx >= p_end) continue;
        ISRS_BOUND(idx - p0, CP);
        const double2 y = sm.ybuf[idx - p0];
        acc.x = fma(w, y.x, acc.x);
        acc.y = fma(w, y.y, acc.y);
      }
      sm.colacc[m1] = acc;
    }
  }
}

// NEXT-1: the Maclaurin closed form (Eq. 4) of one span for one point, times gamma:
//   mu = eta - (P C f3 / alpha)(eta - eta2),  eta = (e^{(i chi - alpha)L} - 1)/(i chi - alpha),
//   eta2 the same with 2 alpha; x = chi h / pi, px = chi h, ah = alpha h, gh = gamma h.
__device__ __forceinline__ void mu_maclaurin(const KParams& p, int s, double x, double px, double ah, double gh,
                                             int Ks, double f3l, double* mr, double* mi) {
  const double aL = __ldg(p.aL + s);
  double sl, cl;
  sincospi_d(x * Ks, &sl, &cl);                  // e^{i chi L}
  const double e1 = exp(-aL), e2 = e1 * e1;
  // eta / h = (e1 cis(chi L) - 1) / ((i chi - alpha) h): multiply by conj(d) / |d|^2
  const double ar = -ah, ai = px;                // d = (i chi - alpha) h
  const double den1 = 1.0 / fma(ai, ai, ar * ar);
  const double n1r = fma(e1, cl, -1.0), n1i = e1 * sl;
  const double eta_r = (n1r * ar + n1i * ai) * den1;
  const double eta_i = (n1i * ar - n1r * ai) * den1;
  const double br = -2.0 * ah;
  const double den2 = 1.0 / fma(ai, ai, br * br);
  const double n2r = fma(e2, cl, -1.0), n2i = e2 * sl;
  const double et2_r = (n2r * br + n2i * ai) * den2;
  const double et2_i = (n2i * br - n2r * ai) * den2;
  const double cf = __ldg(p.mac_c + s) * f3l;
  // (values above are eta / h; gh = gamma h restores the scale)
  *mr = (eta_r - cf * (eta_r - et2_r)) * gh;
  *mi = (eta_i - cf * (eta_i - et2_i)) * gh;
}

// ---- NEXT-2: one span of the integral form for the thread's PPT points (MODE_QUAD)
__device__ __forceinline__ void span_quad(const KParams& p, int s, int ch, double A2, double A3, int Ks,
                                          double f3l, const double (&uv)[PPT], const double (&Ssum)[PPT],
                                          const bool (&valid)[PPT], double (&yr)[PPT], double (&yi)[PPT],
                                          double (&th)[PPT]) {
  // ---- NEXT-2: Eq. 23 mu_s = int_0^L rho_s(z, f3) e^{i chi z} dz by the oracle's rule
  // (reading C12): n = max(64, 4|chi|L/2pi) equal panels rounded up to 2^k, 12-node
  // Gauss-Legendre each; rho_s from Eq. 25 evaluated at every node (the paper's slow
  // baseline: cost grows with the oscillation |chi| L).  Points run one at a time.
  const double Lsp = __ldg(p.Ls + s), al = __ldg(p.alpha + s), gam = __ldg(p.gamma + s);
  const double pcr = __ldg(p.pcr + s);
  for (int q = 0; q < PPT; ++q) {
    const double xq = uv[q] * fma(A3, Ssum[q], A2);       // chi h / pi
    const double xk = xq * Ks;                            // chi L / pi
    double mr = 0.0, mi = 0.0;
    if (valid[q]) {
      const double want = fmax(64.0, ceil(2.0 * fabs(xk)));   // 4 |chi| L / (2 pi)
      long long npan = 64;
      while ((double)npan < want) npan <<= 1;
      const double hp = Lsp / (double)npan, hh = 0.5 * hp;
      const double xz = xk / Lsp;                         // chi / pi per metre
      for (long long j = 0; j < npan; ++j) {
        const double z0 = (double)j * hp;
#pragma unroll
        for (int gq = 0; gq < 12; ++gq) {
          const double z = fma(p.gl_x[gq] + 1.0, hh, z0);
          const double ze = pcr * (-expm1(-al * z)) / al;          // Eq. 2: zeta(z)
          const double xx = p.b_tot * ze;
          // Eq. 25: B P C L_eff e^{-alpha z - zeta f3} / (2 sinh(x/2)), x = B zeta
          const double c = (xx == 0.0) ? 1.0 : xx / (-expm1(-xx));
          const double rho = c * exp(-0.5 * xx - ze * f3l - al * z);
          double sz, cz;
          sincospi_d(xz * z, &sz, &cz);                  // e^{i chi z} (Eq. 24)
          const double wr = p.gl_w[gq] * rho;
          mr = fma(wr, cz, mr);
          mi = fma(wr, sz, mi);
        }
      }
      mr *= hh * gam;
      mi *= hh * gam;
    }
    double ps = 0.0, pc = 1.0;
    if (ch > 0) sincospi_d(th[q], &ps, &pc);
    yr[q] = fma(mr, pc, fma(-mi, ps, yr[q]));
    yi[q] = fma(mr, ps, fma(mi, pc, yi[q]));
    const double t2 = fma(xq, (double)Ks, th[q]);
    th[q] = t2 - 2.0 * rint(0.5 * t2);
  }
}

// ---- row a8: one run of G identical spans in the mixed fp32 variant (MODE_SEG32); rowf is the
// thread's fp32 envelope-table row
__device__ __forceinline__ void span_seg32(const KParams& p, int ch, int G, int cls, double A2, double A3,
                                           double Eh, double ah, double gh, int Ks, const float* rowf,
                                           const double (&uv)[PPT], const double (&Ssum)[PPT],
                                           double (&yr)[PPT], double (&yi)[PPT], double (&th)[PPT]) {
  // ---- row a8: mixed fp32 variant (no span chains).  chi h / pi and its reduction
  // mod 2 stay fp64 (exact); z = cis(pi r) by sincospif; the recurrence runs on pairs
  // of points with packed FFMA2; I_0, mu, the span phase factor and the run's Y sum in fp32;
  // the phase advance and Y across runs in fp64.
  const float Ehf = (float)Eh, ahf = (float)ah, ghf = (float)gh;
  const int Kp4 = (__ldg(p.Kc + cls) + 3) & ~3;
  const float4* rowq = reinterpret_cast<const float4*>(rowf);
  double xs[PPT];
  float sf[PPT], cf[PPT], nrf[PPT], nif[PPT], prr[PPT], pri[PPT], drr[PPT], dri[PPT];
  float2 c2[PPT / 2];
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    xs[q] = uv[q] * fma(A3, Ssum[q], A2);                 // chi h / pi
    const double r = xs[q] - 2.0 * rint(0.5 * xs[q]);     // exact, |r| <= 1
    sincospif((float)r, &sf[q], &cf[q]);
    // I_0 = (w - 1)/(i chi - alpha): the same for every span of the run (G identical spans)
    const float px = (float)(CUDART_PI * xs[q]);
    const float wr1 = fmaf(Ehf, cf[q], -1.f), wi = Ehf * sf[q];
    const float inv = __fdividef(ghf, fmaf(px, px, ahf * ahf));
    nrf[q] = fmaf(wi, px, -ahf * wr1) * inv;
    nif[q] = -fmaf(px, wr1, ahf * wi) * inv;
    // span phase e^{i theta_s} and its per-span step e^{i chi L} (reading C3)
    const double tk = xs[q] * Ks;
    const double rk = tk - 2.0 * rint(0.5 * tk);
    sincospif((float)rk, &dri[q], &drr[q]);
    if (ch > 0) __sincosf(CUDART_PI_F * (float)th[q], &pri[q], &prr[q]);
    else { pri[q] = 0.f; prr[q] = 1.f; }
  }
#pragma unroll
  for (int hq = 0; hq < PPT / 2; ++hq) c2[hq] = make_float2(2.f * cf[2 * hq], 2.f * cf[2 * hq + 1]);
  const int n4 = Kp4 >> 2;
  // the run's Y contribution in fp32 (<= CHAIN_MAX / K spans), added to the fp64 Y once per run
  float ayr[PPT], ayi[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) ayr[q] = ayi[q] = 0.f;
  for (int gi = 0; gi < G; ++gi) {
    // ---- each span's own K-segment recurrence (Eqs. 8-9)
    float2 b1[PPT / 2], b2[PPT / 2];
#pragma unroll
    for (int hq = 0; hq < PPT / 2; ++hq) {
      b1[hq] = make_float2(0.f, 0.f);
      b2[hq] = make_float2(0.f, 0.f);
    }
    auto step = [&](float a) {
#pragma unroll
      for (int hq = 0; hq < PPT / 2; ++hq) {
        // (2cos b_{k+1} + a) - b_{k+2}: the shared a in the addend slot (operand reuse)
        const float2 t = __ffma2_rn(c2[hq], b1[hq], make_float2(a, a));
        // - b_{k+2} as FADD2 with a negated operand (two register pairs read instead of three; the
        // same value as FFMA2 by -1: c2 -0.2 %, c5 -0.1 %, profiles/r02zd_variants_fp32_fadd2.txt)
        const float2 n = __fadd2_rn(t, make_float2(-b2[hq].x, -b2[hq].y));
        b2[hq] = b1[hq];
        b1[hq] = n;
      }
    };
    float4 tc = rowq[0];
#pragma unroll 2
    for (int i4 = 0; i4 < n4 - 1; ++i4) {
      const float4 tn = rowq[i4 + 1];
      step(tc.x);
      step(tc.y);
      step(tc.z);
      step(tc.w);
      tc = tn;
    }
    step(tc.x);
    step(tc.y);
    step(tc.z);                                           // -> b_1, b_2
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const float bb1 = (q & 1) ? b1[q >> 1].y : b1[q >> 1].x;
      const float bb2 = (q & 1) ? b2[q >> 1].y : b2[q >> 1].x;
      const float accr = fmaf(cf[q], bb1, tc.w - bb2);     // a'_0 + z b_1 - b_2
      const float acci = sf[q] * bb1;
      const float mr = nrf[q] * accr - nif[q] * acci;      // mu_s = I_0 sum
      const float mi = nrf[q] * acci + nif[q] * accr;
      ayr[q] += fmaf(mr, prr[q], -mi * pri[q]);            // Y += gamma mu e^{i theta_s}
      ayi[q] += fmaf(mr, pri[q], mi * prr[q]);
      const float npr = fmaf(prr[q], drr[q], -pri[q] * dri[q]);
      pri[q] = fmaf(prr[q], dri[q], pri[q] * drr[q]);
      prr[q] = npr;
    }
  }
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    yr[q] += (double)ayr[q];
    yi[q] += (double)ayi[q];
    const double t2 = fma(xs[q], (double)(Ks * G), th[q]);
    th[q] = t2 - 2.0 * rint(0.5 * t2);
  }
}

// The segment sum of one span chain (Eqs. 8-9 with I_k = I_0 w^k, reading R2 / R9): the chain's G
// spans walk the thread's envelope row G times (rowp[npair] repeats rowp[0] for the wrap) through the
// second-order recurrence b_k = (2cos(chi h) b_{k+1} + a'_k) - b_{k+2}, 1 DFMA + 1 DADD per segment,
// PPT independent recurrences interleaved; returns sum_k a'_k z^k = a'_0 + z b_1 - b_2 per point.
__device__ __forceinline__ void chain_sum(const double2* __restrict__ rowp, int npair, int G,
                                          const double (&c2)[PPT], const double (&sn)[PPT],
                                          double (&accr)[PPT], double (&acci)[PPT]) {
  double b1[PPT], b2[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    b1[q] = 0.0;
    b2[q] = 0.0;
  }
  double2 tc = rowp[0];
  for (int gi = 0; gi < G; ++gi) {
    const int nit = (gi == G - 1) ? npair - 1 : npair;
    ISRS_UNROLL_PRAGMA(ISRS_UNROLL)
    for (int i2 = 0; i2 < nit; ++i2) {
      const double2 tn = rowp[i2 + 1];
      // the coefficient a'_k, shared by the PPT recurrences, sits in the DFMA's addend slot where
      // the operand-reuse cache serves it (tools/fp64_pattern_probe.cu B26)
      double n0[PPT];
#pragma unroll
      for (int q = 0; q < PPT; ++q) n0[q] = fma(c2[q], b1[q], tc.x) - b2[q];
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        const double n1 = fma(c2[q], n0[q], tc.y) - b1[q];
        b2[q] = n0[q];
        b1[q] = n1;
      }
      tc = tn;
    }
  }
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const double n0 = fma(c2[q], b1[q], tc.x) - b2[q];   // b_1
    accr[q] = fma(0.5 * c2[q], n0, tc.y - b1[q]);        // a'_0 + z b_1 - b_2, cos(chi h) = c2 / 2
    acci[q] = sn[q] * n0;
  }
}

// ------------------------------------------------------------------------------------------
// integrand (rows a3-a6)

template <bool COH, int MODE>
__global__ void __launch_bounds__(BLOCK, MIN_BLOCKS)
integrand_kernel(const KParams p, const int* __restrict__ list) {
  extern __shared__ __align__(16) char smem_raw[];
  constexpr bool SEGM = (MODE == MODE_SEGMENT || MODE == MODE_SEGDD || MODE == MODE_SEGLG || MODE == MODE_SEGGRP ||
                         MODE == MODE_SEGDDL || MODE == MODE_SEGSPL || MODE == MODE_SEGGRPSPL);
  constexpr bool SPLIT = (MODE == MODE_SEGSPL || MODE == MODE_SEGGRPSPL);   // k3 line filter (SCI / XCI / MCI)
  constexpr bool LG = (MODE == MODE_SEGLG);   // literal Eq. 22 gain products (NEXT-4b)
  constexpr bool DEDUP = (MODE == MODE_SEGDD || MODE == MODE_SEGDDL);
  constexpr bool DEDUPL = (MODE == MODE_SEGDDL);   // closed-form phased-array factor for runs > 32 spans
  Smem sm;
  constexpr bool grouped = mode_grouped(MODE);   // chain groups (R9): the segment mode when some
                                                     // group holds more than one chain
  smem_layout(p.tstride, p.tw, p.N, COH, grouped, smem_raw, &sm);
  const int tid = threadIdx.x;
  PROF_DECL
  const int rid = list[blockIdx.x];
  const RegionDesc rd = p.desc[rid];
  const int k1 = rd.k1, k2 = rd.k2, flags = rd.flags;
  const int N = p.N;

  const double f = __ldg(p.fv + (flags >> FV_SHIFT));          // NLI frequency (C1 / 3-D f_m)
  const double lo1 = __ldg(p.lo + k1), lo2 = __ldg(p.lo + k2);
  const double d1 = __ldg(p.delta + k1), d2 = __ldg(p.delta + k2);
  // lattice ratio a:b = R1:R2 (coprime); f3 = C + g (a m1 + b m2), exact in fp64 (reading C10)
  const long long r1 = __ldg(p.rate + k1), r2 = __ldg(p.rate + k2);
  const long long g0 = gcd_ll(r1, r2);
  const int a = (int)(r1 / g0), b = (int)(r2 / g0);
  const double g = d1 / a;                                   // = d2 / b, an integer number of Hz
  const double C = __dadd_rn(__dadd_rn(__dadd_rn(lo1, lo2), -f), __dadd_rn(0.5 * d1, 0.5 * d2));
  int inv_a = 0;                                             // a^{-1} mod b
  if (b > 1) {
    for (int x = 1; x < b; ++x)
      if ((long long)a * x % b == 1) { inv_a = x; break; }
  }
  const int J = (a + b) * (N - 1) + 1;

  double Dacc = 0.0;
  double Ghat = 0.0;           // sum_i wD_i |a_i|^2 (G)
  double2 hsum = make_double2(0.0, 0.0);  // sum_i wE_i a_i (H)
  long long npts_total = 0;
  if (COH) {
    for (int m = tid; m < N; m += BLOCK) {
      sm.rowacc[m] = make_double2(0.0, 0.0);
      sm.colacc[m] = make_double2(0.0, 0.0);
    }
  }

  PROF_MARK(0)   // prologue
  for (int seg0 = 0; seg0 < J; seg0 += LINE_CAP) {
    const int nl = min(LINE_CAP, J - seg0);
    // ---- line scan (gates, point counts) and order-preserving compaction of supported lines
    const int4 tot = scan_lines<SPLIT>(p, sm, seg0, nl, N, a, b, inv_a, SPLIT ? rd.kappa : 0, k1, k2, flags, C, g);
    const int S = tot.x, NP = tot.y;
    if (tid == 0) sm.sl_start[S] = NP;
    if (COH) {
      for (int i = tid; i < S; i += BLOCK) sm.lineacc[i] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    npts_total += tot.z;
    if (NP == 0) continue;

    int tb = 0, tn = 0, tcls = -1;  // resident table: compacted lines [tb, tb + tn), class tcls
    PROF_MARK(1)   // line scan + compaction
    int i_first = 0;                // line of slot p0 (carried across chunks: no search)
    for (int p0 = 0; p0 < NP;) {
      // ---- chunk boundaries (block-uniform)
      const int lim = min(i_first + p.tw, S);
      const int p_end = min(p0 + CP, sm.sl_start[lim]);
      const int i_last = line_of(sm.sl_start, lim - 1, p_end - 1, i_first);
      ISRS_BOUND(i_last, S);
      ISRS_BOUND(i_first, i_last + 1);
      PROF_COUNT(10, 1)
      PROF_COUNT(11, p_end - p0)
      PROF_COUNT(12, i_last - i_first + 1)

      // ---- per-thread points: PPT consecutive slots of one line (lines are padded to whole
      // groups), so one envelope-table row serves all PPT recurrences of the thread
      const int slot0 = p0 + PPT * tid;
      const bool gvalid = slot0 < p_end;
      // line of this thread's group: one (warp-uniform, broadcast) search for the line i0 of
      // the warp's first group, then the <= 31 later line starts inside the warp's 32 groups
      // are OR-ed into a position mask (lines are padded to whole groups, so each starts on
      // its own group): line = i0 + #starts at positions <= lane
      const int lane = tid & 31;
      const int wslot0 = p0 + PPT * (tid & ~31);
      const bool wact = wslot0 < p_end;                    // warp has at least one valid group
      const int i0 = wact ? line_of(sm.sl_start, i_last, wslot0, i_first) : i_first;
      int pos = 32;
      if (lane < 31 && i0 + 1 + lane < S) pos = (sm.sl_start[i0 + 1 + lane] - wslot0) / PPT;
      const unsigned starts = __reduce_or_sync(0xffffffffu, (pos < 32) ? (1u << pos) : 0u);
      const int li = gvalid ? i0 + __popc(starts & ((2u << lane) - 1u)) : i_first;
      const int lj = sm.sl_j[li];
      const int kq0 = slot0 - sm.sl_start[li];
      const int lcnt = sm.sl_cnt[li];
      bool valid[PPT];
      double uv[PPT], Ssum[PPT];
      const double f3l = __dadd_rn(C, g * (double)lj);
      // the line's first point (m1f, m2f): one exact division per thread; along the line
      // m1 steps by b and m2 by -a
      const int m1f = sm.sl_first[li];
      const int m2f = (b == 1) ? lj - a * m1f : (lj - a * m1f) / b;
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        valid[q] = gvalid && (kq0 + q < lcnt);
        const int step_q = valid[q] ? kq0 + q : 0;
        const int m1 = m1f + b * step_q;
        const int m2 = m2f - a * step_q;
        const double f1 = __dadd_rn(lo1, __dmul_rn((double)m1 + 0.5, d1));   // C6 bin centres
        const double f2 = __dadd_rn(lo2, __dmul_rn((double)m2 + 0.5, d2));
        const double u = __dadd_rn(f1, -f), w = __dadd_rn(f2, -f);
        uv[q] = __dmul_rn(u, w);
        Ssum[q] = __dadd_rn(f1, f2);
        if constexpr (grouped) {                    // chain groups read them from smem (register room)
          sm.gst[q * BLOCK + tid] = uv[q];
          sm.gst[(PPT + q) * BLOCK + tid] = Ssum[q];
        }
      }

      double yr[PPT], yi[PPT], th[PPT];
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        yr[q] = (MODE == MODE_UNIT) ? 1.0 : 0.0;
        yi[q] = 0.0;
        th[q] = 0.0;
      }

      PROF_MARK(2)   // chunk setup (line lookup, geometry)
      if constexpr (grouped) {
        // ---- chain groups (reading R9): z = e^{i chi h} and I_0 once per group of identical spans;
        // each chain's segment sum is rotated by its span phase e^{i theta_c} (Eq. 22, C3) and summed,
        // then mu = gamma I_0 S once per group
        for (int gr = 0; gr < p.n_grp; ++gr) {
          if (gr > 0) { PROF_MARK(4) }
          const int c0 = __ldg(p.grp_c0 + gr), c1 = __ldg(p.grp_c0 + gr + 1);
          const int s = __ldg(p.chain_s0 + c0);
          const int cls = __ldg(p.cls + s);
          if (cls != tcls || i_first < tb || i_last >= tb + tn) {
            __syncthreads();
            tb = i_first;
            tn = (p.n_cls == 1) ? min(p.tw, S - i_first) : (i_last - i_first + 1);
            tcls = cls;
            build_table<false>(p, sm, cls, tb, tn, C, g);
            PROF_COUNT(8, 1)
            PROF_COUNT(9, tn)
            __syncthreads();
          }
          PROF_MARK(3)
          if (!wact) continue;   // warp-uniform: idle warps of a ragged last chunk skip the math
          const double A2 = __ldg(p.A2 + s), A3 = __ldg(p.A3 + s);
          const int Ks = __ldg(p.K + s);
          const int npair = ((__ldg(p.Kc + cls) + 1) & ~1) >> 1;
          ISRS_BOUND(li - tb, tn);
          const double2* rowp = (const double2*)(sm.T + (li - tb) * p.tstride);
          // thread-private smem slots (column tid: conflict-free) hold what is only needed between
          // chains, so the recurrence runs with the register budget of a single chain
          ISRS_BOUND((5 * PPT - 1) * BLOCK + tid, 5 * PPT * BLOCK);
          double* gu = sm.gst + tid;                        // [q * BLOCK]: (f1 - f)(f2 - f)
          double* gs = sm.gst + PPT * BLOCK + tid;          // f1 + f2
          double* gx = sm.gst + 2 * PPT * BLOCK + tid;      // chi h / pi
          double* gwr = sm.gst + 3 * PPT * BLOCK + tid;     // w = e^{i G0 chi L}, real
          double* gwi = sm.gst + 4 * PPT * BLOCK + tid;     // imaginary
          const int nch = c1 - c0, G0 = __ldg(p.chain_g + c0);
          double c2[PPT], sn[PPT], sr[PPT], si[PPT];
#pragma unroll
          for (int q = 0; q < PPT; ++q) {
            const double x = gu[q * BLOCK] * fma(A3, gs[q * BLOCK], A2);   // chi h / pi (Eq. 5 x h / pi)
            gx[q * BLOCK] = x;
            double cs;
            sincospi_d(x, &sn[q], &cs);                     // z = e^{i chi h}
            c2[q] = cs + cs;
            if (nch > 1) {                                   // w = z^{G0 K} = e^{i G0 chi L}
              const double t = x * (double)(Ks * G0);
              double ss, cc;
              sincospi_d(t - 2.0 * rint(0.5 * t), &ss, &cc);
              gwr[q * BLOCK] = cc;
              gwi[q * BLOCK] = ss;
            }
          }
          // S = sum_c e^{i (theta_c - theta_c0)} sum_c = A_c0 + w (A_c0+1 + w (...)), chains of the
          // group in reverse (Horner over the chains; every chain but the last has G0 spans)
          for (int ch = c1 - 1; ch >= c0; --ch) {
            double accr[PPT], acci[PPT];
            chain_sum(rowp, npair, __ldg(p.chain_g + ch), c2, sn, accr, acci);
            if (ch == c1 - 1) {
#pragma unroll
              for (int q = 0; q < PPT; ++q) {
                sr[q] = accr[q];
                si[q] = acci[q];
              }
            } else {
#pragma unroll
              for (int q = 0; q < PPT; ++q) {
                const double a = gwr[q * BLOCK], b = gwi[q * BLOCK];
                const double t = fma(sr[q], a, fma(-si[q], b, accr[q]));
                si[q] = fma(sr[q], b, fma(si[q], a, acci[q]));
                sr[q] = t;
              }
            }
          }
          const double Eh = __ldg(p.Eh + s), ah = __ldg(p.ah + s), gh = __ldg(p.gh + s);
          int gsum = 0;
          for (int ch = c0; ch < c1; ++ch) gsum += __ldg(p.chain_g + ch);
#pragma unroll
          for (int q = 0; q < PPT; ++q) {
            const double x = gx[q * BLOCK];
            const double px = CUDART_PI * x;     // chi h
            // I_0 = (w - 1)/(i chi - alpha) = h (w - 1) conj(d) / |d|^2, d = -alpha h + i chi h
            const double wr1 = fma(Eh, 0.5 * c2[q], -1.0), wi = Eh * sn[q];
            const double inv = gh * rcp_d(fma(px, px, ah * ah));   // gamma_s h / |d|^2
            const double nr = fma(wi, px, -ah * wr1);
            const double ni = -fma(px, wr1, ah * wi);
            const double mr = (nr * sr[q] - ni * si[q]) * inv;     // gamma mu_group / e^{i theta_c0}
            const double mi = (nr * si[q] + ni * sr[q]) * inv;
            double ps = 0.0, pc = 1.0;                             // theta_1 = 0 for the first group
            if (gr > 0) sincospi_d(th[q], &ps, &pc);
            yr[q] = fma(mr, pc, fma(-mi, ps, yr[q]));              // Y += gamma mu e^{i theta} (Eq. 22, C3)
            yi[q] = fma(mr, ps, fma(mi, pc, yi[q]));
            const double t2 = fma(x, (double)(Ks * gsum), th[q]);  // theta += chi L per span of the group
            th[q] = t2 - 2.0 * rint(0.5 * t2);
          }
        }
      } else if constexpr (MODE != MODE_UNIT) {
        for (int ch = 0; ch < p.n_chain; ++ch) {
          if (ch > 0) { PROF_MARK(4) }   // previous chain's span math
          // chain of G identical consecutive spans starting at s (G = 1 unless chained, R9)
          const int s = __ldg(p.chain_s0 + ch), G = __ldg(p.chain_g + ch);
          const int cls = __ldg(p.cls + s);
#ifdef ISRS_DIAG_NO_REBUILD
          // diagnostic builds only (wrong values): keep the first span's table for every span, to bound
          // what the per-span table costs on multi-class links
          if ((SEGM || MODE == MODE_SEG32) && (tcls < 0 || i_first < tb || i_last >= tb + tn)) {
#else
          if ((SEGM || MODE == MODE_SEG32) &&
              (cls != tcls || i_first < tb || i_last >= tb + tn)) {
#endif
            // ---- (re)build the envelope table rows for compacted lines [tb, tb + tn)
            __syncthreads();
            tb = i_first;
            tn = (p.n_cls == 1) ? min(p.tw, S - i_first) : (i_last - i_first + 1);
            tcls = cls;
            build_table<MODE == MODE_SEG32>(p, sm, cls, tb, tn, C, g);
            PROF_COUNT(8, 1)
            PROF_COUNT(9, tn)
            __syncthreads();
          }
          PROF_MARK(3)   // table (re)build incl. barriers
          if (!wact) continue;   // warp-uniform: idle warps of a ragged last chunk skip the math
          const double A2 = __ldg(p.A2 + s), A3 = __ldg(p.A3 + s);
          const double Eh = __ldg(p.Eh + s), ah = __ldg(p.ah + s), gh = __ldg(p.gh + s);
          const int Ks = __ldg(p.K + s);
          if (MODE == MODE_QUAD) {
            span_quad(p, s, ch, A2, A3, Ks, f3l, uv, Ssum, valid, yr, yi, th);
            continue;
          }
          if (MODE == MODE_SEG32) {
            ISRS_BOUND(li - tb, tn);
            span_seg32(p, ch, G, cls, A2, A3, Eh, ah, gh, Ks,
                       reinterpret_cast<const float*>(sm.T) + (li - tb) * 2 * p.tstride, uv, Ssum, yr, yi,
                       th);
            continue;
          }
          double x[PPT], sn[PPT], cs[PPT];
#pragma unroll
          for (int q = 0; q < PPT; ++q) {
            x[q] = uv[q] * fma(A3, Ssum[q], A2);     // chi h / pi  (Eq. 5 times h / pi)
            sincospi_d(x[q], &sn[q], &cs[q]);        // z = e^{i chi h}
          }
          double accr[PPT], acci[PPT];
          if (SEGM) {
            // ---- Goertzel over the K_s segments (Eqs. 8-9 with I_k = I_0 w^k)
            const int Kp = (__ldg(p.Kc + cls) + 1) & ~1;
            double c2[PPT], b1[PPT], b2[PPT];
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
              c2[q] = cs[q] + cs[q];
              b1[q] = 0.0;
              b2[q] = 0.0;
            }
            const double2* rowp = (const double2*)(sm.T + (li - tb) * p.tstride);
            const int npair = Kp >> 1;
            ISRS_BOUND(li - tb, tn);
            ISRS_BOUND(npair, p.tstride / 2);
            // software-pipelined: the 16-byte loads of pair i2+1 are in flight while the PPT
            // independent recurrences of pair i2 run interleaved (LDS latency ~29 cycles)
            // span chain (R9): the coefficients of G identical spans repeat with period K, so
            // the row is walked G times (rowp[npair] holds a copy of rowp[0] for the wrap)
            double2 tc = rowp[0];
            const int Gr = DEDUP ? 1 : G;        // NEXT-4a: one span's sum, reused below
            // NEXT-4b: span g of the chain carries Lambda_{s+g} = Lambda_s r^g with r = S_L(f3), the
            // SRS gain at the span end (identical spans); blocks run from g = G-1 down, so the
            // recurrence state is scaled by r at every block boundary (linear in the coefficients)
            const double rlg = LG ? exp(__ldg(p.lnc_L + s) - __ldg(p.zeta_L + s) * f3l) : 1.0;
            for (int gi = 0; gi < Gr; ++gi) {
              const int nit = (gi == Gr - 1) ? npair - 1 : npair;
              if (LG && gi > 0) {
#pragma unroll
                for (int q = 0; q < PPT; ++q) {
                  b1[q] *= rlg;
                  b2[q] *= rlg;
                }
              }
              ISRS_UNROLL_PRAGMA(ISRS_UNROLL)
              for (int i2 = 0; i2 < nit; ++i2) {
                const double2 tn = rowp[i2 + 1];
                // b_k = (2cos(chi h) b_{k+1} + a'_k) - b_{k+2}: the coefficient a'_k, shared by the
                // PPT recurrences, sits in the DFMA's addend slot where the operand-reuse cache
                // serves it, so each DFMA fetches two fresh 64-bit registers instead of three (a
                // bank conflict on B200's FP64 path; 83 % -> 89 % of the pipe in isolation,
                // tools/fp64_pattern_probe.cu B26)
                double n0[PPT];
#pragma unroll
                for (int q = 0; q < PPT; ++q) n0[q] = fma(c2[q], b1[q], tc.x) - b2[q];
#pragma unroll
                for (int q = 0; q < PPT; ++q) {
                  const double n1 = fma(c2[q], n0[q], tc.y) - b1[q];
                  b2[q] = n0[q];
                  b1[q] = n1;
                }
                tc = tn;
              }
            }
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
              // x and cos(chi h) were left dead across the recurrence (register room for its
              // schedule): cos = c2 / 2 exactly, x recomputed bitwise (the asm fence stops CSE)
              asm volatile("" : "+d"(uv[q]), "+d"(Ssum[q]));
              x[q] = uv[q] * fma(A3, Ssum[q], A2);
              cs[q] = 0.5 * c2[q];
              const double n0 = fma(c2[q], b1[q], tc.x) - b2[q];   // b_1
              // sum_k a'_k z^k = a'_0 + z b_1 - b_2
              accr[q] = fma(cs[q], n0, tc.y - b1[q]);
              acci[q] = sn[q] * n0;
            }
            if (DEDUPL && G > 32) {
              // NEXT-4a: x sum_{g<G} rho^g, rho = e^{i chi L} (the identical spans' phases, C3); for long
              // runs in closed form e^{i (G-1) chi L / 2} sin(G chi L / 2) / sin(chi L / 2) (3 sincospi and
              // a division instead of G - 1 complex products: c5's run of 50 spans, dedup 10.9 -> 9.0 s
              // for all 200 COIs; slower than the products up to G ~ 30: c3's G = 20 +6 %); within 1e-3
              // of a zero of sin(chi L / 2) (rho ~ 1, the ratio ill-conditioned) the products
#pragma unroll
              for (int q = 0; q < PPT; ++q) {
                const double hx = x[q] * Ks;                       // chi L / pi
                const double hr = hx - 2.0 * rint(0.5 * hx);       // exact, in [-1, 1]
                double s1, c1;
                sincospi_d(0.5 * hr, &s1, &c1);                    // sin, cos (chi L / 2)
                double gr = 1.0, gim = 0.0;
                if (fabs(s1) > 1e-3) {
                  const double tg = 0.5 * (double)G * hr, tp = 0.5 * (double)(G - 1) * hr;
                  double sg, cg, sp, cp;
                  sincospi_d(tg - 2.0 * rint(0.5 * tg), &sg, &cg);
                  sincospi_d(tp - 2.0 * rint(0.5 * tp), &sp, &cp);
                  const double amp = sg / s1;
                  gr = amp * cp;
                  gim = amp * sp;
                } else {
                  const double rc = fma(-2.0 * s1, s1, 1.0), rs = 2.0 * s1 * c1;   // rho
                  for (int g2 = 1; g2 < G; ++g2) {
                    const double t = fma(gr, rc, fma(-gim, rs, 1.0));
                    gim = fma(gr, rs, gim * rc);
                    gr = t;
                  }
                }
                const double ar = accr[q];
                accr[q] = fma(ar, gr, -acci[q] * gim);
                acci[q] = fma(ar, gim, acci[q] * gr);
              }
            } else if (DEDUP && G > 1) {
              // NEXT-4a: x sum_{g<G} rho^g, rho = e^{i chi L} (the identical spans' phases, C3)
#pragma unroll
              for (int q = 0; q < PPT; ++q) {
                double rs, rc;
                sincospi_d(x[q] * Ks, &rs, &rc);
                double gr = 1.0, gim = 0.0;
                for (int g2 = 1; g2 < G; ++g2) {
                  const double t = fma(gr, rc, fma(-gim, rs, 1.0));
                  gim = fma(gr, rs, gim * rc);
                  gr = t;
                }
                const double ar = accr[q];
                accr[q] = fma(ar, gr, -acci[q] * gim);
                acci[q] = fma(ar, gim, acci[q] * gr);
              }
            }
          }
#pragma unroll
          for (int q = 0; q < PPT; ++q) {
            const double px = CUDART_PI * x[q];     // chi h
            double mr, mi;
            if (SEGM) {
              // I_0 = (w - 1)/(i chi - alpha) = h (w - 1) conj(d) / |d|^2, d = -alpha h + i chi h
              const double wr1 = fma(Eh, cs[q], -1.0), wi = Eh * sn[q];
              const double inv = gh * rcp_d(fma(px, px, ah * ah));   // gamma_s h / |d|^2
              const double nr = fma(wi, px, -ah * wr1);
              const double ni = -fma(px, wr1, ah * wi);
              mr = (nr * accr[q] - ni * acci[q]) * inv;
              mi = (nr * acci[q] + ni * accr[q]) * inv;
            } else {
              mu_maclaurin(p, s, x[q], px, ah, gh, Ks, f3l, &mr, &mi);
            }
            if (LG) {   // Lambda_s of the chain's first span (prefix / suffix sums)
              const double lam = exp(0.5 * (fma(-__ldg(p.lgB + s), 2.0 * f3l + f, __ldg(p.lgA + s)) +
                                            fma(-__ldg(p.lgD + s), f, __ldg(p.lgC + s))));
              mr *= lam;
              mi *= lam;
            }
            // Y += gamma_s mu_s e^{i theta_s}, theta_s = pi * th (reading C3)
            double ps = 0.0, pc = 1.0;                  // theta_1 = 0 for the first chain
            if (ch > 0) sincospi_d(th[q], &ps, &pc);
            yr[q] = fma(mr, pc, fma(-mi, ps, yr[q]));
            yi[q] = fma(mr, ps, fma(mi, pc, yi[q]));
            double t2 = fma(x[q], (double)(Ks * G), th[q]);   // theta += chi_s L_s (x G spans)
            th[q] = t2 - 2.0 * rint(0.5 * t2);          // exact reduction mod 2 (units of pi)
          }
        }
      }

      PROF_MARK(4)   // span math (z, recurrence, mu, Y)
      // ---- D accumulation
#pragma unroll
      for (int q = 0; q < PPT; ++q) {
        if (valid[q]) Dacc = fma(sm.wD[li], fma(yr[q], yr[q], yi[q] * yi[q]), Dacc);
      }

      if (COH) {
#pragma unroll
        for (int q = 0; q < PPT; ++q)
          sm.ybuf[PPT * tid + q] = valid[q] ? make_double2(yr[q], yi[q]) : make_double2(0.0, 0.0);
        __syncthreads();
        coherent_chunk(sm, flags, N, a, b, i_first, i_last, p0, p_end);
        __syncthreads();
      }
      p0 = p_end;
      i_first = (sm.sl_start[i_last + 1] <= p_end) ? i_last + 1 : i_last;
    }
    if (COH && (flags & (NEED_G | NEED_H))) {     // block-uniform
      // G and H of this line segment: lines i = tid, tid + BLOCK, ... per thread, then a fixed-order
      // block sum (Eqs. 20-21 with C7: G = sum_lines t |line sum|^2, H = |sum_lines t line sum|^2)
      double v[3] = {0.0, 0.0, 0.0};
      for (int i = tid; i < S; i += BLOCK) {
        const double2 av = sm.lineacc[i];
        v[0] = fma(sm.wD[i], fma(av.x, av.x, av.y * av.y), v[0]);
        v[1] = fma(sm.wE[i], av.x, v[1]);
        v[2] = fma(sm.wE[i], av.y, v[2]);
      }
      block_sum_n<3>(v, sm.red);
      Ghat += v[0];
      hsum.x += v[1];
      hsum.y += v[2];
    }
    __syncthreads();
  }

  PROF_MARK(5)   // D / coherent accumulation, chunk tails
  // D by the fixed smem tree in both kernels (so the D term of a region is bitwise the same whether
  // or not its E/F/G/H are needed, pin P12), the E / F row and column sums of squares (Eqs. 18-19,
  // C7) by fixed-order warp-shuffle block sums
  double tot[3] = {Dacc, 0.0, 0.0};
  if (COH) {
    tot[0] = block_sum(Dacc, sm.red);
    double ef[2] = {0.0, 0.0};
    for (int m = tid; m < N; m += BLOCK) {
      if (flags & NEED_E) ef[0] = fma(sm.rowacc[m].x, sm.rowacc[m].x, fma(sm.rowacc[m].y, sm.rowacc[m].y, ef[0]));
      if (flags & NEED_F) ef[1] = fma(sm.colacc[m].x, sm.colacc[m].x, fma(sm.colacc[m].y, sm.colacc[m].y, ef[1]));
    }
    block_sum_n<2>(ef, sm.red);
    tot[1] = ef[0];
    tot[2] = ef[1];
  } else {
    tot[0] = block_sum(Dacc, sm.red);
  }
  const double Dsum = tot[0];
  if (tid == 0) {
    double* out = p.partials + (size_t)rid * 6;
    const double E = tot[1], F = tot[2];
    out[0] = Dsum * d1 * d2;                                         // D_w
    out[1] = (COH && (flags & NEED_E)) ? E * d1 * d1 * d2 : 0.0;     // E_w
    out[2] = (COH && (flags & NEED_F)) ? F * d2 * d2 * d1 : 0.0;     // F_w
    out[3] = (COH && (flags & NEED_G)) ? Ghat * d1 * d1 * d1 : 0.0;  // G_w (k1 == k2)
    out[4] = (COH && (flags & NEED_H)) ? (hsum.x * hsum.x + hsum.y * hsum.y) * (d1 * d2) * (d1 * d2) : 0.0;
    out[5] = (double)npts_total;
    if (p.mirror) {
      // f1 <-> f2 symmetry (Eqs. 5, 8, 22 are symmetric in f1, f2; pin P2): region (kappa, k2, k1) has
      // the same Y at the mirrored points, hence the same D_w and n_points, with E and F exchanged
      // (its coherent-over-f1 sum is this region's coherent-over-f2 sum); G and H need k1 == k2
      const int mr = __ldg(p.mirror + rid);
      if (mr >= 0) {
        double* o2 = p.partials + (size_t)mr * 6;
        o2[0] = out[0];
        o2[1] = out[2];
        o2[2] = out[1];
        o2[3] = 0.0;
        o2[4] = 0.0;
        o2[5] = out[5];
      }
    }
  }
  PROF_MARK(6)   // epilogue (block sum, partials)
  PROF_FLUSH
}

template <bool COH, int MODE>
static int set_smem(int tstride, int tw, int N) {
  const size_t smem = integrand_smem_bytes(tstride, tw, N, COH, mode_grouped(MODE));
  return cudaFuncSetAttribute(integrand_kernel<COH, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem) == cudaSuccess ? 0 : -1;
}

template <int MODE>
static int prepare_mode(int tstride, int tw, int N) {
  return (set_smem<true, MODE>(tstride, tw, N) || set_smem<false, MODE>(tstride, tw, N)) ? -1 : 0;
}

// Dynamic shared-memory opt-in of both integrand variants of `mode`, before anything is enqueued.
int integrand_prepare(int mode, int tstride, int tw, int N) {
  switch (mode) {
    case MODE_SEGMENT: return prepare_mode<MODE_SEGMENT>(tstride, tw, N);
    case MODE_SEGGRP: return prepare_mode<MODE_SEGGRP>(tstride, tw, N);
    case MODE_SEGSPL: return prepare_mode<MODE_SEGSPL>(tstride, tw, N);
    case MODE_SEGGRPSPL: return prepare_mode<MODE_SEGGRPSPL>(tstride, tw, N);
    case MODE_SEG32: return prepare_mode<MODE_SEG32>(tstride, tw, N);
    case MODE_SEGDD: return prepare_mode<MODE_SEGDD>(tstride, tw, N);
    case MODE_SEGDDL: return prepare_mode<MODE_SEGDDL>(tstride, tw, N);
    case MODE_SEGLG: return prepare_mode<MODE_SEGLG>(tstride, tw, N);
    case MODE_QUAD: return prepare_mode<MODE_QUAD>(tstride, tw, N);
    case MODE_MACLAURIN: return prepare_mode<MODE_MACLAURIN>(tstride, tw, N);
    default: return prepare_mode<MODE_UNIT>(tstride, tw, N);
  }
}

template <bool COH, int MODE>
static int launch_one(const KParams& p, const int* list, long long n_list, cudaStream_t st) {
  const size_t smem = integrand_smem_bytes(p.tstride, p.tw, p.N, COH, mode_grouped(MODE));
  auto kern = integrand_kernel<COH, MODE>;
  const long long max_grid = 0x7fffffffLL;
  for (long long off = 0; off < n_list; off += max_grid) {
    const unsigned grid = (unsigned)std::min(max_grid, n_list - off);
    kern<<<grid, BLOCK, smem, st>>>(p, list + off);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_integrand(const KParams& p, const int* list, long long n_list, bool coherent, void* stream,
                     int* n_launches) {
  if (n_list <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  *n_launches += 1;
  if (coherent) {
    if (p.mode == MODE_SEGMENT) return launch_one<true, MODE_SEGMENT>(p, list, n_list, st);
    if (p.mode == MODE_SEGGRP) return launch_one<true, MODE_SEGGRP>(p, list, n_list, st);
    if (p.mode == MODE_SEGSPL) return launch_one<true, MODE_SEGSPL>(p, list, n_list, st);
    if (p.mode == MODE_SEGGRPSPL) return launch_one<true, MODE_SEGGRPSPL>(p, list, n_list, st);
    if (p.mode == MODE_SEG32) return launch_one<true, MODE_SEG32>(p, list, n_list, st);
    if (p.mode == MODE_SEGDD) return launch_one<true, MODE_SEGDD>(p, list, n_list, st);
    if (p.mode == MODE_SEGDDL) return launch_one<true, MODE_SEGDDL>(p, list, n_list, st);
    if (p.mode == MODE_SEGLG) return launch_one<true, MODE_SEGLG>(p, list, n_list, st);
    if (p.mode == MODE_QUAD) return launch_one<true, MODE_QUAD>(p, list, n_list, st);
    if (p.mode == MODE_MACLAURIN) return launch_one<true, MODE_MACLAURIN>(p, list, n_list, st);
    return launch_one<true, MODE_UNIT>(p, list, n_list, st);
  }
  if (p.mode == MODE_SEGMENT) return launch_one<false, MODE_SEGMENT>(p, list, n_list, st);
  if (p.mode == MODE_SEGGRP) return launch_one<false, MODE_SEGGRP>(p, list, n_list, st);
  if (p.mode == MODE_SEGSPL) return launch_one<false, MODE_SEGSPL>(p, list, n_list, st);
  if (p.mode == MODE_SEGGRPSPL) return launch_one<false, MODE_SEGGRPSPL>(p, list, n_list, st);
  if (p.mode == MODE_SEG32) return launch_one<false, MODE_SEG32>(p, list, n_list, st);
  if (p.mode == MODE_SEGDD) return launch_one<false, MODE_SEGDD>(p, list, n_list, st);
  if (p.mode == MODE_SEGDDL) return launch_one<false, MODE_SEGDDL>(p, list, n_list, st);
  if (p.mode == MODE_SEGLG) return launch_one<false, MODE_SEGLG>(p, list, n_list, st);
  if (p.mode == MODE_QUAD) return launch_one<false, MODE_QUAD>(p, list, n_list, st);
  if (p.mode == MODE_MACLAURIN) return launch_one<false, MODE_MACLAURIN>(p, list, n_list, st);
  return launch_one<false, MODE_UNIT>(p, list, n_list, st);
}

// ------------------------------------------------------------------------------------------
// per-COI assembly (row a7)

__global__ void __launch_bounds__(BLOCK) reduce_kernel(const RParams p) {
  __shared__ double red[6][BLOCK];
  const int ci = blockIdx.x;
  const long long r0 = max(p.coi_off[ci], p.r_lo), r1 = min(p.coi_off[ci + 1], p.r_hi);
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (long long r = r0 + threadIdx.x; r < r1; r += BLOCK) {
    const RegionDesc rd = p.desc[r];
    const double* q = p.partials + (size_t)r * 6;
    const double G1 = p.G[rd.k1], G2 = p.G[rd.k2], R1 = p.R[rd.k1], R2 = p.R[rd.k2];
    const double ph1 = p.phi[rd.k1], ph2 = p.phi[rd.k2], ps1 = p.psi[rd.k1];
    // Eq. 15 with reading C2 (PSD normalisation, one 1/R_i per cumulant-tied channel)
    acc[0] += 16.0 / 27.0 * G1 * G2 * q[0];
    acc[1] += 16.0 / 27.0 * ph1 * G1 * G1 * G2 * q[1] / R1;
    acc[2] += 32.0 / 81.0 * ph2 * G2 * G2 * G1 * q[2] / R2;
    acc[3] += 16.0 / 81.0 * ph1 * G1 * G1 * q[3] / R1;
    acc[4] += 16.0 / 81.0 * ps1 * G1 * G1 * G1 * q[4] / (R1 * R1);
    acc[5] += q[5];
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) red[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int s = BLOCK / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
#pragma unroll
      for (int k = 0; k < 6; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0 && p.part_out) {          // shard mode: raw sums, combined later
    for (int k = 0; k < 6; ++k) p.part_out[(size_t)ci * 6 + k] = red[k][0];
    return;
  }
  if (threadIdx.x == 0) {
    const int kappa = p.coi[ci];
    const double Pk = p.P[kappa];
    // P_NLI = R G_NLI(f_kappa) (C1) or R mean_m G_NLI(f_m) (3-D, NEXT-3); Eq. 11
    const double scale = p.R[kappa] / (Pk * Pk * Pk) * p.inv_fs;
    double e = 0.0;
    for (int k = 0; k < 5; ++k) {
      const double t = __dmul_rn(red[k][0], scale);   // no contraction: eta independent of terms
      if (p.terms) p.terms[(size_t)ci * 5 + k] = t;
      e = __dadd_rn(e, t);
    }
    p.eta[ci] = e;
    p.npts[ci] = red[5][0];
  }
}

// SCI / XCI / MCI parts of eta (ISRS_EGN_FLAG_SPLIT): every region entry of the split work list
// holds islands of ONE class -- the number of distinct interfering channels among (k1, k2, k3): those of
// (k1, k2), plus one for a K3_OUT entry (k3 is none of kappa, k1, k2) -- so its Eq. 15 contribution goes
// to that class; fixed-tree sum per COI in canonical order, Eq. 11 scale.  split_out [n_coi][3].
__global__ void __launch_bounds__(BLOCK) reduce_split_kernel(const RParams p, double* __restrict__ split_out) {
  __shared__ double red[3][BLOCK];
  const int ci = blockIdx.x;
  const int kappa = p.coi[ci];
  const long long r0 = max(p.coi_off[ci], p.r_lo), r1 = min(p.coi_off[ci + 1], p.r_hi);
  double acc[3] = {0, 0, 0};
  for (long long r = r0 + threadIdx.x; r < r1; r += BLOCK) {
    const RegionDesc rd = p.desc[r];
    const double* q = p.partials + (size_t)r * 6;
    const double G1 = p.G[rd.k1], G2 = p.G[rd.k2], R1 = p.R[rd.k1], R2 = p.R[rd.k2];
    const double ph1 = p.phi[rd.k1], ph2 = p.phi[rd.k2], ps1 = p.psi[rd.k1];
    double t = 16.0 / 27.0 * G1 * G2 * q[0];
    t += 16.0 / 27.0 * ph1 * G1 * G1 * G2 * q[1] / R1;
    t += 32.0 / 81.0 * ph2 * G2 * G2 * G1 * q[2] / R2;
    t += 16.0 / 81.0 * ph1 * G1 * G1 * q[3] / R1;
    t += 16.0 / 81.0 * ps1 * G1 * G1 * G1 * q[4] / (R1 * R1);
    const int nint = (rd.k1 != kappa) + (rd.k2 != kappa && rd.k2 != rd.k1) + ((rd.flags & K3_OUT) ? 1 : 0);
    acc[min(nint, 2)] += t;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) red[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int s = BLOCK / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
#pragma unroll
      for (int k = 0; k < 3; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double Pk = p.P[kappa];
    const double scale = p.R[kappa] / (Pk * Pk * Pk) * p.inv_fs;
    for (int k = 0; k < 3; ++k) split_out[(size_t)ci * 3 + k] = __dmul_rn(red[k][0], scale);
  }
}

int launch_reduce_split(const RParams& p, double* split_out, void* stream) {
  if (p.n_coi <= 0) return 0;
  reduce_split_kernel<<<p.n_coi, BLOCK, 0, (cudaStream_t)stream>>>(p, split_out);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// Multi-GPU combine: the per-COI sums of every shard, added in fixed rank order
// (bitwise identical on every rank), then the Eq. 11 scale.
__global__ void combine_kernel(const CParams p) {
  const int ci = blockIdx.x * blockDim.x + threadIdx.x;
  if (ci >= p.n_coi) return;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int r = 0; r < p.world; ++r)
    for (int k = 0; k < 6; ++k) acc[k] += p.gathered[((size_t)r * p.n_coi + ci) * 6 + k];
  const int kappa = p.coi[ci];
  const double Pk = p.P[kappa];
  const double scale = p.R[kappa] / (Pk * Pk * Pk) * p.inv_fs;
  double e = 0.0;
  for (int k = 0; k < 5; ++k) {
    const double t = __dmul_rn(acc[k], scale);   // no contraction: eta independent of terms
    if (p.terms) p.terms[(size_t)ci * 5 + k] = t;
    e = __dadd_rn(e, t);
  }
  p.eta[ci] = e;
  if (p.npts) p.npts[ci] = acc[5];
}

int launch_combine(const CParams& p, void* stream) {
  if (p.n_coi <= 0) return 0;
  combine_kernel<<<(p.n_coi + 127) / 128, 128, 0, (cudaStream_t)stream>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_reduce(const RParams& p, void* stream) {
  if (p.n_coi <= 0) return 0;
  reduce_kernel<<<p.n_coi, BLOCK, 0, (cudaStream_t)stream>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace isrs
