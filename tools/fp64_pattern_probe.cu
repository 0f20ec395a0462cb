// Probe: which instruction pattern caps the integrand kernel's Goertzel loop at ~81% of the
// FP64 pipe on B200?  Each variant runs 4 CTAs x 128 threads per SM; reports DP thread-instr
// per SM-cycle (peak 64) from per-SM clock64 spans.
//   A  Goertzel, PPT chains, coefficient pairs from smem (LDS.128), as in the kernel
//   B  same arithmetic, coefficients from registers (no LDS)
//   C  B with one shared multiplier for all chains (operand reuse)
//   D  DFMA-only: x = fma(y, x, z) with per-chain y, z (3 distinct 64-bit operands)
//   E  DFMA-only with shared y, z (one fresh operand)
//   F  DADD-only chains x = x - y (per-chain y)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_pattern_probe fp64_pattern_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V, int PPT>
__global__ void __launch_bounds__(128, 4) kern(double* out, long long* cyc, int iters) {
  __shared__ __align__(16) double T[128];
  for (int i = threadIdx.x; i < 128; i += 128) T[i] = 1.0 / (1.0 + i);
  __syncthreads();
  double c2[PPT], b1[PPT], b2[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    c2[q] = 2.0 * __cosf(0.001f * (threadIdx.x * PPT + q + 1));
    b1[q] = 0.1 * q;
    b2[q] = 0.2 * q;
  }
  const double2* rowp = (const double2*)T;
  double2 tc = rowp[threadIdx.x & 7];
  const double cs = c2[0];
  double m1;
  asm volatile("mov.b64 %0, 0xBFF0000000000000;" : "=d"(m1));   // -1.0, opaque to ptxas
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int i2 = 0; i2 < 40; ++i2) {
      if (V == 0) {
        const double2 tn = rowp[i2 + 1];
        double n0[PPT];
#pragma unroll
        for (int q = 0; q < PPT; ++q) n0[q] = fma(c2[q], b1[q], tc.x - b2[q]);
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          const double n1 = fma(c2[q], n0[q], tc.y - b1[q]);
          b2[q] = n0[q];
          b1[q] = n1;
        }
        tc = tn;
      } else if (V == 1 || V == 2) {
        double n0[PPT];
#pragma unroll
        for (int q = 0; q < PPT; ++q) n0[q] = fma(V == 2 ? cs : c2[q], b1[q], tc.x - b2[q]);
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          const double n1 = fma(V == 2 ? cs : c2[q], n0[q], tc.y - b1[q]);
          b2[q] = n0[q];
          b1[q] = n1;
        }
      } else if (V == 3) {
#pragma unroll
        for (int q = 0; q < PPT; ++q) { b1[q] = fma(c2[q], b1[q], b2[q]); }
#pragma unroll
        for (int q = 0; q < PPT; ++q) { b1[q] = fma(c2[q], b1[q], b2[q]); }
#pragma unroll
        for (int q = 0; q < PPT; ++q) { b1[q] = fma(c2[q], b1[q], b2[q]); }
#pragma unroll
        for (int q = 0; q < PPT; ++q) { b1[q] = fma(c2[q], b1[q], b2[q]); }
      } else if (V == 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < PPT; ++q) { b1[q] = fma(cs, b1[q], tc.x); }
      } else if (V == 5) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < PPT; ++q) { b1[q] = b1[q] - b2[q]; }
      } else if (V == 6) {   // independent DADD chains and DFMA chains, 1:1
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int q = 0; q < PPT; ++q) { b1[q] = b1[q] - tc.x; b2[q] = fma(b2[q], cs, tc.y); }
      } else if (V == 7) {   // DMUL only
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < PPT; ++q) { b1[q] = b1[q] * c2[q]; }
      } else if (V == 9) {   // Goertzel with the subtraction as DFMA(b2, -1, a): DFMA-only
        const double2 tn = rowp[i2 + 1];
        double n0[PPT];
#pragma unroll
        for (int q = 0; q < PPT; ++q) n0[q] = fma(c2[q], b1[q], fma(b2[q], m1, tc.x));
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          const double n1 = fma(c2[q], n0[q], fma(b1[q], m1, tc.y));
          b2[q] = n0[q];
          b1[q] = n1;
        }
        tc = tn;
      } else if (V == 10) {  // independent DADD-as-DFMA + DFMA 1:1
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int q = 0; q < PPT; ++q) { b1[q] = fma(b1[q], m1, tc.x); b2[q] = fma(b2[q], cs, tc.y); }
      } else if (V == 11) {  // independent DMUL + DFMA 1:1
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int q = 0; q < PPT; ++q) { b1[q] = b1[q] * c2[q]; b2[q] = fma(b2[q], cs, tc.y); }
      } else if (V == 21) {  // per-chain sequential source order
        const double2 tn = rowp[i2 + 1];
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          const double n0 = fma(c2[q], b1[q], tc.x - b2[q]);
          const double n1 = fma(c2[q], n0, tc.y - b1[q]);
          b2[q] = n0;
          b1[q] = n1;
        }
        tc = tn;
      } else if (V == 23) {  // multiplier in the second operand slot
        const double2 tn = rowp[i2 + 1];
        double n0[PPT];
#pragma unroll
        for (int q = 0; q < PPT; ++q) n0[q] = fma(b1[q], c2[q], tc.x - b2[q]);
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          const double n1 = fma(n0[q], c2[q], tc.y - b1[q]);
          b2[q] = n0[q];
          b1[q] = n1;
        }
        tc = tn;
      } else if (V == 24) {  // all subtractions of the pair first, then the FMAs
        const double2 tn = rowp[i2 + 1];
        double t0[PPT], n0[PPT];
#pragma unroll
        for (int q = 0; q < PPT; ++q) t0[q] = tc.x - b2[q];
#pragma unroll
        for (int q = 0; q < PPT; ++q) n0[q] = fma(c2[q], b1[q], t0[q]);
#pragma unroll
        for (int q = 0; q < PPT; ++q) t0[q] = tc.y - b1[q];
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          b1[q] = fma(c2[q], n0[q], t0[q]);
          b2[q] = n0[q];
        }
        tc = tn;
      } else if (V == 25) {  // (c2 b1 - b2) + a : DFMA on per-chain operands, DADD with the shared a
        const double2 tn = rowp[i2 + 1];
        double n0[PPT];
#pragma unroll
        for (int q = 0; q < PPT; ++q) n0[q] = fma(c2[q], b1[q], -b2[q]) + tc.x;
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
          const double n1 = fma(c2[q], n0[q], -b1[q]) + tc.y;
          b2[q] = n0[q];
          b1[q] = n1;
        }
        tc = tn;
      } else if (V == 30) {  // even/odd split: per point two chains in w = z^2 sharing c2w
        const double2 tn = rowp[i2 + 1];
        // (PPT/2 points) x (even, odd): chains 2p, 2p+1 share the multiplier c2[2p]
#pragma unroll
        for (int q = 0; q < PPT; q += 2) {
          const double ne = fma(c2[q], b1[q], tc.y - b2[q]);
          const double no = fma(c2[q], b1[q + 1], tc.x - b2[q + 1]);
          b2[q] = b1[q];
          b1[q] = ne;
          b2[q + 1] = b1[q + 1];
          b1[q + 1] = no;
        }
        tc = tn;
      } else if (V == 31) {  // residue split R = 4: per point 4 chains in w = z^4 sharing c2[p]
        // PPT chains = PPT/4 points; chain 4p + r uses coefficient T[4 j + 3 - r]
        const double2 ta = rowp[2 * (i2 & 15)], tb = rowp[2 * (i2 & 15) + 1];
#pragma unroll
        for (int p4 = 0; p4 < PPT; p4 += 4) {
          const double n0 = fma(c2[p4], b1[p4 + 0], tb.y - b2[p4 + 0]);
          const double n1 = fma(c2[p4], b1[p4 + 1], tb.x - b2[p4 + 1]);
          const double n2 = fma(c2[p4], b1[p4 + 2], ta.y - b2[p4 + 2]);
          const double n3 = fma(c2[p4], b1[p4 + 3], ta.x - b2[p4 + 3]);
          b2[p4 + 0] = b1[p4 + 0]; b1[p4 + 0] = n0;
          b2[p4 + 1] = b1[p4 + 1]; b1[p4 + 1] = n1;
          b2[p4 + 2] = b1[p4 + 2]; b1[p4 + 2] = n2;
          b2[p4 + 3] = b1[p4 + 3]; b1[p4 + 3] = n3;
        }
      } else if (V == 32) {  // block split: one point, 4 chains sharing c2[0]; coefficient
        // streams at two offsets (chains 0,2 / 1,3), two 16-byte loads per pair of steps
        const double2 ta = rowp[i2 & 31], tb = rowp[(i2 + 20) & 31];
#pragma unroll
        for (int p4 = 0; p4 < PPT; p4 += 4) {
          const double c = c2[p4];
          const double n0 = fma(c, b1[p4 + 0], ta.x - b2[p4 + 0]);
          const double n1 = fma(c, b1[p4 + 1], tb.x - b2[p4 + 1]);
          const double n2 = fma(c, b1[p4 + 2], ta.x - b2[p4 + 2]);
          const double n3 = fma(c, b1[p4 + 3], tb.x - b2[p4 + 3]);
          const double m0 = fma(c, n0, ta.y - b1[p4 + 0]);
          const double m1_ = fma(c, n1, tb.y - b1[p4 + 1]);
          const double m2 = fma(c, n2, ta.y - b1[p4 + 2]);
          const double m3 = fma(c, n3, tb.y - b1[p4 + 3]);
          b2[p4 + 0] = n0; b1[p4 + 0] = m0;
          b2[p4 + 1] = n1; b1[p4 + 1] = m1_;
          b2[p4 + 2] = n2; b1[p4 + 2] = m2;
          b2[p4 + 3] = n3; b1[p4 + 3] = m3;
        }
      } else if (V == 26) {  // (c2 b1 + a) - b2: the shared coefficient in the DFMA's addend slot
        const double2 tn = rowp[i2 + 1];
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
      } else if (V == 8) {   // independent 1 DADD : 3 DFMA
#pragma unroll
        for (int q = 0; q < PPT; ++q) { b1[q] = b1[q] - tc.x; b2[q] = fma(b2[q], cs, tc.y); c2[q] = fma(c2[q], cs, tc.x); tc.y = fma(tc.y, cs, tc.x); }
      }
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int q = 0; q < PPT; ++q) s += b1[q] + b2[q];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0) {
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    cyc[3 * blockIdx.x] = t0;
    cyc[3 * blockIdx.x + 1] = t1;
    cyc[3 * blockIdx.x + 2] = smid;
  }
}

template <int V, int PPT>
void run(const char* name, int sms, double* d, long long* dc) {
  const int iters = 400, ctas = 4;
  for (int rep = 0; rep < 2; ++rep) kern<V, PPT><<<sms * ctas, 128>>>(d, dc, iters);
  cudaDeviceSynchronize();
  const int nb = sms * ctas;
  static long long h[3 * 8192];
  cudaMemcpy(h, dc, 3 * nb * sizeof(long long), cudaMemcpyDeviceToHost);
  double span = 0;
  int nsm = 0;
  for (int sm = 0; sm < 4 * sms; ++sm) {
    long long lo = -1, hi = -1;
    int cnt = 0;
    for (int b = 0; b < nb; ++b)
      if (h[3 * b + 2] == sm) {
        if (lo < 0 || h[3 * b] < lo) lo = h[3 * b];
        if (hi < 0 || h[3 * b + 1] > hi) hi = h[3 * b + 1];
        ++cnt;
      }
    if (cnt) { span += (double)(hi - lo) * ctas / cnt; ++nsm; }
  }
  const double c = span / nsm;
  const double per_iter = (V == 30 || V == 31) ? 2.0 * PPT : 4.0 * PPT;   // DP instr per thread per i2
  const double dp = (double)iters * 40 * per_iter * 128 * ctas;
  printf("%-28s PPT=%d  %.1f DP thread-instr per SM-cycle -> %.1f%% of 64   %s\n", name, PPT, dp / c,
         100.0 * dp / c / 64.0, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* d;
  long long* dc;
  cudaMalloc(&d, 8);
  cudaMalloc(&dc, 3 * 8 * 8192);
  const int n = p.multiProcessorCount;
  run<26, 4>("B26 (c2 b1 + a) - b2", n, d, dc);
  run<26, 6>("B26 (c2 b1 + a) - b2", n, d, dc);
  run<26, 8>("B26 (c2 b1 + a) - b2", n, d, dc);
  run<0, 4>("A goertzel + LDS.128", n, d, dc);
  run<32, 4>("Q block split, 1 point", n, d, dc);
  run<32, 8>("Q block split, 2 points", n, d, dc);
  run<31, 4>("R4 residue split, 1 point", n, d, dc);
  run<31, 8>("R4 residue split, 2 points", n, d, dc);
  run<30, 4>("S even/odd shared c2w", n, d, dc);
  run<30, 8>("S even/odd shared c2w", n, d, dc);
  run<30, 6>("S even/odd shared c2w", n, d, dc);
  run<25, 4>("B25 (c2 b1 - b2) + a", n, d, dc);
  run<25, 6>("B25 (c2 b1 - b2) + a", n, d, dc);
  run<25, 8>("B25 (c2 b1 - b2) + a", n, d, dc);
  run<21, 4>("B21 per-chain order", n, d, dc);
  run<23, 4>("B23 mult in slot b", n, d, dc);
  run<24, 4>("B24 subs first", n, d, dc);
  run<21, 3>("B21 per-chain order", n, d, dc);
  run<21, 5>("B21 per-chain order", n, d, dc);
  run<23, 8>("B23 mult in slot b", n, d, dc);
  run<0, 4>("A goertzel + LDS.128", n, d, dc);
  run<9, 4>("J goertzel sub as DFMA", n, d, dc);
  run<10, 4>("K indep DFMA(-1) + DFMA 1:1", n, d, dc);
  run<11, 4>("L indep DMUL + DFMA 1:1", n, d, dc);
  run<5, 8>("F DADD 2 distinct operands", n, d, dc);
  run<6, 4>("G indep DADD + DFMA 1:1", n, d, dc);
  run<6, 8>("G indep DADD + DFMA 1:1", n, d, dc);
  run<7, 8>("H DMUL only", n, d, dc);
  run<8, 4>("I indep 1 DADD : 3 DFMA", n, d, dc);
  run<0, 4>("A goertzel + LDS.128", n, d, dc);
  run<1, 4>("B goertzel, no LDS", n, d, dc);
  run<2, 4>("C goertzel, shared mult", n, d, dc);
  run<3, 4>("D DFMA 3 distinct operands", n, d, dc);
  run<4, 4>("E DFMA shared operands", n, d, dc);
  run<5, 4>("F DADD 2 distinct operands", n, d, dc);
  run<0, 2>("A goertzel + LDS.128", n, d, dc);
  run<1, 2>("B goertzel, no LDS", n, d, dc);
  run<0, 6>("A goertzel + LDS.128", n, d, dc);
  run<1, 6>("B goertzel, no LDS", n, d, dc);
  run<3, 2>("D DFMA 3 distinct operands", n, d, dc);
  run<3, 8>("D DFMA 3 distinct operands", n, d, dc);
  return 0;
}
