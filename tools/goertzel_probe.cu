// Probe: FP64 pipe throughput of the integrand kernel's Goertzel loop in isolation (B200).
// 128-thread CTAs, PPT = 4 independent recurrences per thread, coefficient pairs read from a
// shared-memory row with 16-byte loads; occupancy set with dynamic shared memory.
// Reports DP thread-instructions per SM-cycle (peak 64) for CTAs/SM = 1..4 and two schedules:
//   v0: load pair i+1 while computing pair i (the kernel's source form)
//   v1: load pair i+2 (two pairs in flight)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o goertzel_probe goertzel_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int PPT = 4, K = 80, G = 10;

template <int V>
__global__ void __launch_bounds__(128, 4) loop(double* out, long long* cyc, int reps) {
  extern __shared__ __align__(16) double T[];
  for (int i = threadIdx.x; i < K + 4; i += 128) T[i] = 1.0 / (1.0 + i);
  __syncthreads();
  double c2[PPT], b1[PPT], b2[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) c2[q] = 2.0 * __cosf(0.001f * (threadIdx.x * PPT + q + 1));
  const double2* rowp = (const double2*)T;
  const int npair = K / 2;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int q = 0; q < PPT; ++q) b1[q] = b2[q] = 0.0;
    if (V == 0) {
      double2 tc = rowp[0];
      for (int gi = 0; gi < G; ++gi) {
        const int nit = (gi == G - 1) ? npair - 1 : npair;
#pragma unroll 4
        for (int i2 = 0; i2 < nit; ++i2) {
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
        }
      }
    } else {
      double2 tc = rowp[0], tn = rowp[1];
      for (int gi = 0; gi < G; ++gi) {
        const int nit = (gi == G - 1) ? npair - 1 : npair;
#pragma unroll 4
        for (int i2 = 0; i2 < nit; ++i2) {
          const double2 tnn = rowp[(i2 + 2 < npair + 1) ? i2 + 2 : 0];
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
          tn = tnn;
        }
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

template <int V>
void run(int ctas_per_sm, int sms, double* d, long long* dc) {
  const int reps = 200;
  // occupancy via shared memory: 228 KB per SM / ctas
  size_t smem = (size_t)(220 * 1024) / ctas_per_sm;
  if (smem > 200 * 1024) smem = 200 * 1024;
  cudaFuncSetAttribute(loop<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 2; ++rep) loop<V><<<sms * ctas_per_sm, 128, smem>>>(d, dc, reps);
  cudaDeviceSynchronize();
  const int nb = sms * ctas_per_sm;
  static long long h[3 * 8192];
  cudaMemcpy(h, dc, 3 * nb * sizeof(long long), cudaMemcpyDeviceToHost);
  // per SM: span = max end - min start over its CTAs (clock64 is per SM); average over SMs
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
    if (cnt) { span += (double)(hi - lo) * ctas_per_sm / cnt; ++nsm; }
  }
  const double c = span / nsm;
  const double dp = (double)reps * (G * K - 1) * 2 * PPT * 128 * ctas_per_sm;  // thread DP instr per SM
  printf("v%d ctas/SM=%d  %.1f DP thread-instr per SM-cycle (peak 64) -> %.1f%%   err=%s\n", V, ctas_per_sm,
         dp / c, 100.0 * dp / c / 64.0, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* d;
  long long* dc;
  cudaMalloc(&d, 8);
  cudaMalloc(&dc, 3 * 8 * 8192);
  for (int c = 1; c <= 4; ++c) {
    run<0>(c, p.multiProcessorCount, d, dc);
    run<1>(c, p.multiProcessorCount, d, dc);
  }
  return 0;
}
