// Probe: does FP64 MMA (mma.sync m8n8k4 f64, SASS DMMA) run on a pipe separate from DFMA on B200?
// Measures per-SM throughput (flops per SM clock) of a DMMA loop, a DFMA loop and the two
// interleaved in the same warps.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NM, int NF>
__global__ void loop(double* out, long long* cyc, int iters, double a, double b) {
  double acc[NM > 0 ? NM : 1][2];
  double x[NF > 0 ? NF : 1];
#pragma unroll
  for (int c = 0; c < (NM > 0 ? NM : 1); ++c) acc[c][0] = acc[c][1] = threadIdx.x * 1e-3 + c;
#pragma unroll
  for (int c = 0; c < (NF > 0 ? NF : 1); ++c) x[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < NM; ++c) dmma(acc[c][0], acc[c][1], a, b);
#pragma unroll
    for (int c = 0; c < NF; ++c) x[c] = fma(x[c], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < (NM > 0 ? NM : 1); ++c) s += acc[c][0] + acc[c][1];
#pragma unroll
  for (int c = 0; c < (NF > 0 ? NF : 1); ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NM, int NF>
void run(const char* name, int threads, int sms, double* d, long long* dc) {
  const int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) loop<NM, NF><<<sms, threads>>>(d, dc, iters, 0.999999, 1e-9);
  cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  const double warps = threads / 32;
  const double mma_flops = (double)iters * NM * warps * 512.0;       // 8x8x4 x 2 per warp instr
  const double fma_flops = (double)iters * NF * threads * 2.0;
  printf("%-12s threads=%4d  DMMA %.1f + DFMA %.1f = %.1f flop per SM-cycle (%lld cyc)\n", name, threads,
         mma_flops / c, fma_flops / c, (mma_flops + fma_flops) / c, c);
}

// dependent-chain latency: one warp per SM, a single chain of OP
template <int OP>
__global__ void lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (OP == 0) x = fma(x, a, b);
      if (OP == 1) x = x + b;
      if (OP == 2) x = x * a;
    }
  }
  long long t1 = clock64();
  if (x == 1.2345) out[0] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* d;
  long long* dc;
  cudaMalloc(&d, 8);
  cudaMalloc(&dc, 8 * 4096);
  for (int t : {256, 512, 1024}) {
    run<8, 0>("DMMA", t, p.multiProcessorCount, d, dc);
    run<0, 8>("DFMA", t, p.multiProcessorCount, d, dc);
    run<4, 8>("DMMA+DFMA", t, p.multiProcessorCount, d, dc);
    run<2, 16>("DMMA+2DFMA", t, p.multiProcessorCount, d, dc);
  }
  const char* nm[3] = {"DFMA", "DADD", "DMUL"};
  for (int op = 0; op < 3; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      if (op == 0) lat<0><<<1, 32>>>(d, dc, 1000, 0.999999, 1e-9);
      if (op == 1) lat<1><<<1, 32>>>(d, dc, 1000, 0.999999, 1e-9);
      if (op == 2) lat<2><<<1, 32>>>(d, dc, 1000, 0.999999, 1e-9);
    }
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("%s dependent-chain latency %.2f cycles\n", nm[op], c / 16000.0);
  }
  printf("%s (SM clock %d kHz)\n", cudaGetErrorString(cudaDeviceSynchronize()), p.clockRate);
}
