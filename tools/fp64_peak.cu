// FP64 pipe microbenchmark for B200 (sm_100a): DFMA throughput, DADD throughput,
// and the cost of sincospi/sincos per call. Used to derive the roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>
#include <cmath>

template <int CH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}

__global__ void goertzel_loop(double* out, int iters, double c2) {
  double b1 = threadIdx.x * 1e-3, b2 = 0.5, d1 = 0.25, d2 = 0.125, e1 = 0.3, e2 = 0.1, g1 = 0.2, g2 = 0.7;
  for (int i = 0; i < iters; ++i) {
    double a = 1e-3 * i;
    double t = fma(c2, b1, a - b2); b2 = b1; b1 = t;
    t = fma(c2, d1, a - d2); d2 = d1; d1 = t;
    t = fma(c2, e1, a - e2); e2 = e1; e1 = t;
    t = fma(c2, g1, a - g2); g2 = g1; g1 = t;
  }
  double s = b1 + d1 + e1 + g1;
  if (s == 1.2345) out[0] = s;
}

__global__ void sincospi_loop(double* out, int iters, double x0) {
  double acc = 0, x = x0 + threadIdx.x * 1e-7;
  for (int i = 0; i < iters; ++i) {
    double s, c;
    sincospi(x, &s, &c);
    acc += s * c;
    x += 1.37e3;
  }
  if (acc == 1.2345) out[0] = acc;
}
__global__ void sincos_loop(double* out, int iters, double x0) {
  double acc = 0, x = x0 + threadIdx.x * 1e-7;
  for (int i = 0; i < iters; ++i) {
    double s, c;
    sincos(x, &s, &c);
    acc += s * c;
    x += 1.37e3;
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s sms %d clock %d kHz\n", p.name, sms, clk_khz);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int threads = 512, blocks = sms * 4; int iters = 20000;
  for (int rep = 0; rep < 3; ++rep) {
    dfma_loop<8><<<blocks, threads>>>(d, iters, 0.999999, 1e-9);
    cudaEventRecord(e0);
    dfma_loop<8><<<blocks, threads>>>(d, iters, 0.999999, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)threads * blocks;
    printf("DFMA: %.3f ms  %.2f TFLOP/s  (%.1f DFMA/clk/SM at %d MHz)\n", ms, flops / ms * 1e-9,
           flops / 2 / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1000);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    goertzel_loop<<<blocks, threads>>>(d, iters, 1.7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double dinstr = 2.0 * 4 * iters * (double)threads * blocks + 1.0 * iters * threads * blocks;
    printf("goertzel: %.3f ms  %.2f G DP-thread-instr/s per SM-clk: %.1f\n", ms, dinstr / ms * 1e-6,
           dinstr / (ms * 1e-3) / sms / (clk_khz * 1e3));
  }
  for (int rep = 0; rep < 2; ++rep) {
    int it2 = 2000;
    cudaEventRecord(e0);
    sincospi_loop<<<blocks, threads>>>(d, it2, 0.3);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double calls = (double)it2 * threads * blocks;
    printf("sincospi: %.3f ms  %.3f Gcalls/s -> %.1f DFMA-equiv per call\n", ms, calls / ms * 1e-6,
           (64.0 * sms * clk_khz * 1e3) / (calls / (ms * 1e-3)));
    cudaEventRecord(e0);
    sincos_loop<<<blocks, threads>>>(d, it2, 0.3);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("sincos:   %.3f ms  %.3f Gcalls/s -> %.1f DFMA-equiv per call\n", ms, calls / ms * 1e-6,
           (64.0 * sms * clk_khz * 1e3) / (calls / (ms * 1e-3)));
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
