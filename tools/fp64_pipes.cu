// FP64 pipe model on B200: per-SM throughput of DFMA, DADD, DMUL and a DADD+DFMA mix, measured in
// SM clock cycles (clock64) so the result does not depend on the DVFS clock.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP, int CH>
__global__ void pipe_loop(double* out, long long* cyc, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) x[c] = fma(x[c], a, b);
      if (OP == 1) x[c] = x[c] + b;
      if (OP == 2) x[c] = x[c] * a;
      if (OP == 3) { x[c] = x[c] + b; x[c] = fma(x[c], a, b); }   // mix: DADD then DFMA
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int threads, int blocks_per_sm, int sms, double* d, long long* dc) {
  const int iters = 4000, CH = 8;
  pipe_loop<OP, CH><<<sms * blocks_per_sm, threads>>>(d, dc, iters, 0.999999, 1e-9);
  cudaDeviceSynchronize();
  pipe_loop<OP, CH><<<sms * blocks_per_sm, threads>>>(d, dc, iters, 0.999999, 1e-9);
  cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  double ops = (double)iters * CH * (OP == 3 ? 2 : 1) * threads * blocks_per_sm;  // per SM
  printf("%-8s threads=%4d blk/SM=%d  %.1f DP thread-instr per SM-cycle\n", name, threads, blocks_per_sm, ops / c);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* d; long long* dc;
  cudaMalloc(&d, 8); cudaMalloc(&dc, 8 * 4096);
  for (int w : {256, 512, 1024}) {
    run<0>("DFMA", w, 1, p.multiProcessorCount, d, dc);
    run<1>("DADD", w, 1, p.multiProcessorCount, d, dc);
    run<2>("DMUL", w, 1, p.multiProcessorCount, d, dc);
    run<3>("ADD+FMA", w, 1, p.multiProcessorCount, d, dc);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
