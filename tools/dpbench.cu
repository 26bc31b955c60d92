// FP64 pipe microbenchmark (development tool): dependent-chain latency and
// throughput of DADD/DMUL/DFMA with k independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>

template <int K, int OP>
__global__ void chains(double *out, double a, double b, int iters) {
  double x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = a + threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (OP == 0) x[k] = __dadd_rn(x[k], b);
      if (OP == 1) x[k] = __dmul_rn(x[k], b);
      if (OP == 2) x[k] = __fma_rn(x[k], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int K, int OP>
void run(const char *name, int blocks, int threads) {
  double *out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  const int iters = 4096;
  chains<K, OP><<<blocks, threads>>>(out, 1.0, 1.0000001, iters);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  chains<K, OP><<<blocks, threads>>>(out, 1.0, 1.0000001, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double ops = double(blocks) * threads * K * iters;
  double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-5s K=%2d blocks=%5d thr=%4d: %8.3f ms  %7.1f Gop/s  ", name, K, blocks, threads, ms,
         ops / ms / 1e6);
  if (blocks == 1 && threads == 32)
    printf("latency ~ %.1f cycles/op (at max clock)\n", cycles / (iters * 1.0));
  else
    printf("%.2f warp-op/cycle/SM\n", ops / 32 / cycles / 148);
  cudaFree(out);
}

int main() {
  run<1, 0>("DADD", 1, 32);
  run<1, 1>("DMUL", 1, 32);
  run<1, 2>("DFMA", 1, 32);
  run<8, 2>("DFMA", 148 * 8, 256);
  run<8, 0>("DADD", 148 * 8, 256);
  run<4, 2>("DFMA", 148 * 4, 128);
  run<8, 2>("DFMA", 148 * 2, 128);
  run<8, 2>("DFMA", 148 * 4, 64);
  return 0;
}
