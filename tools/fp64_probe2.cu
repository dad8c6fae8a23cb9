// FP64 pipe probes: chain count, operand patterns, DADD/DMUL vs DFMA.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH, int MODE>
__global__ void probe(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        if (MODE == 0) x[k] = fma(x[k], a, b);
        if (MODE == 1) x[k] = fma(x[k], x[(k + 1) % CH], x[(k + 2) % CH]);
        if (MODE == 2) x[k] = x[k] * a;
        if (MODE == 3) x[k] = x[k] + a;
      }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += x[k];
  if (s == 123.456) out[0] = s;
}
template <int CH, int MODE>
void run(const char* name, int bpsm, int threads) {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d; cudaMalloc(&d, 64);
  int blocks = p.multiProcessorCount * bpsm, iters = 2048;
  for (int w = 0; w < 3; ++w) probe<CH, MODE><<<blocks, threads>>>(d, iters, 0.9999999, 1e-9);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); probe<CH, MODE><<<blocks, threads>>>(d, iters, 0.9999999, 1e-9); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double ops = 4.0 * CH * iters * (double)blocks * threads;
  printf("%-28s ch=%2d blk/SM=%d thr=%4d: %.2f Gop/s = %.1f op/clk/SM (%.2f TFLOP/s if FMA)\n", name, CH, bpsm, threads,
         ops / best * 1e-6, ops / (best * 1e-3) / p.multiProcessorCount / (clk * 1e3), 2 * ops / best * 1e-9);
  cudaFree(d);
}
int main() {
  run<8, 0>("dfma x=fma(x,a,b)", 8, 256);
  run<16, 0>("dfma x=fma(x,a,b)", 4, 256);
  run<4, 0>("dfma x=fma(x,a,b)", 8, 256);
  run<8, 0>("dfma x=fma(x,a,b)", 2, 1024);
  run<8, 1>("dfma reg operands", 8, 256);
  run<16, 1>("dfma reg operands", 4, 256);
  run<8, 2>("dmul", 8, 256);
  run<8, 3>("dadd", 8, 256);
  return 0;
}
