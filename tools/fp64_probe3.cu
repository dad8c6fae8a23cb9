// FP64 operand-pattern probes, second set: does a DFMA that reads the same
// register twice (r2 = fma(dx, dx, acc) in the sweep) or two registers plus a
// constant-bank operand issue at the reuse rate or at the three-register rate?
// And how fast is a DFMA whose third operand is a uniform register (LDCU from
// constant memory)?  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__constant__ double cvals[64];
template <int CH, int MODE>
__global__ void probe(double* out, int iters, double a) {
  double x[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        if (MODE == 0) x[k] = fma(x[(k + 1) % CH], x[(k + 1) % CH], x[k]);   // same register twice
        if (MODE == 1) x[k] = fma(x[k], x[(k + 1) % CH], a);                 // two registers + constant
        if (MODE == 2) x[k] = fma(x[k], x[(k + 1) % CH], cvals[(i + r) & 63]);  // two registers + uniform reg
        if (MODE == 3) x[k] = fma(x[k], x[(k + 1) % CH], x[(k + 2) % CH]);   // three registers
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
  for (int w = 0; w < 3; ++w) probe<CH, MODE><<<blocks, threads>>>(d, iters, 1e-9);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); probe<CH, MODE><<<blocks, threads>>>(d, iters, 1e-9); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double ops = 4.0 * CH * iters * (double)blocks * threads;
  printf("%-36s ch=%2d blk/SM=%d thr=%4d: %.1f op/clk/SM\n", name, CH, bpsm, threads,
         ops / (best * 1e-3) / p.multiProcessorCount / (clk * 1e3));
  cudaFree(d);
}
int main() {
  double h[64];
  for (int i = 0; i < 64; ++i) h[i] = 1e-9 * (i + 1);
  cudaMemcpyToSymbol(cvals, h, sizeof(h));
  run<8, 0>("dfma fma(y, y, x)", 8, 256);
  run<8, 1>("dfma fma(x, y, const)", 8, 256);
  run<8, 2>("dfma fma(x, y, uniform reg)", 8, 256);
  run<8, 3>("dfma fma(x, y, z)", 8, 256);
  return 0;
}
