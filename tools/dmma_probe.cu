// FP64 tensor-core (DMMA m8n8k4) throughput on B200 and overlap with DFMA.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void probe(double* out, int iters, double a, double b) {
  double c[8], x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { c[k] = threadIdx.x + k; x[k] = threadIdx.x * 1e-3 + k; }
  double av = a + threadIdx.x * 1e-9, bv = b + threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (MODE == 0 || MODE == 2) dmma(c[2 * k], c[2 * k + 1], av, bv);
      if (MODE == 1 || MODE == 2) {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = fma(x[q], a, b);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k] + x[k];
  if (s == 123.456) out[0] = s;
}
template <int MODE> void run(const char* name) {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d; cudaMalloc(&d, 64);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 1024;
  for (int w = 0; w < 3; ++w) probe<MODE><<<blocks, threads>>>(d, iters, 0.9999999, 1e-9);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); probe<MODE><<<blocks, threads>>>(d, iters, 0.9999999, 1e-9); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  double warps = (double)blocks * threads / 32;
  double dmma_flops = (MODE == 1) ? 0 : 4.0 * iters * warps * 2 * 8 * 8 * 4;
  double dfma_flops = (MODE == 0) ? 0 : 4.0 * iters * 8 * 2 * (double)blocks * threads;
  printf("%-22s %.3f ms  DMMA %.2f TF/s  DFMA %.2f TF/s  total %.2f\n", name, best, dmma_flops / best * 1e-9,
         dfma_flops / best * 1e-9, (dmma_flops + dfma_flops) / best * 1e-9);
}
int main() {
  run<0>("DMMA only");
  run<1>("DFMA only");
  run<2>("DMMA + DFMA mixed");
  return 0;
}
