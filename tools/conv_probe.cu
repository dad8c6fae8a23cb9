// Throughput of FP64 conversions and whether they contend with DFMA.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void probe(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  int k0 = threadIdx.x, k1 = k0 + 1, k2 = k0 + 2, k3 = k0 + 3;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (MODE == 0) { acc += (double)k0; acc += (double)k1; acc += (double)k2; acc += (double)k3; k0 += 3; k1 += 5; k2 += 7; k3 += 9; }
      if (MODE == 1) { k0 += __double2int_rn(x0); k1 += __double2int_rn(x1); k2 += __double2int_rn(x2); k3 += __double2int_rn(x3); x0 += 1e-9; x1 += 1e-9; x2 += 1e-9; x3 += 1e-9; }
      if (MODE == 2) { x0 = fma(x0, a, (double)k0); x1 = fma(x1, a, (double)k1); x2 = fma(x2, a, (double)k2); x3 = fma(x3, a, (double)k3); k0++; k1++; k2++; k3++; }
      if (MODE == 3) { x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b); k0++; k1++; k2++; k3++; }
      if (MODE == 4) { float f0 = __double2float_rn(x0), f1 = __double2float_rn(x1), f2 = __double2float_rn(x2), f3 = __double2float_rn(x3); k0 += __float_as_int(f0); k1 += __float_as_int(f1); k2 += __float_as_int(f2); k3 += __float_as_int(f3); x0 += 1e-9; x1 += 1e-9; x2 += 1e-9; x3 += 1e-9; }
    }
  }
  double s = x0 + x1 + x2 + x3 + acc + k0 + k1 + k2 + k3;
  if (s == 123.456) out[0] = s;
}
template <int MODE> void run(const char* name, double per_iter_ops) {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d; cudaMalloc(&d, 64);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 2048;
  for (int w = 0; w < 3; ++w) probe<MODE><<<blocks, threads>>>(d, iters, 0.9999999, 1e-9);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); probe<MODE><<<blocks, threads>>>(d, iters, 0.9999999, 1e-9); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  double n = per_iter_ops * 4.0 * iters * (double)blocks * threads;
  printf("%-40s %.3f ms  %.1f op/clk/SM\n", name, best, n / (best * 1e-3) / p.multiProcessorCount / (clk * 1e3));
}
int main() {
  run<0>("I2F.F64 + DADD (4 each)", 4);
  run<1>("F2I (double2int) + DADD", 4);
  run<2>("DFMA with I2F.F64 operand", 4);
  run<3>("DFMA plain (same loop shape)", 4);
  run<4>("F2F.F32.F64 + DADD", 4);
  return 0;
}
