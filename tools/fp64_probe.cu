// FP64 microprobes for B200 (sm_100a): DFMA peak, rsqrt.approx.f64 seed accuracy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_peak(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 123.456) out[0] = s;
}

__device__ __forceinline__ double rsqrt_seed(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

__global__ void rsqrt_err(const double* x, double* err, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = x[i];
  double y = rsqrt_seed(v);
  double ref = 1.0 / sqrt(v);
  err[i] = fabs(y - ref) / ref;
}

__global__ void rsqrt_tp(double* out, int iters) {
  double x0 = 1.0 + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; ++i) {
    x0 = rsqrt_seed(x0) + 1.0; x1 = rsqrt_seed(x1) + 1.0; x2 = rsqrt_seed(x2) + 1.0; x3 = rsqrt_seed(x3) + 1.0;
  }
  double s = x0 + x1 + x2 + x3;
  if (s == 123.456) out[0] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d cc %d.%d clockRate %d kHz\n", p.name, p.multiProcessorCount, p.major, p.minor, clk);
  double* d; CK(cudaMalloc(&d, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int bpsm : {4, 8}) {
    int blocks = p.multiProcessorCount * bpsm, threads = 256;
    for (int w = 0; w < 3; ++w) dfma_peak<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0); dfma_peak<<<blocks, threads>>>(d, iters, 0.999999, 1e-7); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 32.0 * iters * (double)blocks * threads;
    printf("dfma blocks/SM %d: %.3f ms  %.2f TFLOP/s  (%.1f DFMA/clk/SM @ clockRate)\n", bpsm, best, flops / best * 1e-9,
           flops / 2 / (best * 1e-3) / p.multiProcessorCount / (clk * 1e3));
  }
  // sustained 3 s
  {
    int blocks = p.multiProcessorCount * 8, threads = 256;
    cudaEventRecord(e0);
    int n = 0; float ms = 0;
    while (ms < 3000) { dfma_peak<<<blocks, threads>>>(d, iters, 0.999999, 1e-7); ++n; if (n % 20 == 0) { cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);} }
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 32.0 * iters * (double)blocks * threads * n;
    printf("dfma sustained %.0f ms: %.2f TFLOP/s\n", ms, flops / ms * 1e-9);
  }
  // rsqrt seed accuracy
  const int n = 1 << 22;
  double* hx = new double[n];
  for (int i = 0; i < n; ++i) hx[i] = pow(10.0, -8.0 + 16.0 * (i + 0.5) / n) * (1.0 + 0.37 * ((i * 7919LL) % 1000) / 1000.0);
  double *dx, *de; CK(cudaMalloc(&dx, n * 8)); CK(cudaMalloc(&de, n * 8));
  CK(cudaMemcpy(dx, hx, n * 8, cudaMemcpyHostToDevice));
  rsqrt_err<<<(n + 255) / 256, 256>>>(dx, de, n);
  CK(cudaMemcpy(hx, de, n * 8, cudaMemcpyDeviceToHost));
  double mx = 0; for (int i = 0; i < n; ++i) mx = fmax(mx, hx[i]);
  printf("rsqrt.approx.ftz.f64 max rel err %.3e (2^%.1f)\n", mx, log2(mx));
  {
    int blocks = p.multiProcessorCount * 8, threads = 256; int it = 4096;
    rsqrt_tp<<<blocks, threads>>>(d, it); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); rsqrt_tp<<<blocks, threads>>>(d, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 4.0 * it * blocks * threads;
    printf("rsqrt seed: %.2f Gop/s = %.1f /clk/SM\n", ops / ms * 1e-6, ops / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3));
  }
  return 0;
}
