// Dependent-issue latency of the FP64 pipe on B200: one warp runs a chain of
// dependent DFMA / DMUL / DADD (and the MUFU.RSQ64H seed) and reads clock64
// around it.  With 2 cycles of issue per warp-wide FP64 instruction, latency/2
// independent instructions per scheduler keep the pipe full -- the number the
// sweep's tiles provide through targets per thread x sources in flight x warps.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency_probe tools/fp64_latency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, int CHAINS>
__global__ void probe(double* out, long long* cycles, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) x[k] = threadIdx.x * 1e-3 + k + a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int k = 0; k < CHAINS; ++k) {
        if (MODE == 0) x[k] = fma(x[k], a, b);
        if (MODE == 1) x[k] = x[k] * a;
        if (MODE == 2) x[k] = x[k] + b;
        if (MODE == 3) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(x[k]));
      }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += x[k];
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (s == 1.2345) out[0] = s;
}

template <int MODE, int CHAINS>
void run(const char* name) {
  double* d;
  long long* c;
  cudaMalloc(&d, 64);
  cudaMalloc(&c, 64);
  const int iters = 4096;
  probe<MODE, CHAINS><<<1, 32>>>(d, c, iters, 1.0000001, 1e-9);
  probe<MODE, CHAINS><<<1, 32>>>(d, c, iters, 1.0000001, 1e-9);
  long long h = 0;
  cudaMemcpy(&h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const double per = (double)h / ((double)iters * 8 * CHAINS);
  printf("%-14s chains=%2d: %6.2f cycles per instruction per warp (%.1f cycles per round of %d)\n", name, CHAINS,
         per, per * CHAINS, CHAINS);
  cudaFree(d);
  cudaFree(c);
}

int main() {
  run<0, 1>("DFMA");
  run<0, 2>("DFMA");
  run<0, 4>("DFMA");
  run<0, 8>("DFMA");
  run<0, 12>("DFMA");
  run<0, 16>("DFMA");
  run<1, 1>("DMUL");
  run<2, 1>("DADD");
  run<3, 1>("MUFU.RSQ64H");
  run<3, 4>("MUFU.RSQ64H");
  return 0;
}
