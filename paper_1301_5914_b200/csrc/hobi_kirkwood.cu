// Analytic Kirkwood validator on the device: the
// multipole sums of the reference's kirkwood_series (kirkwood.py:159-220)
// at every evaluation point, and its charge-charge energy sum.
//
// The host (kirkwood.py) computes the O(N_c x n_terms) coefficients -- the
// Bessel log-derivative recurrence, alpha, the reaction coefficients A, and
// the trace rows coef_phi / coef_dphi -- exactly as the reference does; the
// O(N_points x N_c x n_terms) Legendre sums run here.  Compiled with
// -fmad=false: the recurrence is written as the reference writes it
// (kirkwood.py:59-71, ((2n+1) x P_n - n P_{n-1}) / (n+1)), so each P_n
// rounds like numpy's.
#include <algorithm>

#include "hobi_internal.cuh"

namespace hobi {
namespace {

constexpr int kKwThreads = 128;
constexpr int kKwTile = 32;  // charges staged in shared memory per pass

// Sum over n of c[n] P_n(x), n = 0..nmax, recurrence as legendre_all
// (kirkwood.py:59-71), accumulated in n order like `coef[k] @ pn`.
__device__ __forceinline__ void legendre_dot2(double x, int nmax, const double* __restrict__ c1,
                                              const double* __restrict__ c2, double& s1, double& s2) {
  double pm = 1.0, p = x;  // P_0, P_1
  s1 = c1[0];
  s2 = c2[0];
  if (nmax < 1) return;
  s1 += c1[1] * p;
  s2 += c2[1] * p;
  for (int n = 1; n < nmax; ++n) {
    const double pn = ((2 * n + 1) * x * p - n * pm) / (n + 1);
    pm = p;
    p = pn;
    s1 += c1[n + 1] * p;
    s2 += c2[n + 1] * p;
  }
}

// phi and dphi/dn traces at m points (kirkwood.py:193-203): for each charge k,
// cos = rad . u_k (1 for a charge at the centre), then coef[k] . P(cos);
// charges accumulate in index order.
__global__ void __launch_bounds__(kKwThreads) kirkwood_trace_kernel(
    const double* __restrict__ pts, int64_t m, const double* __restrict__ units,
    const double* __restrict__ rho, int64_t nc, const double* __restrict__ coef_phi,
    const double* __restrict__ coef_dphi, int nterms, double* __restrict__ phi, double* __restrict__ dphi) {
  extern __shared__ double sm[];
  double* su = sm;                         // [kKwTile][4]: unit vector, rho
  double* sc1 = sm + 4 * kKwTile;          // [kKwTile][nterms]
  double* sc2 = sc1 + kKwTile * nterms;    // [kKwTile][nterms]
  const int64_t i = blockIdx.x * (int64_t)kKwThreads + threadIdx.x;
  const int64_t ii = i < m ? i : m - 1;
  const double x0 = pts[3 * ii], x1 = pts[3 * ii + 1], x2 = pts[3 * ii + 2];
  // radial direction = p / ||p||  (_directions: np.linalg.norm along axis 1
  // is sqrt of an unfused left-to-right sum of squares, then a division)
  const double r = sqrt(x0 * x0 + x1 * x1 + x2 * x2);
  const double r0 = x0 / r, r1 = x1 / r, r2 = x2 / r;
  double o1 = 0.0, o2 = 0.0;
  for (int64_t k0 = 0; k0 < nc; k0 += kKwTile) {
    const int kn = (int)(nc - k0 < kKwTile ? nc - k0 : kKwTile);
    __syncthreads();
    for (int t = threadIdx.x; t < kn * 4; t += kKwThreads) {
      const int k = t / 4, c = t % 4;
      su[t] = c < 3 ? units[3 * (k0 + k) + c] : rho[k0 + k];
    }
    for (int t = threadIdx.x; t < kn * nterms; t += kKwThreads) {
      sc1[t] = coef_phi[k0 * nterms + t];
      sc2[t] = coef_dphi[k0 * nterms + t];
    }
    __syncthreads();
    for (int k = 0; k < kn; ++k) {
      const double* u = su + 4 * k;
      // rad @ units.T is a BLAS dot: fma(z, z', fma(y, y', x*x'))
      const double cs = u[3] > 0.0 ? fma(r2, u[2], fma(r1, u[1], r0 * u[0])) : 1.0;
      double s1, s2;
      legendre_dot2(cs, nterms - 1, sc1 + k * nterms, sc2 + k * nterms, s1, s2);
      o1 += s1;
      o2 += s2;
    }
  }
  if (i < m) {
    phi[i] = o1;
    dphi[i] = o2;
  }
}

// Per-charge energy terms (kirkwood.py:180-188): e_j = 1/2 q_j sum_k sum_n
// A[k,n] rho_j^n P_n(u_k . u_j); the host folds the e_j in charge order.
__global__ void kirkwood_energy_kernel(const double* __restrict__ units, const double* __restrict__ q,
                                       int64_t nc, const double* __restrict__ reac,
                                       const double* __restrict__ rpow, int nterms,
                                       double* __restrict__ ej) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nc) return;
  const double uj0 = units[3 * j], uj1 = units[3 * j + 1], uj2 = units[3 * j + 2];
  const double* rj = rpow + j * nterms;
  double s = 0.0;
  for (int64_t k = 0; k < nc; ++k) {
    const double cs = fma(units[3 * k + 2], uj2, fma(units[3 * k + 1], uj1, units[3 * k] * uj0));
    const double* a = reac + k * nterms;
    double pm = 1.0, p = cs;
    s += a[0] * rj[0] * pm;
    if (nterms > 1) s += a[1] * rj[1] * p;
    for (int n = 1; n + 1 < nterms; ++n) {
      const double pn = ((2 * n + 1) * cs * p - n * pm) / (n + 1);
      pm = p;
      p = pn;
      s += a[n + 1] * rj[n + 1] * p;
    }
  }
  ej[j] = 0.5 * q[j] * s;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace
}  // namespace hobi

using namespace hobi;

extern "C" {

int hobi_kirkwood_traces(int device, const double* points, int64_t m, const double* units, const double* rho,
                         int64_t nc, const double* coef_phi, const double* coef_dphi, int nterms, double* phi,
                         double* dphi) {
  NvtxRange nvtx_("hobi_kirkwood_traces");
  if (m < 0 || nc < 0) return fail(HOBI_ERR_VALUE, "negative sizes");
  if (nterms < 1 || nterms > 256) return fail(HOBI_ERR_VALUE, "n_terms must be in 1..256");
  if (m == 0) return 0;
  HOBI_CUDA(cudaSetDevice(device));
  cudaStream_t s;
  HOBI_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  DevBuf<double> dp, du, dr, c1, c2, o;
  int rc = 0;
  const size_t ncs = (size_t)std::max<int64_t>(nc, 1);
  if (dp.alloc(3 * m) || du.alloc(3 * ncs) || dr.alloc(ncs) || c1.alloc(ncs * nterms) ||
      c2.alloc(ncs * nterms) || o.alloc(2 * m))
    rc = HOBI_ERR_CUDA;
  const size_t smem = (4 + 2 * (size_t)nterms) * kKwTile * sizeof(double);
  cudaError_t e = cudaSuccess;
  if (!rc) {
    e = cudaMemcpyAsync(dp.p, points, 3 * m * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && nc)
      e = cudaMemcpyAsync(du.p, units, 3 * nc * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && nc) e = cudaMemcpyAsync(dr.p, rho, nc * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && nc)
      e = cudaMemcpyAsync(c1.p, coef_phi, nc * nterms * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && nc)
      e = cudaMemcpyAsync(c2.p, coef_dphi, nc * nterms * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && smem > 48 * 1024)
      e = cudaFuncSetAttribute(kirkwood_trace_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) {
      kirkwood_trace_kernel<<<nblk(m, kKwThreads), kKwThreads, smem, s>>>(dp.p, m, du.p, dr.p, nc, c1.p, c2.p,
                                                                         nterms, o.p, o.p + m);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(phi, o.p, m * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dphi, o.p + m, m * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(e, "kirkwood traces");
  }
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return rc;
}

int hobi_kirkwood_energy_terms(int device, const double* units, const double* q, int64_t nc, const double* reac,
                               const double* rpow, int nterms, double* terms) {
  NvtxRange nvtx_("hobi_kirkwood_energy_terms");
  if (nc < 0) return fail(HOBI_ERR_VALUE, "negative sizes");
  if (nterms < 1 || nterms > 256) return fail(HOBI_ERR_VALUE, "n_terms must be in 1..256");
  if (nc == 0) return 0;
  HOBI_CUDA(cudaSetDevice(device));
  cudaStream_t s;
  HOBI_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  DevBuf<double> du, dq, da, dr, o;
  int rc = 0;
  if (du.alloc(3 * nc) || dq.alloc(nc) || da.alloc(nc * nterms) || dr.alloc(nc * nterms) || o.alloc(nc))
    rc = HOBI_ERR_CUDA;
  cudaError_t e = cudaSuccess;
  if (!rc) {
    e = cudaMemcpyAsync(du.p, units, 3 * nc * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dq.p, q, nc * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(da.p, reac, nc * nterms * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(dr.p, rpow, nc * nterms * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
      kirkwood_energy_kernel<<<nblk(nc, 128), 128, 0, s>>>(du.p, dq.p, nc, da.p, dr.p, nterms, o.p);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(terms, o.p, nc * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(e, "kirkwood energy");
  }
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return rc;
}

}  // extern "C"
