// FP64 pair arithmetic of the all-pairs sweep, hand-scheduled
// for the B200 FP64 pipe.  See DESIGN.md "kernel algebra" for the derivation:
// coordinates are pre-scaled by kappa so r' = kappa*r, the physical constants
// (1/4pi, kappa^n, er, 1/er) are folded into the per-source record (the wp
// weight rides on the source normal) and two launch constants, expm1 and exp
// share one table-driven range reduction, and 1/r comes from the MUFU rsqrt
// seed plus one third-order Newton step.  43 FP64 instructions per pair
// (vs ~95 for a literal libdevice transcription of kernels.py:112-130).
#pragma once

#include <cuda_runtime.h>

#include "hobi_internal.cuh"

namespace hobi {

// 1/sqrt(x): MUFU.RSQ64H seed (rel err 2^-20, measured) refined by
// y (1 + e/2 + 3e^2/8), e = 1 - x y^2: error O(e^3) < 1e-17.
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double t = x * y;
  double e = fma(-t, y, 1.0);
  double c = fma(e, 0.375, 0.5);
  double ec = e * c;
  return fma(y, ec, y);  // y read twice: two distinct registers, full DFMA rate
}

// exp(-x) - 1 for 0 <= x < 1e12, computed as S(1+p) - 1 with S = 2^(k/2048)
// from a 2048-entry table (shared memory) and p = e^f - 1 on |f| <= ln2/4096
// (degree-3 Taylor, truncation < 4e-17).  S - 1 is exact for S in [1/2, 1]
// (Sterbenz), so small arguments keep expm1's relative accuracy.  8 FP64 ops.
// K1 = W1 (e^{-kr} - 1)/r needs that accuracy: with kr << 1 and a zero phi
// block, or eps2 ~ eps1, whole rows and the energy are K1 sums (an
// exp-only variant, E - 1 formed after rounding E, lost up to 1e-6 there;
// tests/test_gpu_parity.py::test_small_screening_keeps_expm1_accuracy).
__device__ __forceinline__ double expm1_neg(double x, const double* __restrict__ etab) {
  const double kInv = 2954.6394437405970;      // 2048/ln2
  const double kMagic = 6755399441055744.0;    // 1.5*2^52: rounds to integer in the low word
  const double kStep = 3.3845077175778578e-4;  // ln2/2048
  double kf = fma(-x, kInv, kMagic);
  int k = __double2loint(kf);
  double kd = kf - kMagic;
  double f = fma(kd, -kStep, -x);
  double p = fma(f, 1.6666666666666666e-1, 0.5);
  p = fma(p, f, 1.0);
  p = p * f;
  double T = etab[k & (kExpTable - 1)];
  int n = k >> kExpShift;
  double S = __hiloint2double(__double2hiint(T) + (n << 20), __double2loint(T));
  S = (n < -1000) ? 0.0 : S;
  return fma(S, p, S - 1.0);
}

// Screened pair (kappa > 0), scaled coordinates.  With Ap = er/k and
// Bp = (er-1)/k the source record holds
//   m' = M m with M = Ap k^3 wp/4pi (the source normal carries the wp weight),
//   W1 = -k wd/4pi, C = Ap k^2 wd/(4pi er), D = -Ap k^2 (1-1/er) wd/4pi,
// and one launch constant Bq = Bp/Ap, so M (a + Bq) = k^2 wp (a er + er - 1)/4pi
// and the K2 factor needs a DADD instead of a three-register DFMA.  With
// dny' = d.m' = M dny, u = dny'/r^2:
//   K1 wd + K2 wp = (1/r) (W1 em1 + u (a + Bq))
//   Ap (K3 wd + K4 wp) = (1/r^3) (dnx (t2 - u b) + a nn')
// where t2 = a C + D, b = 3a + kr*kre (kernels.py:119-120), nn' = n.m'; the
// sweep multiplies each stored acc2 partial by 1/Ap.
// acc1 += K1 wd + K2 wp ; acc2 += Ap (K3 wd + K4 wp)   (solver.py:333-334)
// Target normals come as (nx/nz, ny/nz) in the sweep frame (hobi_sweep.cu), so
// d.n and n.m' need no leading DMUL; the sweep scales acc2 by nz per item.
// 43 FP64 instructions per pair (24 DFMA, 12 DMUL, 7 DADD).
template <bool FULL>
__device__ __forceinline__ void pair_screened(double tx, double ty, double tz, double nx, double ny,
                                              double sx, double sy, double sz, double mx,
                                              double my, double mz, double W1, double C, double D,
                                              double Bq, const double* __restrict__ etab,
                                              double& acc1, double& acc2) {
  double dx = tx - sx, dy = ty - sy, dz = tz - sz;
  double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  double dny = fma(dx, mx, fma(dy, my, dz * mz));
  double ir = rsqrt_fast(r2);
  double r = r2 * ir;  // kappa * |x - y|
  double ir2 = ir * ir;
  double em1 = expm1_neg(r, etab);
  double kre = fma(r, em1, r);  // kr e^{-kr}
  double a = em1 + kre;         // (1+kr)e^{-kr} - 1      (kernels.py:119)
  double u = dny * ir2;
  double t = a + Bq;
  acc1 = fma(ir, fma(em1, W1, u * t), acc1);
  if (FULL) {
    double dnx = fma(dx, nx, fma(dy, ny, dz));  // d.n / n_z (sweep frame)
    double nn = fma(nx, mx, fma(ny, my, mz));   // n.m' / n_z
    double b = fma(a, 3.0, r * kre);  // kernels.py:120
    double g = fma(a, C, fma(-u, b, D));
    double X = fma(dnx, g, a * nn);
    acc2 = fma(ir, X * ir2, acc2);
  }
}

// The same arithmetic for R targets against one source, written step-major
// (each operation for all R targets before the next) so consecutive FP64
// instructions share the per-source operand in the same slot and can use the
// register reuse cache: a DFMA reading three fresh register pairs issues at
// only 2/3 of the FP64 rate on B200 (profiles/README.md).
template <int R>
__device__ __forceinline__ void pairs_screened_stepmajor(
    const double (&tx)[R], const double (&ty)[R], const double (&tz)[R], const double (&nx)[R],
    const double (&ny)[R], double sx, double sy, double sz, double mx, double my,
    double mz, double W1, double C, double D, double Bq, const double* __restrict__ etab,
    double (&acc1)[R], double (&acc2)[R]) {
  double dx[R], dy[R], dz[R], r2[R], dny[R], dnx[R], nn[R], ir[R], r[R], em1[R], a[R], kre[R];
#pragma unroll
  for (int q = 0; q < R; ++q) dx[q] = tx[q] - sx;
#pragma unroll
  for (int q = 0; q < R; ++q) dy[q] = ty[q] - sy;
#pragma unroll
  for (int q = 0; q < R; ++q) dz[q] = tz[q] - sz;
#pragma unroll
  for (int q = 0; q < R; ++q) r2[q] = fma(dx[q], dx[q], fma(dy[q], dy[q], dz[q] * dz[q]));
#pragma unroll
  for (int q = 0; q < R; ++q) dny[q] = dz[q] * mz;
#pragma unroll
  for (int q = 0; q < R; ++q) dny[q] = fma(dy[q], my, dny[q]);
#pragma unroll
  for (int q = 0; q < R; ++q) dny[q] = fma(dx[q], mx, dny[q]);
#pragma unroll
  for (int q = 0; q < R; ++q) nn[q] = fma(ny[q], my, mz);
#pragma unroll
  for (int q = 0; q < R; ++q) nn[q] = fma(nx[q], mx, nn[q]);
#pragma unroll
  for (int q = 0; q < R; ++q) dnx[q] = fma(dx[q], nx[q], fma(dy[q], ny[q], dz[q]));
#pragma unroll
  for (int q = 0; q < R; ++q) {
    ir[q] = rsqrt_fast(r2[q]);
    r[q] = r2[q] * ir[q];
  }
#pragma unroll
  for (int q = 0; q < R; ++q) em1[q] = expm1_neg(r[q], etab);
#pragma unroll
  for (int q = 0; q < R; ++q) {
    kre[q] = fma(r[q], em1[q], r[q]);
    a[q] = em1[q] + kre[q];
  }
  double ir2[R], u[R], t[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    ir2[q] = ir[q] * ir[q];
    u[q] = dny[q] * ir2[q];
  }
#pragma unroll
  for (int q = 0; q < R; ++q) t[q] = a[q] + Bq;
#pragma unroll
  for (int q = 0; q < R; ++q) t[q] = u[q] * t[q];
#pragma unroll
  for (int q = 0; q < R; ++q) t[q] = fma(em1[q], W1, t[q]);
#pragma unroll
  for (int q = 0; q < R; ++q) acc1[q] = fma(ir[q], t[q], acc1[q]);
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const double b = fma(a[q], 3.0, r[q] * kre[q]);
    t[q] = fma(-u[q], b, D);
  }
#pragma unroll
  for (int q = 0; q < R; ++q) t[q] = fma(a[q], C, t[q]);
#pragma unroll
  for (int q = 0; q < R; ++q) nn[q] = a[q] * nn[q];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const double X = fma(dnx[q], t[q], nn[q]);
    acc2[q] = fma(ir[q], X * ir2[q], acc2[q]);
  }
}

// Unscreened pair (kappa == 0): K1 = K4 = 0 exactly, as in the reference
// (expm1(0) = 0 makes a = b = 0).  Record: m' = (er-1) wp/4pi m, D = -(1-1/er) wd/4pi.
template <bool FULL>
__device__ __forceinline__ void pair_laplace(double tx, double ty, double tz, double nx, double ny,
                                             double sx, double sy, double sz, double mx,
                                             double my, double mz, double D, double& acc1,
                                             double& acc2) {
  double dx = tx - sx, dy = ty - sy, dz = tz - sz;
  double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  double dny = fma(dx, mx, fma(dy, my, dz * mz));
  double ir = rsqrt_fast(r2);
  double ir3 = (ir * ir) * ir;
  acc1 = fma(dny, ir3, acc1);
  if (FULL) {
    double dnx = fma(dx, nx, fma(dy, ny, dz));  // d.n / n_z (sweep frame)
    acc2 = fma(dnx * ir3, D, acc2);
  }
}

}  // namespace hobi
