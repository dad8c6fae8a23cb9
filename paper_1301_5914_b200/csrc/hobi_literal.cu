// Low-volume kernels written as literal transcriptions of the reference
// arithmetic (compiled with -fmad=false, libdevice exp/expm1/sqrt, IEEE
// division): the charge source terms (K-E), the kernel-value test hook and
// the literal forms of the Duffy singular swap --
// HOBI_SINGULAR=warp|serial, the check the default singular_fast_kernel
// (hobi_singular.cu) is tested against.  These touch O(N) pairs, so fidelity to
// kernels.py beats instruction count here.
#include <cstdlib>
#include <cstring>

#include "hobi_internal.cuh"

namespace hobi {

namespace {

struct K4 {
  double k1, k2, k3, k4;
};

// kernel_values_d, kernels.py:99-130, operation for operation.
__device__ __forceinline__ K4 kernel_values_d(double dx, double dy, double dz, double nxx, double nxy,
                                              double nxz, double nyx, double nyy, double nyz,
                                              double er, double kappa) {
  double r2 = dx * dx + dy * dy + dz * dz;
  double r = sqrt(r2);
  double kr = kappa * r;
  double ekr = exp(-kr);
  double em1 = expm1(-kr);
  double a = em1 + kr * ekr;
  double b = 3.0 * em1 + kr * ekr * (3.0 + kr);
  double dny = dx * nyx + dy * nyy + dz * nyz;
  double dnx = dx * nxx + dy * nxy + dz * nxz;
  double nxny = nxx * nyx + nxy * nyy + nxz * nyz;
  double inv_r3 = 1.0 / (kFourPi * r2 * r);
  K4 k;
  k.k1 = -em1 / (kFourPi * r);
  k.k2 = dny * inv_r3 * ((er - 1.0) + er * a);
  k.k3 = -dnx * inv_r3 * ((1.0 - 1.0 / er) - a / er);
  k.k4 = (-b * dnx * dny / r2 + a * nxny) * inv_r3;
  return k;
}

__global__ void kernel_values_kernel(const double* __restrict__ d, const double* __restrict__ nx,
                                     const double* __restrict__ ny, int64_t n, double er,
                                     double kappa, double* __restrict__ k) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  K4 v = kernel_values_d(d[3 * i], d[3 * i + 1], d[3 * i + 2], nx[3 * i], nx[3 * i + 1], nx[3 * i + 2],
                         ny[3 * i], ny[3 * i + 1], ny[3 * i + 2], er, kappa);
  k[i] = v.k1;
  k[n + i] = v.k2;
  k[2 * n + i] = v.k3;
  k[3 * n + i] = v.k4;
}

__device__ __forceinline__ double interp3(const double* __restrict__ u, int i0, int i1, int i2,
                                          const double* __restrict__ b) {
  return u[i0] * b[0] + u[i1] * b[1] + u[i2] * b[2];  // _interp, solver.py:269-275
}

// One incident pair p: Duffy sum on the rotated element minus the regular-rule
// sum on the rotation-0 element (solver.py:336-361).
__global__ void singular_kernel(int64_t p0, int64_t p1, const int* __restrict__ pair_vertex,
                                const int* __restrict__ pair_face, const int* __restrict__ pair_gverts,
                                const int* __restrict__ faces, const double* __restrict__ vert,
                                const double* __restrict__ vnrm, const double* __restrict__ reg_pos,
                                const double* __restrict__ reg_nrm, const double* __restrict__ reg_w,
                                const double* __restrict__ reg_bary, int nq,
                                const double* __restrict__ duf_pos, const double* __restrict__ duf_nrm,
                                const double* __restrict__ duf_w, const double* __restrict__ duf_bary,
                                int nd, const double* __restrict__ u, int64_t nt, double er,
                                double kappa, double* __restrict__ corr) {
  int64_t p = p0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= p1) return;
  const int v = pair_vertex[p], f = pair_face[p];
  const double x0 = vert[3 * v], x1 = vert[3 * v + 1], x2 = vert[3 * v + 2];
  const double n0 = vnrm[3 * v], n1 = vnrm[3 * v + 1], n2 = vnrm[3 * v + 2];
  const double* dphi = u + nt;
  const int fa = faces[3 * f], fb = faces[3 * f + 1], fc = faces[3 * f + 2];
  double reg1, reg2;
  numpy_row_sum(nq, [&](int m, double& t1, double& t2) {
    const double* y = reg_pos + ((int64_t)f * nq + m) * 3;
    const double* ny = reg_nrm + ((int64_t)f * nq + m) * 3;
    K4 k = kernel_values_d(x0 - y[0], x1 - y[1], x2 - y[2], n0, n1, n2, ny[0], ny[1], ny[2], er, kappa);
    double w = reg_w[(int64_t)f * nq + m];
    double wp = w * interp3(u, fa, fb, fc, reg_bary + 3 * m);
    double wd = w * interp3(dphi, fa, fb, fc, reg_bary + 3 * m);
    t1 = k.k1 * wd + k.k2 * wp;
    t2 = k.k3 * wd + k.k4 * wp;
  }, reg1, reg2);
  const int ga = pair_gverts[3 * p], gb = pair_gverts[3 * p + 1], gc = pair_gverts[3 * p + 2];
  double duf1, duf2;
  numpy_row_sum(nd, [&](int m, double& t1, double& t2) {
    const double* y = duf_pos + (p * nd + m) * 3;
    const double* ny = duf_nrm + (p * nd + m) * 3;
    K4 k = kernel_values_d(x0 - y[0], x1 - y[1], x2 - y[2], n0, n1, n2, ny[0], ny[1], ny[2], er, kappa);
    double w = duf_w[p * nd + m];
    double wp = w * interp3(u, ga, gb, gc, duf_bary + 3 * m);
    double wd = w * interp3(dphi, ga, gb, gc, duf_bary + 3 * m);
    t1 = k.k1 * wd + k.k2 * wp;
    t2 = k.k3 * wd + k.k4 * wp;
  }, duf1, duf2);
  corr[2 * p] = duf1 - reg1;
  corr[2 * p + 1] = duf2 - reg2;
}

// The same correction with one warp per pair: lane m evaluates term m of the
// pair's nq regular + nd Duffy points (looping when nq + nd > 32), the terms
// land in shared memory, and lanes 0 and 1 sum the regular and the Duffy row
// in numpy's order (numpy_row_sum) -- the identical operations in the
// identical order as singular_kernel, so the output is bitwise the same, with
// 20 evaluations in parallel instead of in series (HOBI_SINGULAR=serial
// selects the serial kernel, for the bitwise regression test).
constexpr int kSingWarps = 4;          // pairs per 128-thread block
constexpr int kSingMaxTerms = 16 + 64;  // nq <= 16, nd <= 64 (hobi_create)

__global__ void __launch_bounds__(32 * kSingWarps) singular_warp_kernel(
    int64_t p0, int64_t p1, const int* __restrict__ pair_vertex, const int* __restrict__ pair_face,
    const int* __restrict__ pair_gverts, const int* __restrict__ faces, const double* __restrict__ vert,
    const double* __restrict__ vnrm, const double* __restrict__ reg_pos, const double* __restrict__ reg_nrm,
    const double* __restrict__ reg_w, const double* __restrict__ reg_bary, int nq,
    const double* __restrict__ duf_pos, const double* __restrict__ duf_nrm, const double* __restrict__ duf_w,
    const double* __restrict__ duf_bary, int nd, const double* __restrict__ u, int64_t nt, double er,
    double kappa, double* __restrict__ corr) {
  __shared__ double t1s[kSingWarps][kSingMaxTerms], t2s[kSingWarps][kSingMaxTerms];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = p0 + (int64_t)blockIdx.x * kSingWarps + warp;
  if (p >= p1) return;  // the whole warp leaves together
  const int v = pair_vertex[p], f = pair_face[p];
  const double x0 = vert[3 * v], x1 = vert[3 * v + 1], x2 = vert[3 * v + 2];
  const double n0 = vnrm[3 * v], n1 = vnrm[3 * v + 1], n2 = vnrm[3 * v + 2];
  const double* dphi = u + nt;
  const int nterm = nq + nd;
  for (int m = lane; m < nterm; m += 32) {
    const double *y, *ny, *bary;
    double w;
    int ia, ib, ic;
    if (m < nq) {  // regular point m of the rotation-0 element
      const int64_t q = (int64_t)f * nq + m;
      y = reg_pos + q * 3;
      ny = reg_nrm + q * 3;
      w = reg_w[q];
      ia = faces[3 * f];
      ib = faces[3 * f + 1];
      ic = faces[3 * f + 2];
      bary = reg_bary + 3 * m;
    } else {  // Duffy point m - nq of the rotated element
      const int mm = m - nq;
      const int64_t q = p * nd + mm;
      y = duf_pos + q * 3;
      ny = duf_nrm + q * 3;
      w = duf_w[q];
      ia = pair_gverts[3 * p];
      ib = pair_gverts[3 * p + 1];
      ic = pair_gverts[3 * p + 2];
      bary = duf_bary + 3 * mm;
    }
    K4 k = kernel_values_d(x0 - y[0], x1 - y[1], x2 - y[2], n0, n1, n2, ny[0], ny[1], ny[2], er, kappa);
    double wp = w * interp3(u, ia, ib, ic, bary);
    double wd = w * interp3(dphi, ia, ib, ic, bary);
    t1s[warp][m] = k.k1 * wd + k.k2 * wp;
    t2s[warp][m] = k.k3 * wd + k.k4 * wp;
  }
  __syncwarp();
  double s1 = 0.0, s2 = 0.0;
  if (lane < 2) {
    const int off = lane == 0 ? 0 : nq, n = lane == 0 ? nq : nd;
    const double* a1 = &t1s[warp][off];
    const double* a2 = &t2s[warp][off];
    numpy_row_sum(n, [&](int m, double& t1, double& t2) {
      t1 = a1[m];
      t2 = a2[m];
    }, s1, s2);
  }
  const double duf1 = __shfl_sync(0xffffffffu, s1, 1), duf2 = __shfl_sync(0xffffffffu, s2, 1);
  if (lane == 0) {
    corr[2 * p] = duf1 - s1;
    corr[2 * p + 1] = duf2 - s2;
  }
}

// source_terms_at (kernels.py:159-178) + /eps1 (solver.py:402); one thread per
// collocation point, charges staged through shared memory.
__global__ void rhs_kernel(const double* __restrict__ pos, const double* __restrict__ nrm, int64_t lo,
                           int64_t nt, const double* __restrict__ qpos, const double* __restrict__ q,
                           int64_t nc, double eps1, double* __restrict__ o1, double* __restrict__ o2,
                           unsigned long long* __restrict__ bad) {
  __shared__ double sq[4][256];
  int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // rows [lo, nt) of this launch
  const int64_t ii = i < nt ? i : nt - 1;
  const double x0 = pos[3 * ii], x1 = pos[3 * ii + 1], x2 = pos[3 * ii + 2];
  const double m0 = nrm[3 * ii], m1 = nrm[3 * ii + 1], m2 = nrm[3 * ii + 2];
  double s1 = 0.0, s2 = 0.0;
  for (int64_t k0 = 0; k0 < nc; k0 += 256) {
    __syncthreads();
    int64_t k = k0 + threadIdx.x;
    if (threadIdx.x < 256 && k < nc) {
      sq[0][threadIdx.x] = qpos[3 * k];
      sq[1][threadIdx.x] = qpos[3 * k + 1];
      sq[2][threadIdx.x] = qpos[3 * k + 2];
      sq[3][threadIdx.x] = q[k];
    }
    __syncthreads();
    const int kn = (int)((nc - k0) < 256 ? (nc - k0) : 256);
    for (int j = 0; j < kn; ++j) {
      double d0 = x0 - sq[0][j], d1 = x1 - sq[1][j], d2 = x2 - sq[2][j];
      double r2 = d0 * d0 + d1 * d1 + d2 * d2;
      if (r2 < 1e-300 && i < nt)
        atomicMin(bad, (unsigned long long)i * (unsigned long long)(nc + 1) + (unsigned long long)(k0 + j));
      double r = sqrt(r2);
      double qk = sq[3][j];
      s1 += qk / (kFourPi * r);
      double dnx = d0 * m0 + d1 * m1 + d2 * m2;
      s2 += -qk * dnx / (kFourPi * r2 * r);
    }
  }
  if (i < nt) {
    o1[i - lo] = s1 / eps1;
    o2[i - lo] = s2 / eps1;
  }
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

int launch_singular(hobi_ctx* c, const double* u_dev, int64_t p0, int64_t p1, cudaStream_t stream) {
  if (p1 <= p0) return 0;
  // HOBI_SINGULAR: "fast" (default, hobi_singular.cu), "warp" (literal
  // transcription, one warp per pair) or "serial" (literal, one thread per pair)
  static const int kind = [] {
    const char* e = getenv("HOBI_SINGULAR");
    if (e && !strcmp(e, "serial")) return 2;
    if (e && !strcmp(e, "warp")) return 1;
    return 0;
  }();
  if (kind == 0) {
    int rc = launch_singular_fast(c, u_dev, p0, p1, stream);
    if (rc) return rc;
  } else if (kind == 2)
    singular_kernel<<<nblk(p1 - p0, 128), 128, 0, stream>>>(
        p0, p1, c->pair_vertex.p, c->pair_face.p, c->pair_gverts.p, c->faces.p, c->vert.p, c->vnrm.p,
        c->reg_pos.p, c->reg_nrm.p, c->reg_w.p, c->reg_bary.p, c->nq, c->duf_pos.p, c->duf_nrm.p,
        c->duf_w.p, c->duf_bary.p, c->nd, u_dev, c->nt, c->phys.er, c->phys.kappa, c->corr.p);
  else
    singular_warp_kernel<<<nblk(p1 - p0, kSingWarps), 32 * kSingWarps, 0, stream>>>(
        p0, p1, c->pair_vertex.p, c->pair_face.p, c->pair_gverts.p, c->faces.p, c->vert.p, c->vnrm.p,
        c->reg_pos.p, c->reg_nrm.p, c->reg_w.p, c->reg_bary.p, c->nq, c->duf_pos.p, c->duf_nrm.p,
        c->duf_w.p, c->duf_bary.p, c->nd, u_dev, c->nt, c->phys.er, c->phys.kappa, c->corr.p);
  c->launches++;
  HOBI_CUDA(cudaGetLastError());
  return 0;
}

int rhs_device(hobi_ctx* c, const double* qpos, const double* q, int64_t nc, double* b_dev) {
  const int64_t nt = c->nt;
  if (nc == 0) {
    HOBI_CUDA(cudaMemsetAsync(b_dev, 0, 2 * nt * sizeof(double), c->stream));
    return 0;
  }
  int rc;
  if ((rc = charge_workspace(c, nc))) return rc;
  ChargeWorkspace& w = c->charge_ws;
  double *dq = w.q.p, *dpos = w.qpos.p;
  unsigned long long* bad = w.bad.p;
  HOBI_CUDA(cudaMemcpyAsync(dq, q, nc * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  HOBI_CUDA(cudaMemcpyAsync(dpos, qpos, 3 * nc * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  HOBI_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), c->stream));
  const double* pos = c->scheme == kHobi ? c->vert.p : c->reg_pos.p;
  const double* nrm = c->scheme == kHobi ? c->vnrm.p : c->reg_nrm.p;
  // Under a communicator each rank computes its own rows and the vector is
  // gathered like an operator application (rows are bitwise those of a
  // one-GPU run); the singularity decision is made on every rank from all
  // ranks' first-offender keys.  An emulated split computes every rank's
  // rows here, straight into the gather layout.
  const bool split = c->comm.nccl && c->comm.nranks > 1;
  const bool emul = c->comm.emulated && c->comm.nranks > 1;
  const int64_t m = c->gather_m;
  auto rows = [&](int64_t lo, int64_t hi, double* o1, double* o2) -> int {
    if (hi <= lo) return 0;
    rhs_kernel<<<nblk(hi - lo, 256), 256, 0, c->stream>>>(pos, nrm, lo, hi, dpos, dq, nc,
                                                          c->phys.eps1, o1, o2, bad);
    c->launches++;
    HOBI_CUDA(cudaGetLastError());
    return 0;
  };
  unsigned long long badh = 0;
  if (emul) {
    for (int r = 0; r < c->comm.nranks; ++r) {
      const int64_t base = nt / c->comm.nranks, extra = nt % c->comm.nranks;
      const int64_t lo = r * base + std::min<int64_t>(r, extra), hi = lo + base + (r < extra ? 1 : 0);
      double* slot = c->gather_recv.p + (int64_t)r * 2 * m;
      if ((rc = rows(lo, hi, slot, slot + m))) return rc;
    }
    if ((rc = gather_permute(c, b_dev))) return rc;
    HOBI_CUDA(cudaMemcpyAsync(&badh, bad, sizeof(badh), cudaMemcpyDeviceToHost, c->stream));
  } else if (split) {
    if ((rc = rows(c->lo, c->hi, c->gather_send.p, c->gather_send.p + m))) return rc;
    if ((rc = comm_allgather_bytes(c, bad, w.bad_all.p, sizeof(unsigned long long)))) return rc;
    std::vector<unsigned long long> h(c->comm.nranks);
    HOBI_CUDA(cudaMemcpyAsync(h.data(), w.bad_all.p, h.size() * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, c->stream));
    HOBI_CUDA(cudaStreamSynchronize(c->stream));
    badh = ~0ull;
    for (unsigned long long v : h) badh = v < badh ? v : badh;
    if (badh == ~0ull) {
      if ((rc = comm_allgather(c))) return rc;
      if ((rc = gather_permute(c, b_dev))) return rc;
    }
  } else {
    if ((rc = rows(0, nt, b_dev, b_dev + nt))) return rc;
    HOBI_CUDA(cudaMemcpyAsync(&badh, bad, sizeof(badh), cudaMemcpyDeviceToHost, c->stream));
  }
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  if (badh != ~0ull) {
    unsigned long long i = badh / (unsigned long long)(nc + 1), k = badh % (unsigned long long)(nc + 1);
    return fail(HOBI_ERR_SINGULARITY, "surface point " + std::to_string(i) + " coincides with charge " +
                                          std::to_string(k));
  }
  return 0;
}

int kernel_values_device(const double* d, const double* nx, const double* ny, int64_t n, double eps1,
                         double eps2, double kappa, double* k) {
  if (n == 0) return 0;
  DevBuf<double> dd, dx, dy, dk;
  if (dd.alloc(3 * n) || dx.alloc(3 * n) || dy.alloc(3 * n) || dk.alloc(4 * n)) return HOBI_ERR_CUDA;
  HOBI_CUDA(cudaMemcpy(dd.p, d, 3 * n * sizeof(double), cudaMemcpyHostToDevice));
  HOBI_CUDA(cudaMemcpy(dx.p, nx, 3 * n * sizeof(double), cudaMemcpyHostToDevice));
  HOBI_CUDA(cudaMemcpy(dy.p, ny, 3 * n * sizeof(double), cudaMemcpyHostToDevice));
  kernel_values_kernel<<<nblk(n, 256), 256>>>(dd.p, dx.p, dy.p, n, eps2 / eps1, kappa, dk.p);
  HOBI_CUDA(cudaGetLastError());
  HOBI_CUDA(cudaMemcpy(k, dk.p, 4 * n * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

// kernels.source_terms_at (kernels.py:159-178) at arbitrary surface points:
// the RHS kernel with eps1 = 1 (x/1.0 is exact), on the default stream.
int source_terms_device(const double* points, const double* normals, int64_t m, const double* qpos,
                        const double* q, int64_t nc, double* s1, double* s2) {
  if (m == 0) return 0;
  if (nc == 0) {
    memset(s1, 0, m * sizeof(double));
    memset(s2, 0, m * sizeof(double));
    return 0;
  }
  DevBuf<double> dp, dn, dqp, dq, ds;
  DevBuf<unsigned long long> bad;
  if (dp.alloc(3 * m) || dn.alloc(3 * m) || dqp.alloc(3 * nc) || dq.alloc(nc) || ds.alloc(2 * m) ||
      bad.alloc(1))
    return HOBI_ERR_CUDA;
  HOBI_CUDA(cudaMemcpy(dp.p, points, 3 * m * sizeof(double), cudaMemcpyHostToDevice));
  HOBI_CUDA(cudaMemcpy(dn.p, normals, 3 * m * sizeof(double), cudaMemcpyHostToDevice));
  HOBI_CUDA(cudaMemcpy(dqp.p, qpos, 3 * nc * sizeof(double), cudaMemcpyHostToDevice));
  HOBI_CUDA(cudaMemcpy(dq.p, q, nc * sizeof(double), cudaMemcpyHostToDevice));
  HOBI_CUDA(cudaMemset(bad.p, 0xff, sizeof(unsigned long long)));
  rhs_kernel<<<nblk(m, 256), 256>>>(dp.p, dn.p, 0, m, dqp.p, dq.p, nc, 1.0, ds.p, ds.p + m, bad.p);
  HOBI_CUDA(cudaGetLastError());
  unsigned long long badh = 0;
  HOBI_CUDA(cudaMemcpy(&badh, bad.p, sizeof(badh), cudaMemcpyDeviceToHost));
  if (badh != ~0ull) {
    unsigned long long i = badh / (unsigned long long)(nc + 1), k = badh % (unsigned long long)(nc + 1);
    return fail(HOBI_ERR_SINGULARITY, "surface point " + std::to_string(i) + " coincides with charge " +
                                          std::to_string(k));
  }
  HOBI_CUDA(cudaMemcpy(s1, ds.p, m * sizeof(double), cudaMemcpyDeviceToHost));
  HOBI_CUDA(cudaMemcpy(s2, ds.p + m, m * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

}  // namespace hobi
