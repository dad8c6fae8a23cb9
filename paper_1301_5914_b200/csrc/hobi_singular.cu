// The Duffy singular swap, default form (solver.py:336-363):
// per incident (vertex, face) pair, the Duffy-rule sum over the rotated
// element minus the regular-rule sum over the rotation-0 element.  The
// literal transcriptions (singular_warp_kernel, singular_kernel) are in
// hobi_literal.cu; launch_singular there picks one.
#include <algorithm>
#include <cstdlib>

#include "hobi_fastmath.cuh"
#include "hobi_internal.cuh"
#include "hobi_tma.cuh"

namespace hobi {

namespace {
inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
}  // namespace

// singular_fast_kernel: a block of T threads owns CH chunks of ppb = T /
// (nq + nd) consecutive incident pairs.  Staging: the pairs' Duffy points
// (position, normal, weight: one contiguous range of the pair-ordered caches,
// 56 B per point, the kernel's HBM stream; 1-D TMA bulk copies with an L2
// evict_first hint when the rule sizes are even, 8-byte cp.async otherwise),
// then one thread per pair reads its index record (pair_rec) and fetches the
// target vertex and the six phi/dphi interpolation values, and requests its
// rotation-0 element's regular points.  Compute: per chunk, one thread per
// term evaluates the kernel with the sweep's arithmetic (MUFU rsqrt seed +
// Newton, the table expm1 with expm1-grade relative accuracy,
// hobi_fastmath.cuh) instead of libdevice sqrt/exp/expm1 and five IEEE
// divisions; the pair's regular and Duffy rows are summed in numpy's
// .sum(axis=1) order (numpy_row_sum) and their difference is the correction.
// Against the literal transcription (HOBI_SINGULAR=warp) the matvec agrees
// to 1e-14 (tests/test_gpu_singular.py); profiles/r02_singular.md.

struct SingLayout {  // dynamic shared memory, in doubles (ints at the end)
  int pb, dpos, dnrm, dw, rpos, rnrm, rw, px, uv, t1, t2, r1, r2, ints, bytes;
  __host__ __device__ SingLayout(int ppb, int nq, int nd, int chunks, int threads) {
    pb = ppb * chunks;
    dpos = 0;
    dnrm = dpos + pb * nd * 3;
    dw = dnrm + pb * nd * 3;
    rpos = dw + pb * nd;
    rnrm = rpos + pb * nq * 3;
    rw = rnrm + pb * nq * 3;
    px = rw + pb * nq;         // target vertex position and normal, 6 per pair
    uv = px + pb * 6;          // phi at the 3 regular + 3 Duffy element vertices, then dphi
    t1 = uv + pb * 12;
    t2 = t1 + threads;
    r1 = t2 + threads;
    r2 = r1 + threads;
    ints = r2 + threads;  // face of each pair
    bytes = ints * 8 + pb * 4;
  }
};


// One term of a pair's row (kernels.py:99-130 times the interpolated
// weights, solver.py:350-360) from its target (px: position, normal), its
// point (y, ny, w), the element's phi/dphi at its vertices (uvp[0..2],
// uvp[6..8]) and the point's barycentrics; the sweep's arithmetic.
__device__ __forceinline__ void singular_term(const double* px, const double* y, const double* ny, double w,
                                              const double* uvp, const double* __restrict__ bary, double kappa,
                                              double er, double ier, const double* __restrict__ etab,
                                              double& t1, double& t2) {
  const double n0 = px[3], n1 = px[4], n2 = px[5];
  const double dx = px[0] - y[0], dy = px[1] - y[1], dz = px[2] - y[2];
  const double mx = ny[0], my = ny[1], mz = ny[2];
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  const double ir = rsqrt_fast(r2);
  const double kr = kappa * (r2 * ir);
  const double em1 = expm1_neg(kr, etab);  // e^{-kr} - 1
  const double kre = fma(kr, em1, kr);             // kr e^{-kr}
  const double a = em1 + kre;                      // kernels.py:119
  const double b = fma(a, 3.0, kr * kre);          // kernels.py:120
  const double dny = fma(dx, mx, fma(dy, my, dz * mz));
  const double dnx = fma(dx, n0, fma(dy, n1, dz * n2));
  const double nn = fma(n0, mx, fma(n1, my, n2 * mz));
  const double ir2 = ir * ir;
  const double g3 = (ir * ir2) * (1.0 / kFourPi);  // 1 / (4 pi r^3)
  const double k1 = -em1 * ir * (1.0 / kFourPi);
  const double k2 = dny * g3 * fma(er, a, er - 1.0);
  const double k3 = -dnx * g3 * fma(-a, ier, 1.0 - ier);
  const double k4 = fma(a, nn, -b * dnx * dny * ir2) * g3;
  const double b0 = bary[0], b1 = bary[1], b2 = bary[2];
  const double wp = w * fma(uvp[0], b0, fma(uvp[1], b1, uvp[2] * b2));
  const double wd = w * fma(uvp[6], b0, fma(uvp[7], b1, uvp[8] * b2));
  t1 = fma(k1, wd, k2 * wp);
  t2 = fma(k3, wd, k4 * wp);
}

// NQ = ND = 0: rule sizes at run time; CH chunks of ppb pairs per block
template <int NQ, int ND, int CH, int MINB, int T = 256>
__global__ void __launch_bounds__(T, MINB) singular_fast_kernel(
    int64_t p0, int64_t p1, int ppb_rt, const int4* __restrict__ pair_rec, const double* __restrict__ vert,
    const double* __restrict__ vnrm, const double* __restrict__ reg_pos, const double* __restrict__ reg_nrm,
    const double* __restrict__ reg_w, const double* __restrict__ reg_bary, int nq_rt,
    const double* __restrict__ duf_pos, const double* __restrict__ duf_nrm, const double* __restrict__ duf_w,
    const double* __restrict__ duf_bary, int nd_rt, const double* __restrict__ u, int64_t nt, double kappa,
    double er, double ier, const double* __restrict__ etab, double* __restrict__ corr) {
  extern __shared__ __align__(16) double sm[];
  __shared__ uint64_t bar;
  const int nq = NQ ? NQ : nq_rt, nd = ND ? ND : nd_rt;
  const int ppb = NQ ? T / (NQ + ND) : ppb_rt;
  // 1-D bulk copies (TMA) when every range is 16-byte aligned: even rule sizes
  constexpr bool kBulk = NQ > 0 && NQ % 2 == 0 && ND % 2 == 0;
  const SingLayout L(ppb, nq, nd, CH, T);
  int* sface = reinterpret_cast<int*>(sm + L.ints);
  const int tid = threadIdx.x;
  const int64_t pbase = p0 + (int64_t)blockIdx.x * L.pb;
  const int npairs = (int)(p1 - pbase < L.pb ? p1 - pbase : L.pb);
  // (1) the Duffy points of pairs [pbase, pbase + npairs): one contiguous range
  const int64_t dg0 = pbase * nd;
  if (kBulk) {
    if (tid == 0) {
      mbar_init(&bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      // every byte this block stages: Duffy (56 B per point) + regular (56 B per point)
      mbar_expect_tx(&bar, (uint32_t)npairs * (uint32_t)(nd + nq) * 56u);
      const uint32_t b3 = (uint32_t)npairs * nd * 24u, b1 = (uint32_t)npairs * nd * 8u;
      const uint64_t pol = l2_evict_first();
      bulk_g2s_hint(sm + L.dpos, duf_pos + dg0 * 3, b3, &bar, pol);
      bulk_g2s_hint(sm + L.dnrm, duf_nrm + dg0 * 3, b3, &bar, pol);
      bulk_g2s_hint(sm + L.dw, duf_w + dg0, b1, &bar, pol);
    }
  } else {
    const int n3 = npairs * nd * 3, n1 = npairs * nd;
    for (int k = tid; k < n3; k += T) {
      cp_async8(sm + L.dpos + k, duf_pos + dg0 * 3 + k);
      cp_async8(sm + L.dnrm + k, duf_nrm + dg0 * 3 + k);
    }
    for (int k = tid; k < n1; k += T) cp_async8(sm + L.dw + k, duf_w + dg0 + k);
  }
  if (kBulk) __syncthreads();  // the barrier is initialised before any thread copies on it
  // (2) one thread per pair: index chain and interpolation values
  if (tid < npairs) {
    const int64_t p = pbase + tid;
    const int4 ra = pair_rec[2 * p], rb = pair_rec[2 * p + 1];
    const int v = ra.x, f = ra.y, a0 = ra.z, a1 = ra.w, g0 = rb.x, g1 = rb.y, g2 = rb.z;
    if (kBulk) {  // this pair's rotation-0 element: nq regular points
      bulk_g2s(sm + L.rpos + tid * nq * 3, reg_pos + (int64_t)f * nq * 3, nq * 24u, &bar);
      bulk_g2s(sm + L.rnrm + tid * nq * 3, reg_nrm + (int64_t)f * nq * 3, nq * 24u, &bar);
      bulk_g2s(sm + L.rw + tid * nq, reg_w + (int64_t)f * nq, nq * 8u, &bar);
    }
    sface[tid] = f;
    const int a2 = rb.w;
    double* px = sm + L.px + 6 * tid;
    px[0] = vert[3 * v];
    px[1] = vert[3 * v + 1];
    px[2] = vert[3 * v + 2];
    px[3] = vnrm[3 * v];
    px[4] = vnrm[3 * v + 1];
    px[5] = vnrm[3 * v + 2];
    double* uv = sm + L.uv + 12 * tid;
    const double* dphi = u + nt;
    uv[0] = u[a0];
    uv[1] = u[a1];
    uv[2] = u[a2];
    uv[3] = u[g0];
    uv[4] = u[g1];
    uv[5] = u[g2];
    uv[6] = dphi[a0];
    uv[7] = dphi[a1];
    uv[8] = dphi[a2];
    uv[9] = dphi[g0];
    uv[10] = dphi[g1];
    uv[11] = dphi[g2];
  }
  __syncthreads();
  if (kBulk) {
    mbar_wait(&bar, 0);
  } else {  // (3) the regular points of each pair's rotation-0 element (nq per face)
    for (int k = tid; k < npairs * nq * 3; k += T) {
      const int pr = k / (nq * 3), e = k - pr * nq * 3;
      const int64_t g = (int64_t)sface[pr] * nq * 3 + e;
      cp_async8(sm + L.rpos + k, reg_pos + g);
      cp_async8(sm + L.rnrm + k, reg_nrm + g);
    }
    for (int k = tid; k < npairs * nq; k += T) {
      const int pr = k / nq, e = k - pr * nq;
      cp_async8(sm + L.rw + k, reg_w + (int64_t)sface[pr] * nq + e);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
    __syncthreads();
  }

  const int nterm = nq + nd;
  const int lp = tid / nterm, m = tid - lp * nterm;
  const int j = tid >> 1, row = tid & 1;
  for (int ch = 0; ch < CH; ++ch) {
    const int pr = ch * ppb + lp;  // this thread's pair, block-local
    if (lp < ppb && pr < npairs) {
      const double *y, *ny, *bary, *uvp;
      double w;
      if (m < nq) {
        const int k = pr * nq + m;
        y = sm + L.rpos + 3 * k;
        ny = sm + L.rnrm + 3 * k;
        w = sm[L.rw + k];
        bary = reg_bary + 3 * m;
        uvp = sm + L.uv + 12 * pr;
      } else {
        const int k = pr * nd + (m - nq);
        y = sm + L.dpos + 3 * k;
        ny = sm + L.dnrm + 3 * k;
        w = sm[L.dw + k];
        bary = duf_bary + 3 * (m - nq);
        uvp = sm + L.uv + 12 * pr + 3;
      }
      singular_term(sm + L.px + 6 * pr, y, ny, w, uvp, bary, kappa, er, ier, etab, sm[L.t1 + tid],
                    sm[L.t2 + tid]);
    }
    __syncthreads();
    // rows in numpy's order: thread 2j sums pair j's regular row, 2j+1 its Duffy row
    const bool live = j < ppb && ch * ppb + j < npairs;
    if (live) {
      const int off = j * nterm + (row ? nq : 0), n = row ? nd : nq;
      double s1, s2;
      numpy_row_sum(n, [&](int k, double& a1, double& a2) {
        a1 = sm[L.t1 + off + k];
        a2 = sm[L.t2 + off + k];
      }, s1, s2);
      sm[L.r1 + tid] = s1;
      sm[L.r2 + tid] = s2;
    }
    __syncthreads();
    if (live && row == 0) {  // Duffy row minus regular row (solver.py:362-363)
      const int64_t p = pbase + ch * ppb + j;
      corr[2 * p] = sm[L.r1 + tid + 1] - sm[L.r1 + tid];
      corr[2 * p + 1] = sm[L.r2 + tid + 1] - sm[L.r2 + tid];
    }
  }
}

namespace {
typedef void (*SingFn)(int64_t, int64_t, int, const int4*, const double*, const double*, const double*, const double*, const double*, const double*, int,
                       const double*, const double*, const double*, const double*, int, const double*, int64_t,
                       double, double, double, const double*, double*);
struct SingVariant {
  SingFn fn;
  int chunks, threads;
  const char* name;
};
// [0] is the run-time-rule kernel; the rest are tilings of the default rules
const SingVariant kSingVariants[] = {
    {singular_fast_kernel<0, 0, 3, 4>, 3, 256, "rt_ch3_minb4"},
    {singular_fast_kernel<4, 16, 3, 4>, 3, 256, "q4d16_ch3_minb4"},
    {singular_fast_kernel<4, 16, 2, 5>, 2, 256, "q4d16_ch2_minb5"},
    {singular_fast_kernel<4, 16, 2, 6>, 2, 256, "q4d16_ch2_minb6"},
    {singular_fast_kernel<4, 16, 1, 8>, 1, 256, "q4d16_ch1_minb8"},
    {singular_fast_kernel<4, 16, 4, 3>, 4, 256, "q4d16_ch4_minb3"},
    {singular_fast_kernel<4, 16, 1, 16, 128>, 1, 128, "q4d16_t128_minb16"},
    {singular_fast_kernel<4, 16, 1, 12, 128>, 1, 128, "q4d16_t128_minb12"},
    {singular_fast_kernel<4, 16, 2, 8, 128>, 2, 128, "q4d16_t128_ch2_minb8"},
};
constexpr int kSingVariantCount = sizeof(kSingVariants) / sizeof(kSingVariants[0]);
// config 4 / config 1 per launch (ncu, one B200): 94.0/8.5, 95.0/8.1, 99.1/8.5,
// 90.7/6.7, 95.5/9.0 us for variants 1-5 (profiles/r02_singular.md); 6-8 are 128-thread blocks
constexpr int kSingDefault = 4;
}  // namespace

int launch_singular_fast(hobi_ctx* c, const double* u_dev, int64_t p0, int64_t p1, cudaStream_t stream) {
  if (c->nq + c->nd > 256) return fail(HOBI_ERR_VALUE, "Duffy swap: nq + nd exceeds one block");
  // the default rules (4 regular + 16 Duffy points) get a compile-time
  // instantiation with bulk copies; any other rule the run-time one.
  // HOBI_SINGULAR_VARIANT (1-8) pins a tiling (tuning; bitwise the same)
  static const int tuned = [] {
    const char* e = getenv("HOBI_SINGULAR_VARIANT");
    const int v = e ? atoi(e) : kSingDefault;
    return v >= 1 && v < kSingVariantCount ? v : kSingDefault;
  }();
  const SingVariant& sv = kSingVariants[c->nq == 4 && c->nd == 16 ? tuned : 0];
  const int ppb = sv.threads / (c->nq + c->nd);
  const SingLayout L(ppb, c->nq, c->nd, sv.chunks, sv.threads);
  if (!c->singular_etab) {  // per context: the opt-in and the table address are per device
    for (const auto& v : kSingVariants)
      HOBI_CUDA(cudaFuncSetAttribute(v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    c->singular_etab = exp_table_device();
    if (!c->singular_etab) return fail(HOBI_ERR_CUDA, "Duffy swap: exp table address");
  }
  const unsigned grid = (unsigned)((p1 - p0 + L.pb - 1) / L.pb);
  sv.fn<<<grid, sv.threads, L.bytes, stream>>>(
      p0, p1, ppb, reinterpret_cast<const int4*>(c->pair_rec.p), c->vert.p, c->vnrm.p, c->reg_pos.p,
      c->reg_nrm.p, c->reg_w.p, c->reg_bary.p, c->nq, c->duf_pos.p, c->duf_nrm.p, c->duf_w.p, c->duf_bary.p,
      c->nd, u_dev, c->nt, c->phys.kappa, c->phys.er, c->phys.ier, c->singular_etab, c->corr.p);
  HOBI_CUDA(cudaGetLastError());
  return 0;
}

namespace {
__global__ void pair_rec_kernel(int64_t np, const int* __restrict__ pv, const int* __restrict__ pf,
                                const int* __restrict__ pg, const int* __restrict__ faces, int* __restrict__ rec) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= np) return;
  const int f = pf[p];
  int* r = rec + 8 * p;
  r[0] = pv[p];
  r[1] = f;
  r[2] = faces[3 * f];
  r[3] = faces[3 * f + 1];
  r[4] = pg[3 * p];
  r[5] = pg[3 * p + 1];
  r[6] = pg[3 * p + 2];
  r[7] = faces[3 * f + 2];
}
}  // namespace

// Once per context (hobi_create / hobi_create_from_caches): the Duffy
// swap's per-pair index record, so its staging needs one dependent read
// less (pair -> element vertices -> phi, instead of pair -> face -> ...).
int prepare_singular(hobi_ctx* c) {
  const int64_t np = c->h_pair_starts.empty() ? 0 : c->h_pair_starts.back();
  if (np <= 0 || !c->pair_face.p) return 0;
  if (c->pair_rec.alloc(8 * np)) return HOBI_ERR_CUDA;
  pair_rec_kernel<<<nblk(np, 256), 256, 0, c->stream>>>(np, c->pair_vertex.p, c->pair_face.p, c->pair_gverts.p,
                                                         c->faces.p, c->pair_rec.p);
  HOBI_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace hobi
