// Device-resident restarted GMRES: gmres_solve,
// solver.py:484-560.  The Krylov basis, iterate and residual live in HBM; one
// cooperative kernel per inner step performs the whole modified Gram-Schmidt
// sweep (j+1 dots and axpys plus the normalisation) with grid-wide barriers,
// deterministic fixed-partition reductions and no host round trip except the
// (j+2)-entry Hessenberg column.  Givens rotations, the stopping tests and the
// triangular solve stay on the host in the reference's exact scalar order.
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cmath>
#include <limits>
#include <vector>

#include "hobi_internal.cuh"

namespace cg = cooperative_groups;

namespace hobi {

namespace {

constexpr int kGT = 256;  // threads per block

__device__ __forceinline__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = kGT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  double r = sh[0];
  __syncthreads();
  return r;
}

// Fixed chunk of [0, n) owned by this block.
__device__ __forceinline__ void chunk(int64_t n, int64_t* lo, int64_t* hi) {
  int64_t per = (n + gridDim.x - 1) / gridDim.x;
  *lo = min(n, (int64_t)blockIdx.x * per);
  *hi = min(n, *lo + per);
}

__device__ __forceinline__ double fixed_total(const double* __restrict__ part) {
  double s = 0.0;
  for (unsigned b = 0; b < gridDim.x; ++b) s += part[b];
  return s;
}

// Arnoldi step j: w <- w - sum_i h_ij v_i (MGS), h_{j+1,j} = ||w||,
// v_{j+1} = w / h_{j+1,j} when > 1e-300 (solver.py:538-543).
// `jdev` (graph mode): the step index is read from device memory; `vnext`
// (graph mode): v_{j+1} is also written there, the next application's input.
__global__ void __launch_bounds__(kGT) mgs_kernel(double* __restrict__ V, int64_t ldv, int64_t n, int j,
                                                  double* __restrict__ w, double* __restrict__ part,
                                                  double* __restrict__ hcol, const GmresState* jdev,
                                                  double* __restrict__ vnext) {
  cg::grid_group grid = cg::this_grid();
  if (jdev) j = jdev->j;
  __shared__ double sh[kGT];
  int64_t lo, hi;
  chunk(n, &lo, &hi);
  for (int i = 0; i <= j; ++i) {
    const double* vi = V + (int64_t)i * ldv;
    double acc = 0.0;
    for (int64_t k = lo + threadIdx.x; k < hi; k += kGT) acc = fma(vi[k], w[k], acc);
    double* pb = part + (i & 1) * gridDim.x;
    double bs = block_sum(acc, sh);
    if (threadIdx.x == 0) pb[blockIdx.x] = bs;
    grid.sync();
    const double h = fixed_total(pb);
    if (blockIdx.x == 0 && threadIdx.x == 0) hcol[i] = h;
    for (int64_t k = lo + threadIdx.x; k < hi; k += kGT) w[k] = __dsub_rn(w[k], __dmul_rn(h, vi[k]));
  }
  double acc = 0.0;
  for (int64_t k = lo + threadIdx.x; k < hi; k += kGT) acc = fma(w[k], w[k], acc);
  double* pb = part + ((j + 1) & 1) * gridDim.x;
  double bs = block_sum(acc, sh);
  if (threadIdx.x == 0) pb[blockIdx.x] = bs;
  grid.sync();
  const double nrm = sqrt(fixed_total(pb));
  if (blockIdx.x == 0 && threadIdx.x == 0) hcol[j + 1] = nrm;
  if (nrm > 1e-300) {
    double* vn = V + (int64_t)(j + 1) * ldv;
    for (int64_t k = lo + threadIdx.x; k < hi; k += kGT) {
      const double v = w[k] / nrm;
      vn[k] = v;
      if (vnext) vnext[k] = v;
    }
  }
}

// The same Arnoldi step in one CTA, for small n (<= kSmallN): no cooperative
// launch and no grid-wide barriers -- each dot is a block reduction over a
// fixed thread partition (thread t owns k = t, t + kST, ...; warp shuffles in
// a fixed xor tree, then the 32 warp sums in warp order), so the result is
// deterministic and identical on every rank.  Small problems are latency
// bound: this removes ~15 us per step at config 1 (21 -> ~5 us, ncu).
constexpr int kST = 1024;
constexpr int64_t kSmallN = 32768;

__device__ __forceinline__ double cta_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = sh[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) sh[32] = s;
  }
  __syncthreads();
  s = sh[32];
  __syncthreads();
  return s;
}

__global__ void __launch_bounds__(kST) mgs_small_kernel(double* __restrict__ V, int64_t ldv, int64_t n, int j,
                                                        double* __restrict__ w, double* __restrict__ hcol,
                                                        const GmresState* jdev, double* __restrict__ vnext) {
  __shared__ double sh[33];
  if (jdev) j = jdev->j;
  for (int i = 0; i <= j; ++i) {
    const double* vi = V + (int64_t)i * ldv;
    double acc = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += kST) acc = fma(vi[k], w[k], acc);
    const double h = cta_sum(acc, sh);
    if (threadIdx.x == 0) hcol[i] = h;
    for (int64_t k = threadIdx.x; k < n; k += kST) w[k] = __dsub_rn(w[k], __dmul_rn(h, vi[k]));
  }
  double acc = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += kST) acc = fma(w[k], w[k], acc);
  const double nrm = sqrt(cta_sum(acc, sh));
  if (threadIdx.x == 0) hcol[j + 1] = nrm;
  if (nrm > 1e-300) {
    double* vn = V + (int64_t)(j + 1) * ldv;
    for (int64_t k = threadIdx.x; k < n; k += kST) {
      const double v = w[k] / nrm;
      vn[k] = v;
      if (vnext) vnext[k] = v;
    }
  }
}

// r = b - Ax and block partials of ||r||^2.
__global__ void residual_kernel(const double* __restrict__ b, const double* __restrict__ ax, int64_t n,
                                double* __restrict__ r, double* __restrict__ part) {
  __shared__ double sh[kGT];
  int64_t lo, hi;
  chunk(n, &lo, &hi);
  double acc = 0.0;
  for (int64_t k = lo + threadIdx.x; k < hi; k += kGT) {
    double v = ax ? b[k] - ax[k] : b[k];
    if (r) r[k] = v;
    acc = fma(v, v, acc);
  }
  double bs = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = bs;
}

__global__ void norm_finish_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[b];
  out[0] = sqrt(s);
}

__global__ void scale_kernel(const double* __restrict__ r, int64_t n, double beta, double* __restrict__ v,
                             double* __restrict__ vcopy) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  v[k] = r[k] / beta;
  if (vcopy) vcopy[k] = v[k];
}

// hypot exactly as glibc computes it for double on x86-64 (no FMA; Borges'
// corrected sqrt with the same scaling thresholds), so the device Givens
// rotations round like np.hypot in the reference (solver.py:551) and like
// the host loop's std::hypot: bit-identical on 200,000 sampled argument
// pairs against numpy in this build.
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
  const double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= __dmul_rn(2.0, ay)) {
    const double delta = __dsub_rn(h, ay);
    t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
    t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
  } else {
    const double delta = __dsub_rn(h, ax);
    t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
    t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
  }
  return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

__device__ double glibc_hypot(double x, double y) {
  const double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
  if (isinf(x) || isinf(y)) return INFINITY;
  if (isnan(x) || isnan(y)) return x + y;
  double ax = fabs(x), ay = fabs(y);
  if (ax < ay) {
    const double t = ax;
    ax = ay;
    ay = t;
  }
  if (ax > kLarge) {
    if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
    return __ddiv_rn(hypot_kernel(__dmul_rn(ax, kScale), __dmul_rn(ay, kScale)), kScale);
  }
  if (ay < kTiny) {
    if (ax >= __ddiv_rn(ay, kEps)) return __dadd_rn(ax, ay);
    ax = __dmul_rn(ax, 0x1p600);
    ay = __dmul_rn(ay, 0x1p600);
    return __dmul_rn(hypot_kernel(ax, ay), kScale);
  }
  if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
  return hypot_kernel(ax, ay);
}

// One inner step's Givens update and stopping test (solver.py:544-558) in
// the host loop's exact scalar order, then the loop condition for the
// graph's WHILE node: continue while j < m, total < max_it and
// |g_j| / ||b|| > tol.
__global__ void givens_kernel(GmresState* __restrict__ st, const double* __restrict__ hcol,
                              double* __restrict__ H, double* __restrict__ cs, double* __restrict__ sn,
                              double* __restrict__ g, cudaGraphConditionalHandle cond) {
  if (threadIdx.x || blockIdx.x) return;
  const int j = st->j, m = st->m;
  auto Hat = [&](int i, int jj) -> double& { return H[(size_t)i * m + jj]; };
  for (int i = 0; i <= j + 1; ++i) Hat(i, j) = hcol[i];
  for (int i = 0; i < j; ++i) {
    const double tmp = __dadd_rn(__dmul_rn(cs[i], Hat(i, j)), __dmul_rn(sn[i], Hat(i + 1, j)));
    Hat(i + 1, j) = __dadd_rn(__dmul_rn(-sn[i], Hat(i, j)), __dmul_rn(cs[i], Hat(i + 1, j)));
    Hat(i, j) = tmp;
  }
  const double denom = glibc_hypot(Hat(j, j), Hat(j + 1, j));
  cs[j] = __ddiv_rn(Hat(j, j), denom);
  sn[j] = __ddiv_rn(Hat(j + 1, j), denom);
  Hat(j, j) = denom;
  Hat(j + 1, j) = 0.0;
  g[j + 1] = __dmul_rn(-sn[j], g[j]);
  g[j] = __dmul_rn(cs[j], g[j]);
  const int jn = j + 1, total = st->total + 1;
  st->j = jn;
  st->total = total;
  const bool converged = __ddiv_rn(fabs(g[jn]), st->norm_b) <= st->tol;
  cudaGraphSetConditional(cond, (!converged && jn < m && total < st->max_it) ? 1u : 0u);
}

// Test hook: glibc_hypot on n argument pairs (the bitwise check against the
// host's std::hypot, hobi_hypot_check).
__global__ void hypot_check_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                                   double* __restrict__ out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) out[k] = glibc_hypot(a[k], b[k]);
}

// x += V[:j]^T y  (solver.py:560)
__global__ void update_kernel(const double* __restrict__ V, int64_t ldv, int64_t n, int j,
                              const double* __restrict__ y, double* __restrict__ x) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double s = 0.0;
  for (int i = 0; i < j; ++i) s = fma(V[(int64_t)i * ldv + k], y[i], s);
  x[k] = x[k] + s;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

int gmres_device(int device, cudaStream_t stream, int64_t n, DeviceOperator* op, const double* b_host,
                 double tol, int restart, int max_it, double* x_host, int* iterations,
                 double* residual, double* best_out, int* matvecs, int64_t* launch_counter,
                 GmresWorkspace* cached) {
  if (n % 2) return fail(HOBI_ERR_VALUE, "vector length must be even: (phi, dphi/dn) halves");
  if (!(tol > 0.0 && tol < 1.0)) return fail(HOBI_ERR_VALUE, "tolerance must be in (0, 1)");
  if (restart < 1) return fail(HOBI_ERR_VALUE, "restart must be >= 1");
  if (max_it < 1) return fail(HOBI_ERR_VALUE, "max_iterations must be >= 1");
  *iterations = 0;
  *residual = 0.0;
  *best_out = std::numeric_limits<double>::infinity();
  *matvecs = 0;
  int64_t launches = 0;
  const int m = restart;
  GmresWorkspace local;
  GmresWorkspace& ws = cached ? *cached : local;
  if (ws.n != n || ws.m != m) {
    int sms = 0, occ = 0;
    HOBI_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    HOBI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mgs_kernel, kGT, 0));
    ws.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * std::max(occ, 1),
                                                           std::min<int64_t>(2 * sms, (n + 1023) / 1024)));
    ws.ldv = ((n + 31) / 32) * 32;
    ws.n = -1;
    ws.cycle.reset();  // its nodes point at the buffers being replaced
    if (ws.V.alloc((size_t)(m + 1) * ws.ldv) || ws.w.alloc(n) || ws.x.alloc(n) || ws.r.alloc(n) ||
        ws.b.alloc(n) || ws.part.alloc(2 * ws.grid) || ws.hcol.alloc(m + 2) || ws.nrm.alloc(1) ||
        ws.y.alloc(m) || ws.hcol_h.alloc(m + 2) || ws.nrm_h.alloc(1) || ws.vin.alloc(n) ||
        ws.H.alloc((size_t)(m + 1) * m) || ws.cs.alloc(m) || ws.sn.alloc(m) || ws.g.alloc(m + 1) ||
        ws.st.alloc(1) || ws.st_h.alloc(1) || ws.H_h.alloc((size_t)(m + 1) * m) || ws.g_h.alloc(m + 1))
      return HOBI_ERR_CUDA;
    ws.n = n;
    ws.m = m;
  }
  HOBI_CUDA(cudaMemcpyAsync(ws.b.p, b_host, n * sizeof(double), cudaMemcpyHostToDevice, stream));

  auto norm_of = [&](const double* ax, double* rout, double* val) -> int {
    residual_kernel<<<ws.grid, kGT, 0, stream>>>(ws.b.p, ax, n, rout, ws.part.p);
    norm_finish_kernel<<<1, 32, 0, stream>>>(ws.part.p, ws.grid, ws.nrm.p);
    launches += 2;
    HOBI_CUDA(cudaGetLastError());
    HOBI_CUDA(cudaMemcpyAsync(ws.nrm_h.p, ws.nrm.p, sizeof(double), cudaMemcpyDeviceToHost, stream));
    HOBI_CUDA(cudaStreamSynchronize(stream));
    *val = ws.nrm_h.p[0];
    return 0;
  };
  int rc;
  double norm_b = 0.0;
  if ((rc = norm_of(nullptr, nullptr, &norm_b))) return rc;
  if (norm_b == 0.0) {
    std::fill(x_host, x_host + n, 0.0);
    if (launch_counter) *launch_counter += launches;
    return 0;
  }
  HOBI_CUDA(cudaMemsetAsync(ws.x.p, 0, n * sizeof(double), stream));
  int total = 0;
  double best = std::numeric_limits<double>::infinity();
  const bool trace = getenv("HOBI_GMRES_TRACE") && getenv("HOBI_GMRES_TRACE")[0] == '1';
  auto now = [] { return std::chrono::duration<double, std::milli>(
                      std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double t_mv = 0.0, t_orth = 0.0;
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), hcol(m + 2), y(m);
  auto Hat = [&](int i, int j) -> double& { return H[(size_t)i * m + j]; };

  // Device-driven inner cycle (CUDA graph with a WHILE conditional node):
  // body = operator application on ws.vin -> w, MGS (step index read from
  // device memory, v_{j+1} also written to ws.vin), Givens + stopping test
  // (givens_kernel), which sets the loop condition.  No host round trip per
  // step; the host reads the rotated Hessenberg matrix, g and the step count
  // once per cycle and does the triangular solve as before.  Captured once
  // per workspace and operator (graph_key) and replayed.
  const uint64_t key = cached ? op->graph_key() : 0;
  const bool use_graph = key != 0;
  auto build_graph = [&]() -> int {
    ws.cycle.reset();
    cudaGraph_t graph = nullptr;
    HOBI_CUDA(cudaGraphCreate(&graph, 0));
    ws.cycle.graph = graph;
    cudaGraphConditionalHandle cond;
    HOBI_CUDA(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    HOBI_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    const int64_t l0 = launch_counter ? *launch_counter : 0;
    HOBI_CUDA(cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    op->begin_capture();
    int arc = op->apply(ws.vin.p, ws.w.p);
    op->end_capture();
    if (!arc) {
      if (n <= kSmallN) {
        mgs_small_kernel<<<1, kST, 0, stream>>>(ws.V.p, ws.ldv, n, 0, ws.w.p, ws.hcol.p, ws.st.p, ws.vin.p);
      } else {
        double* Vp = ws.V.p;
        int64_t ldv = ws.ldv, nn = n;
        int jj = 0;
        double *wp = ws.w.p, *pp = ws.part.p, *hp = ws.hcol.p, *vn = ws.vin.p;
        const GmresState* jd = ws.st.p;
        void* args[] = {&Vp, &ldv, &nn, &jj, &wp, &pp, &hp, &jd, &vn};
        cudaLaunchCooperativeKernel((const void*)mgs_kernel, dim3(ws.grid), dim3(kGT), args, 0, stream);
      }
      givens_kernel<<<1, 1, 0, stream>>>(ws.st.p, ws.hcol.p, ws.H.p, ws.cs.p, ws.sn.p, ws.g.p, cond);
    }
    cudaGraph_t captured = nullptr;
    cudaError_t ce = cudaStreamEndCapture(stream, &captured);
    if (arc) return arc;
    if (ce != cudaSuccess) return cuda_fail(ce, "GMRES cycle capture");
    HOBI_CUDA(cudaGetLastError());
    ws.cycle.step_launches = (launch_counter ? *launch_counter - l0 : 0) + 2;
    if (launch_counter) *launch_counter = l0;  // counted per executed step instead
    HOBI_CUDA(cudaGraphInstantiate(&ws.cycle.exec, graph, 0));
    ws.cycle.key = key;
    return 0;
  };
  auto run_cycle_graph = [&](double beta, int& total_io, int& j_out) -> int {
    if (ws.cycle.key != key || !ws.cycle.exec) {
      int brc = build_graph();
      if (brc) {
        ws.cycle.reset();
        return brc;
      }
    }
    *ws.st_h.p = GmresState{0, total_io, m, max_it, norm_b, tol};
    HOBI_CUDA(cudaMemcpyAsync(ws.st.p, ws.st_h.p, sizeof(GmresState), cudaMemcpyHostToDevice, stream));
    HOBI_CUDA(cudaMemcpyAsync(ws.g.p, &beta, sizeof(double), cudaMemcpyHostToDevice, stream));
    HOBI_CUDA(cudaGraphLaunch(ws.cycle.exec, stream));
    HOBI_CUDA(cudaMemcpyAsync(ws.st_h.p, ws.st.p, sizeof(GmresState), cudaMemcpyDeviceToHost, stream));
    HOBI_CUDA(cudaMemcpyAsync(ws.H_h.p, ws.H.p, (size_t)(m + 1) * m * sizeof(double), cudaMemcpyDeviceToHost,
                              stream));
    HOBI_CUDA(cudaMemcpyAsync(ws.g_h.p, ws.g.p, (m + 1) * sizeof(double), cudaMemcpyDeviceToHost, stream));
    HOBI_CUDA(cudaStreamSynchronize(stream));
    j_out = ws.st_h.p->j;
    total_io = ws.st_h.p->total;
    return 0;
  };
  while (true) {
    if ((rc = op->apply(ws.x.p, ws.w.p))) return rc;
    ++*matvecs;
    double rn = 0.0;
    if ((rc = norm_of(ws.w.p, ws.r.p, &rn))) return rc;
    const double rel = rn / norm_b;
    best = std::min(best, rel);
    if (rel <= tol) {
      *iterations = total;
      *residual = rel;
      *best_out = best;
      HOBI_CUDA(cudaMemcpyAsync(x_host, ws.x.p, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
      HOBI_CUDA(cudaStreamSynchronize(stream));
      if (launch_counter) *launch_counter += launches;
      return 0;
    }
    if (total >= max_it) {
      *iterations = total;
      *residual = rel;
      *best_out = best;
      if (launch_counter) *launch_counter += launches;
      char msg[160];
      snprintf(msg, sizeof(msg), "no convergence in %d iterations (best residual %.3e, tolerance %.3e)",
               total, best, tol);
      return fail(HOBI_ERR_NONCONVERGENCE, msg);
    }
    const double beta = rn;
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(cs.begin(), cs.end(), 0.0);
    std::fill(sn.begin(), sn.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    const bool graph = use_graph && !trace;
    scale_kernel<<<nblk(n, 256), 256, 0, stream>>>(ws.r.p, n, beta, ws.V.p, graph ? ws.vin.p : nullptr);
    launches++;
    g[0] = beta;
    int j = 0;
    if (graph) {  // the whole inner cycle on the device: one graph launch, one read-back
      if ((rc = run_cycle_graph(beta, total, j))) return rc;
      *matvecs += j;
      launches += j * ws.cycle.step_launches;
      if (trace) fprintf(stderr, "gmres cycle (graph): %d steps, total %d\n", j, total);
      for (int i = 0; i <= j && i <= m; ++i)
        for (int k = 0; k < m; ++k) Hat(i, k) = ws.H_h.p[(size_t)i * m + k];
      for (int i = 0; i <= j && i <= m; ++i) g[i] = ws.g_h.p[i];
    }
    while (!graph && j < m && total < max_it) {
      double ta = trace ? (cudaStreamSynchronize(stream), now()) : 0.0;
      if ((rc = op->apply(ws.V.p + (int64_t)j * ws.ldv, ws.w.p))) return rc;
      ++*matvecs;
      double tb = trace ? (cudaStreamSynchronize(stream), now()) : 0.0;
      if (n <= kSmallN) {
        mgs_small_kernel<<<1, kST, 0, stream>>>(ws.V.p, ws.ldv, n, j, ws.w.p, ws.hcol.p, nullptr, nullptr);
        HOBI_CUDA(cudaGetLastError());
        launches++;
      } else {
        double* Vp = ws.V.p;
        int64_t ldv = ws.ldv, nn = n;
        int jj = j;
        double *wp = ws.w.p, *pp = ws.part.p, *hp = ws.hcol.p;
        const GmresState* jd = nullptr;
        double* vn = nullptr;
        void* args[] = {&Vp, &ldv, &nn, &jj, &wp, &pp, &hp, &jd, &vn};
        HOBI_CUDA(cudaLaunchCooperativeKernel((const void*)mgs_kernel, dim3(ws.grid), dim3(kGT), args, 0,
                                              stream));
        launches++;
      }
      HOBI_CUDA(cudaMemcpyAsync(ws.hcol_h.p, ws.hcol.p, (j + 2) * sizeof(double),
                                cudaMemcpyDeviceToHost, stream));
      HOBI_CUDA(cudaStreamSynchronize(stream));
      std::copy(ws.hcol_h.p, ws.hcol_h.p + j + 2, hcol.begin());
      if (trace) {
        double tc = now();
        t_mv += tb - ta;
        t_orth += tc - tb;
        fprintf(stderr, "gmres it %d j %d matvec %.3f ms orth+sync %.3f ms\n", total, j, tb - ta, tc - tb);
      }
      for (int i = 0; i <= j + 1; ++i) Hat(i, j) = hcol[i];
      for (int i = 0; i < j; ++i) {  // apply previous rotations (solver.py:544-547)
        double tmp = cs[i] * Hat(i, j) + sn[i] * Hat(i + 1, j);
        Hat(i + 1, j) = -sn[i] * Hat(i, j) + cs[i] * Hat(i + 1, j);
        Hat(i, j) = tmp;
      }
      double denom = std::hypot(Hat(j, j), Hat(j + 1, j));
      cs[j] = Hat(j, j) / denom;
      sn[j] = Hat(j + 1, j) / denom;
      Hat(j, j) = denom;
      Hat(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++total;
      ++j;
      if (std::fabs(g[j]) / norm_b <= tol) break;
    }
    // y = triu(H[:j,:j]) \ g[:j], column-oriented back substitution (solver.py:559)
    for (int i = 0; i < j; ++i) y[i] = g[i];
    for (int k = j - 1; k >= 0; --k) {
      y[k] /= Hat(k, k);
      for (int i = 0; i < k; ++i) y[i] -= y[k] * Hat(i, k);
    }
    if (j) {
      HOBI_CUDA(cudaMemcpyAsync(ws.y.p, y.data(), j * sizeof(double), cudaMemcpyHostToDevice, stream));
      update_kernel<<<nblk(n, 256), 256, 0, stream>>>(ws.V.p, ws.ldv, n, j, ws.y.p, ws.x.p);
      launches++;
      HOBI_CUDA(cudaGetLastError());
    }
  }
}

}  // namespace hobi

extern "C" int hobi_hypot_check(int device, const double* a, const double* b, int64_t n, double* out) {
  using namespace hobi;
  if (n < 0) return fail(HOBI_ERR_VALUE, "negative size");
  if (n == 0) return 0;
  HOBI_CUDA(cudaSetDevice(device));
  DevBuf<double> da, db, dout;
  if (da.alloc(n) || db.alloc(n) || dout.alloc(n)) return HOBI_ERR_CUDA;
  HOBI_CUDA(cudaMemcpy(da.p, a, n * sizeof(double), cudaMemcpyHostToDevice));
  HOBI_CUDA(cudaMemcpy(db.p, b, n * sizeof(double), cudaMemcpyHostToDevice));
  hypot_check_kernel<<<nblk(n, 256), 256>>>(da.p, db.p, n, dout.p);
  HOBI_CUDA(cudaGetLastError());
  HOBI_CUDA(cudaMemcpy(out, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}
