// All-pairs regular sweep with its prologue (K-C: source
// weights from u) and epilogue (K-D: group reduction + Duffy swap + diagonal),
// plus the energy reduction (K-F) that reuses the sweep.
//
// Reference: _apply_range (solver.py:278-367) -> kernel_values_d
// (kernels.py:99-130); solvation_energy (solver.py:581-614).
//
// Layout in HBM:
//   tgt  : SoA (6, nt_pad)  x', y', z', nx'/nz', ny'/nz', nz'
//          (x' = len_scale * Q x, n' = Q n: the sweep frame, Physics::q)
//   src  : AoS (ns_pad, 10) x', y', z', M n'x, M n'y, M n'z, W1, C, D, 0
//          (M = k^3 wp/4pi screened, (er-1) wp/4pi unscreened; hobi_fastmath.cuh)
//   part : (n_groups, 2, nt_pad) per-source-group partial sums
// The sweep is persistent: each resident CTA pulls work items (a tile of
// 128*R targets held R per thread in registers, x one fixed source group)
// from an atomic ticket; source tiles of kSrcTile records stream through a
// kStages-deep shared-memory ring filled by the TMA bulk-copy engine
// (cp.async.bulk + mbarrier).  Source groups depend only on the problem, never
// on the row split or the tiling, so every row's sum is bitwise identical for
// any number of GPUs (solver.py:12-17).
//
// Instantiations: MODE (screened / kappa = 0), FULL (K3/K4 block too, or the
// K1/K2-only energy sweep), SELF (LOBI self-pair mask, applied only on source
// tiles that overlap the item's rows), R targets per thread, MINB CTAs per SM,
// UNROLL of the source loop, STEP (step-major pair arithmetic).  launch_sweep
// picks an 896-row or a 512-row tile (whichever leaves fewer rows past the last
// whole tile; small ranges: 128-row tiles, or one wide launch), and runs the rows past the
// last whole tile as a second 128-row-tile launch on a second side stream.
#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>

#include "hobi_fastmath.cuh"
#include "hobi_internal.cuh"
#include "hobi_tma.cuh"

namespace hobi {

__device__ __align__(128) double g_exp_table[kExpTable];  // 16-byte aligned for the bulk copy

// Once per device (the table never changes; a sweep running in another
// context reads it, so it is not rewritten under it).
int upload_exp_table() {
  static std::mutex m;
  static std::vector<int> done;
  int dev = 0;
  HOBI_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(m);
  if (dev < (int)done.size() && done[dev]) return 0;
  double t[kExpTable];
  for (int j = 0; j < kExpTable; ++j) t[j] = (double)exp2l((long double)j / kExpTable);
  HOBI_CUDA(cudaMemcpyToSymbol(g_exp_table, t, sizeof(t)));
  if (dev >= (int)done.size()) done.resize(dev + 1, 0);
  done[dev] = 1;
  return 0;
}

// Device address of the table on the current device (for kernels in other
// translation units, which take it as an argument).
const double* exp_table_device() {
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, g_exp_table) != cudaSuccess) return nullptr;
  return static_cast<const double*>(p);
}

namespace {

constexpr uint32_t kTileBytes = kSrcTile * kSrcStride * sizeof(double);
constexpr uint32_t kExpBytes = kExpTable * sizeof(double);
constexpr size_t kSweepSmem =
    (size_t)kStages * kTileBytes + kExpBytes + (kStages + 1) * sizeof(uint64_t);  // ring, exp table, barriers

// Persistent, dynamically scheduled sweep.  Work item = (target tile, source
// group); items are numbered group-major so CTAs running concurrently share a
// source group in L2, and handed out by an atomic ticket so every SM stays busy
// to the end of the launch at any row split (no wave quantisation).  Each
// item's result depends only on its (tile, group), never on which CTA ran it,
// so the sums stay deterministic.  Source tiles of every item flow through one
// continuous kStages-deep TMA ring: `seq` counts tiles across items.
template <int MODE, bool FULL, bool SELF, int R, int MINB, int UNROLL, bool STEP = false>
__global__ void __launch_bounds__(kSweepThreads, MINB) sweep_kernel(
    const double* __restrict__ tgt, int64_t ldt, int64_t t_begin, int64_t t_end,
    const double* __restrict__ src, const int2* __restrict__ groups, int n_groups,
    double* __restrict__ part, int64_t ldp, unsigned* __restrict__ ticket, double Bq, double s2) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);
  double* etab = ring + kStages * kSrcTile * kSrcStride;
  uint64_t* bars = reinterpret_cast<uint64_t*>(etab + kExpTable);
  __shared__ int item_sh;

  constexpr int kTile = kSweepThreads * R;
  const int n_ttiles = (int)((t_end - t_begin + kTile - 1) / kTile);
  const int n_items = n_ttiles * n_groups;

  // The 128-row tile (R == 1) serves small problems and remainder rows, where a
  // CTA runs one or two 64-source items and its start-up is on the critical
  // path (profiles/r02_small_sweep.md): there the exp table arrives by one
  // bulk copy behind its own barrier instead of 16 loads and stores per
  // thread, and the first item is the CTA's own index, so no CTA waits on a
  // ticket round trip before its first tile (nor after its last one when the
  // grid covers every item).  The wide tiles keep the plain prologue: their
  // start-up is amortised over hundreds of tiles, and ptxas schedules their
  // loop measurably worse next to the other prologue (same file).
  constexpr bool kLean = R == 1;
  if (!kLean && MODE == kScreened)
    for (int i = threadIdx.x; i < kExpTable; i += kSweepThreads) etab[i] = g_exp_table[i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages + (kLean ? 1 : 0); ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (kLean && MODE == kScreened) {
      mbar_expect_tx(&bars[kStages], kExpBytes);
      bulk_g2s(etab, g_exp_table, kExpBytes, &bars[kStages]);
    }
  }
  bool etab_pending = kLean && MODE == kScreened;
  uint32_t seq = 0;  // source tiles consumed so far by this CTA (ring position)
  for (int pass = 0;; ++pass) {
    int item;
    if (kLean && pass == 0) {
      item = (int)blockIdx.x;
      __syncthreads();  // barriers initialised
    } else {
      if (kLean && (int)gridDim.x >= n_items) break;  // one item per CTA: nothing left to hand out
      if (threadIdx.x == 0) item_sh = (kLean ? (int)gridDim.x : 0) + (int)atomicAdd(ticket, 1u);
      __syncthreads();
      item = item_sh;
      __syncthreads();
    }
    if (item >= n_items) break;
    const int g = item / n_ttiles;
    const int tt = item - g * n_ttiles;
    const int2 grp = groups[g];  // (first source tile, tile count)
    const int tile0 = grp.x;
    const int ntl = grp.y;
    // thread owns R consecutive targets; warps entirely past the end skip the math
    const int64_t tb = t_begin + (int64_t)tt * kTile + (int64_t)threadIdx.x * R;
    const bool warp_live = t_begin + (int64_t)tt * kTile + (int64_t)(threadIdx.x & ~31) * R < t_end;
    const double* gsrc = src + (int64_t)tile0 * kSrcTile * kSrcStride;
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int s = 0; s < kStages - 1 && s < ntl; ++s) {
        const int st = (int)((seq + s) % kStages);
        mbar_expect_tx(&bars[st], kTileBytes);
        bulk_g2s(ring + st * kSrcTile * kSrcStride, gsrc + (int64_t)s * kSrcTile * kSrcStride,
                 kTileBytes, &bars[st]);
      }
    }
    double tx[R], ty[R], tz[R], nx[R], ny[R];  // normals as (n'x/n'z, n'y/n'z)
    double a1[R], a2[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      int64_t t = min(tb + q, t_end - 1);  // padded slots recompute the last row
      tx[q] = tgt[t];
      ty[q] = tgt[ldt + t];
      tz[q] = tgt[2 * ldt + t];
      nx[q] = tgt[3 * ldt + t];
      ny[q] = tgt[4 * ldt + t];
      a1[q] = 0.0;
      a2[q] = 0.0;
    }
    if (kLean && etab_pending) {  // first item only: the table's bulk copy has landed
      mbar_wait(&bars[kStages], 0u);
      etab_pending = false;
    }
    for (int it = 0; it < ntl; ++it) {
      if (threadIdx.x == 0 && it + kStages - 1 < ntl) {
        const int nxt = it + kStages - 1;
        const int st = (int)((seq + nxt) % kStages);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bars[st], kTileBytes);
        bulk_g2s(ring + st * kSrcTile * kSrcStride, gsrc + (int64_t)nxt * kSrcTile * kSrcStride,
                 kTileBytes, &bars[st]);
      }
      const uint32_t pos = seq + it;
      const int st = (int)(pos % kStages);
      mbar_wait(&bars[st], (pos / kStages) & 1u);
      const double2* rec = reinterpret_cast<const double2*>(ring + st * kSrcTile * kSrcStride);
      // LOBI: only source tiles overlapping this item's target rows hold a
      // self pair; every other tile takes the unmasked path (step-major where
      // the instantiation has one), a branch uniform per CTA.  Both paths give
      // bitwise the same sums.
      bool masked = false;
      if constexpr (SELF) {
        const int64_t s0 = (int64_t)(tile0 + it) * kSrcTile;
        const int64_t tlo = t_begin + (int64_t)tt * kTile;
        masked = s0 < tlo + kTile && s0 + kSrcTile > tlo;
      }
      const bool fast = STEP && !masked;
      if constexpr (STEP) {
        if (fast) {
#pragma unroll UNROLL
          for (int j = 0; j < (warp_live ? kSrcTile : 0); ++j) {
            const double2 p01 = rec[5 * j + 0], p2m0 = rec[5 * j + 1], m12 = rec[5 * j + 2];
            const double2 w01 = rec[5 * j + 3], w2x = rec[5 * j + 4];
            pairs_screened_stepmajor<R>(tx, ty, tz, nx, ny, p01.x, p01.y, p2m0.x, p2m0.y, m12.x,
                                        m12.y, w01.x, w01.y, w2x.x, Bq, etab, a1, a2);
          }
        }
      }
      if (!fast) {
#pragma unroll UNROLL
        for (int j = 0; j < (warp_live ? kSrcTile : 0); ++j) {
          const double2 p01 = rec[5 * j + 0], p2m0 = rec[5 * j + 1], m12 = rec[5 * j + 2];
          const double2 w01 = rec[5 * j + 3], w2x = rec[5 * j + 4];
#pragma unroll
          for (int q = 0; q < R; ++q) {
            double sx = p01.x, sy = p01.y, sz = p2m0.x;
            double mx = p2m0.y, my = m12.x, mz = m12.y, W1 = w01.x, C = w01.y, D = w2x.x;
            if (SELF && masked) {
              // LOBI self pair: displacement forced to (1,0,0) and every weight
              // (the weighted normal included) to 0, so it contributes exactly +0
              // (solver.py:303-310).
              const bool self = ((int64_t)(tile0 + it) * kSrcTile + j) == tb + q;
              if (self) {
                sx = tx[q] - 1.0;
                sy = ty[q];
                sz = tz[q];
                mx = my = mz = W1 = C = D = 0.0;
              }
            }
            if (MODE == kScreened)
              pair_screened<FULL>(tx[q], ty[q], tz[q], nx[q], ny[q], sx, sy, sz, mx, my, mz, W1,
                                  C, D, Bq, etab, a1[q], a2[q]);
            else
              pair_laplace<FULL>(tx[q], ty[q], tz[q], nx[q], ny[q], sx, sy, sz, mx, my, mz, D,
                                 a1[q], a2[q]);
          }
        }
      }
      __syncthreads();
    }
    seq += (uint32_t)ntl;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      int64_t t = tb + q;
      if (t < t_end) {
        part[(2 * (int64_t)g) * ldp + t] = a1[q];
        // acc2 accumulated d.n/n'z terms (the sweep frame) and, screened, a
        // record scaled by Ap = er/kappa (weight_constants): one multiply by
        // n'z * s2 per row and item restores the K3+K4 sum
        if (FULL) part[(2 * (int64_t)g + 1) * ldp + t] = a2[q] * (tgt[5 * ldt + t] * s2);
      }
    }
  }
}

// Scaled static source positions: record fields 0..2; padding records get
// zero weights (fields 3..9), so they contribute exactly +-0.
__device__ __forceinline__ double row3(const Mat3& a, int i, double x, double y, double z) {
  return fma(a.m[3 * i], x, fma(a.m[3 * i + 1], y, a.m[3 * i + 2] * z));
}

__global__ void static_sources_kernel(const double* __restrict__ pos, int64_t ns, int64_t ns_pad,
                                      Mat3 sq, double* __restrict__ src) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= ns_pad) return;
  double* rec = src + s * kSrcStride;
  if (s < ns) {  // x' = (len_scale Q) x
    const double x = pos[3 * s], y = pos[3 * s + 1], z = pos[3 * s + 2];
    rec[0] = row3(sq, 0, x, y, z);
    rec[1] = row3(sq, 1, x, y, z);
    rec[2] = row3(sq, 2, x, y, z);
  } else {  // padding: far away
    rec[0] = 1e6 + (double)(s - ns);
    rec[1] = 1e6;
    rec[2] = 1e6;
  }
  for (int k = 3; k < kSrcStride; ++k) rec[k] = 0.0;
}

// Targets SoA in the sweep frame: x' = (len_scale Q) x, n' = Q n stored as
// (n'x/n'z, n'y/n'z, n'z).  A target whose n'z is zero or below 1e-150 in
// magnitude sets *bad (the caller then picks the next frame).  Charges (no
// normal) get n' = (0, 0, 1).
__global__ void targets_kernel(const double* __restrict__ pos, const double* __restrict__ nrm,
                               int64_t nt, int64_t ldt, Mat3 sq, Mat3 q, double* __restrict__ tgt,
                               int* __restrict__ bad) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= ldt) return;
  int64_t i = t < nt ? t : nt - 1;
  const double x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
  tgt[t] = row3(sq, 0, x, y, z);
  tgt[ldt + t] = row3(sq, 1, x, y, z);
  tgt[2 * ldt + t] = row3(sq, 2, x, y, z);
  double px = 0.0, py = 0.0, nz = 1.0;
  if (nrm) {
    const double a = nrm[3 * i], b = nrm[3 * i + 1], c = nrm[3 * i + 2];
    nz = row3(q, 2, a, b, c);
    if (!(fabs(nz) >= 1e-150)) {
      if (bad) atomicExch(bad, 1);
      nz = 1.0;
    }
    px = row3(q, 0, a, b, c) / nz;
    py = row3(q, 1, a, b, c) / nz;
  }
  tgt[3 * ldt + t] = px;
  tgt[4 * ldt + t] = py;
  tgt[5 * ldt + t] = nz;
}

// K-C: interpolate u onto the regular points and fold the physics into the
// per-source record.  phi_q = v0 b0 + v1 b1 + v2 b2 (solver.py:269-275),
// wphi = reg_w * phi_q (solver.py:321-322); the wp-weighted terms ride on the
// source normal (fields 3..5), the wd-weighted ones are W1, C, D.
__global__ void source_weights_kernel(const double* __restrict__ u, int64_t nt,
                                      const int* __restrict__ faces, const double* __restrict__ reg_w,
                                      const double* __restrict__ bary, int nq, int64_t ns,
                                      const double* __restrict__ area, const double* __restrict__ nrm,
                                      double kM, double kW1, double kC, double kD, Mat3 q,
                                      double* __restrict__ src) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= ns) return;
  double wp, wd;
  if (area) {  // LOBI: centroid collocation, weight = flat area (solver.py:297-298)
    wp = area[s] * u[s];
    wd = area[s] * u[nt + s];
  } else {
    int64_t f = s / nq;
    int m = (int)(s - f * nq);
    int i0 = faces[3 * f], i1 = faces[3 * f + 1], i2 = faces[3 * f + 2];
    double b0 = bary[3 * m], b1 = bary[3 * m + 1], b2 = bary[3 * m + 2];
    double ph = __dadd_rn(__dadd_rn(__dmul_rn(u[i0], b0), __dmul_rn(u[i1], b1)), __dmul_rn(u[i2], b2));
    double dp = __dadd_rn(__dadd_rn(__dmul_rn(u[nt + i0], b0), __dmul_rn(u[nt + i1], b1)),
                          __dmul_rn(u[nt + i2], b2));
    double w = reg_w[s];
    wp = w * ph;
    wd = w * dp;
  }
  double* rec = src + s * kSrcStride;
  const double M = kM * wp;
  const double a = nrm[3 * s], b = nrm[3 * s + 1], c = nrm[3 * s + 2];
  rec[3] = M * row3(q, 0, a, b, c);  // weighted normal in the sweep frame
  rec[4] = M * row3(q, 1, a, b, c);
  rec[5] = M * row3(q, 2, a, b, c);
  rec[6] = kW1 * wd;
  rec[7] = kC * wd;
  rec[8] = kD * wd;
  rec[9] = 0.0;
}

// K-D: fixed-order group reduction + Duffy swap (solver.py:362-363) + diagonal
// (solver.py:365-366).  A block covers 32 consecutive rows (threadIdx.x, so
// every partial-sum load is a coalesced 256-byte row segment) x 8 group
// slices (threadIdx.y: groups y, y+8, ...); the 8 slice sums are folded in a
// fixed order, so each row's result is independent of the row split.
// Row v of [lo, hi) is written to o1[v-lo], o2[v-lo].
constexpr int kEpiRows = 32, kEpiSlices = 8;
__global__ void __launch_bounds__(kEpiRows* kEpiSlices) epilogue_kernel(
    const double* __restrict__ part, int64_t ldp, int n_groups, const double* __restrict__ corr,
    const int* __restrict__ pair_starts, const double* __restrict__ u, int64_t nt, int64_t lo,
    int64_t hi, double diag1, double diag2, double* __restrict__ o1, double* __restrict__ o2) {
  __shared__ double s1[kEpiSlices][kEpiRows], s2[kEpiSlices][kEpiRows];
  const int64_t v = lo + (int64_t)blockIdx.x * kEpiRows + threadIdx.x;
  const int64_t vv = v < hi ? v : hi - 1;
  double a1 = 0.0, a2 = 0.0;
  // unrolled so the independent partial loads issue back to back (the adds
  // keep their group order: same bits, a fraction of the load latency)
#pragma unroll 4
  for (int g = threadIdx.y; g < n_groups; g += kEpiSlices) {
    a1 += part[(2 * (int64_t)g) * ldp + vv];
    a2 += part[(2 * (int64_t)g + 1) * ldp + vv];
  }
  s1[threadIdx.y][threadIdx.x] = a1;
  s2[threadIdx.y][threadIdx.x] = a2;
  __syncthreads();
  if (threadIdx.y != 0 || v >= hi) return;
  double acc1 = ((s1[0][threadIdx.x] + s1[1][threadIdx.x]) + (s1[2][threadIdx.x] + s1[3][threadIdx.x])) +
                ((s1[4][threadIdx.x] + s1[5][threadIdx.x]) + (s1[6][threadIdx.x] + s1[7][threadIdx.x]));
  double acc2 = ((s2[0][threadIdx.x] + s2[1][threadIdx.x]) + (s2[2][threadIdx.x] + s2[3][threadIdx.x])) +
                ((s2[4][threadIdx.x] + s2[5][threadIdx.x]) + (s2[6][threadIdx.x] + s2[7][threadIdx.x]));
  if (corr) {
    double c1 = 0.0, c2 = 0.0;
    for (int p = pair_starts[v]; p < pair_starts[v + 1]; ++p) {
      c1 += corr[2 * (int64_t)p];
      c2 += corr[2 * (int64_t)p + 1];
    }
    acc1 += c1;
    acc2 += c2;
  }
  o1[v - lo] = __dsub_rn(__dmul_rn(diag1, u[v]), acc1);
  o2[v - lo] = __dsub_rn(__dmul_rn(diag2, u[nt + v]), acc2);
}

// Fused epilogue + gather over NVLink (P2P mode): the same fixed-order row
// reduction as epilogue_kernel, but every finished row is stored straight
// into all ranks' receive buffers (final layout, phi rows then dphi rows) by
// peer stores; the last block to finish fences and bumps every rank's
// arrival counter for this epoch parity with a system-scope atomic.
__global__ void __launch_bounds__(kEpiRows* kEpiSlices) epilogue_p2p_kernel(
    const double* __restrict__ part, int64_t ldp, int n_groups, const double* __restrict__ corr,
    const int* __restrict__ pair_starts, const double* __restrict__ u, int64_t nt, int64_t lo,
    int64_t hi, double diag1, double diag2, double* const* __restrict__ peers, int nranks, int rank,
    int parity, unsigned* __restrict__ done) {
  __shared__ double s1[kEpiSlices][kEpiRows], s2[kEpiSlices][kEpiRows];
  const int64_t v = lo + (int64_t)blockIdx.x * kEpiRows + threadIdx.x;
  const int64_t vv = v < hi ? v : hi - 1;
  double a1 = 0.0, a2 = 0.0;
#pragma unroll 4
  for (int g = threadIdx.y; hi > lo && g < n_groups; g += kEpiSlices) {
    a1 += part[(2 * (int64_t)g) * ldp + vv];
    a2 += part[(2 * (int64_t)g + 1) * ldp + vv];
  }
  s1[threadIdx.y][threadIdx.x] = a1;
  s2[threadIdx.y][threadIdx.x] = a2;
  __syncthreads();
  if (threadIdx.y == 0 && v < hi) {
    double acc1 = ((s1[0][threadIdx.x] + s1[1][threadIdx.x]) + (s1[2][threadIdx.x] + s1[3][threadIdx.x])) +
                  ((s1[4][threadIdx.x] + s1[5][threadIdx.x]) + (s1[6][threadIdx.x] + s1[7][threadIdx.x]));
    double acc2 = ((s2[0][threadIdx.x] + s2[1][threadIdx.x]) + (s2[2][threadIdx.x] + s2[3][threadIdx.x])) +
                  ((s2[4][threadIdx.x] + s2[5][threadIdx.x]) + (s2[6][threadIdx.x] + s2[7][threadIdx.x]));
    if (corr) {
      double c1 = 0.0, c2 = 0.0;
      for (int p = pair_starts[v]; p < pair_starts[v + 1]; ++p) {
        c1 += corr[2 * (int64_t)p];
        c2 += corr[2 * (int64_t)p + 1];
      }
      acc1 += c1;
      acc2 += c2;
    }
    const double r1 = __dsub_rn(__dmul_rn(diag1, u[v]), acc1);
    const double r2 = __dsub_rn(__dmul_rn(diag2, u[nt + v]), acc2);
    const int64_t off = (int64_t)parity * 2 * nt;
    for (int r = 0; r < nranks; ++r) {  // peer stores over NVLink (own buffer for r == rank)
      peers[r][off + v] = r1;
      peers[r][off + nt + v] = r2;
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    const unsigned prev = atomicAdd(done, 1u);
    if (prev == gridDim.x - 1) {  // last block: every row of this rank is out
      __threadfence_system();
      // counter (parity, this rank) in every rank's area: one writer per
      // counter, so a rank running ahead can never stand in for a late one
      for (int r = 0; r < nranks; ++r) {
        unsigned long long* flag =
            reinterpret_cast<unsigned long long*>(peers[r] + 4 * nt) + parity * kMaxRanks + rank;
        atomicAdd_system(flag, 1ull);
      }
      *done = 0u;
    }
  }
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Wait until all ranks' rows of this epoch have arrived, then hand the
// gathered vector to the caller's buffer.  A watchdog bounds the wait: after
// timeout_ns the kernel raises *err (mapped host memory) and exits.
__global__ void p2p_wait_copy_kernel(const double* __restrict__ area, int64_t nt, int nranks, int parity,
                                     unsigned long long target, unsigned long long timeout_ns,
                                     int* err, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    volatile unsigned long long* flag =
        reinterpret_cast<volatile unsigned long long*>(const_cast<double*>(area) + 4 * nt) +
        parity * kMaxRanks;
    const unsigned long long t0 = global_ns();
    bool late = false;
    for (int r = 0; r < nranks && !late; ++r)
      while (flag[r] < target) {
        if (global_ns() - t0 > timeout_ns) {  // a peer is gone: report instead of hanging the GPU
          *reinterpret_cast<volatile int*>(err) = 1;
          late = true;
          break;
        }
        __nanosleep(128);
      }
    __threadfence_system();
  }
  __syncthreads();
  const double* buf = area + (int64_t)parity * 2 * nt;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 2 * nt;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = __ldcv(buf + k);
}

// Gathered rank-major rows [r][2][m] -> out[0:nt] ++ out[nt:2nt].
__global__ void permute_kernel(const double* __restrict__ recv, int64_t m, int64_t nt, int nranks,
                               double* __restrict__ out) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nt) return;
  int64_t base = nt / nranks, extra = nt % nranks;
  int64_t cut = extra * (base + 1);
  int64_t r = v < cut ? v / (base + 1) : extra + (v - cut) / (base ? base : 1);
  int64_t lo = r < extra ? r * (base + 1) : cut + (r - extra) * base;
  out[v] = recv[(r * 2) * m + (v - lo)];
  out[nt + v] = recv[(r * 2 + 1) * m + (v - lo)];
}

// Energy (solver.py:608-614): per-charge group sums in fixed group order,
// q_k * sum_k, then one block folds the charges in a fixed tree order.
__global__ void energy_charge_kernel(const double* __restrict__ part, int64_t ldp, int n_groups,
                                     const double* __restrict__ q, int64_t k0, int64_t k1,
                                     double* __restrict__ v) {
  int64_t k = k0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= k1) return;
  double s = part[k];
  for (int g = 1; g < n_groups; ++g) s += part[(2 * (int64_t)g) * ldp + k];
  v[k - k0] = q[k] * s;
}

// rank-major [r][m] slots of per-charge values -> charge order
__global__ void permute1_kernel(const double* __restrict__ recv, int64_t m, int64_t n, int nranks,
                                double* __restrict__ out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int64_t base = n / nranks, extra = n % nranks, cut = extra * (base + 1);
  int64_t r = k < cut ? k / (base + 1) : extra + (k - cut) / (base ? base : 1);
  int64_t lo = r < extra ? r * (base + 1) : cut + (r - extra) * base;
  out[k] = recv[r * m + (k - lo)];
}

__global__ void energy_fold_kernel(const double* __restrict__ v, int64_t nc, double* __restrict__ out) {
  __shared__ double sh[1024];
  double acc = 0.0;
  for (int64_t k = threadIdx.x; k < nc; k += blockDim.x) acc += v[k];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = 0.5 * kFourPi * kKcal * sh[0];
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

int collect_sweep_timing(hobi_ctx* c) {
  for (size_t k = 0; k + 1 < c->ev_used; k += 2) {
    HOBI_CUDA(cudaEventSynchronize(c->ev_pool[k + 1]));
    float ms = 0.f;
    HOBI_CUDA(cudaEventElapsedTime(&ms, c->ev_pool[k], c->ev_pool[k + 1]));
    c->sweep_ms += ms;
    c->sweep_launches++;
  }
  c->ev_used = 0;
  return 0;
}

namespace {

typedef void (*SweepFn)(const double*, int64_t, int64_t, int64_t, const double*, const int2*, int,
                        double*, int64_t, unsigned*, double, double);

struct SweepVariant {
  SweepFn fn;
  int r;  // targets per thread
  const char* name;
};

// Tuning variants of the hot instantiation (screened, full, no self mask):
// targets per thread x min CTAs per SM (register cap) x source unroll.
#define HOBI_V(R, M, U) \
  { sweep_kernel<kScreened, true, false, R, M, U>, R, "R" #R "_minb" #M "_unroll" #U }
#define HOBI_VS(R, M, U) \
  { sweep_kernel<kScreened, true, false, R, M, U, true>, R, "step_R" #R "_minb" #M "_unroll" #U }
static const SweepVariant kVariants[] = {
    HOBI_V(2, 1, 2), HOBI_V(2, 6, 2), HOBI_V(4, 3, 2), HOBI_V(1, 8, 2), HOBI_V(4, 3, 1),
    HOBI_V(4, 4, 1), HOBI_V(3, 4, 1), HOBI_V(6, 2, 1), HOBI_V(8, 2, 1), HOBI_V(3, 4, 2),
    HOBI_V(4, 4, 2), HOBI_V(5, 3, 1), HOBI_VS(6, 2, 1), HOBI_VS(4, 3, 1), HOBI_VS(3, 4, 1),
    HOBI_VS(4, 3, 2), HOBI_VS(4, 3, 4), HOBI_VS(6, 2, 2), HOBI_VS(3, 4, 2), HOBI_VS(5, 3, 2),
    HOBI_VS(8, 2, 2), HOBI_VS(6, 2, 3), HOBI_VS(7, 2, 3), HOBI_V(1, 8, 4), HOBI_V(1, 8, 8),
    HOBI_V(1, 6, 4), HOBI_V(1, 4, 8), HOBI_V(1, 5, 6), HOBI_V(1, 3, 12),
};
#undef HOBI_V
#undef HOBI_VS
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);
// LOBI (self-pair mask) counterparts of the wide / narrow / small tiles.
static const SweepVariant kSelfVariants[] = {
    {sweep_kernel<kScreened, true, true, 7, 2, 3, true>, 7, "self_step_R7_minb2_unroll3"},
    {sweep_kernel<kScreened, true, true, 4, 3, 2, true>, 4, "self_step_R4_minb3_unroll2"},
    {sweep_kernel<kScreened, true, true, 1, 3, 12>, 1, "self_R1_minb3_unroll12"},
};
// kappa = 0 (Laplace instantiation, no step-major form needed): wide / narrow
// / small tiles, without and with the LOBI self mask.
static const SweepVariant kLaplaceVariants[] = {
    {sweep_kernel<kLaplace, true, false, 7, 2, 3>, 7, "laplace_R7_minb2_unroll3"},
    {sweep_kernel<kLaplace, true, false, 4, 3, 2>, 4, "laplace_R4_minb3_unroll2"},
    {sweep_kernel<kLaplace, true, false, 1, 3, 12>, 1, "laplace_R1_minb3_unroll12"},
};
// energy sweeps (K1/K2 only, charges as targets), screened and kappa = 0
static const SweepVariant kEnergyVariants[] = {
    {sweep_kernel<kScreened, false, false, 7, 2, 3>, 7, "energy_R7_minb2_unroll3"},
    {sweep_kernel<kScreened, false, false, 4, 3, 2>, 4, "energy_R4_minb3_unroll2"},
    {sweep_kernel<kScreened, false, false, 1, 3, 12>, 1, "energy_R1_minb3_unroll12"},
};
static const SweepVariant kEnergyLaplaceVariants[] = {
    {sweep_kernel<kLaplace, false, false, 7, 2, 3>, 7, "energy_laplace_R7_minb2_unroll3"},
    {sweep_kernel<kLaplace, false, false, 4, 3, 2>, 4, "energy_laplace_R4_minb3_unroll2"},
    {sweep_kernel<kLaplace, false, false, 1, 3, 12>, 1, "energy_laplace_R1_minb3_unroll12"},
};
static const SweepVariant kLaplaceSelfVariants[] = {
    {sweep_kernel<kLaplace, true, true, 7, 2, 3>, 7, "laplace_self_R7_minb2_unroll3"},
    {sweep_kernel<kLaplace, true, true, 4, 3, 2>, 4, "laplace_self_R4_minb3_unroll2"},
    {sweep_kernel<kLaplace, true, true, 1, 3, 12>, 1, "laplace_self_R1_minb3_unroll12"},
};
// R1_minb3_unroll12: 128-row tiles with twelve sources in flight per thread
// (112 registers): the 128-row tile runs with few warps per SM, so its FP64
// dependence chains need the instruction-level parallelism (config 1: 0.026 ms
// vs 0.030 for unroll 4 and 0.039 for unroll 2; pinned on config 4: 38.9 vs
// 39.7 ms; profiles/r02_small_configs.md)
constexpr int kSmallVariant = 28;
constexpr int kWideVariant = 22;   // step_R7_minb2_unroll3: 896-row tiles, the default
constexpr int kNarrowVariant = 15; // step_R4_minb3_unroll2: 512-row tiles
static_assert(kWideVariant < kNumVariants && kNarrowVariant < kNumVariants && kSmallVariant < kNumVariants,
              "variant table");

// Physics folded into the per-source record and two launch constants (see
// hobi_fastmath.cuh).  Screened: with Ap = er/k, Bp = (er-1)/k the wp-weighted
// normal carries M = Ap k^3 wp/4pi, so M' (a + Bq) with Bq = Bp/Ap is the K2
// factor u (a Ap + Bp) of the unscaled record and the a*Ap DFMA becomes a DADD;
// C and D carry the same Ap so the K3+K4 sum comes out scaled by Ap, undone by
// s2 = 1/Ap when an item stores its row partials.
struct WeightConstants {
  double kM, kW1, kC, kD, Bq, s2;
};
WeightConstants weight_constants(const Physics& p) {
  WeightConstants w{};
  w.s2 = 1.0;
  if (p.mode == kScreened) {
    const double k = p.kappa, k4 = k / kFourPi;
    w.kM = k * k4 * p.er;             // Ap k^3/4pi = er k^2/4pi
    w.kW1 = -k4;                      // -k/4pi
    w.kC = k4;                        // Ap k^2/(4pi er) = k/4pi
    w.kD = -k4 * (p.er - 1.0);        // -Ap k^2 (1-1/er)/4pi
    w.Bq = (p.er - 1.0) / p.er;       // Bp/Ap
    w.s2 = k / p.er;                  // 1/Ap
  } else {
    w.kM = (p.er - 1.0) / kFourPi;
    w.kD = -(1.0 - 1.0 / p.er) / kFourPi;
  }
  return w;
}

// Sweep phase of one operator application over rows [t0, t1).  The tuned
// wide-tile sweep runs on the main stream; concurrently, on the side stream,
// the Duffy swap of those rows (when swap_u is given: it needs only u) and the
// remainder rows past the last whole wide tile, with 128-row tiles.  The side
// stream is joined before returning (in stream order).
int launch_sweep(hobi_ctx* c, const double* tgt, int64_t ldt, int64_t t0, int64_t t1, bool full,
                 double* part, int64_t ldp, const int2* groups, int n_groups,
                 const double* swap_u = nullptr) {
  if (t1 <= t0) return 0;
  const bool self = c->scheme == kLobi && full;
  // up to two launches over disjoint row ranges: the tuned tile over whole
  // tiles, and 128-row tiles over the remainder.  An item costs the same
  // whether its tile is full or not, so a part-filled last wide tile would
  // waste up to a tile's worth of time per source group (4.8% of a 4-way
  // split of config 4); splitting it off keeps every row's sum unchanged.
  struct Seg {
    SweepFn fn;
    int r;
    int64_t a, b;
  } seg[2];
  int nseg = 1;
  seg[0] = {nullptr, kSweepR, t0, t1};
  {
    {
      // the tuning table for screened HOBI; LOBI (self mask), kappa = 0 and
      // the energy sweep run the same tile choice on their own wide / narrow /
      // small instantiations
      const bool scr = c->phys.mode == kScreened;
      const bool tuned = scr && full && !self;
      const SweepVariant* tab = tuned ? kVariants
                                : !full ? (scr ? kEnergyVariants : kEnergyLaplaceVariants)
                                : scr ? kSelfVariants
                                : self ? kLaplaceSelfVariants : kLaplaceVariants;
      const int wide = tuned ? kWideVariant : 0, narrow = tuned ? kNarrowVariant : 1,
                small = tuned ? kSmallVariant : 2;
      int vi = tuned ? c->sweep_variant : wide;
      const bool pinned = c->variant_pinned && tuned;
      // the wide tile is ~2% faster per pair, but the rows past the last
      // whole tile cost more than their share (a side launch of 128-row
      // tiles beside the persistent main launch): switch to the narrow tile
      // when the wide one would leave more than 5% of the rows and the narrow
      // one fewer (config 4 keeps 896-row tiles and 642 remainder rows, as
      // do its 2- and 4-way splits; the 8-way split leaves 641 of 5,121 rows
      // vs 1 and switches).
      if (!pinned && vi == wide) {
        const int64_t rows = t1 - t0;
        const int64_t rem_w = rows % (kSweepThreads * tab[wide].r);
        const int64_t rem_n = rows % (kSweepThreads * tab[narrow].r);
        if (rem_n < rem_w && rem_w * 20 > rows) vi = narrow;
      }
      // small problems: if the tuned tile leaves too few work items for 148
      // SMs, use 128-row tiles (same sums bitwise, more parallelism) -- unless
      // the wide tile, run as one launch with a part-filled last tile, still
      // gives every CTA slot two items: then the wide tile's cheaper pairs win
      // (config 2: 0.182 vs 0.197 ms per sweep; config 1 keeps the 128-row
      // tile, 0.033 vs 0.052 ms; profiles/r02_small_configs.md)
      const int64_t items = (int64_t)nblk(t1 - t0, kSweepThreads * tab[vi].r) * n_groups;
      const int64_t wide_items = (int64_t)nblk(t1 - t0, kSweepThreads * tab[wide].r) * n_groups;
      bool single = false;
      if (!pinned && items < 8 * 296) {
        single = wide_items >= 2 * 296;
        vi = single ? wide : small;
      }
      seg[0].fn = tab[vi].fn;
      seg[0].r = tab[vi].r;
      const int64_t tile = (int64_t)kSweepThreads * seg[0].r;
      const int64_t whole = (t1 - t0) / tile * tile;
      if (!pinned && !single && seg[0].r > 1 && whole > 0 && whole < t1 - t0) {
        seg[0].b = t0 + whole;
        seg[1] = {tab[small].fn, tab[small].r, t0 + whole, t1};
        nseg = 2;
      }
    }
  }
  if (!c->sms) HOBI_CUDA(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device));
  const int sms = c->sms;
  const WeightConstants wc = weight_constants(c->phys);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->timing) {  // brackets are read lazily by collect_sweep_timing: no sync here
    if (c->ev_used + 2 > c->ev_pool.size()) {
      for (int k = 0; k < 2; ++k) {
        cudaEvent_t e;
        HOBI_CUDA(cudaEventCreate(&e));
        c->ev_pool.push_back(e);
      }
    }
    e0 = c->ev_pool[c->ev_used];
    e1 = c->ev_pool[c->ev_used + 1];
    c->ev_used += 2;
    HOBI_CUDA(cudaEventRecord(e0, c->stream));
  }
  // Duffy swap on the side stream, remainder rows on a second side stream
  // (behind the swap they would start only after the swap, typically at the
  // end of the persistent main launch: 1.7% of an 8-way split's rank time)
  const bool use_side = nseg == 2 || swap_u;
  if (use_side) {
    HOBI_CUDA(cudaEventRecord(c->fork, c->stream));
    if (swap_u) {
      HOBI_CUDA(cudaStreamWaitEvent(c->side, c->fork, 0));
      int rc = launch_singular(c, swap_u, c->h_pair_starts[t0], c->h_pair_starts[t1], c->side);
      if (rc) return rc;
    }
    if (nseg == 2) HOBI_CUDA(cudaStreamWaitEvent(c->side2, c->fork, 0));
  }
  for (int k = nseg - 1; k >= 0; --k) {  // remainder first, so it is queued early
    const Seg& sg = seg[k];
    cudaStream_t st = k == 1 ? c->side2 : c->stream;
    unsigned* ticket = k == 1 ? c->ticket.p + 1 : c->ticket.p;
    int per_sm = -1;
    for (const auto& o : c->occupancy)
      if (o.first == (const void*)sg.fn) per_sm = o.second;
    if (per_sm < 0) {
      HOBI_CUDA(cudaFuncSetAttribute(sg.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem));
      HOBI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sg.fn, kSweepThreads, kSweepSmem));
      c->occupancy.emplace_back((const void*)sg.fn, per_sm);
    }
    const int64_t items = (int64_t)nblk(sg.b - sg.a, kSweepThreads * sg.r) * n_groups;
    const unsigned grid =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)std::max(per_sm, 1) * sms));
    HOBI_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), st));
    sg.fn<<<grid, kSweepThreads, kSweepSmem, st>>>(tgt, ldt, sg.a, sg.b, c->src.p, groups, n_groups, part,
                                                   ldp, ticket, wc.Bq, wc.s2);
    HOBI_CUDA(cudaGetLastError());
    c->launches++;
  }
  if (swap_u) {
    HOBI_CUDA(cudaEventRecord(c->join, c->side));
    HOBI_CUDA(cudaStreamWaitEvent(c->stream, c->join, 0));
  }
  if (nseg == 2) {
    HOBI_CUDA(cudaEventRecord(c->join2, c->side2));
    HOBI_CUDA(cudaStreamWaitEvent(c->stream, c->join2, 0));
  }
  if (c->timing) {
    HOBI_CUDA(cudaEventRecord(e1, c->stream));
    if (c->ev_used >= 256 && collect_sweep_timing(c)) return HOBI_ERR_CUDA;
  }
  return 0;
}


}  // namespace

// Fixed partition of the source tiles into groups -- a function of the
// problem size only, so row sums never depend on the row split.  Bulk groups
// of B tiles come first; the end of the source axis is cut into groups that
// halve in size (B/2, B/2, B/4, B/4, ..., 1, 1), so the group-major work queue
// of the persistent sweep ends with small items and the dynamic tail is short.
// B gives an 8-way split with `tiles8` reference tiles per rank ~16 work
// items per 2 x 148 CTA slots (more with the tuned 3-CTA/SM, 512-row tile).
std::vector<int2> make_groups(int n_src_tiles, int64_t tiles8) {
  std::vector<int2> g;
  if (n_src_tiles <= 0) return g;
  const int64_t want = std::max<int64_t>(1, (16 * 2 * 148 + tiles8 - 1) / tiles8);
  // large problems get at least 4 tiles (256 sources) per group, so the
  // partial sums cost <= 1/16 B of HBM traffic per pair.  Coarser groups
  // shrink the partial-sum buffer but starve split ranks of work items: a
  // 32-tile floor (config 4: 169 groups, 111 MB instead of 645 / 423 MB) cut
  // the one-GPU model of a 4- and 8-way split of config 4 from 98.1% and 96.1% to 88.5%
  // and 85.5% efficiency (profiles/r02_group_floor.md), so the floor stays 4.
  const int floor = n_src_tiles >= 1024 ? 4 : 1;
  const int B = (int)std::max<int64_t>(floor, (n_src_tiles + want - 1) / want);
  std::vector<int> tail;
  int tail_sum = 0;
  for (int s = 1; s < B; s *= 2) {
    if (tail_sum + 2 * s > n_src_tiles / 2) break;
    tail.push_back(s);
    tail.push_back(s);
    tail_sum += 2 * s;
  }
  int t = 0;
  const int bulk = n_src_tiles - tail_sum;
  for (; t + B <= bulk; t += B) g.push_back(make_int2(t, B));
  if (t < bulk) {
    g.push_back(make_int2(t, bulk - t));
    t = bulk;
  }
  for (int k = (int)tail.size() - 1; k >= 0; --k) {
    g.push_back(make_int2(t, tail[k]));
    t += tail[k];
  }
  return g;
}

int sweep_variant_count() { return kNumVariants; }
const char* sweep_variant_name(int v) { return (v >= 0 && v < kNumVariants) ? kVariants[v].name : ""; }


// Rotation k of a fixed sequence of generic frames (Rodrigues; axis and angle
// chosen away from the coordinate planes that icosphere and MSMS meshes tend
// to populate with exactly zero normal components).
void set_frame(Physics& p, int k) {
  const double ax = 1.0, ay = 1.0 + 0.37 * k, az = 1.61 + 0.23 * k;
  const double n = std::sqrt(ax * ax + ay * ay + az * az);
  const double x = ax / n, y = ay / n, z = az / n;
  const double th = 0.0625 * (1.0 + 0.5 * k), co = std::cos(th), si = std::sin(th), t = 1.0 - co;
  const double q[9] = {t * x * x + co,     t * x * y - si * z, t * x * z + si * y,
                       t * x * y + si * z, t * y * y + co,     t * y * z - si * x,
                       t * x * z - si * y, t * y * z + si * x, t * z * z + co};
  p.frame = k;
  for (int i = 0; i < 9; ++i) p.q[i] = q[i];
}

static Mat3 frame_rot(const Physics& p) {
  Mat3 m;
  for (int i = 0; i < 9; ++i) m.m[i] = p.q[i];
  return m;
}
static Mat3 frame_pos(const Physics& p) {  // len_scale * Q for positions
  Mat3 m;
  for (int i = 0; i < 9; ++i) m.m[i] = p.len_scale * p.q[i];
  return m;
}

int prepare_targets(hobi_ctx* c) {
  const double* pos = c->scheme == kHobi ? c->vert.p : c->reg_pos.p;  // lobi: centroids
  const double* nrm = c->scheme == kHobi ? c->vnrm.p : c->reg_nrm.p;
  DevBuf<int> bad;
  if (bad.alloc(1)) return HOBI_ERR_CUDA;
  // test hook: frames below this index count as rejected (exercises the retry)
  const char* rej = getenv("HOBI_TEST_FRAME_REJECT");
  const int reject_below = rej ? atoi(rej) : 0;
  for (int k = c->phys.frame; k < kNumFrames; ++k) {
    set_frame(c->phys, k);
    HOBI_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c->stream));
    targets_kernel<<<nblk(c->nt_pad, 256), 256, 0, c->stream>>>(
        pos, nrm, c->nt, c->nt_pad, frame_pos(c->phys), frame_rot(c->phys), c->tgt.p, bad.p);
    c->launches++;
    HOBI_CUDA(cudaGetLastError());
    int h = 0;
    HOBI_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    HOBI_CUDA(cudaStreamSynchronize(c->stream));
    if (!h && k >= reject_below) return 0;
  }
  return fail(HOBI_ERR_VALUE, "no sweep frame gives every collocation normal a nonzero z component");
}

int prepare_static_sources(hobi_ctx* c) {
  static_sources_kernel<<<nblk(c->ns_pad, 256), 256, 0, c->stream>>>(
      c->reg_pos.p, c->ns, c->ns_pad, frame_pos(c->phys), c->src.p);
  c->launches++;
  HOBI_CUDA(cudaGetLastError());
  return 0;
}

static int update_weights(hobi_ctx* c, const double* u_dev) {
  const WeightConstants w = weight_constants(c->phys);
  source_weights_kernel<<<nblk(c->ns, 256), 256, 0, c->stream>>>(
      u_dev, c->nt, c->faces.p, c->reg_w.p, c->reg_bary.p, c->nq, c->ns,
      c->scheme == kLobi ? c->lobi_area.p : nullptr, c->reg_nrm.p, w.kM, w.kW1, w.kC, w.kD,
      frame_rot(c->phys), c->src.p);
  c->launches++;
  HOBI_CUDA(cudaGetLastError());
  return 0;
}

int matvec_rows_device(hobi_ctx* c, const double* u_dev, int64_t lo, int64_t hi, double* o1,
                       double* o2) {
  if (hi <= lo) return 0;
  int rc;
  const bool hobi = c->scheme == kHobi;
  if ((rc = update_weights(c, u_dev))) return rc;
  if ((rc = launch_sweep(c, c->tgt.p, c->nt_pad, lo, hi, true, c->part.p, c->nt_pad, c->groups.p,
                         c->n_groups, hobi ? u_dev : nullptr)))
    return rc;
  const double* corr = hobi ? c->corr.p : nullptr;
  const int* starts = hobi ? c->pair_starts.p : nullptr;
  epilogue_kernel<<<nblk(hi - lo, kEpiRows), dim3(kEpiRows, kEpiSlices), 0, c->stream>>>(
      c->part.p, c->nt_pad, c->n_groups, corr, starts, u_dev, c->nt, lo, hi, c->phys.diag1,
      c->phys.diag2, o1, o2);
  c->launches++;
  HOBI_CUDA(cudaGetLastError());
  return 0;
}

// Row split with the gather fused into the epilogue (peer stores + arrival
// counters) instead of ncclAllGather + permutation.  Two halves: the send
// half computes this rank's rows and stores them into every rank's receive
// area (bumping the arrival counters); the receive half waits for every
// rank's arrivals of this epoch and copies the gathered vector out.
int matvec_p2p_send(hobi_ctx* c, const double* u_dev) {
  const int64_t lo = c->lo, hi = c->hi;
  const int parity = (int)(c->comm.epoch & 1);
  int rc;
  const bool hobi = c->scheme == kHobi;
  if (hi > lo) {
    if ((rc = update_weights(c, u_dev))) return rc;
    if ((rc = launch_sweep(c, c->tgt.p, c->nt_pad, lo, hi, true, c->part.p, c->nt_pad, c->groups.p,
                           c->n_groups, hobi ? u_dev : nullptr)))
      return rc;
  }
  // an empty range still launches one block so this rank signals its arrival
  const unsigned blocks = hi > lo ? nblk(hi - lo, kEpiRows) : 1;
  epilogue_p2p_kernel<<<blocks, dim3(kEpiRows, kEpiSlices), 0, c->stream>>>(
      c->part.p, c->nt_pad, c->n_groups, hobi ? c->corr.p : nullptr,
      hobi ? c->pair_starts.p : nullptr, u_dev, c->nt, lo, hi,
      c->phys.diag1, c->phys.diag2, c->p2p_peers.p, c->comm.nranks, c->comm.rank, parity,
      c->p2p_done.p);
  c->launches++;
  HOBI_CUDA(cudaGetLastError());
  return 0;
}

int matvec_p2p_recv(hobi_ctx* c, double* out_dev) {
  const int parity = (int)(c->comm.epoch & 1);
  const unsigned long long target = c->comm.epoch / 2 + 1 + c->p2p_extra;  // arrivals per rank
  p2p_wait_copy_kernel<<<std::max(1u, nblk(2 * c->nt, 1024)), 256, 0, c->stream>>>(
      c->p2p_area.p, c->nt, c->comm.nranks, parity, target, c->p2p_timeout_ns, c->p2p_err_dev, out_dev);
  c->launches++;
  HOBI_CUDA(cudaGetLastError());
  c->comm.epoch++;
  return 0;
}

static int matvec_p2p(hobi_ctx* c, const double* u_dev, double* out_dev) {
  int rc = matvec_p2p_send(c, u_dev);
  return rc ? rc : matvec_p2p_recv(c, out_dev);
}

int matvec_full_device(hobi_ctx* c, const double* u_dev, double* out_dev) {
  int rc;
  if (c->comm.p2p) {
    if (c->comm.p2p_pending) return fail(HOBI_ERR_STATE, "a P2P send phase is pending (hobi_matvec_p2p_phase)");
    return matvec_p2p(c, u_dev, out_dev);
  }
  if (c->comm.nranks == 1 && !c->comm.nccl)
    return matvec_rows_device(c, u_dev, 0, c->nt, out_dev, out_dev + c->nt);
  if (!c->comm.emulated && !c->comm.nccl)
    return fail(HOBI_ERR_STATE, "row split without a gather: the P2P communicator's peer areas are not open");
  const int64_t m = c->gather_m;
  if (c->comm.emulated) {  // every rank's rows, computed here, in the gather layout
    for (int r = 0; r < c->comm.nranks; ++r) {
      int64_t base = c->nt / c->comm.nranks, extra = c->nt % c->comm.nranks;
      int64_t lo = r * base + (r < extra ? r : extra);
      int64_t hi = lo + base + (r < extra ? 1 : 0);
      double* slot = c->gather_recv.p + (int64_t)r * 2 * m;
      if ((rc = matvec_rows_device(c, u_dev, lo, hi, slot, slot + m))) return rc;
    }
  } else {
    if ((rc = matvec_rows_device(c, u_dev, c->lo, c->hi, c->gather_send.p, c->gather_send.p + m)))
      return rc;
    if ((rc = comm_allgather(c))) return rc;
  }
  return gather_permute(c, out_dev);
}

// Called after a synchronisation: did a P2P wait give up on a peer?
int p2p_check(hobi_ctx* c) {
  if (c->comm.p2p && c->p2p_err && *reinterpret_cast<volatile int*>(c->p2p_err))
    return fail(HOBI_ERR_NCCL,
                "P2P gather: rows of a peer rank did not arrive within HOBI_P2P_TIMEOUT_MS");
  return 0;
}

int gather_permute(hobi_ctx* c, double* out_dev) {
  permute_kernel<<<nblk(c->nt, 256), 256, 0, c->stream>>>(c->gather_recv.p, c->gather_m, c->nt,
                                                           c->comm.nranks, out_dev);
  c->launches++;
  HOBI_CUDA(cudaGetLastError());
  return 0;
}

// Buffers for a charge set of size nc, kept by the context (see GmresWorkspace).
int charge_workspace(hobi_ctx* c, int64_t nc) {
  ChargeWorkspace& w = c->charge_ws;
  if (w.nc == nc) return 0;
  const int64_t ldc = ((nc + kTargetTile - 1) / kTargetTile) * kTargetTile;
  std::vector<int2> gtab = make_groups(c->n_src_tiles, std::max<int64_t>(1, (nc + 767) / 768));
  w.nc = -1;
  w.n_groups = (int)gtab.size();
  if (w.q.alloc(nc) || w.qpos.alloc(3 * nc) || w.tq.alloc(6 * ldc) || w.e.alloc(1) ||
      w.groups.alloc(gtab.size()) || w.part.alloc((size_t)w.n_groups * 2 * ldc) || w.v.alloc(nc) ||
      w.recv.alloc(nc + 64) || w.bad.alloc(1) ||
      w.bad_all.alloc(std::max<int64_t>(1024, c->comm.nranks)))
    return HOBI_ERR_CUDA;
  HOBI_CUDA(cudaMemcpy(w.groups.p, gtab.data(), gtab.size() * sizeof(int2), cudaMemcpyHostToDevice));
  w.nc = nc;
  return 0;
}

int energy_device(hobi_ctx* c, const double* qpos, const double* q, int64_t nc, const double* x_dev,
                  double* energy) {
  *energy = 0.0;
  if (nc == 0) return 0;
  // charges act as targets of a K1/K2-only sweep over the regular points
  // (solver.py:609-613); their "normal" is unused.
  const int64_t ldc = ((nc + kTargetTile - 1) / kTargetTile) * kTargetTile;
  int rc;
  if ((rc = charge_workspace(c, nc))) return rc;
  ChargeWorkspace& w = c->charge_ws;
  const int groups = w.n_groups;
  HOBI_CUDA(cudaMemcpyAsync(w.q.p, q, nc * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  HOBI_CUDA(cudaMemcpyAsync(w.qpos.p, qpos, 3 * nc * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  double *tq = w.tq.p, *part = w.part.p, *dq = w.q.p;
  const int2* dgroups = w.groups.p;
  targets_kernel<<<nblk(ldc, 256), 256, 0, c->stream>>>(w.qpos.p, nullptr, nc, ldc, frame_pos(c->phys),
                                                        frame_rot(c->phys), tq, nullptr);
  c->launches++;
  if ((rc = update_weights(c, x_dev))) return rc;
  // Under a communicator the charges are split across ranks; the per-charge
  // values are gathered and folded in charge order on every rank, so the
  // energy is bitwise that of a one-GPU run.  An emulated split computes
  // every rank's slot here.
  const bool split = c->comm.nccl && c->comm.nranks > 1;
  const bool emul = c->comm.emulated && c->comm.nranks > 1;
  const int nr = (split || emul) ? c->comm.nranks : 1;
  const int64_t mc = (nc + nr - 1) / nr;
  if ((size_t)nr * mc > w.recv.n && w.recv.alloc((size_t)nr * mc)) return HOBI_ERR_CUDA;
  double *v = w.v.p, *recv = w.recv.p, *e = w.e.p;
  bool timing = c->timing;
  c->timing = false;
  for (int r = 0; r < nr; ++r) {
    if (split && r != c->comm.rank) continue;
    const int64_t base = nc / nr, extra = nc % nr;
    const int64_t k0 = r * base + std::min<int64_t>(r, extra), k1 = k0 + base + (r < extra ? 1 : 0);
    if (k1 <= k0) continue;
    if ((rc = launch_sweep(c, tq, ldc, k0, k1, false, part, ldc, dgroups, groups))) break;
    double* dst = nr == 1 ? v : (split ? recv + (int64_t)c->comm.rank * mc : recv + (int64_t)r * mc);
    energy_charge_kernel<<<nblk(k1 - k0, 256), 256, 0, c->stream>>>(part, ldc, groups, dq, k0, k1, dst);
    c->launches++;
  }
  c->timing = timing;
  if (rc) return rc;
  if (split) {  // each rank contributes its slot (in place inside recv)
    if ((rc = comm_allgather_bytes(c, recv + (int64_t)c->comm.rank * mc, recv, mc * sizeof(double))))
      return rc;
  }
  if (nr > 1) {
    permute1_kernel<<<nblk(nc, 256), 256, 0, c->stream>>>(recv, mc, nc, nr, v);
    c->launches++;
  }
  energy_fold_kernel<<<1, 1024, 0, c->stream>>>(v, nc, e);
  c->launches++;
  HOBI_CUDA(cudaGetLastError());
  HOBI_CUDA(cudaMemcpyAsync(energy, e, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

}  // namespace hobi
