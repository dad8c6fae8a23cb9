// C ABI (include/hobi.h): context lifecycle, host-side pair tables, the
// operator entry points, GMRES drivers and the NCCL row-gather.
//
// Reference mapping (paths relative to /root/reference/pkg/src/pbbem):
//   hobi_create        <- solver.discretize            solver.py:165-266
//   hobi_matvec*       <- _Operator.__call__/_apply_range solver.py:447-459, 278-367
//   hobi_rhs           <- assemble_rhs                 solver.py:393-402
//   hobi_gmres         <- gmres_solve                  solver.py:484-560
//   hobi_energy        <- solvation_energy             solver.py:581-614
//   hobi_comm_*        <- the fork-pool row split      solver.py:405-459
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "hobi_internal.cuh"

namespace hobi {

static thread_local std::string g_last_error;

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(HOBI_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                                 cudaGetErrorString(e) + ") in " + what);
}

// ---------------------------------------------------------------------------
// NCCL, resolved at run time from the process (torch loads libnccl.so.2) so
// the library has no link-time dependency and single-GPU use never needs it.

namespace nccl {
typedef struct {
  char internal[128];
} UniqueId;
typedef int (*GetUniqueIdFn)(UniqueId*);
typedef int (*CommInitRankFn)(void**, int, UniqueId, int);
typedef int (*AllGatherFn)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef int (*CommDestroyFn)(void*);
typedef const char* (*GetErrorStringFn)(int);
constexpr int kFloat64 = 8;  // ncclFloat64

struct Api {
  bool loaded = false;
  GetUniqueIdFn get_unique_id = nullptr;
  CommInitRankFn init_rank = nullptr;
  AllGatherFn all_gather = nullptr;
  CommDestroyFn destroy = nullptr;
  GetErrorStringFn err = nullptr;
};

static Api& api() {
  static Api a;
  if (a.loaded) return a;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names)
    if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) return a;
  a.get_unique_id = (GetUniqueIdFn)dlsym(h, "ncclGetUniqueId");
  a.init_rank = (CommInitRankFn)dlsym(h, "ncclCommInitRank");
  a.all_gather = (AllGatherFn)dlsym(h, "ncclAllGather");
  a.destroy = (CommDestroyFn)dlsym(h, "ncclCommDestroy");
  a.err = (GetErrorStringFn)dlsym(h, "ncclGetErrorString");
  a.loaded = a.get_unique_id && a.init_rank && a.all_gather && a.destroy;
  return a;
}

static int check(int r, const char* what) {
  if (r == 0) return 0;
  const char* s = api().err ? api().err(r) : "unknown";
  return fail(HOBI_ERR_NCCL, std::string("NCCL error in ") + what + ": " + s);
}
}  // namespace nccl

int comm_allgather(hobi_ctx* c) {
  auto& a = nccl::api();
  return nccl::check(a.all_gather(c->gather_send.p, c->gather_recv.p, (size_t)(2 * c->gather_m),
                                  nccl::kFloat64, c->comm.nccl, c->stream),
                     "ncclAllGather");
}

int comm_allgather_bytes(hobi_ctx* c, const void* send, void* recv, size_t bytes) {
  auto& a = nccl::api();
  constexpr int kUint8 = 1;  // ncclUint8
  return nccl::check(a.all_gather(send, recv, bytes, kUint8, c->comm.nccl, c->stream), "ncclAllGather");
}

static void row_range(int64_t n, int nranks, int rank, int64_t* lo, int64_t* hi) {
  int64_t base = n / nranks, extra = n % nranks;
  *lo = rank * base + std::min<int64_t>(rank, extra);
  *hi = *lo + base + (rank < extra ? 1 : 0);
}

static int setup_gather(hobi_ctx* c, int nranks) {
  c->gather_m = (c->nt + nranks - 1) / nranks;
  if (c->gather_send.alloc(2 * c->gather_m) || c->gather_recv.alloc((size_t)nranks * 2 * c->gather_m))
    return HOBI_ERR_CUDA;
  // on the context stream (non-blocking, so not ordered after the legacy
  // stream), finished before any later work can touch the buffer
  HOBI_CUDA(cudaMemsetAsync(c->gather_recv.p, 0, (size_t)nranks * 2 * c->gather_m * sizeof(double), c->stream));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

// ---------------------------------------------------------------------------
// source-group partition: a function of the problem size only (never of the
// row split or the tuned tile), chosen so an 8-way split still fills 148 SMs
// several times.  768 rows is a fixed reference tile for that sizing, not the
// sweep's tile: retuning the sweep must not move group boundaries.

static int choose_groups(hobi_ctx* c) {
  c->n_src_tiles = (int)(c->ns_pad / kSrcTile);
  std::vector<int2> g = make_groups(c->n_src_tiles, std::max<int64_t>(1, ((c->nt + 7) / 8 + 767) / 768));
  c->n_groups = (int)g.size();
  if (c->groups.alloc(g.size())) return HOBI_ERR_CUDA;
  HOBI_CUDA(cudaMemcpy(c->groups.p, g.data(), g.size() * sizeof(int2), cudaMemcpyHostToDevice));
  return 0;
}

static int common_init(hobi_ctx* c, int device, double eps1, double eps2, double kappa) {
  if (!(eps1 > 0.0)) return fail(HOBI_ERR_VALUE, "eps1 must be positive, got " + std::to_string(eps1));
  if (!(eps2 > 0.0)) return fail(HOBI_ERR_VALUE, "eps2 must be positive, got " + std::to_string(eps2));
  if (!(kappa >= 0.0))
    return fail(HOBI_ERR_VALUE, "kappa must be nonnegative, got " + std::to_string(kappa));
  c->device = device;
  HOBI_CUDA(cudaSetDevice(device));
  HOBI_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  HOBI_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  HOBI_CUDA(cudaStreamCreateWithFlags(&c->side2, cudaStreamNonBlocking));
  HOBI_CUDA(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
  HOBI_CUDA(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
  HOBI_CUDA(cudaEventCreateWithFlags(&c->join2, cudaEventDisableTiming));
  HOBI_CUDA(cudaEventCreate(&c->ev0));
  HOBI_CUDA(cudaEventCreate(&c->ev1));
  if (const char* v = getenv("HOBI_SWEEP_VARIANT")) {  // tuning: default tile, still auto-switched
    const int vi = atoi(v);
    if (vi < 0 || vi >= sweep_variant_count()) return fail(HOBI_ERR_VALUE, "HOBI_SWEEP_VARIANT out of range");
    c->sweep_variant = vi;
  }
  Physics& p = c->phys;
  p.eps1 = eps1;
  p.eps2 = eps2;
  p.kappa = kappa;
  p.er = eps2 / eps1;  // kernels.py:109
  p.ier = 1.0 / p.er;
  p.diag1 = 0.5 * (1.0 + p.er);
  p.diag2 = 0.5 * (1.0 + 1.0 / p.er);
  p.mode = kappa > 0.0 ? kScreened : kLaplace;
  p.len_scale = p.mode == kScreened ? kappa : 1.0;
  if (const char* f = getenv("HOBI_SWEEP_FRAME")) {  // testing: first sweep frame tried
    const int k = atoi(f);
    if (k < 0 || k >= kNumFrames) return fail(HOBI_ERR_VALUE, "HOBI_SWEEP_FRAME out of range");
    p.frame = k;
  }
  int rc;
  if ((rc = upload_exp_table())) return rc;
  return 0;
}

static int alloc_operands(hobi_ctx* c) {
  c->nt_pad = ((c->nt + kTargetTile - 1) / kTargetTile) * kTargetTile;
  c->ns_pad = std::max<int64_t>(kSrcTile, ((c->ns + kSrcTile - 1) / kSrcTile) * kSrcTile);
  int rcg = choose_groups(c);
  if (rcg) return rcg;
  if (c->tgt.alloc(6 * c->nt_pad) || c->src.alloc(c->ns_pad * kSrcStride) ||
      c->part.alloc((size_t)c->n_groups * 2 * c->nt_pad) || c->ticket.alloc(2) ||
      c->u.alloc(std::max<int64_t>(1, 2 * c->nt)) ||
      c->out.alloc(std::max<int64_t>(1, 2 * c->nt)))
    return HOBI_ERR_CUDA;
  c->lo = 0;
  c->hi = c->nt;
  int rc;
  if (c->nt > 0 && (rc = prepare_targets(c))) return rc;
  if ((rc = prepare_static_sources(c))) return rc;
  if ((rc = prepare_singular(c))) return rc;
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

// HOBI_TRACE_INIT=1: wall time of each stage of context creation (stderr).
struct InitTrace {
  bool on = getenv("HOBI_TRACE_INIT") && getenv("HOBI_TRACE_INIT")[0] == '1';
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what, cudaStream_t s = nullptr) {
    if (!on) return;
    if (s) cudaStreamSynchronize(s);
    auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "hobi init %-16s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// Scale check for the table-driven exp (valid for kappa*r < 1e12).
static int check_extent(hobi_ctx* c, const double* v, int64_t n) {
  if (c->phys.mode != kScreened) return 0;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::min(lo[k], v[3 * i + k]);
      hi[k] = std::max(hi[k], v[3 * i + k]);
    }
  double diag = 0.0;
  for (int k = 0; k < 3; ++k) diag += (hi[k] - lo[k]) * (hi[k] - lo[k]);
  if (c->phys.kappa * std::sqrt(diag) > 1e9)
    return fail(HOBI_ERR_VALUE, "kappa * mesh extent exceeds the supported range (1e9)");
  if (c->phys.kappa * std::sqrt(diag) < 1e-30) {
    // screening this weak changes every kernel value by a relative O(kappa r)
    // <= 1e-30, far below double rounding, while kappa-scaled coordinates and
    // the k^3-weighted source normals would head for underflow: use the
    // kappa = 0 instantiation (K1 = K4 = 0) for the sweep
    c->phys.mode = kLaplace;
    c->phys.len_scale = 1.0;
  }
  return 0;
}

}  // namespace hobi

using namespace hobi;

// ---------------------------------------------------------------------------

extern "C" {

const char* hobi_last_error(void) { return g_last_error.c_str(); }

int hobi_abi_version(void) { return HOBI_ABI_VERSION; }

int hobi_device_count(int* count) {
  *count = 0;
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  return 0;
}

int hobi_device_sms(int device, int* sms) {
  *sms = 0;
  HOBI_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, device));
  return 0;
}

// Mesh-size and face-index checks shared by every constructor: sizes must fit
// the device's int32 indices, and every face must reference vertices in [0, nv).
static int check_faces(const int64_t* faces, int64_t nv, int64_t nf) {
  if (nv < 1 || nf < 1) return fail(HOBI_ERR_VALUE, "mesh must have vertices and faces");
  if (nv >= (1ll << 31) || 3 * nf >= (1ll << 31)) return fail(HOBI_ERR_VALUE, "mesh too large");
  for (int64_t i = 0; i < 3 * nf; ++i)
    if (faces[i] < 0 || faces[i] >= nv)
      return fail(HOBI_ERR_VALUE, "face " + std::to_string(i / 3) + " references a vertex outside [0, " +
                                      std::to_string(nv) + ")");
  return 0;
}

int hobi_create(int device, const double* vertices, const double* normals, int64_t nv,
                const int64_t* faces, int64_t nf, double eps1, double eps2, double kappa,
                const double* reg_pts, const double* reg_wts, const double* reg_shape, int nq,
                const double* duf_pts, const double* duf_wts, const double* duf_shape, int nd,
                hobi_ctx** out) {
  NvtxRange nvtx_("hobi_create");
  *out = nullptr;
  if (nq < 1 || nq > 16) return fail(HOBI_ERR_VALUE, "regular rule must have 1..16 points");
  if (nd < 1 || nd > 64) return fail(HOBI_ERR_VALUE, "Duffy rule must have 1..64 points");
  int rc;
  if ((rc = check_faces(faces, nv, nf))) return rc;
  InitTrace tr;
  hobi_ctx* c = new hobi_ctx();
  auto bail = [&](int r) {
    hobi_destroy(c);
    return r;
  };
  if ((rc = common_init(c, device, eps1, eps2, kappa))) return bail(rc);
  tr.mark("common_init", c->stream);
  if ((rc = check_extent(c, vertices, nv))) return bail(rc);
  c->scheme = kHobi;
  c->nv = nv;
  c->nf = nf;
  c->nt = nv;
  c->nq = nq;
  c->nd = nd;
  c->ns = nf * nq;
  const int64_t np = 3 * nf;
  // Pair tables (solver.py:229-243): slot 3f+k couples faces[f,k] with face f;
  // a stable counting sort by vertex realises lexsort((pair_face, pair_vertex)).
  std::vector<int> count(nv + 1, 0), pv(np), pf(np), pg(3 * np), slot_to_pair(np);
  for (int64_t s = 0; s < np; ++s) count[faces[s] + 1]++;
  for (int64_t v = 0; v < nv; ++v) count[v + 1] += count[v];
  c->h_pair_starts.assign(count.begin(), count.end());
  std::vector<int> fill(count.begin(), count.end() - 1);
  for (int64_t s = 0; s < np; ++s) {
    const int64_t f = s / 3, k = s % 3;
    const int v = (int)faces[s];
    const int p = fill[v]++;
    slot_to_pair[s] = p;
    pv[p] = v;
    pf[p] = (int)f;
    for (int q = 0; q < 3; ++q) pg[3 * p + q] = (int)faces[3 * f + (k + q) % 3];
  }
  std::vector<int> faces32(3 * nf);
  for (int64_t i = 0; i < 3 * nf; ++i) faces32[i] = (int)faces[i];
  std::vector<double> rbary(3 * nq), dbary(3 * nd);
  for (int m = 0; m < nq; ++m) {  // _barycentric (solver.py:158-162)
    rbary[3 * m] = 1.0 - reg_pts[2 * m] - reg_pts[2 * m + 1];
    rbary[3 * m + 1] = reg_pts[2 * m];
    rbary[3 * m + 2] = reg_pts[2 * m + 1];
  }
  for (int m = 0; m < nd; ++m) {
    dbary[3 * m] = 1.0 - duf_pts[2 * m] - duf_pts[2 * m + 1];
    dbary[3 * m + 1] = duf_pts[2 * m];
    dbary[3 * m + 2] = duf_pts[2 * m + 1];
  }
  if (c->vert.alloc(3 * nv) || c->vnrm.alloc(3 * nv) || c->faces.alloc(3 * nf) ||
      c->reg_pos.alloc(3 * nf * nq) || c->reg_nrm.alloc(3 * nf * nq) || c->reg_w.alloc(nf * nq) ||
      c->duf_pos.alloc(3 * np * nd) || c->duf_nrm.alloc(3 * np * nd) || c->duf_w.alloc(np * nd) ||
      c->pair_vertex.alloc(np) || c->pair_face.alloc(np) || c->pair_gverts.alloc(3 * np) ||
      c->pair_starts.alloc(nv + 1) || c->reg_bary.alloc(3 * nq) || c->duf_bary.alloc(3 * nd) ||
      c->corr.alloc(2 * np))
    return bail(HOBI_ERR_CUDA);
  auto up = [&](void* d, const void* h, size_t bytes) {
    return cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->stream);
  };
  cudaError_t e = cudaSuccess;
  if (!e) e = up(c->vert.p, vertices, 3 * nv * sizeof(double));
  if (!e) e = up(c->vnrm.p, normals, 3 * nv * sizeof(double));
  if (!e) e = up(c->faces.p, faces32.data(), 3 * nf * sizeof(int));
  if (!e) e = up(c->pair_vertex.p, pv.data(), np * sizeof(int));
  if (!e) e = up(c->pair_face.p, pf.data(), np * sizeof(int));
  if (!e) e = up(c->pair_gverts.p, pg.data(), 3 * np * sizeof(int));
  if (!e) e = up(c->pair_starts.p, count.data(), (nv + 1) * sizeof(int));
  if (!e) e = up(c->reg_bary.p, rbary.data(), 3 * nq * sizeof(double));
  if (!e) e = up(c->duf_bary.p, dbary.data(), 3 * nd * sizeof(double));
  if (e) return bail(cuda_fail(e, "cudaMemcpyAsync(upload)"));
  tr.mark("alloc+upload", c->stream);
  int bad_slot = -1, bad_code = 0;
  {
    // the rule tables live in __constant__ memory shared by every context on
    // the device: concurrent creations take turns until their geometry
    // kernels have finished reading them (build_geometry synchronises)
    static std::mutex rule_tables_mutex;
    std::lock_guard<std::mutex> lock(rule_tables_mutex);
    if ((rc = upload_rule_tables(reg_shape, nq, duf_shape, nd, reg_wts, duf_wts))) return bail(rc);
    tr.mark("rule tables", c->stream);
    if ((rc = build_geometry(c, slot_to_pair.data(), &bad_slot, &bad_code))) return bail(rc);
  }
  tr.mark("geometry", c->stream);
  if (bad_slot >= 0) {
    static const char* msgs[] = {"", "arc endpoints coincide",
                                 "endpoint normal is nearly parallel to the chord",
                                 "endpoint normals are antiparallel"};
    return bail(fail(HOBI_ERR_DEGENERATE_ARC,
                     "face " + std::to_string(bad_slot / 3) + ": " + msgs[bad_code & 3]));
  }
  if ((rc = alloc_operands(c))) return bail(rc);
  tr.mark("operands", c->stream);
  *out = c;
  return 0;
}

namespace {
#include "hobi_default_rules.inc"
}  // namespace

int hobi_create_default(int device, const double* vertices, const double* normals, int64_t nv,
                        const int64_t* faces, int64_t nf, double eps1, double eps2, double kappa,
                        int duffy_points, hobi_ctx** out) {
  *out = nullptr;
  for (const DefDuffy& d : kDefDuffy)
    if (d.n == duffy_points)
      return hobi_create(device, vertices, normals, nv, faces, nf, eps1, eps2, kappa, kDefRegPts, kDefRegWts,
                         kDefRegShape, 4, d.pts, d.wts, d.shape, d.n * d.n, out);
  return fail(HOBI_ERR_VALUE, "hobi_create_default: duffy_points must be 4, 6 or 8, got " +
                                  std::to_string(duffy_points));
}

int hobi_create_from_caches(int device, const double* vertices, const double* normals, int64_t nv,
                            const int64_t* faces, int64_t nf, double eps1, double eps2, double kappa,
                            const double* reg_pos, const double* reg_nrm, const double* reg_w,
                            const double* reg_bary, int nq, const double* duf_pos,
                            const double* duf_nrm, const double* duf_w, const double* duf_bary, int nd,
                            const int64_t* pair_vertex, const int64_t* pair_face,
                            const int64_t* pair_gverts, const int64_t* pair_starts, hobi_ctx** out) {
  *out = nullptr;
  if (nq < 1 || nq > 16 || nd < 1 || nd > 64) return fail(HOBI_ERR_VALUE, "rule sizes out of range");
  int rc;
  if ((rc = check_faces(faces, nv, nf))) return rc;
  const int64_t np = 3 * nf;
  // the pair tables index device arrays in the Duffy swap and the epilogue:
  // a CSR over vertices, pairs in range, each pair's vertex inside its segment
  if (pair_starts[0] != 0 || pair_starts[nv] != np)
    return fail(HOBI_ERR_VALUE, "pair_starts must run from 0 to 3*n_faces");
  for (int64_t v = 0; v < nv; ++v) {
    if (pair_starts[v + 1] < pair_starts[v]) return fail(HOBI_ERR_VALUE, "pair_starts must be non-decreasing");
    for (int64_t p = pair_starts[v]; p < pair_starts[v + 1]; ++p)
      if (pair_vertex[p] != v) return fail(HOBI_ERR_VALUE, "pair_vertex disagrees with pair_starts");
  }
  for (int64_t p = 0; p < np; ++p) {
    if (pair_face[p] < 0 || pair_face[p] >= nf) return fail(HOBI_ERR_VALUE, "pair_face out of range");
    for (int k = 0; k < 3; ++k)
      if (pair_gverts[3 * p + k] < 0 || pair_gverts[3 * p + k] >= nv)
        return fail(HOBI_ERR_VALUE, "pair_gverts out of range");
  }
  hobi_ctx* c = new hobi_ctx();
  auto bail = [&](int r) {
    hobi_destroy(c);
    return r;
  };
  if ((rc = common_init(c, device, eps1, eps2, kappa))) return bail(rc);
  if ((rc = check_extent(c, vertices, nv))) return bail(rc);
  c->scheme = kHobi;
  c->nv = nv;
  c->nf = nf;
  c->nt = nv;
  c->nq = nq;
  c->nd = nd;
  c->ns = nf * nq;
  auto narrow = [](const int64_t* a, int64_t n) {
    std::vector<int> v(n);
    for (int64_t i = 0; i < n; ++i) v[i] = (int)a[i];
    return v;
  };
  std::vector<int> f32 = narrow(faces, 3 * nf), pv = narrow(pair_vertex, np), pf = narrow(pair_face, np),
                   pg = narrow(pair_gverts, 3 * np), ps = narrow(pair_starts, nv + 1);
  c->h_pair_starts = ps;
  if (c->vert.alloc(3 * nv) || c->vnrm.alloc(3 * nv) || c->faces.alloc(3 * nf) ||
      c->reg_pos.alloc(3 * nf * nq) || c->reg_nrm.alloc(3 * nf * nq) || c->reg_w.alloc(nf * nq) ||
      c->duf_pos.alloc(3 * np * nd) || c->duf_nrm.alloc(3 * np * nd) || c->duf_w.alloc(np * nd) ||
      c->pair_vertex.alloc(np) || c->pair_face.alloc(np) || c->pair_gverts.alloc(3 * np) ||
      c->pair_starts.alloc(nv + 1) || c->reg_bary.alloc(3 * nq) || c->duf_bary.alloc(3 * nd) ||
      c->corr.alloc(2 * np))
    return bail(HOBI_ERR_CUDA);
  struct Up {
    void* d;
    const void* h;
    size_t bytes;
  } ups[] = {{c->vert.p, vertices, 3 * nv * sizeof(double)},
             {c->vnrm.p, normals, 3 * nv * sizeof(double)},
             {c->faces.p, f32.data(), 3 * nf * sizeof(int)},
             {c->reg_pos.p, reg_pos, 3 * nf * nq * sizeof(double)},
             {c->reg_nrm.p, reg_nrm, 3 * nf * nq * sizeof(double)},
             {c->reg_w.p, reg_w, nf * nq * sizeof(double)},
             {c->reg_bary.p, reg_bary, 3 * nq * sizeof(double)},
             {c->duf_pos.p, duf_pos, 3 * np * nd * sizeof(double)},
             {c->duf_nrm.p, duf_nrm, 3 * np * nd * sizeof(double)},
             {c->duf_w.p, duf_w, np * nd * sizeof(double)},
             {c->duf_bary.p, duf_bary, 3 * nd * sizeof(double)},
             {c->pair_vertex.p, pv.data(), np * sizeof(int)},
             {c->pair_face.p, pf.data(), np * sizeof(int)},
             {c->pair_gverts.p, pg.data(), 3 * np * sizeof(int)},
             {c->pair_starts.p, ps.data(), (nv + 1) * sizeof(int)}};
  for (const Up& u : ups) {
    cudaError_t e = cudaMemcpy(u.d, u.h, u.bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaMemcpy(upload caches)"));
  }
  if ((rc = alloc_operands(c))) return bail(rc);
  *out = c;
  return 0;
}

int hobi_create_lobi(int device, const double* vertices, const double* normals, int64_t nv,
                     const int64_t* faces, int64_t nf, double eps1, double eps2, double kappa,
                     hobi_ctx** out) {
  (void)normals;
  *out = nullptr;
  int rc;
  if ((rc = check_faces(faces, nv, nf))) return rc;
  hobi_ctx* c = new hobi_ctx();
  auto bail = [&](int r) {
    hobi_destroy(c);
    return r;
  };
  if ((rc = common_init(c, device, eps1, eps2, kappa))) return bail(rc);
  if ((rc = check_extent(c, vertices, nv))) return bail(rc);
  c->scheme = kLobi;
  c->nv = nv;
  c->nf = nf;
  c->nt = nf;
  c->ns = nf;
  c->nq = 1;
  // flat centroids, unit normals, areas (solver.py:173-186)
  std::vector<double> cen(3 * nf), nrm(3 * nf), area(nf);
  for (int64_t f = 0; f < nf; ++f) {
    const double* a = vertices + 3 * faces[3 * f];
    const double* b = vertices + 3 * faces[3 * f + 1];
    const double* d = vertices + 3 * faces[3 * f + 2];
    double e1[3], e2[3];
    for (int k = 0; k < 3; ++k) {
      cen[3 * f + k] = ((a[k] + b[k]) + d[k]) / 3.0;
      e1[k] = b[k] - a[k];
      e2[k] = d[k] - a[k];
    }
    double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                    e1[0] * e2[1] - e1[1] * e2[0]};
    volatile double s = cr[0] * cr[0];  // unfused left-to-right, like np.linalg.norm(axis=1)
    s = s + cr[1] * cr[1];
    s = s + cr[2] * cr[2];
    double two = std::sqrt((double)s);
    for (int k = 0; k < 3; ++k) nrm[3 * f + k] = cr[k] / two;
    area[f] = 0.5 * two;
  }
  if (c->reg_pos.alloc(3 * nf) || c->reg_nrm.alloc(3 * nf) || c->lobi_area.alloc(nf))
    return bail(HOBI_ERR_CUDA);
  HOBI_CUDA(cudaMemcpy(c->reg_pos.p, cen.data(), 3 * nf * sizeof(double), cudaMemcpyHostToDevice));
  HOBI_CUDA(cudaMemcpy(c->reg_nrm.p, nrm.data(), 3 * nf * sizeof(double), cudaMemcpyHostToDevice));
  HOBI_CUDA(cudaMemcpy(c->lobi_area.p, area.data(), nf * sizeof(double), cudaMemcpyHostToDevice));
  if ((rc = alloc_operands(c))) return bail(rc);
  *out = c;
  return 0;
}

int hobi_destroy(hobi_ctx* c) {
  if (!c) return 0;
  cudaSetDevice(c->device);
  if (c->comm.nccl && nccl::api().loaded) nccl::api().destroy(c->comm.nccl);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : c->comm.opened) cudaIpcCloseMemHandle(p);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->p2p_err) cudaFreeHost(c->p2p_err);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->side) cudaStreamSynchronize(c->side);
  if (c->side2) cudaStreamSynchronize(c->side2);
  if (c->fork) cudaEventDestroy(c->fork);
  if (c->join) cudaEventDestroy(c->join);
  if (c->join2) cudaEventDestroy(c->join2);
  cudaStream_t s = c->stream, side = c->side, side2 = c->side2;
  delete c;  // DevBufs free themselves
  if (s) cudaStreamDestroy(s);
  if (side) cudaStreamDestroy(side);
  if (side2) cudaStreamDestroy(side2);
  return 0;
}

int hobi_size(hobi_ctx* c, int64_t* n_colloc, int64_t* n_sources) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (n_colloc) *n_colloc = c->nt;
  if (n_sources) *n_sources = c->ns;
  return 0;
}

int hobi_matvec_device(hobi_ctx* c, const double* u_dev, double* out_dev) {
  NvtxRange nvtx_("hobi_matvec_device");
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  HOBI_CUDA(cudaSetDevice(c->device));
  return matvec_full_device(c, u_dev, out_dev);
}

// Host-buffer application of a small problem: a latency-bound call (config 1:
// 0.03 ms of kernels) spends more time in two pageable copies, five launches
// and their gaps than in the sweep, so the whole call -- H2D from a pinned
// staging vector, the matvec's kernels on their streams, D2H into a pinned
// staging vector -- is captured once and replayed as one graph launch.  Same
// kernels, same arguments, same order: results are bitwise those of the
// plain path.  HOBI_MATVEC_GRAPH=0 turns it off.
static const size_t kHostGraphBytes = 256 << 10;

static bool host_graph_eligible(const hobi_ctx* c, size_t bytes) {
  if (bytes > kHostGraphBytes || c->host_calls < 1 || c->host_graph_off) return false;  // first call: plain path
  if (c->comm.nranks != 1 || c->comm.nccl || c->comm.p2p || c->comm.emulated) return false;
  static const bool off = [] {
    const char* e = getenv("HOBI_MATVEC_GRAPH");
    return e && e[0] == '0';
  }();
  return !off;
}

static int matvec_host_graph(hobi_ctx* c, const double* u, double* out, size_t bytes) {
  if (!c->host_in.p && (c->host_in.alloc(2 * c->nt) || c->host_out.alloc(2 * c->nt))) return HOBI_ERR_CUDA;
  const uint64_t key = 1 ^ ((uint64_t)(c->sweep_variant + 1) << 48) ^ ((uint64_t)c->variant_pinned << 60);
  if (!c->host_graph.exec || c->host_graph.key != key) {
    c->host_graph.reset();
    const bool saved_timing = c->timing;
    const int64_t l0 = c->launches;
    c->timing = false;  // no event pairs inside a capture
    HOBI_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = cudaMemcpyAsync(c->u.p, c->host_in.p, bytes, cudaMemcpyHostToDevice, c->stream);
    int rc = e == cudaSuccess ? matvec_full_device(c, c->u.p, c->out.p) : cuda_fail(e, "cudaMemcpyAsync");
    if (!rc) {
      e = cudaMemcpyAsync(c->host_out.p, c->out.p, bytes, cudaMemcpyDeviceToHost, c->stream);
      if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpyAsync");
    }
    cudaGraph_t captured = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &captured);  // always leave capture mode
    c->timing = saved_timing;
    c->host_graph.graph = captured;
    c->host_graph.step_launches = c->launches - l0;
    c->launches = l0;  // counted per replay instead
    cudaError_t ie = cudaSuccess;
    if (!rc && ce == cudaSuccess) ie = cudaGraphInstantiate(&c->host_graph.exec, captured, 0);
    if (rc || ce != cudaSuccess || ie != cudaSuccess) {
      // not fatal: this context applies through the plain path from now on
      c->host_graph.reset();
      c->host_graph_off = true;
      cudaGetLastError();
      return hobi_matvec(c, u, out);
    }
    c->host_graph.key = key;
  }
  memcpy(c->host_in.p, u, bytes);
  HOBI_CUDA(cudaGraphLaunch(c->host_graph.exec, c->stream));
  c->launches += c->host_graph.step_launches;
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  memcpy(out, c->host_out.p, bytes);
  return 0;
}

int hobi_matvec(hobi_ctx* c, const double* u, double* out) {
  NvtxRange nvtx_("hobi_matvec");
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  HOBI_CUDA(cudaSetDevice(c->device));
  const size_t bytes = 2 * c->nt * sizeof(double);
  if (c->nt == 0) return 0;
  if (host_graph_eligible(c, bytes)) return matvec_host_graph(c, u, out, bytes);
  c->host_calls++;
  HOBI_CUDA(cudaMemcpyAsync(c->u.p, u, bytes, cudaMemcpyHostToDevice, c->stream));
  int rc = matvec_full_device(c, c->u.p, c->out.p);
  if (rc) return rc;
  HOBI_CUDA(cudaMemcpyAsync(out, c->out.p, bytes, cudaMemcpyDeviceToHost, c->stream));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  return p2p_check(c);
}

int hobi_matvec_rows(hobi_ctx* c, const double* u, int64_t lo, int64_t hi, double* o1, double* o2) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (lo < 0 || hi > c->nt || lo > hi) return fail(HOBI_ERR_VALUE, "row range outside [0, n)");
  HOBI_CUDA(cudaSetDevice(c->device));
  if (hi == lo) return 0;
  HOBI_CUDA(cudaMemcpyAsync(c->u.p, u, 2 * c->nt * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  int rc = matvec_rows_device(c, c->u.p, lo, hi, c->out.p, c->out.p + (hi - lo));
  if (rc) return rc;
  HOBI_CUDA(cudaMemcpyAsync(o1, c->out.p, (hi - lo) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  HOBI_CUDA(cudaMemcpyAsync(o2, c->out.p + (hi - lo), (hi - lo) * sizeof(double), cudaMemcpyDeviceToHost,
                            c->stream));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int hobi_rhs(hobi_ctx* c, const double* qpos, const double* q, int64_t nc, double* b) {
  NvtxRange nvtx_("hobi_rhs");
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  HOBI_CUDA(cudaSetDevice(c->device));
  int rc = rhs_device(c, qpos, q, nc, c->out.p);
  if (rc) return rc;
  HOBI_CUDA(cudaMemcpyAsync(b, c->out.p, 2 * c->nt * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int hobi_energy(hobi_ctx* c, const double* qpos, const double* q, int64_t nc, const double* phi,
                const double* dphi, double* energy) {
  NvtxRange nvtx_("hobi_energy");
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  HOBI_CUDA(cudaSetDevice(c->device));
  HOBI_CUDA(cudaMemcpyAsync(c->u.p, phi, c->nt * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  HOBI_CUDA(cudaMemcpyAsync(c->u.p + c->nt, dphi, c->nt * sizeof(double), cudaMemcpyHostToDevice,
                            c->stream));
  return energy_device(c, qpos, q, nc, c->u.p, energy);
}

namespace {
struct CtxOperator : DeviceOperator {
  hobi_ctx* c;
  explicit CtxOperator(hobi_ctx* ctx) : c(ctx) {}
  int apply(const double* in, double* out) override {
    int rc = p2p_check(c);  // GMRES has synchronised on the previous application
    return rc ? rc : matvec_full_device(c, in, out);
  }
  // One unsplit context (no collective, no P2P epochs, no emulated split):
  // its matvec is stream work only, so GMRES may replay it from a graph.
  uint64_t graph_key() override {
    if (c->comm.nranks != 1 || c->comm.nccl || c->comm.p2p || c->comm.emulated) return 0;
    if (getenv("HOBI_GMRES_GRAPH") && getenv("HOBI_GMRES_GRAPH")[0] == '0') return 0;
    return reinterpret_cast<uintptr_t>(c) ^ ((uint64_t)(c->sweep_variant + 1) << 48) ^
           ((uint64_t)c->variant_pinned << 60);
  }
  bool saved_timing = true;
  void begin_capture() override {
    saved_timing = c->timing;
    c->timing = false;
  }
  void end_capture() override { c->timing = saved_timing; }
};

struct HostOperator : DeviceOperator {
  hobi_apply_fn fn;
  void* user;
  int64_t n;
  cudaStream_t stream;
  std::vector<double> hin, hout;
  HostOperator(hobi_apply_fn f, void* u, int64_t nn, cudaStream_t s)
      : fn(f), user(u), n(nn), stream(s), hin(nn), hout(nn) {}
  int apply(const double* in, double* out) override {
    HOBI_CUDA(cudaMemcpyAsync(hin.data(), in, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
    HOBI_CUDA(cudaStreamSynchronize(stream));
    if (fn(user, hin.data(), hout.data(), n)) return fail(HOBI_ERR_VALUE, "operator callback failed");
    HOBI_CUDA(cudaMemcpyAsync(out, hout.data(), n * sizeof(double), cudaMemcpyHostToDevice, stream));
    HOBI_CUDA(cudaStreamSynchronize(stream));
    return 0;
  }
};
}  // namespace

int hobi_gmres(hobi_ctx* c, const double* b, double tol, int restart, int max_it, double* x,
               int* iterations, double* residual, double* best, int* matvecs) {
  NvtxRange nvtx_("hobi_gmres");
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  HOBI_CUDA(cudaSetDevice(c->device));
  CtxOperator op(c);
  int rc = gmres_device(c->device, c->stream, 2 * c->nt, &op, b, tol, restart, max_it, x, iterations,
                        residual, best, matvecs, &c->launches, &c->gmres_ws);
  int rc2 = p2p_check(c);
  return rc2 ? rc2 : rc;
}

int hobi_solve(hobi_ctx* c, const double* qpos, const double* q, int64_t nc, double tol, int restart,
               int max_it, double* phi, double* dphi, double* energy, int* iterations, double* residual,
               int* matvecs) {
  NvtxRange nvtx_("hobi_solve");
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  *energy = 0.0;
  std::vector<double> b(2 * c->nt), x(2 * c->nt);
  int rc = hobi_rhs(c, qpos, q, nc, b.data());
  if (rc) return rc;
  double best = 0.0;
  rc = hobi_gmres(c, b.data(), tol, restart, max_it, x.data(), iterations, residual, &best, matvecs);
  std::copy(x.begin(), x.begin() + c->nt, phi);
  std::copy(x.begin() + c->nt, x.end(), dphi);
  if (rc) return rc;
  return hobi_energy(c, qpos, q, nc, phi, dphi, energy);
}

int hobi_gmres_host_operator(int device, int64_t n, hobi_apply_fn apply, void* user, const double* b,
                             double tol, int restart, int max_it, double* x, int* iterations,
                             double* residual, double* best, int* matvecs) {
  HOBI_CUDA(cudaSetDevice(device));
  cudaStream_t s;
  HOBI_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int rc;
  {
    HostOperator op(apply, user, n, s);
    rc = gmres_device(device, s, n, &op, b, tol, restart, max_it, x, iterations, residual, best,
                      matvecs, nullptr);
  }
  cudaStreamDestroy(s);
  return rc;
}

int hobi_export_caches(hobi_ctx* c, double* reg_pos, double* reg_nrm, double* reg_w, double* duf_pos,
                       double* duf_nrm, double* duf_w, int64_t* pair_vertex, int64_t* pair_face,
                       int64_t* pair_gverts, int64_t* pair_starts) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (c->scheme != kHobi) return fail(HOBI_ERR_VALUE, "caches exist only for scheme 'hobi'");
  HOBI_CUDA(cudaSetDevice(c->device));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  const int64_t np = 3 * c->nf;
  auto dn = [&](void* h, const void* d, size_t bytes) -> int {
    if (!h) return 0;
    HOBI_CUDA(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost));
    return 0;
  };
  auto di = [&](int64_t* h, const int* d, int64_t n) -> int {
    if (!h) return 0;
    std::vector<int> t(n);
    HOBI_CUDA(cudaMemcpy(t.data(), d, n * sizeof(int), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) h[i] = t[i];
    return 0;
  };
  int rc;
  if ((rc = dn(reg_pos, c->reg_pos.p, 3 * c->nf * c->nq * sizeof(double)))) return rc;
  if ((rc = dn(reg_nrm, c->reg_nrm.p, 3 * c->nf * c->nq * sizeof(double)))) return rc;
  if ((rc = dn(reg_w, c->reg_w.p, c->nf * c->nq * sizeof(double)))) return rc;
  if ((rc = dn(duf_pos, c->duf_pos.p, 3 * np * c->nd * sizeof(double)))) return rc;
  if ((rc = dn(duf_nrm, c->duf_nrm.p, 3 * np * c->nd * sizeof(double)))) return rc;
  if ((rc = dn(duf_w, c->duf_w.p, np * c->nd * sizeof(double)))) return rc;
  if ((rc = di(pair_vertex, c->pair_vertex.p, np))) return rc;
  if ((rc = di(pair_face, c->pair_face.p, np))) return rc;
  if ((rc = di(pair_gverts, c->pair_gverts.p, 3 * np))) return rc;
  if ((rc = di(pair_starts, c->pair_starts.p, c->nv + 1))) return rc;
  return 0;
}

int hobi_export_nodes(hobi_ctx* c, double* node_pos, double* node_nrm) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (c->scheme != kHobi) return fail(HOBI_ERR_VALUE, "curved nodes exist only for scheme 'hobi'");
  if (!c->node0_pos.p)
    return fail(HOBI_ERR_STATE, "curved nodes are not kept for a context built from caches");
  HOBI_CUDA(cudaSetDevice(c->device));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  if (node_pos) HOBI_CUDA(cudaMemcpy(node_pos, c->node0_pos.p, 30 * c->nf * sizeof(double), cudaMemcpyDeviceToHost));
  if (node_nrm) HOBI_CUDA(cudaMemcpy(node_nrm, c->node0_nrm.p, 30 * c->nf * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

int hobi_kernel_values(int device, const double* d, const double* nx, const double* ny, int64_t n,
                       double eps1, double eps2, double kappa, double* k) {
  HOBI_CUDA(cudaSetDevice(device));
  return kernel_values_device(d, nx, ny, n, eps1, eps2, kappa, k);
}

int hobi_source_terms(int device, const double* points, const double* normals, int64_t m,
                      const double* qpos, const double* q, int64_t nc, double* s1, double* s2) {
  if (m < 0 || nc < 0) return fail(HOBI_ERR_VALUE, "negative point or charge count");
  if ((m && (!points || !normals || !s1 || !s2)) || (nc && (!qpos || !q)))
    return fail(HOBI_ERR_VALUE, "null array");
  HOBI_CUDA(cudaSetDevice(device));
  return source_terms_device(points, normals, m, qpos, q, nc, s1, s2);
}

int hobi_geometry_fit_arcs(int device, const double* p0, const double* n0, const double* p1,
                           const double* n1, int64_t n, double* coef, int* code) {
  if (n < 0) return fail(HOBI_ERR_VALUE, "negative count");
  if (n && (!p0 || !n0 || !p1 || !n1 || !coef || !code)) return fail(HOBI_ERR_VALUE, "null array");
  HOBI_CUDA(cudaSetDevice(device));
  return geometry_fit_arcs(p0, n0, p1, n1, n, coef, code);
}

int hobi_geometry_arc_normals(int device, const double* coef, const double* t, const double* reference,
                              int64_t n, double* normals, int* straight) {
  if (n < 0) return fail(HOBI_ERR_VALUE, "negative count");
  if (n && (!coef || !t || !reference || !normals || !straight)) return fail(HOBI_ERR_VALUE, "null array");
  HOBI_CUDA(cudaSetDevice(device));
  return geometry_arc_normals(coef, t, reference, n, normals, straight);
}

int hobi_geometry_nodes(int device, const double* vertex_pos, const double* vertex_nrm, int64_t n,
                        double* node_pos, double* node_nrm, int64_t* first_bad, int* bad_code) {
  if (n < 0) return fail(HOBI_ERR_VALUE, "negative count");
  if (!first_bad || !bad_code || (n && (!vertex_pos || !vertex_nrm || !node_pos || !node_nrm)))
    return fail(HOBI_ERR_VALUE, "null array");
  HOBI_CUDA(cudaSetDevice(device));
  return geometry_nodes(vertex_pos, vertex_nrm, n, node_pos, node_nrm, first_bad, bad_code);
}

int hobi_geometry_frames(int device, const double* node_pos, const double* node_nrm, int64_t n_elements,
                         const double* shape, int n_points, double* pos, double* nrm, double* jac,
                         double* d_dr, double* d_ds) {
  if (n_elements < 0 || n_points < 0) return fail(HOBI_ERR_VALUE, "negative count");
  if (n_elements && n_points && (!node_pos || !node_nrm || !shape || !pos || !nrm || !jac))
    return fail(HOBI_ERR_VALUE, "null array");
  HOBI_CUDA(cudaSetDevice(device));
  return geometry_frames(node_pos, node_nrm, n_elements, shape, n_points, pos, nrm, jac, d_dr, d_ds);
}

int hobi_comm_unique_id(unsigned char id[128]) {
  auto& a = nccl::api();
  if (!a.loaded) return fail(HOBI_ERR_NCCL, "libnccl.so.2 could not be loaded");
  nccl::UniqueId u;
  int rc = nccl::check(a.get_unique_id(&u), "ncclGetUniqueId");
  if (rc) return rc;
  memcpy(id, u.internal, 128);
  return 0;
}

int hobi_comm_init(hobi_ctx* c, const unsigned char id[128], int nranks, int rank) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(HOBI_ERR_VALUE, "bad rank/nranks");
  HOBI_CUDA(cudaSetDevice(c->device));
  c->comm = Comm();
  c->comm.nranks = nranks;
  c->comm.rank = rank;
  row_range(c->nt, nranks, rank, &c->lo, &c->hi);
  // A single rank needs no collective; HOBI_FORCE_NCCL=1 still builds a
  // one-rank communicator so the NCCL gather path can be exercised on one GPU.
  const char* force = getenv("HOBI_FORCE_NCCL");
  if (nranks == 1 && !(force && force[0] == '1')) return 0;
  auto& a = nccl::api();
  if (!a.loaded) return fail(HOBI_ERR_NCCL, "libnccl.so.2 could not be loaded");
  nccl::UniqueId u;
  memcpy(u.internal, id, 128);
  int rc = nccl::check(a.init_rank(&c->comm.nccl, nranks, u, rank), "ncclCommInitRank");
  if (rc) return rc;
  return setup_gather(c, nranks);
}

int hobi_comm_init_p2p(hobi_ctx* c, int nranks, int rank) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(HOBI_ERR_VALUE, "bad rank/nranks");
  if (nranks > kMaxRanks) return fail(HOBI_ERR_VALUE, "P2P gather supports at most 64 ranks");
  HOBI_CUDA(cudaSetDevice(c->device));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  if (c->comm.nccl && nccl::api().loaded) nccl::api().destroy(c->comm.nccl);
  c->comm = Comm();
  c->comm.nranks = nranks;
  c->comm.rank = rank;
  c->comm.p2p_only = true;
  row_range(c->nt, nranks, rank, &c->lo, &c->hi);
  return 0;
}

int hobi_comm_p2p_handle(hobi_ctx* c, unsigned char handle[64]) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  HOBI_CUDA(cudaSetDevice(c->device));
  // two (2 nt) receive buffers + arrival counters [parity][source rank]
  if (c->comm.nranks > kMaxRanks) return fail(HOBI_ERR_VALUE, "P2P gather supports at most 64 ranks");
  if (c->comm.p2p) return fail(HOBI_ERR_STATE, "the P2P gather is active: its area cannot be re-exported");
  const size_t n = 4 * (size_t)c->nt + 2 * kMaxRanks;
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  if (c->p2p_area.alloc(n)) return HOBI_ERR_CUDA;
  HOBI_CUDA(cudaMemsetAsync(c->p2p_area.p, 0, n * sizeof(double), c->stream));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  c->comm.p2p_fresh = true;
  cudaIpcMemHandle_t h;
  HOBI_CUDA(cudaIpcGetMemHandle(&h, c->p2p_area.p));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle, &h, 64);
  return 0;
}

int hobi_comm_p2p_open(hobi_ctx* c, const unsigned char* handles, int nranks, int rank) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (!c->p2p_area.p) return fail(HOBI_ERR_STATE, "hobi_comm_p2p_handle must be called first");
  // the arrival counters count from zero: an area that was opened before (even
  // if the gather was disabled since) needs a fresh hobi_comm_p2p_handle and a
  // new exchange, or stale counts would release rows before they arrive
  if (!c->comm.p2p_fresh)
    return fail(HOBI_ERR_STATE, "P2P receive area already used: call hobi_comm_p2p_handle again first");
  if (nranks != c->comm.nranks || rank != c->comm.rank)
    return fail(HOBI_ERR_STATE, "P2P ranks differ from the communicator (call hobi_comm_init first)");
  HOBI_CUDA(cudaSetDevice(c->device));
  std::vector<double*> ptrs(nranks);
  for (int r = 0; r < nranks; ++r) {
    if (r == rank) {
      ptrs[r] = c->p2p_area.p;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + 64 * (size_t)r, 64);
    void* p = nullptr;
    HOBI_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->comm.opened.push_back(p);
    ptrs[r] = static_cast<double*>(p);
  }
  if (c->p2p_peers.alloc(nranks) || c->p2p_done.alloc(1)) return HOBI_ERR_CUDA;
  HOBI_CUDA(cudaMemcpyAsync(c->p2p_peers.p, ptrs.data(), nranks * sizeof(double*), cudaMemcpyHostToDevice,
                            c->stream));
  HOBI_CUDA(cudaMemsetAsync(c->p2p_done.p, 0, sizeof(unsigned), c->stream));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  if (!c->p2p_err) {
    HOBI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->p2p_err), sizeof(int), cudaHostAllocMapped));
    HOBI_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->p2p_err_dev), c->p2p_err, 0));
  }
  *c->p2p_err = 0;
  const char* tmo = getenv("HOBI_P2P_TIMEOUT_MS");
  const double ms = tmo ? atof(tmo) : 60000.0;
  c->p2p_timeout_ns = (unsigned long long)((ms > 0 ? ms : 60000.0) * 1e6);
  const char* extra = getenv("HOBI_P2P_TEST_MISSING_ARRIVALS");
  c->p2p_extra = extra ? (unsigned long long)atoll(extra) : 0;
  c->comm.p2p = true;
  c->comm.p2p_fresh = false;
  c->comm.p2p_pending = false;
  c->comm.epoch = 0;
  return 0;
}

int hobi_matvec_p2p_phase(hobi_ctx* c, const double* u, double* out, int phase) {
  NvtxRange nvtx_("hobi_matvec_p2p_phase");
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (!c->comm.p2p) return fail(HOBI_ERR_STATE, "the P2P gather is not active");
  if (phase != 0 && phase != 1) return fail(HOBI_ERR_VALUE, "phase must be 0 (send) or 1 (receive)");
  if ((phase == 0) == c->comm.p2p_pending)
    return fail(HOBI_ERR_STATE, phase == 0 ? "the previous send phase has no receive phase yet"
                                           : "no send phase is pending");
  HOBI_CUDA(cudaSetDevice(c->device));
  const size_t bytes = 2 * c->nt * sizeof(double);
  int rc;
  if (phase == 0) {
    HOBI_CUDA(cudaMemcpyAsync(c->u.p, u, bytes, cudaMemcpyHostToDevice, c->stream));
    if ((rc = matvec_p2p_send(c, c->u.p))) return rc;
    HOBI_CUDA(cudaStreamSynchronize(c->stream));  // rows and arrival counts are out
    c->comm.p2p_pending = true;
    return 0;
  }
  c->comm.p2p_pending = false;
  if ((rc = matvec_p2p_recv(c, c->out.p))) return rc;
  HOBI_CUDA(cudaMemcpyAsync(out, c->out.p, bytes, cudaMemcpyDeviceToHost, c->stream));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  return p2p_check(c);
}

int hobi_comm_p2p_disable(hobi_ctx* c) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  HOBI_CUDA(cudaSetDevice(c->device));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  c->comm.p2p = false;  // the NCCL gather (set up by hobi_comm_init) takes over
  c->comm.p2p_pending = false;
  return 0;
}

int hobi_comm_info(hobi_ctx* c, int* nranks, int* rank, int* p2p) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (nranks) *nranks = c->comm.nranks;
  if (rank) *rank = c->comm.rank;
  if (p2p) *p2p = c->comm.p2p ? 1 : 0;
  return 0;
}

int hobi_emulate_ranks(hobi_ctx* c, int nranks) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (nranks < 1) return fail(HOBI_ERR_VALUE, "nranks must be >= 1");
  HOBI_CUDA(cudaSetDevice(c->device));
  c->comm = Comm();
  c->comm.nranks = nranks;
  c->comm.emulated = nranks > 1;
  c->lo = 0;
  c->hi = c->nt;
  if (nranks == 1) return 0;
  return setup_gather(c, nranks);
}

int hobi_timing_reset(hobi_ctx* c) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  HOBI_CUDA(cudaSetDevice(c->device));
  if (collect_sweep_timing(c)) return HOBI_ERR_CUDA;
  c->sweep_ms = 0.0;
  c->sweep_launches = 0;
  c->launches = 0;
  return 0;
}

int hobi_timing(hobi_ctx* c, double* sweep_ms, int64_t* sweep_launches, int64_t* all_launches) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  HOBI_CUDA(cudaSetDevice(c->device));
  if (collect_sweep_timing(c)) return HOBI_ERR_CUDA;
  if (sweep_ms) *sweep_ms = c->sweep_ms;
  if (sweep_launches) *sweep_launches = c->sweep_launches;
  if (all_launches) *all_launches = c->launches;
  return 0;
}

int hobi_bench(hobi_ctx* c, const double* u, double* out, int steps, int mode, int flush_l2,
               double* ms) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (steps < 0 || (mode != 0 && mode != 1)) return fail(HOBI_ERR_VALUE, "bad bench arguments");
  HOBI_CUDA(cudaSetDevice(c->device));
  const size_t bytes = 2 * c->nt * sizeof(double);
  DevBuf<unsigned char> scratch;
  const size_t flush_bytes = (size_t)512 << 20;
  if (flush_l2 && scratch.alloc(flush_bytes)) return HOBI_ERR_CUDA;
  EventPair ev;
  HOBI_CUDA(ev.create());
  cudaEvent_t e0 = ev.a, e1 = ev.b;
  int rc = 0;
  if (mode == 0) HOBI_CUDA(cudaMemcpyAsync(c->u.p, u, bytes, cudaMemcpyHostToDevice, c->stream));
  for (int i = 0; i < steps && !rc; ++i) {
    if (flush_l2) HOBI_CUDA(cudaMemsetAsync(scratch.p, i & 0xff, flush_bytes, c->stream));
    HOBI_CUDA(cudaEventRecord(e0, c->stream));
    if (mode == 1) HOBI_CUDA(cudaMemcpyAsync(c->u.p, u, bytes, cudaMemcpyHostToDevice, c->stream));
    rc = matvec_full_device(c, c->u.p, c->out.p);
    if (rc) break;
    if (mode == 1) HOBI_CUDA(cudaMemcpyAsync(out, c->out.p, bytes, cudaMemcpyDeviceToHost, c->stream));
    HOBI_CUDA(cudaEventRecord(e1, c->stream));
    HOBI_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    HOBI_CUDA(cudaEventElapsedTime(&t, e0, e1));
    ms[i] = t;
    rc = p2p_check(c);
  }
  if (!rc && mode == 0 && out) {
    HOBI_CUDA(cudaMemcpyAsync(out, c->out.p, bytes, cudaMemcpyDeviceToHost, c->stream));
    HOBI_CUDA(cudaStreamSynchronize(c->stream));
  }
  return rc;
}

int hobi_sweep_variant(hobi_ctx* c, int variant, int* count, char* name, int name_len) {
  if (count) *count = sweep_variant_count();
  if (!c) return 0;
  if (variant >= 0) {
    if (variant >= sweep_variant_count()) return fail(HOBI_ERR_VALUE, "no such sweep variant");
    c->sweep_variant = variant;
    c->variant_pinned = true;
  }
  if (name && name_len > 0) {
    snprintf(name, name_len, "%s", sweep_variant_name(c->sweep_variant));
  }
  return 0;
}

int hobi_bench_rows(hobi_ctx* c, const double* u, int64_t lo, int64_t hi, int steps, int flush_l2,
                    double* ms) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (lo < 0 || hi > c->nt || lo > hi || steps < 0) return fail(HOBI_ERR_VALUE, "bad bench_rows arguments");
  HOBI_CUDA(cudaSetDevice(c->device));
  DevBuf<unsigned char> scratch;
  const size_t flush_bytes = (size_t)512 << 20;
  if (flush_l2 && scratch.alloc(flush_bytes)) return HOBI_ERR_CUDA;
  EventPair ev;
  HOBI_CUDA(ev.create());
  cudaEvent_t e0 = ev.a, e1 = ev.b;
  HOBI_CUDA(cudaMemcpyAsync(c->u.p, u, 2 * c->nt * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  int rc = 0;
  for (int i = 0; i < steps && !rc; ++i) {
    if (flush_l2) HOBI_CUDA(cudaMemsetAsync(scratch.p, i & 0xff, flush_bytes, c->stream));
    HOBI_CUDA(cudaEventRecord(e0, c->stream));
    rc = matvec_rows_device(c, c->u.p, lo, hi, c->out.p, c->out.p + (hi - lo));
    if (rc) break;
    HOBI_CUDA(cudaEventRecord(e1, c->stream));
    HOBI_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    HOBI_CUDA(cudaEventElapsedTime(&t, e0, e1));
    ms[i] = t;
  }
  return rc;
}

int hobi_sweep_layout(hobi_ctx* c, int* n_groups, int64_t* n_sources_padded) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  if (n_groups) *n_groups = c->n_groups;
  if (n_sources_padded) *n_sources_padded = c->ns_pad;
  return 0;
}

int hobi_pairs_per_matvec(hobi_ctx* c, double* pairs) {
  if (!c) return fail(HOBI_ERR_STATE, "null context");
  *pairs = (double)c->nt * (double)c->ns;
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// FP64 roofline probe: 8 independent DFMA chains per thread, each DFMA
// reading two vector registers and one uniform register (the addend).  That
// operand pattern issues at the FP64 pipe's full 64 lanes/clk/SM (measured
// 63.5, the DMUL/DADD rate); a DFMA reading three vector registers without
// reuse-cache hits runs at 2/3 of it, and x = fma(x, a, b) with a, b in
// reused vector registers at ~58.6 (tools/fp64_probe2.cu, fp64_probe3.cu).

namespace {
__global__ void dfma_probe_kernel(double* out, int iters, double c) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = 0.5 + 1e-4 * k + 1e-7 * threadIdx.x;  // decays to ~c: no inf or subnormals
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], x[(k + 1) & 7], c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 123.456) out[0] = s;
}
}  // namespace

extern "C" int hobi_probe_fp64_tflops(int device, double ms, double* tflops) {
  *tflops = 0.0;
  HOBI_CUDA(cudaSetDevice(device));
  int sms = 0;
  HOBI_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  DevBuf<double> d;
  if (d.alloc(1)) return HOBI_ERR_CUDA;
  const int blocks = sms * 8, threads = 256, iters = 2048;
  EventPair ev;
  HOBI_CUDA(ev.create());
  cudaEvent_t e0 = ev.a, e1 = ev.b;
  for (int w = 0; w < 3; ++w) dfma_probe_kernel<<<blocks, threads>>>(d.p, iters, 1e-9);
  HOBI_CUDA(cudaDeviceSynchronize());
  double total_ms = 0.0, flops = 0.0;
  float best = 1e30f;
  while (total_ms < ms) {
    HOBI_CUDA(cudaEventRecord(e0));
    dfma_probe_kernel<<<blocks, threads>>>(d.p, iters, 1e-9);
    HOBI_CUDA(cudaEventRecord(e1));
    HOBI_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    HOBI_CUDA(cudaEventElapsedTime(&t, e0, e1));
    best = std::min(best, t);
    total_ms += t;
    flops = 2.0 * 32.0 * iters * (double)blocks * threads;
  }
  *tflops = flops / (best * 1e-3) * 1e-12;
  return 0;
}
