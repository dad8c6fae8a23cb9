// Internal declarations shared by the HOBI-PB CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/hobi.h"

namespace hobi {

// NVTX range for timeline tools (header-only NVTX v3; a no-op without a tool attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

constexpr double kFourPi = 12.566370614359172;  // 4.0 * np.pi (kernels.py:27)
constexpr double kKcal = 332.0716;               // kernels.py:33

// Sweep tiling.
constexpr int kSweepThreads = 128;  // threads per CTA
constexpr int kSweepR = 2;          // targets held in registers per thread
constexpr int kTargetTile = kSweepThreads * kSweepR;
constexpr int kSrcTile = 64;        // sources per shared-memory stage
constexpr int kSrcStride = 10;      // doubles per source record
constexpr int kStages = 4;          // TMA bulk-copy pipeline depth
constexpr int kMaxRanks = 64;      // P2P gather: arrival counters per buffer parity
constexpr int kExpShift = 11;
constexpr int kExpTable = 1 << kExpShift;  // 2^(j/2048) table for the FP64 exp

enum Scheme { kHobi = 0, kLobi = 1 };
enum KernelMode { kLaplace = 0, kScreened = 1 };

// Record `msg` as this thread's last error and return `status`.
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define HOBI_CUDA(call)                                   \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return hobi::cuda_fail(e_, #call); \
  } while (0)

// A pair of timing events destroyed on every exit path.
struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaError_t create() {
    cudaError_t e = cudaEventCreate(&a);
    return e != cudaSuccess ? e : cudaEventCreate(&b);
  }
  ~EventPair() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  int alloc(size_t count) {
    release();
    n = count;
    if (count == 0) return 0;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
};

// Page-locked host buffer (small per-iteration device->host reads).
template <typename T>
struct HostBuf {
  T* p = nullptr;
  size_t n = 0;
  int alloc(size_t count) {
    release();
    n = count;
    if (count == 0) return 0;
    cudaError_t e = cudaMallocHost(&p, count * sizeof(T));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocHost");
    return 0;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
  }
  ~HostBuf() { release(); }
};

// Constant physics, folded per scheme.
struct Physics {
  double eps1, eps2, kappa, er, ier;
  double diag1, diag2;  // 0.5*(1+er), 0.5*(1+1/er)  (solver.py:365-366)
  int mode;             // kLaplace when kappa == 0
  double len_scale;     // kappa for kScreened (coordinates are pre-scaled), 1 otherwise
  // Sweep frame: a fixed rotation q (row-major) applied to every sweep
  // position and normal, chosen so that no target normal has a zero (or
  // subnormal) z component in it; the sweep then holds target normals as
  // (nx/nz, ny/nz) and scales the K3+K4 row sum by nz once per item, which
  // saves two DMULs per pair (hobi_fastmath.cuh).  Distances and dot products
  // do not depend on the frame.
  int frame = 0;
  double q[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
};

// 3x3 matrix by value for kernel arguments.
struct Mat3 {
  double m[9];
};
constexpr int kNumFrames = 8;
void set_frame(Physics& p, int k);  // rotation k of a fixed generic sequence

struct Comm {
  void* nccl = nullptr;  // ncclComm_t
  int nranks = 1;
  int rank = 0;
  bool emulated = false;
  // fused epilogue + NVLink peer-store gather (hobi_comm_p2p_*)
  bool p2p = false;
  uint64_t epoch = 0;                 // operator applications gathered so far
  bool p2p_only = false;              // hobi_comm_init_p2p: ranks without an NCCL communicator
  bool p2p_fresh = false;             // receive area zeroed and not yet opened (hobi_comm_p2p_handle)
  bool p2p_pending = false;           // hobi_matvec_p2p_phase: send half done, receive half due
  std::vector<void*> opened;          // peer areas opened through CUDA IPC
};

// Device workspaces kept by a context across calls: cudaMalloc/cudaFree on
// every solve showed 0.1-0.3 s stalls on the B200 hosts.
// Inner-cycle state of the device-driven Arnoldi loop (hobi_gmres.cu).
struct GmresState {
  int j, total, m, max_it;
  double norm_b, tol;
};

// An instantiated CUDA graph, destroyed with its owner.
struct GraphHolder {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint64_t key = 0;           // DeviceOperator::graph_key() it was captured for
  int64_t step_launches = 0;  // kernels one loop iteration launches
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
    key = 0;
  }
  ~GraphHolder() { reset(); }
};

struct GmresWorkspace {
  DevBuf<double> V, w, x, r, b, part, hcol, nrm, y;
  HostBuf<double> hcol_h, nrm_h;  // pinned landing slots of the per-step reads
  // device-driven inner cycle: iterate copy, rotated Hessenberg, Givens
  // factors, rhs g, loop state (+ pinned mirrors) and the cycle's graph
  DevBuf<double> vin, H, cs, sn, g;
  DevBuf<GmresState> st;
  HostBuf<GmresState> st_h;
  HostBuf<double> H_h, g_h;
  GraphHolder cycle;
  int64_t n = -1, ldv = 0;
  int m = -1, grid = 1;
};

// numpy's float64 add.reduce over a short contiguous row (n <= 128): a
// left-to-right sum for n < 8, otherwise eight interleaved accumulators folded
// as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail -- the order
// `.sum(axis=1)` uses for the 4- and 16-point rows of solver.py:350-360.
template <typename Term>
__device__ __forceinline__ void numpy_row_sum(int n, Term term, double& s1, double& s2) {
  if (n < 8) {
    s1 = 0.0;
    s2 = 0.0;
    for (int m = 0; m < n; ++m) {
      double t1, t2;
      term(m, t1, t2);
      s1 += t1;
      s2 += t2;
    }
    return;
  }
  double r1[8], r2[8];
  const int nb = n - n % 8;
#pragma unroll
  for (int j = 0; j < 8; ++j) term(j, r1[j], r2[j]);
  for (int i = 8; i < nb; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double t1, t2;
      term(i + j, t1, t2);
      r1[j] += t1;
      r2[j] += t2;
    }
  }
  s1 = ((r1[0] + r1[1]) + (r1[2] + r1[3])) + ((r1[4] + r1[5]) + (r1[6] + r1[7]));
  s2 = ((r2[0] + r2[1]) + (r2[2] + r2[3])) + ((r2[4] + r2[5]) + (r2[6] + r2[7]));
  for (int m = nb; m < n; ++m) {
    double t1, t2;
    term(m, t1, t2);
    s1 += t1;
    s2 += t2;
  }
}

struct ChargeWorkspace {  // energy / RHS buffers for one charge set size
  int64_t nc = -1;
  DevBuf<double> q, qpos, tq, part, v, recv, e;
  DevBuf<int2> groups;
  DevBuf<unsigned long long> bad, bad_all;
  int n_groups = 0;
};

}  // namespace hobi

struct hobi_ctx {
  int device = 0;
  int scheme = hobi::kHobi;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;              // Duffy swap runs here, concurrent with the sweep
  cudaStream_t side2 = nullptr;             // rows past the last whole sweep tile, concurrent too
  cudaEvent_t fork = nullptr, join = nullptr, join2 = nullptr;
  hobi::Physics phys{};
  int64_t nv = 0, nf = 0;  // mesh sizes
  int64_t nt = 0;          // collocation points (targets)
  int64_t ns = 0;          // regular sources (nf*nq for hobi, nf for lobi)
  int nq = 0, nd = 0;
  int64_t ns_pad = 0, nt_pad = 0;
  int n_src_tiles = 0, n_groups = 0;
  hobi::DevBuf<int2> groups;                 // source groups: (first tile, tile count)
  int64_t lo = 0, hi = 0;  // owned rows

  // geometry (physical units)
  hobi::DevBuf<double> vert, vnrm;           // (nv,3)
  hobi::DevBuf<int> faces;                   // (nf,3)
  hobi::DevBuf<double> reg_pos, reg_nrm, reg_w;  // (nf,nq,3),(nf,nq,3),(nf,nq)
  hobi::DevBuf<double> duf_pos, duf_nrm, duf_w;  // pair order (3nf,nd,3)...
  hobi::DevBuf<double> node0_pos, node0_nrm;     // rotation-0 curved nodes (nf,10,3)
  hobi::DevBuf<int> pair_vertex, pair_face, pair_gverts, pair_starts;
  // per incident pair, 8 ints: vertex, face, the face's vertices, the rotated
  // element's vertices (prepare_singular; one 32-byte read per pair)
  hobi::DevBuf<int> pair_rec;
  std::vector<int> h_pair_starts;
  hobi::DevBuf<double> reg_bary, duf_bary;   // (nq,3), (nd,3)
  hobi::DevBuf<double> lobi_area;            // (nf)
  // sweep operands
  hobi::DevBuf<double> tgt;                  // (6, nt_pad) scaled SoA
  hobi::DevBuf<double> src;                  // (ns_pad, 12) scaled AoS records
  hobi::DevBuf<double> part;                 // (n_groups, 2, nt_pad)
  hobi::DevBuf<unsigned> ticket;             // work-item counter of the persistent sweep
  hobi::DevBuf<double> corr;                 // (3nf, 2) Duffy-minus-regular per pair
  hobi::DevBuf<double> u, out;               // (2nt)
  hobi::DevBuf<double> gather_send, gather_recv;  // (2*m), (nranks*2*m)
  // P2P area: two (2*nt) receive buffers (epoch parity) + 2 arrival counters,
  // exported to the peers through CUDA IPC; p2p_peers[r] = rank r's area.
  hobi::DevBuf<double> p2p_area;
  hobi::DevBuf<double*> p2p_peers;
  hobi::DevBuf<unsigned> p2p_done;
  // peer-arrival watchdog: the wait kernel gives up after p2p_timeout_ns and
  // raises *p2p_err (mapped pinned host memory), which synchronising calls check
  int* p2p_err = nullptr;
  int* p2p_err_dev = nullptr;
  unsigned long long p2p_timeout_ns = 0;
  unsigned long long p2p_extra = 0;  // test hook: wait for arrivals that never come
  int64_t gather_m = 0;
  hobi::Comm comm;

  // instrumentation
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<cudaEvent_t> ev_pool;   // recorded sweep brackets, read lazily
  // launch bookkeeping cached per sweep instantiation: (kernel, CTAs per SM)
  std::vector<std::pair<const void*, int>> occupancy;
  const double* singular_etab = nullptr;  // exp table on this device; set once singular_fast_kernel is opted in
  int sms = 0;
  size_t ev_used = 0;                  // pairs of ev_pool in flight
  double sweep_ms = 0.0;
  int64_t sweep_launches = 0;
  int64_t launches = 0;
  bool timing = true;
  int sweep_variant = 22;  // index into the sweep tuning table (hobi_sweep.cu): step_R7_minb2_unroll3
  bool variant_pinned = false;  // set by hobi_sweep_variant: no small-problem switch
  hobi::GmresWorkspace gmres_ws;
  hobi::ChargeWorkspace charge_ws;
  // Small host-buffer applications (hobi_matvec up to kHostGraphBytes): pinned
  // staging vectors and one captured graph, H2D -> matvec -> D2H, replayed per call.
  hobi::GraphHolder host_graph;
  hobi::HostBuf<double> host_in, host_out;
  int64_t host_calls = 0;
  bool host_graph_off = false;  // a capture failed once: this context keeps the plain path
};

namespace hobi {

// geometry (hobi_geometry.cu)
int upload_rule_tables(const double* reg_shape, int nq, const double* duf_shape, int nd,
                       const double* reg_wts, const double* duf_wts);
int build_geometry(hobi_ctx* c, const int* pair_of_slot, int* first_bad_slot, int* bad_code);
// function-level geometry (geometry.py) on caller arrays, current device, default stream
int geometry_fit_arcs(const double* p0, const double* n0, const double* p1, const double* n1, int64_t n,
                      double* coef, int* code);
int geometry_arc_normals(const double* coef, const double* t, const double* ref, int64_t n, double* nrm,
                         int* straight);
int geometry_nodes(const double* vdata, const double* ndata, int64_t n, double* node_pos,
                   double* node_nrm, int64_t* first_bad, int* bad_code);
int geometry_frames(const double* node_pos, const double* node_nrm, int64_t nelem, const double* shape,
                    int m, double* pos, double* nrm, double* jac, double* d_dr, double* d_ds);

// sweep (hobi_sweep.cu)
int upload_exp_table();
const double* exp_table_device();
int collect_sweep_timing(hobi_ctx* c);
int charge_workspace(hobi_ctx* c, int64_t nc);
std::vector<int2> make_groups(int n_src_tiles, int64_t target_tiles_at_8);
int sweep_variant_count();
const char* sweep_variant_name(int v);
int prepare_targets(hobi_ctx* c);
int prepare_static_sources(hobi_ctx* c);
int prepare_singular(hobi_ctx* c);
int matvec_rows_device(hobi_ctx* c, const double* u_dev, int64_t lo, int64_t hi, double* o1,
                       double* o2);
int matvec_full_device(hobi_ctx* c, const double* u_dev, double* out_dev);
int energy_device(hobi_ctx* c, const double* qpos, const double* q, int64_t nc,
                  const double* x_dev, double* energy);
int rhs_device(hobi_ctx* c, const double* qpos, const double* q, int64_t nc, double* b_dev);
int source_terms_device(const double* points, const double* normals, int64_t m, const double* qpos,
                        const double* q, int64_t nc, double* s1, double* s2);
int kernel_values_device(const double* d, const double* nx, const double* ny, int64_t n,
                         double eps1, double eps2, double kappa, double* k);

// Duffy swap over pairs [p0, p1) on `stream` (hobi_literal.cu)
int launch_singular(hobi_ctx* c, const double* u_dev, int64_t p0, int64_t p1, cudaStream_t stream);
int launch_singular_fast(hobi_ctx* c, const double* u_dev, int64_t p0, int64_t p1, cudaStream_t stream);

// GMRES (hobi_gmres.cu)
struct DeviceOperator {
  virtual int apply(const double* in_dev, double* out_dev) = 0;
  // Non-zero when apply() is a pure sequence of stream work on the GMRES
  // stream that may be captured into a CUDA graph and replayed; the value
  // changes whenever the captured work would (operator, tiling, ...).
  virtual uint64_t graph_key() { return 0; }
  // Bracket the capture: the operator stops recording its instrumentation
  // events (a captured cudaEventRecord never fires on replay).
  virtual void begin_capture() {}
  virtual void end_capture() {}
  virtual ~DeviceOperator() {}
};
int gmres_device(int device, cudaStream_t stream, int64_t n, DeviceOperator* op,
                 const double* b_host, double tol, int restart, int max_it, double* x_host,
                 int* iterations, double* residual, double* best, int* matvecs,
                 int64_t* launch_counter, GmresWorkspace* cached = nullptr);

// comm (hobi_api.cu): the operator's row gather, and a raw byte allgather
// (`bytes` per rank, rank-major into recv) on the context stream
int comm_allgather(hobi_ctx* c);
int comm_allgather_bytes(hobi_ctx* c, const void* send, void* recv, size_t bytes);
// gathered [rank][2][m] slots -> out[0:nt] ++ out[nt:2nt] (hobi_sweep.cu)
int gather_permute(hobi_ctx* c, double* out_dev);
int p2p_check(hobi_ctx* c);
// halves of the fused P2P gather (hobi_sweep.cu), for hobi_matvec_p2p_phase
int matvec_p2p_send(hobi_ctx* c, const double* u_dev);
int matvec_p2p_recv(hobi_ctx* c, double* out_dev);

}  // namespace hobi
