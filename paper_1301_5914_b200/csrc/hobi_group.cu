// Single-process multi-GPU operator (SolverConfig.workers -> GPUs, the
// reference's fork-pool row split, solver.py:405-477, without torchrun).
//
// A group holds one context per device, each with the full caches
// (replicated, as in the one-process-per-GPU mode).  Member i owns rows
// partition_targets(n, size)[i].  One application: the leader's input is
// copied peer-to-peer to every member (NVLink on an NVSwitch box), each member
// runs the sweep + epilogue of its rows on its own streams, and the epilogue
// kernel stores its finished rows straight into the leader's output vector
// over peer memory -- the gather is fused into the compute kernel, in final
// layout, with no staging buffer and no permutation; the leader waits on
// every member's event.  Without peer access a member stages its [2][m] slot
// and copies it over instead.  Only event waits order the devices --
// no kernel waits on another -- so members may share a device (that is how
// the path is tested on one GPU).  Rows are bitwise identical for any split,
// so a group solve equals the one-GPU solve bit for bit.  GMRES runs on the
// leader through the same device-resident solver.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "hobi_internal.cuh"

namespace hobi {
namespace {

struct Member {
  hobi_ctx* c = nullptr;
  int device = 0;       // kept so the group can be released after its members
  bool direct = false;  // epilogue stores straight into the leader's output (peer access)
  int64_t lo = 0, hi = 0;
  DevBuf<double> u, slot;  // input copy and [2][m] output slot on the member's device
  cudaEvent_t done = nullptr;
};

}  // namespace
}  // namespace hobi

struct hobi_group {
  std::vector<hobi::Member> m;
  int64_t nt = 0, slot_m = 0;
  hobi::DevBuf<double> recv;  // leader: [size][2][slot_m]
  cudaEvent_t in_ready = nullptr;
  hobi::GmresWorkspace gmres_ws;
};

using namespace hobi;

namespace {

struct GroupOperator : DeviceOperator {
  hobi_group* g;
  explicit GroupOperator(hobi_group* grp) : g(grp) {}
  int apply(const double* in, double* out) override {
    hobi_ctx* lead = g->m[0].c;
    const size_t bytes = 2 * g->nt * sizeof(double);
    HOBI_CUDA(cudaSetDevice(lead->device));
    HOBI_CUDA(cudaEventRecord(g->in_ready, lead->stream));
    for (size_t i = 0; i < g->m.size(); ++i) {
      Member& mb = g->m[i];
      hobi_ctx* c = mb.c;
      HOBI_CUDA(cudaSetDevice(c->device));
      HOBI_CUDA(cudaStreamWaitEvent(c->stream, g->in_ready, 0));
      const double* u = in;
      if (i > 0) {  // peer copy of the iterate (NVLink), then the member's own rows
        HOBI_CUDA(cudaMemcpyPeerAsync(mb.u.p, c->device, in, lead->device, bytes, c->stream));
        u = mb.u.p;
      }
      int rc;
      if (mb.direct) {
        // fused gather: the epilogue kernel's row stores land in the leader's
        // output vector (NVLink peer stores), final layout, nothing to permute
        rc = matvec_rows_device(c, u, mb.lo, mb.hi, out + mb.lo, out + g->nt + mb.lo);
        if (rc) return rc;
      } else {  // no peer access: stage the rows and copy them over
        rc = matvec_rows_device(c, u, mb.lo, mb.hi, mb.slot.p, mb.slot.p + g->slot_m);
        if (rc) return rc;
        HOBI_CUDA(cudaMemcpyPeerAsync(g->recv.p + i * 2 * g->slot_m, lead->device, mb.slot.p, c->device,
                                      2 * g->slot_m * sizeof(double), c->stream));
      }
      HOBI_CUDA(cudaEventRecord(mb.done, c->stream));
    }
    HOBI_CUDA(cudaSetDevice(lead->device));
    bool staged = false;
    for (Member& mb : g->m) {
      HOBI_CUDA(cudaStreamWaitEvent(lead->stream, mb.done, 0));
      staged |= !mb.direct;
    }
    if (!staged) return 0;
    // staged members: their slots arrived in the leader's receive buffer
    for (size_t i = 0; i < g->m.size(); ++i) {
      const Member& mb = g->m[i];
      if (mb.direct || mb.hi <= mb.lo) continue;
      const double* slot = g->recv.p + i * 2 * g->slot_m;
      HOBI_CUDA(cudaMemcpyAsync(out + mb.lo, slot, (mb.hi - mb.lo) * sizeof(double),
                                cudaMemcpyDeviceToDevice, lead->stream));
      HOBI_CUDA(cudaMemcpyAsync(out + g->nt + mb.lo, slot + g->slot_m, (mb.hi - mb.lo) * sizeof(double),
                                cudaMemcpyDeviceToDevice, lead->stream));
    }
    return 0;
  }
};

}  // namespace

extern "C" {

int hobi_group_create(hobi_ctx* const* members, int size, hobi_group** out) {
  *out = nullptr;
  if (size < 1 || !members) return fail(HOBI_ERR_VALUE, "a group needs at least one context");
  for (int i = 0; i < size; ++i) {
    const hobi_ctx* c = members[i];
    if (!c) return fail(HOBI_ERR_STATE, "null context in group");
    const hobi_ctx* l = members[0];
    if (c->nt != l->nt || c->ns != l->ns || c->scheme != l->scheme || c->nq != l->nq)
      return fail(HOBI_ERR_VALUE, "group members must discretise the same problem");
    if (c->comm.nranks != 1 || c->comm.emulated)
      return fail(HOBI_ERR_STATE, "group members must not be in a communicator or emulated split");
  }
  hobi_group* g = new hobi_group();
  auto bail = [&](int rc) {
    hobi_group_destroy(g);
    return rc;
  };
  g->nt = members[0]->nt;
  g->slot_m = std::max<int64_t>(1, (g->nt + size - 1) / size);
  g->m.resize(size);
  for (int i = 0; i < size; ++i) {
    Member& mb = g->m[i];
    mb.c = members[i];
    mb.device = mb.c->device;
    const int64_t base = g->nt / size, extra = g->nt % size;
    mb.lo = i * base + std::min<int64_t>(i, extra);
    mb.hi = mb.lo + base + (i < extra ? 1 : 0);
    if (cudaSetDevice(mb.c->device) != cudaSuccess) return bail(cuda_fail(cudaGetLastError(), "cudaSetDevice"));
    if (mb.u.alloc(2 * g->nt) || mb.slot.alloc(2 * g->slot_m)) return bail(HOBI_ERR_CUDA);
    cudaError_t e = cudaEventCreateWithFlags(&mb.done, cudaEventDisableTiming);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaEventCreate"));
  }
  hobi_ctx* lead = members[0];
  if (cudaSetDevice(lead->device) != cudaSuccess) return bail(cuda_fail(cudaGetLastError(), "cudaSetDevice"));
  if (g->recv.alloc((size_t)size * 2 * g->slot_m)) return bail(HOBI_ERR_CUDA);
  cudaError_t e = cudaEventCreateWithFlags(&g->in_ready, cudaEventDisableTiming);
  if (e != cudaSuccess) return bail(cuda_fail(e, "cudaEventCreate"));
  // peer access between distinct devices (NVLink); same-device members need none
  g->m[0].direct = true;
  for (int i = 1; i < size; ++i) {
    const int d = members[i]->device;
    if (d == lead->device) {
      g->m[i].direct = !getenv("HOBI_GROUP_STAGED");  // test hook: force the staged path
      continue;
    }
    int ok = 0;
    cudaDeviceCanAccessPeer(&ok, d, lead->device);
    g->m[i].direct = ok && !getenv("HOBI_GROUP_STAGED");
    if (ok) {
      cudaSetDevice(lead->device);
      e = cudaDeviceEnablePeerAccess(d, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return bail(cuda_fail(e, "peer access"));
      cudaSetDevice(d);
      e = cudaDeviceEnablePeerAccess(lead->device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return bail(cuda_fail(e, "peer access"));
      cudaGetLastError();  // clear a tolerated "already enabled"
    }
  }
  *out = g;
  return 0;
}

// Touches only the group's own resources (never the member contexts), so it
// is safe after the members are gone.
int hobi_group_destroy(hobi_group* g) {
  if (!g) return 0;
  for (Member& mb : g->m) {
    if (!mb.c) continue;
    cudaSetDevice(mb.device);
    cudaDeviceSynchronize();
    if (mb.done) cudaEventDestroy(mb.done);
    mb.u.release();
    mb.slot.release();
  }
  if (!g->m.empty()) cudaSetDevice(g->m[0].device);
  if (g->in_ready) cudaEventDestroy(g->in_ready);
  delete g;  // leader-device buffers free themselves (leader is current)
  return 0;
}

int hobi_group_matvec(hobi_group* g, const double* u, double* out) {
  if (!g) return fail(HOBI_ERR_STATE, "null group");
  hobi_ctx* lead = g->m[0].c;
  HOBI_CUDA(cudaSetDevice(lead->device));
  const size_t bytes = 2 * g->nt * sizeof(double);
  HOBI_CUDA(cudaMemcpyAsync(lead->u.p, u, bytes, cudaMemcpyHostToDevice, lead->stream));
  GroupOperator op(g);
  int rc = op.apply(lead->u.p, lead->out.p);
  if (rc) return rc;
  HOBI_CUDA(cudaSetDevice(lead->device));
  HOBI_CUDA(cudaMemcpyAsync(out, lead->out.p, bytes, cudaMemcpyDeviceToHost, lead->stream));
  HOBI_CUDA(cudaStreamSynchronize(lead->stream));
  return 0;
}

int hobi_group_info(hobi_group* g, int* size, int* devices, int64_t* lo, int64_t* hi, int* direct) {
  if (!g) return fail(HOBI_ERR_STATE, "null group");
  if (size) *size = (int)g->m.size();
  for (size_t i = 0; i < g->m.size(); ++i) {
    if (devices) devices[i] = g->m[i].device;
    if (lo) lo[i] = g->m[i].lo;
    if (hi) hi[i] = g->m[i].hi;
    if (direct) direct[i] = g->m[i].direct ? 1 : 0;
  }
  return 0;
}

// Timed group applications, the group analogue of hobi_bench: each step is
// bracketed by CUDA events on the leader's stream, and the leader's stream
// waits for every member's finishing event before the closing event, so a
// step's time is the slowest device's (max over the group).  Every member's
// L2 is flushed before the step (outside the brackets) when flush_l2 != 0.
int hobi_group_bench(hobi_group* g, const double* u, double* out, int steps, int mode, int flush_l2,
                     double* ms) {
  if (!g) return fail(HOBI_ERR_STATE, "null group");
  if (steps < 0 || (mode != 0 && mode != 1)) return fail(HOBI_ERR_VALUE, "bad bench arguments");
  hobi_ctx* lead = g->m[0].c;
  const size_t bytes = 2 * g->nt * sizeof(double);
  const size_t flush_bytes = (size_t)512 << 20;
  const size_t n = g->m.size();
  std::vector<DevBuf<unsigned char>> scratch(n);
  std::vector<cudaEvent_t> flushed(n, nullptr);
  auto cleanup = [&]() {
    for (size_t i = 0; i < n; ++i) {
      cudaSetDevice(g->m[i].device);
      if (flushed[i]) cudaEventDestroy(flushed[i]);
      scratch[i].release();
    }
    cudaSetDevice(lead->device);
  };
  int rc = 0;
  for (size_t i = 0; i < n && !rc; ++i) {
    if (cudaSetDevice(g->m[i].device) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "cudaSetDevice");
    if (!rc && flush_l2) rc = scratch[i].alloc(flush_bytes);
    if (!rc) {
      cudaError_t e = cudaEventCreateWithFlags(&flushed[i], cudaEventDisableTiming);
      if (e != cudaSuccess) rc = cuda_fail(e, "cudaEventCreate");
    }
  }
  if (rc) {
    cleanup();
    return rc;
  }
  EventPair ev;
  cudaSetDevice(lead->device);
  cudaError_t e = ev.create();
  if (e != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "cudaEventCreate");
  }
  GroupOperator op(g);
  if (mode == 0) {
    e = cudaMemcpyAsync(lead->u.p, u, bytes, cudaMemcpyHostToDevice, lead->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpyAsync");
  }
  for (int s = 0; s < steps && !rc; ++s) {
    for (size_t i = 0; i < n && !rc; ++i) {  // flush every member's L2, outside the brackets
      Member& mb = g->m[i];
      cudaSetDevice(mb.device);
      if (flush_l2) e = cudaMemsetAsync(scratch[i].p, s & 0xff, flush_bytes, mb.c->stream);
      if (e == cudaSuccess) e = cudaEventRecord(flushed[i], mb.c->stream);
      if (e != cudaSuccess) rc = cuda_fail(e, "flush");
    }
    if (rc) break;
    cudaSetDevice(lead->device);
    for (size_t i = 0; i < n; ++i) cudaStreamWaitEvent(lead->stream, flushed[i], 0);
    e = cudaEventRecord(ev.a, lead->stream);
    if (e == cudaSuccess && mode == 1)
      e = cudaMemcpyAsync(lead->u.p, u, bytes, cudaMemcpyHostToDevice, lead->stream);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "bench step");
      break;
    }
    rc = op.apply(lead->u.p, lead->out.p);  // ends with the leader waiting on every member
    if (rc) break;
    cudaSetDevice(lead->device);
    if (mode == 1) e = cudaMemcpyAsync(out, lead->out.p, bytes, cudaMemcpyDeviceToHost, lead->stream);
    if (e == cudaSuccess) e = cudaEventRecord(ev.b, lead->stream);
    if (e == cudaSuccess) e = cudaEventSynchronize(ev.b);
    float t = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, ev.a, ev.b);
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "bench step");
      break;
    }
    ms[s] = t;
  }
  if (!rc && mode == 0 && out) {
    cudaSetDevice(lead->device);
    e = cudaMemcpyAsync(out, lead->out.p, bytes, cudaMemcpyDeviceToHost, lead->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(lead->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "bench readback");
  }
  for (size_t i = 0; i < n; ++i) {  // the scratch buffers must not be freed under a pending memset
    cudaSetDevice(g->m[i].device);
    cudaStreamSynchronize(g->m[i].c->stream);
  }
  cleanup();
  return rc;
}

int hobi_group_gmres(hobi_group* g, const double* b, double tol, int restart, int max_it, double* x,
                     int* iterations, double* residual, double* best, int* matvecs) {
  if (!g) return fail(HOBI_ERR_STATE, "null group");
  hobi_ctx* lead = g->m[0].c;
  HOBI_CUDA(cudaSetDevice(lead->device));
  GroupOperator op(g);
  int rc = gmres_device(lead->device, lead->stream, 2 * g->nt, &op, b, tol, restart, max_it, x, iterations,
                        residual, best, matvecs, &lead->launches, &g->gmres_ws);
  cudaSetDevice(lead->device);
  return rc;
}

}  // extern "C"
