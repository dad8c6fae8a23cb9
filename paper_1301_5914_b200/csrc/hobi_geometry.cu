// Geometry precompute: curved cubic 10-node elements for every
// (face, rotation) slot and their frames at the regular and Duffy points.
//
// Reference: nodes_from_vertex_data (geometry.py:261-302) called from
// discretize (solver.py:194-206), frames_at (geometry.py:342-359) called at
// solver.py:217-227.  This translation unit is compiled with -fmad=false and
// writes every fused multiply-add explicitly, so it rounds exactly like the
// reference: np.dot / np.linalg.norm of a 3-vector are BLAS ddot
// (fma(z,z',fma(y,y',x*x'))), elementwise numpy arithmetic never fuses, and
// einsum over the 10 nodes is a left-to-right sum.  With IEEE sqrt and
// division on both sides the device caches reproduce the reference bit for bit.
#include "hobi_internal.cuh"

namespace hobi {

__constant__ double c_reg_shape[3][16][10];  // N, dN/dr, dN/ds at the regular points
__constant__ double c_duf_shape[3][64][10];  // same at the Duffy points
__constant__ double c_reg_wts[16];
__constant__ double c_duf_wts[64];

namespace {

struct V3 {
  double x, y, z;
};

__device__ __forceinline__ V3 ld3(const double* p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ void st3(double* p, V3 v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}
__device__ __forceinline__ V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 scl(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ V3 divs(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
// BLAS ddot rounding of np.dot on two 3-vectors.
__device__ __forceinline__ double bdot(V3 a, V3 b) { return fma(a.z, b.z, fma(a.y, b.y, a.x * b.x)); }
__device__ __forceinline__ double bnorm(V3 a) { return sqrt(bdot(a, a)); }

struct Arc {
  V3 c0, c1, c2, c3;
};

enum { kOk = 0, kCoincide = 1, kParallel = 2, kAntiparallel = 3 };

// fit_arc (geometry.py:46-84)
__device__ Arc fit_arc(V3 p0, V3 n0, V3 p1, V3 n1, int* code) {
  V3 chord = sub(p1, p0);
  double clen = bnorm(chord);
  if (clen < 1e-300 && *code == kOk) *code = kCoincide;
  V3 t0 = sub(chord, scl(bdot(chord, n0), n0));
  V3 t1 = sub(chord, scl(bdot(chord, n1), n1));
  double l0 = bnorm(t0), l1 = bnorm(t1);
  if ((l0 < 1e-12 * clen || l1 < 1e-12 * clen) && *code == kOk) *code = kParallel;
  t0 = divs(t0, l0);
  t1 = divs(t1, l1);
  double cos2t = fmin(fmax(bdot(t0, t1), -1.0), 1.0);
  double cost = sqrt(0.5 * (1.0 + cos2t));
  double mag = 2.0 * clen / (1.0 + cost);
  V3 m0 = scl(mag, t0), m1 = scl(mag, t1);
  Arc a;
  a.c0 = p0;
  a.c1 = m0;
  a.c2 = sub(sub(add(scl(-3.0, p0), scl(3.0, p1)), scl(2.0, m0)), m1);
  a.c3 = add(add(sub(scl(2.0, p0), scl(2.0, p1)), m0), m1);
  return a;
}

// arc_point (geometry.py:87-88)
__device__ __forceinline__ V3 arc_point(const Arc& a, double t) {
  return add(a.c0, scl(t, add(a.c1, scl(t, add(a.c2, scl(t, a.c3))))));
}

// arc_normal (geometry.py:99-121)
__device__ V3 arc_normal(const Arc& a, double t, V3 ref, int* straight = nullptr) {
  V3 v = add(a.c1, scl(t, add(scl(2.0, a.c2), scl(t, scl(3.0, a.c3)))));
  V3 acc = add(scl(2.0, a.c2), scl(6.0 * t, a.c3));
  double v2 = bdot(v, v);
  if (straight) *straight = 1;
  if (v2 < 1e-300) return ref;
  V3 k = divs(sub(acc, scl(bdot(v, acc) / v2, v)), sqrt(v2));
  double kl = bnorm(k);
  if (kl < 1e-12) return ref;
  if (straight) *straight = 0;
  V3 n = divs(k, kl);
  if (bdot(n, ref) < 0.0) n = {-n.x, -n.y, -n.z};
  return n;
}

// _blend_reference (geometry.py:252-258)
__device__ V3 blend(V3 n0, V3 n1, double t, int* code) {
  V3 r = add(scl(1.0 - t, n0), scl(t, n1));
  double len = bnorm(r);
  if (len < 1e-12 && *code == kOk) *code = kAntiparallel;
  return divs(r, len);
}

// One slot s = rot f + k: rotation k puts local vertex k of face f at node 1
// (solver.py:198-206; rot = 3 slots per face, or rot = 1 for the rotation-0
// element alone).  Writes 10 node positions and normals.
__global__ void nodes_kernel(const double* __restrict__ vert, const double* __restrict__ vnrm,
                             const int* __restrict__ faces, int64_t nslots, int rot,
                             double* __restrict__ node_pos, double* __restrict__ node_nrm,
                             unsigned long long* __restrict__ bad) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= nslots) return;
  int64_t f = s / rot;
  int k = (int)(s - rot * f);
  int i1 = faces[3 * f + k], i2 = faces[3 * f + (k + 1) % 3], i3 = faces[3 * f + (k + 2) % 3];
  V3 x1 = ld3(vert + 3 * i1), n1 = ld3(vnrm + 3 * i1);
  V3 x2 = ld3(vert + 3 * i2), n2 = ld3(vnrm + 3 * i2);
  V3 x3 = ld3(vert + 3 * i3), n3 = ld3(vnrm + 3 * i3);
  int code = kOk;
  V3 P[10], N[10];
  P[0] = x1; N[0] = n1;
  P[3] = x2; N[3] = n2;
  P[8] = x3; N[8] = n3;
  Arc a12 = fit_arc(x1, n1, x2, n2, &code);
  Arc a13 = fit_arc(x1, n1, x3, n3, &code);
  const double third = 1.0 / 3.0;
  const double tt[2] = {third, 2 * third};
  const int on12[2] = {1, 4}, on13[2] = {2, 5}, oncross[2] = {6, 7};
  for (int q = 0; q < 2; ++q) {
    P[on12[q]] = arc_point(a12, tt[q]);
    N[on12[q]] = arc_normal(a12, tt[q], blend(n1, n2, tt[q], &code));
  }
  for (int q = 0; q < 2; ++q) {
    P[on13[q]] = arc_point(a13, tt[q]);
    N[on13[q]] = arc_normal(a13, tt[q], blend(n1, n3, tt[q], &code));
  }
  V3 y1 = arc_point(a12, 1.0), y2 = arc_point(a13, 1.0);
  V3 ny1 = arc_normal(a12, 1.0, n2), ny2 = arc_normal(a13, 1.0, n3);
  Arc cr = fit_arc(y1, ny1, y2, ny2, &code);
  for (int q = 0; q < 2; ++q) {
    P[oncross[q]] = arc_point(cr, tt[q]);
    N[oncross[q]] = arc_normal(cr, tt[q], blend(ny1, ny2, tt[q], &code));
  }
  Arc mid = fit_arc(P[4], N[4], P[5], N[5], &code);
  P[9] = arc_point(mid, 0.5);
  N[9] = arc_normal(mid, 0.5, blend(N[4], N[5], 0.5, &code));
  for (int n = 0; n < 10; ++n) {
    st3(node_pos + (s * 10 + n) * 3, P[n]);
    st3(node_nrm + (s * 10 + n) * 3, N[n]);
  }
  if (code != kOk) atomicMin(bad, (unsigned long long)(s * 4 + code));
}

// frames_at (geometry.py:342-359) at one point: position, tangents, oriented
// unit normal and Jacobian from the element's 10 nodes and the three shape rows.
__device__ __forceinline__ void frame_eval(const double* __restrict__ P, const double* __restrict__ Nn,
                                           const double* __restrict__ B, const double* __restrict__ Br,
                                           const double* __restrict__ Bs, V3& x, V3& xr, V3& xs, V3& n,
                                           double& jac) {
  x = {0, 0, 0};
  xr = {0, 0, 0};
  xs = {0, 0, 0};
  V3 h = {0, 0, 0};
  for (int k = 0; k < 10; ++k) {  // einsum "mk,eki->emi": left-to-right, unfused
    V3 pk = ld3(P + 3 * k), nk = ld3(Nn + 3 * k);
    x = add(x, scl(B[k], pk));
    xr = add(xr, scl(Br[k], pk));
    xs = add(xs, scl(Bs[k], pk));
    h = add(h, scl(B[k], nk));
  }
  V3 c = {xr.y * xs.z - xr.z * xs.y, xr.z * xs.x - xr.x * xs.z, xr.x * xs.y - xr.y * xs.x};
  jac = sqrt(c.x * c.x + c.y * c.y + c.z * c.z);
  n = divs(c, jac);
  double sd = 0.0;
  sd = sd + n.x * h.x;
  sd = sd + n.y * h.y;
  sd = sd + n.z * h.z;
  if (sd < 0.0) n = {-n.x, -n.y, -n.z};
}

// Element e at point m of a rule.  Writes position, oriented unit normal and
// weight*Jacobian at `dst`.
template <bool DUFFY>
__global__ void frames_kernel(const double* __restrict__ node_pos, const double* __restrict__ node_nrm,
                              int64_t nelem, int nslot_stride, int npts,
                              const int* __restrict__ dst_of_elem, double* __restrict__ pos,
                              double* __restrict__ nrm, double* __restrict__ w) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nelem * npts) return;
  int64_t e = t / npts;
  int m = (int)(t - e * npts);
  // element e reads slot e*nslot_stride (rotation 0 only for the regular rule)
  const double* P = node_pos + (e * nslot_stride) * 30;
  const double* Nn = node_nrm + (e * nslot_stride) * 30;
  const double* B = DUFFY ? c_duf_shape[0][m] : c_reg_shape[0][m];
  const double* Br = DUFFY ? c_duf_shape[1][m] : c_reg_shape[1][m];
  const double* Bs = DUFFY ? c_duf_shape[2][m] : c_reg_shape[2][m];
  V3 x, xr, xs, n;
  double jac;
  frame_eval(P, Nn, B, Br, Bs, x, xr, xs, n, jac);
  int64_t d = DUFFY ? dst_of_elem[e] : e;
  st3(pos + (d * npts + m) * 3, x);
  st3(nrm + (d * npts + m) * 3, n);
  w[d * npts + m] = (DUFFY ? c_duf_wts[m] : c_reg_wts[m]) * jac;
}

// The geometry module's function-level forms (geometry.py), batched: the same
// device functions the precompute uses, on caller-supplied arrays.
__global__ void fit_arcs_kernel(const double* __restrict__ p0, const double* __restrict__ n0,
                                const double* __restrict__ p1, const double* __restrict__ n1, int64_t n,
                                double* __restrict__ coef, int* __restrict__ code) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = kOk;
  Arc a = fit_arc(ld3(p0 + 3 * i), ld3(n0 + 3 * i), ld3(p1 + 3 * i), ld3(n1 + 3 * i), &c);
  st3(coef + 12 * i, a.c0);
  st3(coef + 12 * i + 3, a.c1);
  st3(coef + 12 * i + 6, a.c2);
  st3(coef + 12 * i + 9, a.c3);
  code[i] = c;
}

__global__ void arc_normals_kernel(const double* __restrict__ coef, const double* __restrict__ t,
                                   const double* __restrict__ ref, int64_t n, double* __restrict__ nrm,
                                   int* __restrict__ straight) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  Arc a = {ld3(coef + 12 * i), ld3(coef + 12 * i + 3), ld3(coef + 12 * i + 6), ld3(coef + 12 * i + 9)};
  int flag = 0;
  st3(nrm + 3 * i, arc_normal(a, t[i], ld3(ref + 3 * i), &flag));
  straight[i] = flag;
}

// frames_at for nelem elements at m caller-chosen reference points; shape is
// the (3, m, 10) table N, dN/dr, dN/ds in global memory.
__global__ void frames_at_kernel(const double* __restrict__ node_pos, const double* __restrict__ node_nrm,
                                 int64_t nelem, const double* __restrict__ shape, int m,
                                 double* __restrict__ pos, double* __restrict__ nrm,
                                 double* __restrict__ jac, double* __restrict__ d_dr,
                                 double* __restrict__ d_ds) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nelem * m) return;
  int64_t e = t / m;
  int q = (int)(t - e * m);
  V3 x, xr, xs, n;
  double j;
  frame_eval(node_pos + e * 30, node_nrm + e * 30, shape + (int64_t)q * 10,
             shape + ((int64_t)m + q) * 10, shape + (2 * (int64_t)m + q) * 10, x, xr, xs, n, j);
  st3(pos + 3 * t, x);
  st3(nrm + 3 * t, n);
  jac[t] = j;
  if (d_dr) st3(d_dr + 3 * t, xr);
  if (d_ds) st3(d_ds + 3 * t, xs);
}

}  // namespace

int upload_rule_tables(const double* reg_shape, int nq, const double* duf_shape, int nd,
                       const double* reg_wts, const double* duf_wts) {
  double rs[3][16][10] = {}, ds[3][64][10] = {}, rw[16] = {}, dw[64] = {};
  for (int c = 0; c < 3; ++c) {
    for (int m = 0; m < nq; ++m)
      for (int k = 0; k < 10; ++k) rs[c][m][k] = reg_shape[(c * nq + m) * 10 + k];
    for (int m = 0; m < nd; ++m)
      for (int k = 0; k < 10; ++k) ds[c][m][k] = duf_shape[(c * nd + m) * 10 + k];
  }
  for (int m = 0; m < nq; ++m) rw[m] = reg_wts[m];
  for (int m = 0; m < nd; ++m) dw[m] = duf_wts[m];
  HOBI_CUDA(cudaMemcpyToSymbol(c_reg_shape, rs, sizeof(rs)));
  HOBI_CUDA(cudaMemcpyToSymbol(c_duf_shape, ds, sizeof(ds)));
  HOBI_CUDA(cudaMemcpyToSymbol(c_reg_wts, rw, sizeof(rw)));
  HOBI_CUDA(cudaMemcpyToSymbol(c_duf_wts, dw, sizeof(dw)));
  return 0;
}

int build_geometry(hobi_ctx* c, const int* pair_of_slot_host, int* first_bad_slot, int* bad_code) {
  const int64_t nslots = 3 * c->nf;
  *first_bad_slot = -1;
  *bad_code = 0;
  if (nslots == 0) return 0;
  DevBuf<double> npos, nnrm;
  DevBuf<int> perm;
  DevBuf<unsigned long long> bad;
  if (npos.alloc(nslots * 30) || nnrm.alloc(nslots * 30) || perm.alloc(nslots) || bad.alloc(1))
    return HOBI_ERR_CUDA;
  HOBI_CUDA(cudaMemcpyAsync(perm.p, pair_of_slot_host, nslots * sizeof(int), cudaMemcpyHostToDevice,
                            c->stream));
  HOBI_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), c->stream));
  const int T = 128;
  nodes_kernel<<<(unsigned)((nslots + T - 1) / T), T, 0, c->stream>>>(
      c->vert.p, c->vnrm.p, c->faces.p, nslots, 3, npos.p, nnrm.p, bad.p);
  c->launches++;
  HOBI_CUDA(cudaGetLastError());
  unsigned long long badh = 0;
  HOBI_CUDA(cudaMemcpyAsync(&badh, bad.p, sizeof(badh), cudaMemcpyDeviceToHost, c->stream));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  if (badh != ~0ull) {
    *first_bad_slot = (int)(badh / 4);
    *bad_code = (int)(badh % 4);
    return 0;
  }
  int64_t nreg = c->nf * c->nq;
  frames_kernel<false><<<(unsigned)((nreg + T - 1) / T), T, 0, c->stream>>>(
      npos.p, nnrm.p, c->nf, 3, c->nq, nullptr, c->reg_pos.p, c->reg_nrm.p, c->reg_w.p);
  c->launches++;
  int64_t nduf = nslots * c->nd;
  frames_kernel<true><<<(unsigned)((nduf + T - 1) / T), T, 0, c->stream>>>(
      npos.p, nnrm.p, nslots, 1, c->nd, perm.p, c->duf_pos.p, c->duf_nrm.p, c->duf_w.p);
  c->launches++;
  HOBI_CUDA(cudaGetLastError());
  // keep the rotation-0 nodes (the reference's CurvedElement per face)
  if (c->node0_pos.alloc(30 * c->nf) || c->node0_nrm.alloc(30 * c->nf)) return HOBI_ERR_CUDA;
  HOBI_CUDA(cudaMemcpy2DAsync(c->node0_pos.p, 30 * sizeof(double), npos.p, 90 * sizeof(double),
                              30 * sizeof(double), c->nf, cudaMemcpyDeviceToDevice, c->stream));
  HOBI_CUDA(cudaMemcpy2DAsync(c->node0_nrm.p, 30 * sizeof(double), nnrm.p, 90 * sizeof(double),
                              30 * sizeof(double), c->nf, cudaMemcpyDeviceToDevice, c->stream));
  HOBI_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

namespace {
template <class T>
int to_device(DevBuf<T>& b, const T* h, int64_t n) {
  if (b.alloc(n)) return HOBI_ERR_CUDA;
  HOBI_CUDA(cudaMemcpy(b.p, h, n * sizeof(T), cudaMemcpyHostToDevice));
  return 0;
}
template <class T>
int to_host(T* h, const DevBuf<T>& b, int64_t n) {
  HOBI_CUDA(cudaMemcpy(h, b.p, n * sizeof(T), cudaMemcpyDeviceToHost));
  return 0;
}
inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
}  // namespace

int geometry_fit_arcs(const double* p0, const double* n0, const double* p1, const double* n1, int64_t n,
                      double* coef, int* code) {
  if (n == 0) return 0;
  DevBuf<double> a, b, c, d, o;
  DevBuf<int> k;
  int rc;
  if ((rc = to_device(a, p0, 3 * n)) || (rc = to_device(b, n0, 3 * n)) || (rc = to_device(c, p1, 3 * n)) ||
      (rc = to_device(d, n1, 3 * n)))
    return rc;
  if (o.alloc(12 * n) || k.alloc(n)) return HOBI_ERR_CUDA;
  fit_arcs_kernel<<<blocks(n, 128), 128>>>(a.p, b.p, c.p, d.p, n, o.p, k.p);
  HOBI_CUDA(cudaGetLastError());
  if ((rc = to_host(coef, o, 12 * n)) || (rc = to_host(code, k, n))) return rc;
  return 0;
}

int geometry_arc_normals(const double* coef, const double* t, const double* ref, int64_t n, double* nrm,
                         int* straight) {
  if (n == 0) return 0;
  DevBuf<double> a, b, c, o;
  DevBuf<int> k;
  int rc;
  if ((rc = to_device(a, coef, 12 * n)) || (rc = to_device(b, t, n)) || (rc = to_device(c, ref, 3 * n)))
    return rc;
  if (o.alloc(3 * n) || k.alloc(n)) return HOBI_ERR_CUDA;
  arc_normals_kernel<<<blocks(n, 128), 128>>>(a.p, b.p, c.p, n, o.p, k.p);
  HOBI_CUDA(cudaGetLastError());
  if ((rc = to_host(nrm, o, 3 * n)) || (rc = to_host(straight, k, n))) return rc;
  return 0;
}

// nodes_from_vertex_data for n vertex triples: vdata is (n, 3, 3) positions,
// ndata (n, 3, 3) unit normals (triangle i has vertices 3i, 3i+1, 3i+2).
int geometry_nodes(const double* vdata, const double* ndata, int64_t n, double* node_pos,
                   double* node_nrm, int64_t* first_bad, int* bad_code) {
  *first_bad = -1;
  *bad_code = 0;
  if (n == 0) return 0;
  if (3 * n > 0x7fffffffll) return fail(HOBI_ERR_VALUE, "too many elements for 32-bit vertex ids");
  DevBuf<double> v, nn, op, on;
  DevBuf<int> f;
  DevBuf<unsigned long long> bad;
  int rc;
  if ((rc = to_device(v, vdata, 9 * n)) || (rc = to_device(nn, ndata, 9 * n))) return rc;
  std::vector<int> faces(3 * n);
  for (int64_t i = 0; i < 3 * n; ++i) faces[i] = (int)i;
  if ((rc = to_device(f, faces.data(), 3 * n))) return rc;
  if (op.alloc(30 * n) || on.alloc(30 * n) || bad.alloc(1)) return HOBI_ERR_CUDA;
  HOBI_CUDA(cudaMemset(bad.p, 0xff, sizeof(unsigned long long)));
  nodes_kernel<<<blocks(n, 128), 128>>>(v.p, nn.p, f.p, n, 1, op.p, on.p, bad.p);
  HOBI_CUDA(cudaGetLastError());
  unsigned long long badh = 0;
  HOBI_CUDA(cudaMemcpy(&badh, bad.p, sizeof(badh), cudaMemcpyDeviceToHost));
  if (badh != ~0ull) {
    *first_bad = (int64_t)(badh / 4);
    *bad_code = (int)(badh % 4);
    return 0;
  }
  if ((rc = to_host(node_pos, op, 30 * n)) || (rc = to_host(node_nrm, on, 30 * n))) return rc;
  return 0;
}

int geometry_frames(const double* node_pos, const double* node_nrm, int64_t nelem, const double* shape,
                    int m, double* pos, double* nrm, double* jac, double* d_dr, double* d_ds) {
  const int64_t total = nelem * m;
  if (total == 0) return 0;
  DevBuf<double> p, nn, sh, op, on, oj, or_, os;
  int rc;
  if ((rc = to_device(p, node_pos, 30 * nelem)) || (rc = to_device(nn, node_nrm, 30 * nelem)) ||
      (rc = to_device(sh, shape, 30 * (int64_t)m)))
    return rc;
  if (op.alloc(3 * total) || on.alloc(3 * total) || oj.alloc(total)) return HOBI_ERR_CUDA;
  if (d_dr && or_.alloc(3 * total)) return HOBI_ERR_CUDA;
  if (d_ds && os.alloc(3 * total)) return HOBI_ERR_CUDA;
  frames_at_kernel<<<blocks(total, 128), 128>>>(p.p, nn.p, nelem, sh.p, m, op.p, on.p, oj.p,
                                                d_dr ? or_.p : nullptr, d_ds ? os.p : nullptr);
  HOBI_CUDA(cudaGetLastError());
  if ((rc = to_host(pos, op, 3 * total)) || (rc = to_host(nrm, on, 3 * total)) ||
      (rc = to_host(jac, oj, total)))
    return rc;
  if (d_dr && (rc = to_host(d_dr, or_, 3 * total))) return rc;
  if (d_ds && (rc = to_host(d_ds, os, 3 * total))) return rc;
  return 0;
}

}  // namespace hobi
