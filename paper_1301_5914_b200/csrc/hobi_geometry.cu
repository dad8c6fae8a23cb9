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
__device__ V3 arc_normal(const Arc& a, double t, V3 ref) {
  V3 v = add(a.c1, scl(t, add(scl(2.0, a.c2), scl(t, scl(3.0, a.c3)))));
  V3 acc = add(scl(2.0, a.c2), scl(6.0 * t, a.c3));
  double v2 = bdot(v, v);
  if (v2 < 1e-300) return ref;
  V3 k = divs(sub(acc, scl(bdot(v, acc) / v2, v)), sqrt(v2));
  double kl = bnorm(k);
  if (kl < 1e-12) return ref;
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

// One slot s = 3 f + k: rotation k puts local vertex k of face f at node 1
// (solver.py:198-206).  Writes 10 node positions and normals.
__global__ void nodes_kernel(const double* __restrict__ vert, const double* __restrict__ vnrm,
                             const int* __restrict__ faces, int64_t nslots,
                             double* __restrict__ node_pos, double* __restrict__ node_nrm,
                             unsigned long long* __restrict__ bad) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= nslots) return;
  int64_t f = s / 3;
  int k = (int)(s - 3 * f);
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

// frames_at (geometry.py:342-359) for element e at point m of a rule.
// Writes position, oriented unit normal and weight*Jacobian at `dst`.
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
  V3 x = {0, 0, 0}, xr = {0, 0, 0}, xs = {0, 0, 0}, h = {0, 0, 0};
  for (int k = 0; k < 10; ++k) {  // einsum "mk,eki->emi": left-to-right, unfused
    V3 pk = ld3(P + 3 * k), nk = ld3(Nn + 3 * k);
    x = add(x, scl(B[k], pk));
    xr = add(xr, scl(Br[k], pk));
    xs = add(xs, scl(Bs[k], pk));
    h = add(h, scl(B[k], nk));
  }
  V3 c = {xr.y * xs.z - xr.z * xs.y, xr.z * xs.x - xr.x * xs.z, xr.x * xs.y - xr.y * xs.x};
  double jac = sqrt(c.x * c.x + c.y * c.y + c.z * c.z);
  V3 n = divs(c, jac);
  double sd = 0.0;
  sd = sd + n.x * h.x;
  sd = sd + n.y * h.y;
  sd = sd + n.z * h.z;
  if (sd < 0.0) n = {-n.x, -n.y, -n.z};
  int64_t d = DUFFY ? dst_of_elem[e] : e;
  st3(pos + (d * npts + m) * 3, x);
  st3(nrm + (d * npts + m) * 3, n);
  w[d * npts + m] = (DUFFY ? c_duf_wts[m] : c_reg_wts[m]) * jac;
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
      c->vert.p, c->vnrm.p, c->faces.p, nslots, npos.p, nnrm.p, bad.p);
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

}  // namespace hobi
