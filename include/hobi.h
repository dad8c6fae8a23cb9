/*
 * hobi.h -- C ABI of the B200-native HOBI-PB boundary-integral hot path.
 *
 * The reference (arXiv 1301.5914 restated as the Python package `pbbem`, see
 * SURVEY.md) has no native boundary: its hot path is the Python operator
 * protocol in /root/reference/pkg/src/pbbem/solver.py.  Each entry point below
 * replaces one reference interface, cited as file:line relative to that
 * package.  Plain pointers and sizes only; every array is C-contiguous
 * float64 / int64 in the reference's layout; all pointers are HOST pointers
 * unless the name ends in `_device`.  The library owns its device buffers
 * for the lifetime of a context.  Contexts are not thread-safe.
 *
 * Status codes map 1:1 to the reference's exception types (hobi_last_error()
 * returns the message text, formatted like the reference's).
 */
#ifndef HOBI_H
#define HOBI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HOBI_ABI_VERSION 1

enum hobi_status {
  HOBI_OK = 0,
  HOBI_ERR_VALUE = 1,          /* ValueError (solver.py:373-374, 381-382, 493-494)          */
  HOBI_ERR_DEGENERATE_ARC = 2, /* geometry.DegenerateArcError ("face f: ...", solver.py:205) */
  HOBI_ERR_SINGULARITY = 3,    /* kernels.SingularityError (kernels.py:167-172)             */
  HOBI_ERR_NONCONVERGENCE = 4, /* solver.GmresNonConvergence (solver.py:521-526)             */
  HOBI_ERR_CUDA = 5,           /* device / driver failure                                    */
  HOBI_ERR_NCCL = 6,           /* collective failure                                         */
  HOBI_ERR_STATE = 7           /* misuse of the API (wrong order of calls, bad handle)       */
};

/* A context owns its streams and workspaces: use one from one thread at a time;
 * different contexts may be driven from different threads concurrently. */
typedef struct hobi_ctx hobi_ctx;

/* Message of the last failing call on this thread ("" if none). */
const char* hobi_last_error(void);
int hobi_abi_version(void);
int hobi_device_count(int* count);
/* Streaming multiprocessors of a device (roofline bookkeeping). */
int hobi_device_sms(int device, int* sms);

/*
 * Build every discretisation cache on `device`: curved cubic nodes for the
 * three rotations of every face, frames at the regular and Duffy points,
 * incident-pair tables.  Replaces solver.discretize (solver.py:165-266) for
 * scheme "hobi" (the mesh must already have passed FlatMesh.validate,
 * mesh.py:50-75, which the host wrapper calls first).
 *   vertices, normals : (nv, 3)      faces : (nf, 3) int64
 *   reg_pts (nq, 2), reg_wts (nq), reg_shape (3, nq, 10): N, dN/dr, dN/ds
 *   (quadrature.py:68-87, geometry.py:197-205); duf_* likewise for the
 *   Duffy rule (quadrature.py:101-116).  nq <= 16, nd <= 64.
 * Fails with HOBI_ERR_DEGENERATE_ARC at the first failing face in face
 * order, rotations 0,1,2 (solver.py:198-206).
 */
int hobi_create(int device, const double* vertices, const double* normals, int64_t nv,
                const int64_t* faces, int64_t nf, double eps1, double eps2, double kappa,
                const double* reg_pts, const double* reg_wts, const double* reg_shape, int nq,
                const double* duf_pts, const double* duf_wts, const double* duf_shape, int nd,
                hobi_ctx** out);

/*
 * hobi_create with the reference's default rules built in: the 4-point
 * conical Gauss-Radau regular rule and the duffy_points x duffy_points Duffy
 * rule (duffy_points in {4, 6, 8}; SolverConfig's default is 4), with their
 * cubic shape tables (quadrature.py:68-116, geometry.py:197-205) -- the same
 * bits the Python host computes, so a C/C++ integrator gets the same caches
 * without any quadrature code of its own.
 */
int hobi_create_default(int device, const double* vertices, const double* normals, int64_t nv,
                        const int64_t* faces, int64_t nf, double eps1, double eps2, double kappa,
                        int duffy_points, hobi_ctx** out);

/*
 * Build a HOBI context from caches computed elsewhere -- e.g. the fields of
 * the reference's own DiscretizedProblem (solver.py:122-140: reg_pos/nrm/w,
 * reg_bary, duf_pos/nrm/w, duf_bary, pair_vertex/face/gverts/starts, in the
 * reference's layouts) -- so a pbbem installation can keep its discretize
 * and swap in only the operator, GMRES, RHS and energy.
 */
int hobi_create_from_caches(int device, const double* vertices, const double* normals, int64_t nv,
                            const int64_t* faces, int64_t nf, double eps1, double eps2, double kappa,
                            const double* reg_pos, const double* reg_nrm, const double* reg_w,
                            const double* reg_bary, int nq, const double* duf_pos,
                            const double* duf_nrm, const double* duf_w, const double* duf_bary, int nd,
                            const int64_t* pair_vertex, const int64_t* pair_face,
                            const int64_t* pair_gverts, const int64_t* pair_starts, hobi_ctx** out);

/* LOBI (flat centroid) discretisation: solver.py:177-186.  No rules needed. */
int hobi_create_lobi(int device, const double* vertices, const double* normals, int64_t nv,
                     const int64_t* faces, int64_t nf, double eps1, double eps2, double kappa,
                     hobi_ctx** out);

/* Release the context: _Operator.close (solver.py:461-466). */
int hobi_destroy(hobi_ctx* ctx);

/* n_collocation (solver.py:142-144): N_v for hobi, N_f for lobi. */
int hobi_size(hobi_ctx* ctx, int64_t* n_colloc, int64_t* n_sources);

/*
 * One operator application u -> A u over HOST buffers of length 2*n_colloc,
 * including both copies: _Operator.__call__ / matvec_hobi / matvec_lobi
 * (solver.py:447-459, 370-390).  Under a communicator (hobi_comm_init) every
 * rank passes the full u and receives the full A u.
 */
int hobi_matvec(hobi_ctx* ctx, const double* u, double* out);
/* Same on device pointers already resident in HBM (the ctx's stream). */
int hobi_matvec_device(hobi_ctx* ctx, const double* u_device, double* out_device);
/*
 * Rows [lo, hi) of both blocks only: _apply_range (solver.py:278-367).
 * out_phi, out_dphi have hi-lo entries each.  Results are bitwise
 * independent of how [0, n) is split (solver.py:12-17).
 */
int hobi_matvec_rows(hobi_ctx* ctx, const double* u, int64_t lo, int64_t hi, double* out_phi,
                     double* out_dphi);

/* b = (S1, S2)/eps1 at the collocation points: assemble_rhs (solver.py:393-402)
 * over source_terms_at (kernels.py:159-178).  b has 2*n_colloc entries. */
int hobi_rhs(hobi_ctx* ctx, const double* qpos, const double* q, int64_t nc, double* b);

/* Reaction-field energy in kcal/mol: solvation_energy (solver.py:581-614). */
int hobi_energy(hobi_ctx* ctx, const double* qpos, const double* q, int64_t nc, const double* phi,
                const double* dphi, double* energy);

/*
 * Device-resident restarted GMRES with MGS + Givens and true-residual restarts:
 * gmres_solve (solver.py:484-560) applied to this context's operator.  x has
 * 2*n_colloc entries.  On HOBI_ERR_NONCONVERGENCE `best` holds the best
 * relative residual (GmresNonConvergence.best_residual).
 */
int hobi_gmres(hobi_ctx* ctx, const double* b, double tol, int restart, int max_it, double* x,
               int* iterations, double* residual, double* best, int* matvecs);

/*
 * solve() after discretize (solver.py:563-574) in one call, for C/C++
 * integrators: RHS, GMRES to `tol`, then the energy.  phi and dphi receive
 * n_colloc entries each; iterations/residual/matvecs as hobi_gmres.  Status
 * codes as the three calls it chains (a non-converged solve returns
 * HOBI_ERR_NONCONVERGENCE; phi, dphi and energy are then unspecified).
 */
int hobi_solve(hobi_ctx* ctx, const double* qpos, const double* q, int64_t nc, double tol, int restart,
               int max_it, double* phi, double* dphi, double* energy, int* iterations, double* residual,
               int* matvecs);

/*
 * The same GMRES on an arbitrary operator supplied as a host callback
 * (gmres_solve accepts any callable, solver.py:484).  `apply` receives host
 * arrays of length n and returns 0 on success.
 */
typedef int (*hobi_apply_fn)(void* user, const double* in, double* out, int64_t n);
int hobi_gmres_host_operator(int device, int64_t n, hobi_apply_fn apply, void* user,
                             const double* b, double tol, int restart, int max_it, double* x,
                             int* iterations, double* residual, double* best, int* matvecs);

/* Copy device caches back in the reference's layout (DiscretizedProblem fields,
 * solver.py:122-140).  Any pointer may be NULL. */
int hobi_export_caches(hobi_ctx* ctx, double* reg_pos, double* reg_nrm, double* reg_w,
                       double* duf_pos, double* duf_nrm, double* duf_w, int64_t* pair_vertex,
                       int64_t* pair_face, int64_t* pair_gverts, int64_t* pair_starts);

/* The rotation-0 curved element of every face, (nf, 10, 3) node positions and
 * unit node normals: DiscretizedProblem.elements (solver.py:208-215). */
int hobi_export_nodes(hobi_ctx* ctx, double* node_pos, double* node_nrm);

/* K1..K4 of kernels.kernel_values_d (kernels.py:99-130) on the device, for n
 * displacement/normal triples (n,3); k has shape (4, n).  Test hook. */
int hobi_kernel_values(int device, const double* d, const double* nx, const double* ny, int64_t n,
                       double eps1, double eps2, double kappa, double* k);

/* kernels.source_terms_at (kernels.py:159-178): S1 = sum_k q_k G0 and
 * S2 = sum_k q_k dG0/dn_x at m surface points (m,3) with unit normals (m,3),
 * unscaled.  HOBI_ERR_SINGULARITY ("surface point i coincides with charge k")
 * when a point sits on a charge. */
int hobi_source_terms(int device, const double* points, const double* normals, int64_t m,
                      const double* qpos, const double* q, int64_t nc, double* s1, double* s2);

/*
 * The geometry module's functions (geometry.py) on caller arrays: the device
 * functions the precompute of hobi_create runs, batched over n items.
 *
 * hobi_geometry_fit_arcs: fit_arc (geometry.py:46-84) for n endpoint pairs
 *   (n,3) each; coef is (n, 4, 3) = c0..c3, code[i] is 0, 1 (endpoints
 *   coincide) or 2 (endpoint normal nearly parallel to the chord).
 * hobi_geometry_arc_normals: arc_normal (geometry.py:99-121) at parameter t[i]
 *   of arc coef[i] with sign reference (n,3); straight[i] = 1 where the
 *   reference itself was returned.
 * hobi_geometry_nodes: nodes_from_vertex_data (geometry.py:261-302) for n
 *   vertex triples, vertex_pos / vertex_nrm (n, 3, 3); node_pos / node_nrm are
 *   (n, 10, 3).  first_bad = -1, or the first triple whose arcs are degenerate
 *   with bad_code 1, 2 or 3 (endpoint normals antiparallel); the node arrays
 *   are not written then.
 * hobi_geometry_frames: frames_at (geometry.py:342-359) for n_elements
 *   elements (n, 10, 3) at n_points reference points given as the (3,
 *   n_points, 10) table N, dN/dr, dN/ds; pos / nrm are (n, n_points, 3), jac
 *   (n, n_points); d_dr / d_ds (n, n_points, 3) may be NULL.
 */
int hobi_geometry_fit_arcs(int device, const double* p0, const double* n0, const double* p1,
                           const double* n1, int64_t n, double* coef, int* code);
int hobi_geometry_arc_normals(int device, const double* coef, const double* t, const double* reference,
                              int64_t n, double* normals, int* straight);
int hobi_geometry_nodes(int device, const double* vertex_pos, const double* vertex_nrm, int64_t n,
                        double* node_pos, double* node_nrm, int64_t* first_bad, int* bad_code);
int hobi_geometry_frames(int device, const double* node_pos, const double* node_nrm, int64_t n_elements,
                         const double* shape, int n_points, double* pos, double* nrm, double* jac,
                         double* d_dr, double* d_ds);

/*
 * Multi-GPU row split: one process per GPU.  Rank r owns rows
 * partition_targets(n_colloc, nranks)[r] (solver.py:405-418); each matvec
 * ends with one ncclAllGather of the owned rows over NVLink.
 * hobi_comm_unique_id is called on rank 0; the 128 bytes are broadcast by the
 * host (torch.distributed) and passed to hobi_comm_init on every rank.
 */
int hobi_comm_unique_id(unsigned char id[128]);
int hobi_comm_init(hobi_ctx* ctx, const unsigned char id[128], int nranks, int rank);
/*
 * Opt-in alternative to the NCCL allgather: the epilogue kernel stores every
 * finished row directly into all ranks' receive buffers over NVLink (CUDA IPC
 * peer memory) and signals arrival with system-scope atomics; a wait kernel
 * hands the gathered vector on.  After hobi_comm_init, every rank calls
 * hobi_comm_p2p_handle, the host all-gathers the 64-byte handles (rank
 * order), and every rank calls hobi_comm_p2p_open with all of them.  If a
 * peer's rows do not arrive within HOBI_P2P_TIMEOUT_MS (environment, default
 * 60000, read at open) the wait gives up and the next synchronising call
 * returns HOBI_ERR_NCCL; the context's P2P gather is unusable afterwards.
 */
int hobi_comm_p2p_handle(hobi_ctx* ctx, unsigned char handle[64]);
int hobi_comm_p2p_open(hobi_ctx* ctx, const unsigned char* handles, int nranks, int rank);
/* Fall back from the peer-store gather to the communicator's ncclAllGather
 * (permanently, e.g. when a start-up check of the P2P path fails). */
int hobi_comm_p2p_disable(hobi_ctx* ctx);
/*
 * P2P-only row split (no NCCL communicator): this context owns rows
 * partition_targets(n, nranks)[rank]; follow with hobi_comm_p2p_handle /
 * hobi_comm_p2p_open.  For ranks that have no NCCL (or share a device, where
 * NCCL refuses two ranks).  Until the peers are open a matvec fails with
 * HOBI_ERR_STATE; RHS and energy run unsplit (bitwise the same values).
 */
int hobi_comm_init_p2p(hobi_ctx* ctx, int nranks, int rank);
/*
 * One P2P-gathered operator application in two host-ordered halves, for
 * ranks whose kernels must not wait on one another (several ranks on one
 * time-sliced GPU): phase 0 copies u in, computes this rank's rows and stores
 * them into every rank's receive area (arrival counters bumped), then
 * synchronises; phase 1 -- called once every rank has finished phase 0 (a
 * host barrier) -- finds every arrival in place, copies the gathered A u out
 * and checks the watchdog.  hobi_matvec == phase 0 + phase 1 without the
 * host round trip.  Phases must alternate (HOBI_ERR_STATE otherwise).
 */
int hobi_matvec_p2p_phase(hobi_ctx* ctx, const double* u, double* out, int phase);
/* Row-split state: ranks, this rank, and whether the P2P gather is active. */
int hobi_comm_info(hobi_ctx* ctx, int* nranks, int* rank, int* p2p);

/*
 * Single-process multi-GPU group (SolverConfig.workers -> GPUs without
 * torchrun; replaces the fork pool of solver.py:405-477 inside one process).
 * `members` are contexts of the same problem, usually one per device
 * (member 0 leads: inputs, outputs and GMRES live there); member i owns rows
 * partition_targets(n_colloc, size)[i].  Each application copies the iterate
 * peer-to-peer to the members and runs every member's rows on its own device;
 * each member's epilogue kernel stores its rows straight into the leader's
 * output over peer memory (a staged copy where peer access is unavailable).
 * Devices are ordered by events only, so members may also
 * share a device.  Results are bitwise those of one context.  Members must
 * outlive every group call and must not be in a communicator or emulated
 * split; hobi_group_destroy touches only the group's own buffers.
 */
typedef struct hobi_group hobi_group;
int hobi_group_create(hobi_ctx* const* members, int size, hobi_group** out);
int hobi_group_destroy(hobi_group* group);
int hobi_group_matvec(hobi_group* group, const double* u, double* out);
int hobi_group_gmres(hobi_group* group, const double* b, double tol, int restart, int max_it, double* x,
                     int* iterations, double* residual, double* best, int* matvecs);
/* Placement of a group: member count, and per member (arrays of `size`, any
 * may be NULL) its device, row range [lo, hi) and whether its epilogue stores
 * straight into the leader's output (1) or stages a copy (0). */
int hobi_group_info(hobi_group* group, int* size, int* devices, int64_t* lo, int64_t* hi, int* direct);
/* hobi_bench for a group: each step bracketed by CUDA events on the leader's
 * stream, which waits for every member, so ms[i] is the slowest device's
 * time; flush_l2 flushes every member's L2 between steps. */
int hobi_group_bench(hobi_group* group, const double* u, double* out, int steps, int mode, int flush_l2,
                     double* ms);
/* Single-GPU emulation of an nranks-way split (same buffers, same gather
 * layout and permutation kernel, no NCCL): for determinism tests. */
int hobi_emulate_ranks(hobi_ctx* ctx, int nranks);

/* Instrumentation: device time of the all-pairs sweep kernel (CUDA events on
 * the launching stream) accumulated since the last reset, its launch count,
 * and the count of every kernel this library launched. */
int hobi_timing_reset(hobi_ctx* ctx);
int hobi_timing(hobi_ctx* ctx, double* sweep_ms, int64_t* sweep_launches, int64_t* all_launches);
/* Tuning hook: select all-pairs sweep variant `variant` (< 0 keeps the
 * current one); reports the number of variants and the active one's name.
 * A selected variant is pinned: it runs every row range as is.  Unpinned
 * (default), the 896-row tile falls back to 512-row tiles for ranges that
 * leave fewer rows past the last whole tile that way, and to 128-row
 * tiles (or one wide-tile launch with a part-filled last tile) when a range
 * has too few work items; all variants and fallbacks
 * produce bitwise identical results (the environment variable
 * HOBI_SWEEP_VARIANT sets the unpinned default at context creation). */
int hobi_sweep_variant(hobi_ctx* ctx, int variant, int* count, char* name, int name_len);

/* Sweep layout: number of fixed source groups (partial sums per row) and the
 * padded source count -- for the algorithmic-bytes accounting of bench.py. */
int hobi_sweep_layout(hobi_ctx* ctx, int* n_groups, int64_t* n_sources_padded);

/*
 * MSMS ingest fast path (host only, no device needed): parse_msms's record
 * rules (mesh.py; reference mesh.py:141-185) on the .vert/.face texts, one pass.
 * Fills vdata (up to vert_cap rows of x y z nx ny nz as written) and faces
 * (up to face_cap rows, 0-based) and reports the record counts; the number of
 * lines of each text is a sufficient capacity.  Returns HOBI_ERR_VALUE
 * ("irregular") whenever the text has anything the Python parser might read
 * differently or would reject -- the caller then runs the Python parser,
 * which gives the reference's exact result or error.
 */
int hobi_msms_parse(const char* vert, int64_t vert_len, const char* face, int64_t face_len, double* vdata,
                    int64_t vert_cap, int64_t* faces, int64_t face_cap, int64_t* n_vert, int64_t* n_face);

/*
 * Analytic Kirkwood validator on the device (kirkwood.py:159-220; the
 * O(points x charges x terms) sums of kirkwood_series).  The caller supplies
 * what the reference computes per charge: unit directions (nc, 3), radii
 * rho (nc), and rows of nterms coefficients per charge.
 * hobi_kirkwood_traces: phi[i] = sum_k coef_phi[k] . P(rad_i . u_k) and the
 * same for dphi (kirkwood.py:193-203), P by the reference's recurrence
 * (kirkwood.py:59-71), cos = 1 for a charge at the centre.
 * hobi_kirkwood_energy_terms: terms[j] = 1/2 q_j sum_k sum_n
 * reac[k,n] rpow[j,n] P_n(u_k . u_j) (kirkwood.py:180-188); the energy is
 * 4 pi 332.0716 sum_j terms[j].  nterms <= 256.
 */
int hobi_kirkwood_traces(int device, const double* points, int64_t m, const double* units, const double* rho,
                         int64_t nc, const double* coef_phi, const double* coef_dphi, int nterms, double* phi,
                         double* dphi);
int hobi_kirkwood_energy_terms(int device, const double* units, const double* q, int64_t nc, const double* reac,
                               const double* rpow, int nterms, double* terms);

/* Regular pairs per full matvec (N_v x N_f x nq for hobi), for throughput. */
int hobi_pairs_per_matvec(hobi_ctx* ctx, double* pairs);

/*
 * Benchmark helper: `steps` operator applications, each bracketed by CUDA
 * events on the context stream; ms[i] receives step i's device time.
 * mode 0: u is copied to HBM once before the loop, each step is
 *         HBM-resident u -> A u (the kernel-level `value`);
 * mode 1: each step is the host-buffer call of hobi_matvec: H2D of u,
 *         operator, D2H of A u (the end-to-end `e2e`).
 * flush_l2 != 0 writes a 512 MiB scratch buffer between steps (outside the
 * brackets) so no step starts with the previous step's data in L2.
 */
int hobi_bench(hobi_ctx* ctx, const double* u, double* out, int steps, int mode, int flush_l2,
               double* ms);

/* Per-rank cost model of a p-way split on one GPU: `steps` device-timed
 * applications restricted to rows [lo, hi) (source weights, sweep, Duffy
 * swap, diagonal -- everything a rank computes before the allgather). */
int hobi_bench_rows(hobi_ctx* ctx, const double* u, int64_t lo, int64_t hi, int steps, int flush_l2,
                    double* ms);

/* Test hook: the device hypot used by the device-driven GMRES cycle (glibc's
 * double hypot restated, so Givens rotations round like np.hypot,
 * solver.py:551) on n argument pairs; out[i] = hypot(a[i], b[i]). */
int hobi_hypot_check(int device, const double* a, const double* b, int64_t n, double* out);

/* DFMA throughput probe (FP64 roofline denominator), TFLOP/s over ~`ms` ms. */
int hobi_probe_fp64_tflops(int device, double ms, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* HOBI_H */
