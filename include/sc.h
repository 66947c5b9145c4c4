/*
 * sc.h -- C-ABI of the B200-native condensed spectral-element Helmholtz solver
 * (arXiv 1601.08179, "TPT" transformed tensor-product factorisation + solver "BT").
 *
 * Problem (Eq. eq:helmholtz_equation): lambda u - Laplace(u) = f,
 * lambda >= 0, on a Cartesian grid of cuboidal elements of polynomial degree p with
 * GLL Lagrange bases, homogeneous Dirichlet boundaries.  After static
 * condensation only element-boundary ("skeleton") unknowns remain; in the
 * basis transformed by S = diag(1, S_II, 1) along every direction the
 * condensed operator is applied in 13 n_I^3 multiplications per element (Table 2,
 * P:406-440) and the paper's block preconditioner is diagonal.
 *
 * Conventions (all functions):
 *  - Every function returns sc_status; SC_OK == 0.
 *  - Pointers named d_* are DEVICE pointers (caller-owned, e.g. torch tensors on the
 *    ctx's device); pointers named h_* are HOST pointers.  Vectors are fp64.
 *  - "skeleton vector": length sc_layout_info.n_total, the entity-structured layout of
 *    DESIGN.md §3 (x/y/z-faces, x/y/z-edges, vertices of the rank-local slab, each entity
 *    contiguous, including both bounding z-planes).  Dirichlet entities are stored as 0;
 *    inputs there are ignored, outputs there are written as 0.  Padding entries between
 *    sub-arrays are ignored on input and written as 0 on output.
 *  - "lattice vector": the rank-local GLL lattice, (n_x p+1)(n_y p+1)(n_zloc p+1) values,
 *    x fastest, nodal basis.
 *  - All device work is stream-ordered on `stream` (a cudaStream_t; NULL = legacy default
 *    stream).  No function synchronises the device except where stated.
 *  - A ctx is not thread-safe.  x and y arguments must not alias.
 *  - Invalid arguments return SC_EINVAL with no side effect; CUDA / NCCL failures return
 *    SC_ECUDA / SC_ENCCL and leave the ctx unusable (sc_destroy is still safe).
 *  - Multi-GPU: every rank calls the same functions with its own slab (z-slab of whole
 *    element layers); the ctx performs the interface-plane halo exchange and
 *    the scalar all-reduces with NCCL (communicator passed in sc_params.nccl_comm).
 */
#ifndef SC_H
#define SC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SC_OK = 0,
  SC_EINVAL = 1,      /* invalid argument (no side effects)                            */
  SC_ENOMEM = 2,      /* host or device allocation failed / workspace too small        */
  SC_ECUDA = 3,       /* CUDA runtime error                                            */
  SC_ENCCL = 4,       /* NCCL error or NCCL library not loadable                       */
  SC_EBREAKDOWN = 5,  /* PCG: p^T A p <= 0 (operator not SPD on the free set)          */
  SC_ESTATE = 6       /* call sequence error (e.g. workspace not bound)                */
} sc_status;

typedef struct sc_ctx sc_ctx;   /* opaque; owns the small device tables (<= 1 MB) */

typedef struct {
  int p;                 /* polynomial degree, 2 <= p <= 32                                 */
  int ne[3];             /* GLOBAL element counts (n_x, n_y, n_z), each >= 1                */
  const double* h[3];    /* HOST arrays of GLOBAL element widths, h[d] has ne[d] entries >0 */
  double lambda;         /* Helmholtz parameter, finite and >= 0                    */
  int device;            /* CUDA device ordinal                                             */
  void* nccl_comm;       /* ncclComm_t or NULL (single GPU)                                 */
  int rank, nranks;      /* z-slab partition: rank r owns element layers [z0_r, z1_r)       */
} sc_params;

typedef struct {
  long long n_total;          /* skeleton vector length (entries, incl. padding)            */
  long long n_free;           /* free (non-Dirichlet) skeleton unknowns in this slab        */
  long long n_lattice;        /* rank-local lattice vector length                           */
  long long n_lattice_global; /* global lattice size N (the paper's "N")                    */
  long long off_face[3];      /* offsets of x-, y-, z-face arrays                           */
  long long n_faces[3];       /* number of x-, y-, z-faces (each (p-1)^2 entries)           */
  long long off_edge[3];      /* offsets of x-, y-, z-edge arrays (edge "along" x, y, z)    */
  long long n_edges[3];       /* number of x-, y-, z-edges (each p-1 entries)               */
  long long off_vertex;       /* offset of the vertex array                                 */
  long long n_vertices;
  int ne_local[3];            /* rank-local element counts                                  */
  int z_begin, z_end;         /* global element-layer range of this slab                    */
  int p, n_i;                 /* degree, n_I = p-1                                          */
} sc_layout_info;

typedef struct {
  int iters;          /* number of operator applications A p performed                     */
  int converged;      /* 1 if ||r_k||_2 <= rtol ||r_0||_2 was reached                      */
  double relres;      /* ||r_k||_2 / ||r_0||_2 (recursively updated residual, transformed) */
  double r0norm;      /* ||r_0||_2 = ||b||_2                                               */
  double t_solve_s;   /* wall time of the solve on the host (incl. convergence polling)    */
} sc_pcg_report;

/* Conversion modes for sc_to_transformed / sc_from_transformed:
 *  SC_PERM   : pure permutation lattice <-> skeleton layout (no basis change)
 *  SC_PRIMAL : solution-like vectors. to: x~ = Shat^{-T} x ;  from: x = Shat^T x~
 *  SC_DUAL   : residual/RHS-like vectors. to: b~ = Shat b ;   from: b = Shat^{-1} b~
 * Shat = block-diag over skeleton entities of S_II(x)S_II (faces), S_II (edges), 1 (vertices);
 * S_II M_II S_II^T = I (Eq. eq:generalized_eigenvalues) so S_II^{-1} = M_II S_II^T. */
typedef enum { SC_PERM = 0, SC_PRIMAL = 1, SC_DUAL = 2 } sc_basis_mode;

/* Validate params, build the 1-D transformed basis (GLL, K, generalized eigenpairs with
 * sign rule a0_m > 0, ascending Lambda) and the geometry tables (d_e, D^{-1}); allocate small
 * device tables.  Synchronous.  The diagonal (BT) preconditioner 1/diag(Rhat Htilde Rhat^T)
 * is built by sc_bind_workspace (it lives in the caller-owned workspace). */
sc_status sc_setup(const sc_params* prm, sc_ctx** out);
sc_status sc_destroy(sc_ctx* ctx);

/* Host-only: validate params and return the rank-local slab layout sc_setup would use
 * (no GPU, no allocation; nccl_comm may be NULL).  Used by multi-rank host logic and tests. */
sc_status sc_layout_query(const sc_params* prm, sc_layout_info* out);
sc_status sc_layout(const sc_ctx* ctx, sc_layout_info* out);

/* Workspace for sc_pcg_solve and sc_apply_condensed (caller-owned device memory,
 * e.g. a torch tensor).  Must be bound before those calls; bytes >= sc_workspace_bytes.
 * Binding computes the BT preconditioner diagonal into the workspace (synchronous).
 * Re-binding is allowed; it discards the cached PCG graph (which refers to the old buffers). */
size_t sc_workspace_bytes(const sc_ctx* ctx);
sc_status sc_bind_workspace(sc_ctx* ctx, void* d_ws, size_t bytes);

/* 1-D data of the transformed basis (host copies), for tests and diagnostics.
 * out arrays: lam[n_I], a0[n_I], ap[n_I], S[n_I*n_I] (row-major, S_II), w[p+1] (GLL weights),
 * kt[4] = {K00, K0p, w0, sigma-consistency error}.  Any pointer may be NULL. */
sc_status sc_basis_1d(const sc_ctx* ctx, double* lam, double* a0, double* ap, double* S,
                      double* w, double* kt);

/* Same data computed on the host for degree p without a ctx or a GPU (L0 only).
 * Returns SC_EINVAL for p outside [2, 32]. */
sc_status sc_basis_1d_host(int p, double* lam, double* a0, double* ap, double* S, double* w,
                           double* kt);

/* y~ = Rhat Htilde Rhat^T x~ : the assembled condensed operator in the transformed basis
 * (Table 2 suboperators + Eq. 26 primary part), including the interface halo exchange.
 * d_x, d_y: skeleton vectors. */
sc_status sc_apply_condensed(sc_ctx* ctx, const double* d_x, double* d_y, void* stream);

/* Solver BT: PCG with the diagonal preconditioner 1/diag(Rhat Htilde Rhat^T) in the
 * transformed system, x0 = 0, stop when ||r_k||_2 <= rtol ||b||_2 (recursive residual) or
 * after maxit iterations; rtol <= 0 runs exactly maxit iterations.  d_b, d_x: skeleton
 * vectors.  Synchronises the stream to poll convergence (every 8 iterations).  Non-convergence
 * is SC_OK with rep->converged = 0; p^T A p <= 0 returns SC_EBREAKDOWN.  Single GPU: from the
 * second 8-iteration chunk on, the chunk is replayed from a CUDA graph captured for d_x (the
 * ctx owns the graph; a different d_x re-captures; environment SC_NO_GRAPH=1 disables it). */
sc_status sc_pcg_solve(sc_ctx* ctx, const double* d_b, double* d_x, double rtol, int maxit,
                       sc_pcg_report* rep, void* stream);

/* Split form of sc_pcg_solve for fixed-iteration runs (benchmarks, checkpointing):
 * sc_pcg_start initialises r = b, x = 0, p = Pinv r and the device scalars (rtol / maxit
 * as in sc_pcg_solve); sc_pcg_iterate enqueues `niter` further iterations without any
 * host synchronisation (iterations after convergence are no-ops on the device);
 * sc_pcg_status synchronises the stream and fills `rep`.  d_x must stay valid between
 * the calls. */
sc_status sc_pcg_start(sc_ctx* ctx, const double* d_b, double* d_x, double rtol, int maxit, void* stream);
sc_status sc_pcg_iterate(sc_ctx* ctx, int niter, void* stream);
sc_status sc_pcg_status(sc_ctx* ctx, sc_pcg_report* rep, void* stream);

/* Kernel timing of the condensed-operator kernel with CUDA events recorded on the launch
 * stream around every launch while enabled (at most 8192 launches are recorded).
 * sc_profile_read synchronises the device and returns the summed duration in ms and the
 * number of launches since the last enable, then clears the record. */
sc_status sc_profile_enable(sc_ctx* ctx, int on);
sc_status sc_profile_read(sc_ctx* ctx, double* h_total_ms, long long* h_count);

/* Same as sc_pcg_solve, but h_b / h_x are HOST buffers (pinned for best speed); the
 * host->device and device->host copies happen inside the call, on `stream`, using the
 * workspace.  For end-to-end timing through the public API. */
sc_status sc_pcg_solve_host(sc_ctx* ctx, const double* h_b, double* h_x, double rtol,
                            int maxit, sc_pcg_report* rep, void* stream);

/* Alg. 4 pre-processing (transform of F corrected per DESIGN.md reading R3):
 * F_e = (h1h2h3/8)(w(x)w(x)w) f on the element's lattice nodes; F~ = (S(x)S(x)S) F_e;
 * b~ = Rhat (F~_B - Htilde_BI D^{-1} F~_I).  d_f: lattice vector, d_b: skeleton vector. */
sc_status sc_condense_rhs(sc_ctx* ctx, const double* d_f, double* d_b, void* stream);

/* Alg. 4 post-processing: u~_I = D^{-1}(F~_I - Htilde_IB u~_B),
 * u_e = (S(x)S(x)S)^T u~_e, written to every lattice node.  d_f: lattice f (as given to
 * sc_condense_rhs), d_x: skeleton solution, d_u: lattice output. */
sc_status sc_recover(sc_ctx* ctx, const double* d_f, const double* d_x, double* d_u, void* stream);

/* Inhomogeneous Dirichlet data (the paper's solver benchmark: u = u_ex on the domain
 * boundary).  d_g: lattice vector whose values on the domain-boundary nodes are the Dirichlet data
 * (other nodes ignored).  sc_condense_rhs_dirichlet: b~ = b~(f) - (Rhat Htilde Rhat^T g~)_F with
 * g~ = Shat^{-T} g on the Dirichlet entities (A_FF x_F = b_F - A_FD g_D; reading R17),
 * Dirichlet entries of d_b set to 0; solve with sc_pcg_solve as usual.  sc_recover_dirichlet:
 * as sc_recover with the skeleton completed by g~ on the Dirichlet entities, so d_u equals g on the
 * boundary.  Both use the PCG buffers of the workspace as scratch (not between sc_pcg_start and
 * sc_pcg_status).  Any geometry; p as in sc_setup. */
sc_status sc_condense_rhs_dirichlet(sc_ctx* ctx, const double* d_f, const double* d_g, double* d_b, void* stream);
sc_status sc_recover_dirichlet(sc_ctx* ctx, const double* d_f, const double* d_g, const double* d_x, double* d_u,
                               void* stream);

/* Basis / layout conversions (untimed helpers for parity).
 * to:   lattice -> skeleton;  from: skeleton -> lattice (element-interior lattice nodes
 * are written as 0). */
sc_status sc_to_transformed(sc_ctx* ctx, const double* d_lattice, double* d_skel, int mode, void* stream);
sc_status sc_from_transformed(sc_ctx* ctx, const double* d_skel, double* d_lattice, int mode, void* stream);

/* Seeded uniform[-1,1) skeleton vector (counter-based splitmix64, reading R9):
 * entry at skeleton node with GLOBAL lattice index g = uniform(seed, g); Dirichlet 0. */
sc_status sc_fill_random(sc_ctx* ctx, uint64_t seed, double* d_skel, void* stream);

/* Deterministic fp64 dot product over owned free skeleton entries, all-reduced over ranks.
 * Result written to *h_out (synchronises the stream). */
sc_status sc_dot(sc_ctx* ctx, const double* d_a, const double* d_b, double* h_out, void* stream);

/* The diagonal preconditioner table: d_pinv[i] = 1 / diag(Rhat Htilde Rhat^T)_ii at free
 * entries, 0 elsewhere (skeleton vector). */
sc_status sc_preconditioner(sc_ctx* ctx, double* d_pinv, void* stream);

/* NCCL bootstrap (multi-GPU): rank 0 calls sc_nccl_unique_id, the 128-byte id is broadcast
 * by the caller (e.g. torch.distributed), then every rank calls sc_nccl_comm_init on its
 * device.  The communicator is passed in sc_params.nccl_comm and freed by
 * sc_nccl_comm_destroy.  libnccl.so.2 is loaded at run time (SC_ENCCL if absent). */
sc_status sc_nccl_unique_id(unsigned char h_id[128]);
sc_status sc_nccl_comm_init(const unsigned char h_id[128], int nranks, int rank, int device, void** comm_out);
sc_status sc_nccl_comm_destroy(void* comm);

/* In-process loopback group (tests): creates nranks communicator handles in comms_out[0..nranks-1]
 * that stand in for NCCL communicators in sc_params.nccl_comm when the ranks are host threads
 * of ONE process (one context and stream per thread, any device).  The halo exchange and the
 * scalar all-reduce then move data with cudaMemcpyAsync between host barriers, summing the
 * scalars in rank order -- every collective becomes a host synchronisation point, so this is
 * for exercising the multi-rank path on one GPU, not for speed.  Every rank of the
 * group must take part in each collective.  The caller owns the handles and frees them all at
 * once with sc_loopback_comms_destroy after every context using them is destroyed.
 * SC_EINVAL on nranks < 1, NULL pointers or handles not from one create call. */
sc_status sc_loopback_comms_create(int nranks, void** comms_out);
sc_status sc_loopback_comms_destroy(void** comms, int nranks);

/* ---- Operator variants of the paper's operator comparison (§7 "Efficiency of operators",
 * P:493-504, Table 3), in the NODAL GLL basis:  d_y = Rhat Hhat Rhat^T d_x  with the element
 * Schur complement Hhat_e = H_BB - H_BI H_II^{-1} H_IB.  d_x, d_y: skeleton vectors in
 * the entity layout of sc_layout (nodal values, no basis change); Dirichlet entries ignored on input
 * and written as 0; multi-GPU halo exchange as in sc_apply_condensed.  Results equal those of the
 * transformed operator converted to the nodal basis, up to rounding.
 *
 * sc_apply_tpc -- variant TPC: Alg. 3 (`alg:face_to_eigenspace`) with the
 *   Table 1 tensor-product suboperators, 37 n_I^3 multiplications for the condensed part plus the
 *   nodal primary part (12 n_I^3, Eqs. eq:east_east_primary_part / eq:east_west_primary_part); one
 *   CTA per element, assembly by fp64 atomics into d_y (zeroed first).  Any geometry.
 * sc_mmc_bytes / sc_mmc_bind / sc_apply_mmc -- variant MMC (Alg. 2 `alg:face_to_face`):
 *   sc_mmc_bind precomputes the element matrix Hhat_e (all 6 n_I^2 + 12 n_I + 8 shell nodes; one
 *   matrix for a uniform grid, one per element otherwise: the paper's memory argument) into
 *   the caller-owned device buffer d_buf of at least sc_mmc_bytes(ctx) bytes (SC_ENOMEM if smaller:
 *   the memory guard), synchronously; the buffer also holds the gathered element shells.  The buffer
 *   must stay valid while sc_apply_mmc is used; re-binding replaces it.  sc_apply_mmc gathers every
 *   element's shell (R^T), applies all elements with ONE cuBLAS DGEMM (a strided batch for
 *   per-element matrices) and assembles (R) entity by entity in a fixed order (deterministic).
 *   SC_ESTATE if sc_mmc_bind was not called; SC_ECUDA if libcublas.so.12 cannot be loaded. */
sc_status sc_apply_tpc(sc_ctx* ctx, const double* d_x, double* d_y, void* stream);
size_t sc_mmc_bytes(const sc_ctx* ctx);
sc_status sc_mmc_bind(sc_ctx* ctx, void* d_buf, size_t bytes, void* stream);
sc_status sc_apply_mmc(sc_ctx* ctx, const double* d_x, double* d_y, void* stream);

/* Solvers UC / DC / BC of the paper's solver comparison (§8 "Performance of solvers", P:602-607,
 * Table 4 `tab:solver_complexities`) on the NODAL condensed system:  PCG (x0 = 0, Hestenes-Stiefel as
 * sc_pcg_solve) with operator `op` (SC_OP_TPC as in the paper, or SC_OP_MMC after sc_mmc_bind) and
 * preconditioner `prec`: SC_PREC_NONE (UC), SC_PREC_DIAG (DC: 1/diag(Rhat Hhat Rhat^T), built per call),
 * SC_PREC_BLOCK (BC: the exact inverse of every assembled face / edge / vertex self-block, P:597-600,
 * applied in tensor-product form as Shat^T Ptilde Shat, 24 n_I^3 per element).  Stops when
 * ||r_k||_2 <= rtol ||r_0||_2 for the recursively updated NODAL residual, or after maxit iterations.
 * d_b, d_x: nodal skeleton vectors (sc_layout, SC_PERM conversions).  Uses the bound workspace (not
 * between sc_pcg_start and sc_pcg_status); synchronises the stream every 8 iterations.  Errors as
 * sc_pcg_solve; SC_EINVAL for an unknown op / prec, SC_ESTATE for MMC without sc_mmc_bind. */
enum { SC_OP_TPC = 1, SC_OP_MMC = 2 };
enum { SC_PREC_NONE = 0, SC_PREC_DIAG = 1, SC_PREC_BLOCK = 2 };
sc_status sc_pcg_solve_nodal(sc_ctx* ctx, int op, int prec, const double* d_b, double* d_x, double rtol,
                             int maxit, sc_pcg_report* rep, void* stream);

/* Operator kernel family this ctx runs: "v7" (two passes: element condensed parts, then
 * entity-wise primary part + assembly; the default for 3 <= p <= 16 on uniform grids), "v6" / "v6h8"
 * (halo-recompute tile columns, 3 <= p <= 8), "v3" (tile columns with look-back), "rw" (row-warp, p = 3, 4),
 * "p2s" (owner-computes stencil, p = 2, one rank) / "p2" (colour-scheduled row-warp, p = 2),
 * "v4" (colour-scheduled element CTAs, p >= 9; the default for p >= 17 and non-uniform grids), "v1" (one CTA
 * per element, any geometry). */
const char* sc_operator_kernel(const sc_ctx* ctx);

/* Number of kernels launched by this ctx since setup (for the bench's gpu_launches). */
long long sc_launch_count(const sc_ctx* ctx);

/* Human-readable message of the last error on this ctx ("" if none). */
const char* sc_last_error(const sc_ctx* ctx);

/* Library build identifier (compile flags, arch). */
const char* sc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SC_H */
