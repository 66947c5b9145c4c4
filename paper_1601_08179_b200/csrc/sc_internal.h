// Internal declarations shared by the host (api.cu, basis1d.cpp) and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#define SC_PMAX 32
#define SC_NIMAX (SC_PMAX - 1)

namespace sc {

// Kernel attributes (dynamic shared-memory opt-in) and occupancy queries are per device: the
// launchers cache them per device ordinal, not in one process-wide static.
constexpr int kMaxDev = 64;
inline int dev_slot() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDev) ? d : 0;
}

// 1-D transformed basis (host, double), see basis1d.cpp.
struct Basis1D {
  int p = 0, ni = 0;
  double x[SC_PMAX + 1], w[SC_PMAX + 1];
  double K[(SC_PMAX + 1) * (SC_PMAX + 1)];
  double lam[SC_NIMAX], a0[SC_NIMAX], ap[SC_NIMAX];
  double S[SC_NIMAX * SC_NIMAX];      // S_II, row-major, rows = M-orthonormal eigenvectors
  int sigma[SC_NIMAX];                // ap = sigma * a0 (parity of eigenvector m)
  double K00 = 0, K0p = 0, w0 = 0;
  double parity_err = 0, eig_err = 0;
};

bool build_basis_1d(int p, Basis1D& B, std::string& err);

// Device-side description of the rank-local slab (passed by value to kernels).
struct Geom {
  int p, ni, nx, ny, nz;        // local element counts
  int dir_bot, dir_top;         // z-planes 0 / nz are Dirichlet (physical boundary)
  long long off_f[3], off_e[3], off_v, n_total;
  long long n_f[3], n_e[3], n_v;
  int nx1, ny1, nz1;            // local lattice dims
  int z_begin;                  // global element layer of local layer 0
  int uniform;                  // all elements share one geometry (D^{-1} table valid)
  double lam_h;                 // Helmholtz lambda
  const double* hx;             // device arrays of local element widths
  const double* hy;
  const double* hz;
  const double* tab;            // device 1-D tables, see TAB_* offsets
  const double* dinv;           // uniform grids: D^{-1}(i,j,k), i fastest (n_I^3); else null
  double d_uni[4];              // uniform grids: d_e
  int nodir;                    // 1: Dirichlet entities are NOT masked (inhomogeneous-Dirichlet lifting
                                //    in the v1 operator, the conversions and the recovery; api.cu)
};

// Offsets into the device 1-D table (doubles).
enum {
  TAB_LAM = 0,
  TAB_A0 = TAB_LAM + SC_NIMAX,
  TAB_AP = TAB_A0 + SC_NIMAX,
  TAB_SIG = TAB_AP + SC_NIMAX,
  TAB_W = TAB_SIG + SC_NIMAX,                 // GLL weights w[0..p]
  TAB_SCAL = TAB_W + SC_PMAX + 1,             // K00, K0p, w0
  TAB_MAT = TAB_SCAL + 8,                     // 5 matrices n_I x n_I for conversions
  TAB_SIZE = TAB_MAT + 5 * SC_NIMAX * SC_NIMAX
};
// Conversion matrices: 0 identity, 1 S M (to primal = S^{-T}), 2 S (to dual),
// 3 S^T (from primal), 4 M S^T (from dual = S^{-1}).
enum { MAT_I = 0, MAT_SM = 1, MAT_S = 2, MAT_ST = 3, MAT_MST = 4 };

// Nodal-basis operator variants (kernels_var.cu, §7): device table layout (doubles).
enum {
  VT_SM = 0,                                  // (S_II M_II)[m][q] = S_mq w_q, row-major n_I x n_I
  VT_A0 = VT_SM + SC_NIMAX * SC_NIMAX,        // a0 = S_II K_I0
  VT_AP = VT_A0 + SC_NIMAX,                   // ap = S_II K_Ip
  VT_LAM = VT_AP + SC_NIMAX,                  // Lambda
  VT_K = VT_LAM + SC_NIMAX,                   // nodal K, (p+1) x (p+1) row-major
  VT_W = VT_K + (SC_PMAX + 1) * (SC_PMAX + 1),  // GLL weights w[0..p]
  VT_SIZE = VT_W + SC_PMAX + 1
};

// PCG device scalars (doubles in the workspace).
enum {
  SCAL_RZ = 0, SCAL_RZNEW, SCAL_PQ, SCAL_ALPHA, SCAL_BETA, SCAL_RR, SCAL_RR0,
  SCAL_DONE, SCAL_ITERS, SCAL_BREAK, SCAL_TOL2, SCAL_MAXIT, SCAL_RED0, SCAL_RED1, SCAL_RED2,
  SCAL_RAN,   // 1 if this iteration's alpha step ran (guards the x / p update)
  SCAL_COUNT = 32
};

#define SC_RED_BLOCKS 1184   // fixed grid of the deterministic 2-stage reductions (8 x 148)

// ---- kernel launchers (kernels_*.cu); all return cudaError_t as int ----
int launch_apply(const Geom& g, const double* x, double* y, const double* done, void* stream, int* nlaunch,
                 void* events = nullptr);
int launch_diag(const Geom& g, double* diag, void* stream, int* nlaunch);
bool p2s_make_coef(const double d[4], double lam, double a0, double ap, double K00, double K0p, double w0,
                   std::vector<double>& coef, std::string& err);
int launch_apply_p2s(const Geom& g, const double* x, double* y, const double* done, const double* coef, void* stream,
                     int* nlaunch, void* events = nullptr);
bool v7_supported(int ni);
void v7_make_coef(int ni, const double* d, const double* a0, const double* ap, const double* lam, double K00,
                  double K0p, double w0, std::vector<unsigned char>& out, std::vector<double>& dinv);
void v7_set_dinv(std::vector<unsigned char>& coef, const double* d_dinv);
long long v7_dot_parts(const Geom& g);
int launch_apply_v7(const Geom& g, const double* x, double* y, double* u0, double* u1, const double* done,
                    const void* coef, double* dotp, void* stream, int* nlaunch, void* events = nullptr);
int launch_apply_tpc(const Geom& g, const double* vt, const double* x, double* y, void* stream, int* nlaunch,
                     void* events = nullptr);
int launch_mmc_columns(const Geom& g, const double* vt, double* H, int nB, long long ngeom, void* stream, int* nlaunch);
int launch_mmc_gather(const Geom& g, const double* x, double* X, int nB, void* stream, int* nlaunch);
int launch_mmc_assemble(const Geom& g, const double* Y, double* y, int nB, void* stream, int* nlaunch);
int launch_var_diag(const Geom& g, const double* vt, double* diag, void* stream, int* nlaunch);
int launch_var_prec(const Geom& g, int mode, const double* m, const double* r, double* z, void* stream, int* nlaunch);
int launch_unit_mask(const double* mask, double* m, long long n, void* stream, int* nlaunch);
int launch_var_init(const double* b, const double* mask, double* r, double* x, long long n, void* stream, int* nlaunch);
int launch_var_update(double* r, const double* q, long long n, const double* scal, void* stream, int* nlaunch);
int launch_var_direction(double* x, double* p, const double* z, long long n, const double* scal, int first,
                         void* stream, int* nlaunch);
int launch_invert_diag(const Geom& g, double* diag, void* stream, int* nlaunch);
int launch_convert(const Geom& g, const double* in, double* out, int to_skel, int mat, void* stream, int* nlaunch);
int launch_fill_random(const Geom& g, uint64_t seed, double* v, void* stream, int* nlaunch);
int launch_dir_split(const Geom& g, double* a, const double* b, int mode, void* stream, int* nlaunch);
int launch_condense(const Geom& g, const double* f, double* b, double* scratch, long long scratch_elems,
                    void* stream, int* nlaunch);
int launch_recover(const Geom& g, const double* f, const double* x, double* u, double* scratch,
                   long long scratch_elems, void* stream, int* nlaunch);

// PCG vector kernels (kernels_vec.cu). `own_lo/own_hi`: [lo, hi) skeleton ranges excluded
// from dot products (interface plane owned by the lower rank), up to 4 ranges.
struct OwnMask { long long lo[4], hi[4]; int n; };
// Uniform geometry: the assembled diagonal (hence Pinv) of every non-Dirichlet entry depends only
// on its entity class (x/y/z faces, x/y/z edges, vertices) and its index inside the entity, so the
// PCG kernels read Pinv from a small table instead of streaming an N_c vector.  Dirichlet and
// padding entries of r are 0, so the table value there is irrelevant.
struct PinvTab { long long off[7], len[7]; int n[7], base[7]; const double* tab; };
int launch_dot_partial(const double* a, const double* b, long long n, OwnMask m, double* partials,
                       const double* done, void* stream, int* nlaunch);
int launch_reduce_partials(const double* partials, int nparts, double* out, const double* done,
                           void* stream, int* nlaunch);
int launch_pcg_init(const double* b, const double* pinv, double* x, double* r, double* p, long long n,
                    OwnMask m, double* partials, void* stream, int* nlaunch);
int launch_pcg_init_finalize(double* scal, const double* partials, double tol2, int maxit, void* stream, int* nlaunch);
int launch_pcg_alpha(double* scal, void* stream, int* nlaunch);
int launch_pcg_update_tab(double* r, const double* q, const PinvTab& T, OwnMask m, const double* scal,
                          double* partials, void* stream, int* nlaunch);
int launch_pcg_direction_tab(double* x, double* p, const double* r, const PinvTab& T, const double* scal,
                             void* stream, int* nlaunch);
int launch_pcg_update(double* r, const double* q, const double* pinv, long long n, OwnMask m, const double* scal,
                      double* partials, void* stream, int* nlaunch);
int launch_pcg_beta(double* scal, void* stream, int* nlaunch);
int launch_pcg_direction(double* x, double* p, const double* r, const double* pinv, long long n, const double* scal,
                         void* stream, int* nlaunch);
int launch_reduce2(const double* partials, double* scal, int slot0, int nvals, const double* done,
                   void* stream, int* nlaunch);

}  // namespace sc

namespace sc {
struct ColState;
// v3 tile-column operator (kernels_col.cu), n_I <= 7, uniform geometry.
bool col_supported(int ni);
void col_tile(int ni, int* tx, int* ty, int* pend);
void col_make_coef(int ni, const double* d, const double* a0, const double* lam, double K00, double K0p, double w0,
                   std::vector<unsigned char>& out);
int launch_apply_col_raw(const Geom& g, const double* x, double* y, const double* done, void* state, void* flags,
                         double* corner, double* pending, int ntx, int nty, int nseg, int zseg, const void* coef,
                         double* dotp, void* stream, int* nlaunch, void* events);
// Uniform-geometry coefficient block of the element-scheduled operators (v4, p2)
struct BigCoef {
  double c[3][32];   // c[d][m] = d_{d+1} a0_m          (condensed part)
  double e[3][32];   // e[d][m] = d_{d+1} w0 a0_m       (face <- bounding edges)
  double L[3][32];   // L[d][m] = d_{d+1} w0 Lam_m      (face self term)
  double a0[32], lam[32];
  double dl[3][32];  // dl[d][m] = d_{d+1} Lam_m          (D = d0 + dl[0][i] + dl[1][j] + dl[2][k])
  double F0[3];      // d0 w0 + d_{d+1} K00             (face self term)
  double k0p[3];     // d_{d+1} K0p                     (opposite face)
  double d[4];
  double K00, K0p, w0;
};
// v4 operator (n_I >= 8, uniform geometry): colour-scheduled one-CTA-per-element kernels
bool big_supported(int ni);
void big_make_coef(int ni, const double* d, const double* a0, const double* lam, double K00, double K0p, double w0,
                   std::vector<unsigned char>& coef);
int launch_apply_big(const Geom& g, const double* x, double* y, const double* done, const void* coef, void* stream,
                     int* nlaunch, void* events);
// p = 3, 4 operator (uniform geometry): row-warp scheme with shared-memory staging
bool rw_supported(int ni);
int launch_apply_rw(const Geom& g, const double* x, double* y, const double* done, const void* coef, void* stream,
                    int* nlaunch, void* events);
// p = 2 operator (uniform geometry): warp = 32 consecutive elements of an x-row, colour-scheduled
int launch_apply_p2(const Geom& g, const double* x, double* y, const double* done, const void* coef, void* stream,
                    int* nlaunch, void* events);
// v6 operator (2 <= n_I <= 7, uniform geometry): tile columns with a recomputed halo, uniform class
// lanes (kernels_v6.cu); h = compute-tile height (4: 8 x 4 elements, 2 CTAs per SM; 8: 8 x 8, 1 CTA)
bool v6_supported(int ni);
void v6_tiles(int nx, int ny, int h, int* ntx, int* nty);
void v6_segments(int ntiles, int nz, int nslots, int* nseg, int* zseg);
void v6_make_coef(int ni, const double* d, const double* a0, const double* lam, double K00, double K0p, double w0,
                  std::vector<unsigned char>& out);
int launch_apply_v6(const Geom& g, const double* x, double* y, const double* done, int ntx, int nty, int nseg,
                    int zseg, const void* coef, double* dotp, void* stream, int* nl, void* events, int h);
// z-segments of the tile columns: ntiles columns of nz layers on nsm persistent CTAs
void col_choose_segments(int ntiles, int nz, int nsm, int* nseg, int* zseg);
int col_slots();   // step slots of the parked look-back partials (look-back distance + 1)
// sum of v[0..n) in a fixed order into scal[slot] (deterministic), skipped when *done != 0
int launch_sum_ordered(const double* v, int n, double* scal, int slot, const double* done, void* stream, int* nl);
int launch_add_segments(double* y, const double* add, const long long* off, const long long* len, int n,
                        void* stream, int* nlaunch);
}
