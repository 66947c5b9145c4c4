// C-ABI entry points (include/sc.h): context, layout, workspace, operator, BT-PCG loop,
// conversions, NCCL bootstrap and interface-plane halo exchange.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <set>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sc.h"
#include "sc_internal.h"

using namespace sc;

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

bool load_nccl() {
  if (g_nccl.loaded) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    const char* env = getenv("SC_NCCL_LIB");
    if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) return false;
#define SYM(name, field) g_nccl.field = (decltype(g_nccl.field))dlsym(h, name); if (!g_nccl.field) return false;
  SYM("ncclGetUniqueId", GetUniqueId)
  SYM("ncclCommInitRank", CommInitRank)
  SYM("ncclCommDestroy", CommDestroy)
  SYM("ncclAllReduce", AllReduce)
  SYM("ncclSend", Send)
  SYM("ncclRecv", Recv)
  SYM("ncclGroupStart", GroupStart)
  SYM("ncclGroupEnd", GroupEnd)
  SYM("ncclGetErrorString", GetErrorString)
#undef SYM
  g_nccl.loaded = true;
  return true;
}
// ---------------------------------------------------------------- loopback group
// In-process stand-in for the NCCL communicator (sc_loopback_comms_create): G ranks are
// host threads of one process, each with its own context and stream; the halo and the scalar
// all-reduce move data with cudaMemcpyAsync (UVA, any device) between host barriers.  Test
// infrastructure for the multi-rank path on one GPU -- every collective is a host sync point.
struct LoopGroup {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const double*> seg;        // [rank][side][q] published segment pointers
  std::vector<const double*> val;        // [rank] published scalar pointers
  bool broken = false;                   // a rank missed a barrier: every later collective fails
  bool barrier() {                       // false after a 120 s timeout (a rank left the group)
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    long long g = gen;
    if (++arrived == nranks) { arrived = 0; ++gen; cv.notify_all(); return true; }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};
struct LoopComm {
  LoopGroup* grp;
  int rank;
};
std::mutex g_loop_mu;
std::set<const void*> g_loop_comms;      // live LoopComm handles (distinguishes them from ncclComm_t)
bool is_loop_comm(const void* c) {
  std::lock_guard<std::mutex> lk(g_loop_mu);
  return c && g_loop_comms.count(c);
}
}  // namespace

// ------------------------------------------------------------------ cuBLAS (dlopen)
// MMC's "single call to DGEMM" is a plain library GEMM: cuBLAS, loaded at run time
// (the copy torch already mapped if present), so the library does not link against one cuBLAS build.
namespace {
struct CublasApi {
  bool tried = false, loaded = false;
  int (*Create)(void**) = nullptr;
  int (*Destroy)(void*) = nullptr;
  int (*SetStream)(void*, cudaStream_t) = nullptr;
  int (*Dgemm)(void*, int, int, int, int, int, const double*, const double*, int, const double*, int,
               const double*, double*, int) = nullptr;
  int (*DgemmStridedBatched)(void*, int, int, int, int, int, const double*, const double*, int, long long,
                             const double*, int, long long, const double*, double*, int, long long, int) = nullptr;
};
CublasApi g_cublas;
std::mutex g_cublas_mu;

bool load_cublas() {
  std::lock_guard<std::mutex> lk(g_cublas_mu);
  if (g_cublas.tried) return g_cublas.loaded;
  g_cublas.tried = true;
  void* h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("/usr/local/cuda/lib64/libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
#define SYM(name, field) g_cublas.field = (decltype(g_cublas.field))dlsym(h, name); if (!g_cublas.field) return false;
  SYM("cublasCreate_v2", Create)
  SYM("cublasDestroy_v2", Destroy)
  SYM("cublasSetStream_v2", SetStream)
  SYM("cublasDgemm_v2", Dgemm)
  SYM("cublasDgemmStridedBatched", DgemmStridedBatched)
#undef SYM
  g_cublas.loaded = true;
  return true;
}
void cublas_destroy(void* h) {
  if (h && g_cublas.loaded) g_cublas.Destroy(h);
}
}  // namespace

// ------------------------------------------------------------------ context
struct sc_ctx {
  sc_params prm;
  std::vector<double> hx, hy, hz;       // global widths
  Basis1D B;
  Geom g;
  sc_layout_info L;
  double* d_tab = nullptr;              // 1-D tables
  double* d_h = nullptr;                // local widths hx | hy | hz
  double* d_dinv = nullptr;             // uniform D^{-1} table
  // v3 tile-column operator state (kernels_col.cu)
  bool use_col = false;
  bool use_big = false;
  bool use_p2 = false;                  // p = 2 row-warp operator (kernels_p2.cu)
  bool use_p2s = false;                 // p = 2 owner-computes stencil (kernels_p2s.cu, one rank)
  std::vector<double> p2s_coef;
  bool use_rw = false;                  // p = 3, 4 row-warp operator (kernels_rw.cu)
  bool use_v6 = false;                  // 3 <= p <= 8 halo-recompute tile columns (kernels_v6.cu)
  bool use_v7 = false;                  // 3 <= p <= 8 two-pass operator (kernels_v7.cu, one rank)
  std::vector<unsigned char> v7_coef;
  double* d_u7 = nullptr;               // v7 face-part vectors u0 | u1 (2 n_total doubles)
  std::vector<unsigned char> v6_coef;
  int v6_ntx = 0, v6_nty = 0, v6_nseg = 1, v6_zseg = 0;
  int v6_h = 4;                         // compute-tile height: 4 (2 CTAs per SM) or 8 (1 CTA of 16 warps)
  bool use_ptab = false;                // PCG reads Pinv from the per-class table (uniform geometry)
  PinvTab ptab;                 // v4 colour-scheduled element operator (n_I >= 8, uniform geometry)
  std::vector<unsigned char> big_coef;
  std::vector<unsigned char> col_coef;  // kernel-parameter coefficient block
  int col_ntx = 0, col_nty = 0;
  int col_nseg = 1, col_zseg = 0;       // z-segments per tile column (load balance over the SMs)
  void* d_colstate = nullptr;
  int* d_flags = nullptr;
  double* d_corner = nullptr;
  double* d_pending = nullptr;
  double* d_dotp = nullptr;             // per-tile x . y partials of the operator (PCG p . q)
  bool fused_dot = true;                // p . q from the operator's per-tile partials (SC_FUSED_DOT=0: dot kernel)
  // workspace (caller-owned)
  double* ws = nullptr;
  size_t ws_bytes = 0;
  double *pinv = nullptr, *r = nullptr, *pv = nullptr, *q = nullptr, *bdev = nullptr, *xdev = nullptr;
  double *scal = nullptr, *partials = nullptr, *halo = nullptr, *scratch = nullptr;
  long long scratch_elems = 0;
  long long plane_len = 0;              // entries of one interface plane
  long long seg_off[2][4], seg_len[4];  // bottom / top plane segments
  OwnMask own;
  ncclComm_t comm = nullptr;
  LoopComm* loop = nullptr;             // in-process loopback group instead of NCCL (tests)
  long long nlaunch = 0;
  double* x_cur = nullptr;              // PCG iterate between sc_pcg_start / sc_pcg_iterate
  // CUDA graph of kPcgChunk PCG iterations (single GPU, no kernel profiling), captured for the
  // iterate x_cur it was built with
  cudaGraphExec_t pcg_graph = nullptr;
  const double* pcg_graph_x = nullptr;   // iterate the graph was captured for
  const double* pcg_seen_x = nullptr;    // iterate of the last eager chunk
  int pcg_graph_launches = 0;
  cudaStream_t cap_stream = nullptr;
  double tol2 = -1.0;
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_ev;     // pairs (start, stop)
  int prof_n = 0;
  // nodal-basis operator variants of PAPER.md §7 (kernels_var.cu): TPC and MMC
  double* d_vt = nullptr;               // VT_* tables (S M, a0, ap, Lambda, nodal K, w)
  double* mmc_H = nullptr;              // caller-owned buffer: element matrices | X | Y
  double* mmc_X = nullptr;
  double* mmc_Y = nullptr;
  long long mmc_ngeom = 0;              // 1 (uniform geometry) or n_e (one matrix per element)
  int mmc_nB = 0;                       // shell nodes per element, 6 n_I^2 + 12 n_I + 8
  void* cublas = nullptr;               // cublasHandle_t (libcublas.so.12 loaded at run time)
  std::string err;
  bool broken = false;
};

static const long long kAlign = 32;   // entries (256 B)
static long long align_up(long long v) { return (v + kAlign - 1) / kAlign * kAlign; }

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (cudaError_t)(call);                                          \
    if (e_ != cudaSuccess) {                                                       \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);               \
      ctx->broken = true;                                                          \
      return SC_ECUDA;                                                             \
    }                                                                              \
  } while (0)

#define NK(call)                                                                   \
  do {                                                                             \
    ncclResult_t r_ = (call);                                                      \
    if (r_ != ncclSuccess) {                                                       \
      ctx->err = std::string(#call) + ": " + g_nccl.GetErrorString(r_);            \
      ctx->broken = true;                                                          \
      return SC_ENCCL;                                                             \
    }                                                                              \
  } while (0)

#define LAUNCH(expr)                                                               \
  do {                                                                             \
    int nl_ = 0;                                                                   \
    int e2_ = (expr);                                                              \
    ctx->nlaunch += nl_;                                                           \
    if (e2_ != 0) {                                                                \
      ctx->err = std::string(#expr) + ": " + cudaGetErrorString((cudaError_t)e2_); \
      ctx->broken = true;                                                          \
      return SC_ECUDA;                                                             \
    }                                                                              \
  } while (0)
// (launchers take `&nl_` as their last argument)

static bool finite_pos(double v) { return std::isfinite(v) && v > 0; }

// Validate the parameters and compute the rank-local slab geometry and skeleton layout
// (host only; shared by sc_setup and sc_layout_query).
static sc_status layout_compute(const sc_params* prm, bool need_comm, Geom& g, sc_layout_info& L) {
  if (!prm) return SC_EINVAL;
  const int p = prm->p;
  if (p < 2 || p > SC_PMAX) return SC_EINVAL;
  for (int d = 0; d < 3; ++d) {
    if (prm->ne[d] < 1 || !prm->h[d]) return SC_EINVAL;
    for (int e = 0; e < prm->ne[d]; ++e)
      if (!finite_pos(prm->h[d][e])) return SC_EINVAL;
  }
  if (!std::isfinite(prm->lambda) || prm->lambda < 0) return SC_EINVAL;
  if (prm->nranks < 1 || prm->rank < 0 || prm->rank >= prm->nranks) return SC_EINVAL;
  if (prm->nranks > prm->ne[2]) return SC_EINVAL;
  // SC_TEST_LOCAL_SLAB=1 (tests only): a rank's slab without a communicator -- the operator
  // then returns the slab's local partial sums on its interface planes (no halo exchange) and
  // dots are rank-local, which is what the single-GPU slab parity tests compare against
  const char* ls = getenv("SC_TEST_LOCAL_SLAB");
  if (need_comm && prm->nranks > 1 && !prm->nccl_comm && !(ls && ls[0] == '1')) return SC_EINVAL;
  const int ni = p - 1;
  // slab partition: rank r owns element layers [z0, z1) (balanced, contiguous)
  const int nzg = prm->ne[2], R = prm->nranks, r = prm->rank;
  const int z0 = (int)((long long)nzg * r / R), z1 = (int)((long long)nzg * (r + 1) / R);
  const int nx = prm->ne[0], ny = prm->ne[1], nz = z1 - z0;
  memset(&g, 0, sizeof(g));
  g.p = p; g.ni = ni; g.nx = nx; g.ny = ny; g.nz = nz;
  g.dir_bot = (r == 0); g.dir_top = (r == R - 1);
  g.z_begin = z0;
  g.nx1 = nx * p + 1; g.ny1 = ny * p + 1; g.nz1 = nz * p + 1;
  g.lam_h = prm->lambda;
  const long long n2 = (long long)ni * ni;
  g.n_f[0] = (long long)(nx + 1) * ny * nz;
  g.n_f[1] = (long long)nx * (ny + 1) * nz;
  g.n_f[2] = (long long)nx * ny * (nz + 1);
  g.n_e[0] = (long long)nx * (ny + 1) * (nz + 1);
  g.n_e[1] = (long long)(nx + 1) * ny * (nz + 1);
  g.n_e[2] = (long long)(nx + 1) * (ny + 1) * nz;
  g.n_v = (long long)(nx + 1) * (ny + 1) * (nz + 1);
  long long off = 0;
  for (int d = 0; d < 3; ++d) { g.off_f[d] = off; off = align_up(off + g.n_f[d] * n2); }
  for (int d = 0; d < 3; ++d) { g.off_e[d] = off; off = align_up(off + g.n_e[d] * ni); }
  g.off_v = off;
  off = align_up(off + g.n_v);
  g.n_total = off;
  memset(&L, 0, sizeof(L));
  L.n_total = g.n_total;
  L.n_lattice = (long long)g.nx1 * g.ny1 * g.nz1;
  L.n_lattice_global = (long long)(nx * p + 1) * (ny * p + 1) * ((long long)nzg * p + 1);
  for (int d = 0; d < 3; ++d) {
    L.off_face[d] = g.off_f[d]; L.n_faces[d] = g.n_f[d];
    L.off_edge[d] = g.off_e[d]; L.n_edges[d] = g.n_e[d];
  }
  L.off_vertex = g.off_v; L.n_vertices = g.n_v;
  L.ne_local[0] = nx; L.ne_local[1] = ny; L.ne_local[2] = nz;
  L.z_begin = z0; L.z_end = z1; L.p = p; L.n_i = ni;
  {  // free unknowns owned by this rank (the lower rank owns each interface plane):
     // free lattice box gx in [1, nx p - 1], gy in [1, ny p - 1], gz in [1, gz_hi] minus element interiors
    long long gz_hi = g.dir_top ? (long long)nz * p - 1 : (long long)nz * p;
    long long tot = ((long long)nx * p - 1) * ((long long)ny * p - 1) * gz_hi;
    L.n_free = tot - (long long)nx * ny * nz * (long long)ni * ni * ni;
  }
  return SC_OK;
}

extern "C" sc_status sc_layout_query(const sc_params* prm, sc_layout_info* out) {
  if (!prm || !out) return SC_EINVAL;
  Geom g;
  return layout_compute(prm, false, g, *out);
}

extern "C" sc_status sc_setup(const sc_params* prm, sc_ctx** out) {
  if (!prm || !out) return SC_EINVAL;
  *out = nullptr;
  {
    Geom gq;
    sc_layout_info lq;
    sc_status st = layout_compute(prm, true, gq, lq);
    if (st != SC_OK) return st;
  }
  const int p = prm->p;
  sc_ctx* ctx = new sc_ctx();
  ctx->prm = *prm;
  for (int d = 0; d < 3; ++d) {
    std::vector<double>& h = d == 0 ? ctx->hx : (d == 1 ? ctx->hy : ctx->hz);
    h.assign(prm->h[d], prm->h[d] + prm->ne[d]);
    ctx->prm.h[d] = h.data();
  }
  std::string berr;
  if (!build_basis_1d(p, ctx->B, berr)) {
    ctx->err = berr;
    delete ctx;
    return SC_EINVAL;
  }
  const int ni = p - 1;
  Geom& g = ctx->g;
  sc_layout_info& L = ctx->L;
  layout_compute(prm, true, g, L);
  const int R = prm->nranks, r = prm->rank;
  const int z0 = L.z_begin, z1 = L.z_end;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long n2 = (long long)ni * ni;
  // ---- device tables
  std::vector<double> tab(TAB_SIZE, 0.0);
  const Basis1D& B = ctx->B;
  for (int m = 0; m < ni; ++m) {
    tab[TAB_LAM + m] = B.lam[m];
    tab[TAB_A0 + m] = B.a0[m];
    tab[TAB_AP + m] = B.ap[m];
    tab[TAB_SIG + m] = B.sigma[m];
  }
  for (int i = 0; i <= p; ++i) tab[TAB_W + i] = B.w[i];
  tab[TAB_SCAL + 0] = B.K00;
  tab[TAB_SCAL + 1] = B.K0p;
  tab[TAB_SCAL + 2] = B.w0;
  const int MS = SC_NIMAX * SC_NIMAX;
  for (int a = 0; a < ni; ++a)
    for (int b = 0; b < ni; ++b) {
      double s_ab = B.S[a * ni + b], s_ba = B.S[b * ni + a];
      tab[TAB_MAT + MAT_I * MS + a * ni + b] = (a == b) ? 1.0 : 0.0;
      tab[TAB_MAT + MAT_SM * MS + a * ni + b] = s_ab * B.w[b + 1];    // (S M)[a][b]
      tab[TAB_MAT + MAT_S * MS + a * ni + b] = s_ab;                  // S[a][b]
      tab[TAB_MAT + MAT_ST * MS + a * ni + b] = s_ba;                 // S^T[a][b]
      tab[TAB_MAT + MAT_MST * MS + a * ni + b] = B.w[a + 1] * s_ba;   // (M S^T)[a][b]
    }
  bool uniform = true;
  for (double v : ctx->hx) uniform &= (v == ctx->hx[0]);
  for (double v : ctx->hy) uniform &= (v == ctx->hy[0]);
  for (double v : ctx->hz) uniform &= (v == ctx->hz[0]);
  g.uniform = uniform;
  if (cudaSetDevice(prm->device) != cudaSuccess) { ctx->err = "cudaSetDevice"; delete ctx; return SC_ECUDA; }
  auto fail = [&](const char* what) { ctx->err = what; sc_destroy(ctx); return SC_ECUDA; };
  if (cudaMalloc(&ctx->d_tab, sizeof(double) * TAB_SIZE) != cudaSuccess) return fail("cudaMalloc tab");
  if (cudaMemcpy(ctx->d_tab, tab.data(), sizeof(double) * TAB_SIZE, cudaMemcpyHostToDevice) != cudaSuccess)
    return fail("cudaMemcpy tab");
  {  // nodal-basis variant tables (kernels_var.cu)
    std::vector<double> vt(VT_SIZE, 0.0);
    for (int a = 0; a < ni; ++a) {
      for (int b = 0; b < ni; ++b) vt[VT_SM + a * ni + b] = B.S[a * ni + b] * B.w[b + 1];
      vt[VT_A0 + a] = B.a0[a];
      vt[VT_AP + a] = B.ap[a];
      vt[VT_LAM + a] = B.lam[a];
    }
    for (int i = 0; i <= p; ++i) {
      vt[VT_W + i] = B.w[i];
      for (int j = 0; j <= p; ++j) vt[VT_K + i * (p + 1) + j] = B.K[i * (p + 1) + j];
    }
    if (cudaMalloc(&ctx->d_vt, sizeof(double) * VT_SIZE) != cudaSuccess) return fail("cudaMalloc vt");
    if (cudaMemcpy(ctx->d_vt, vt.data(), sizeof(double) * VT_SIZE, cudaMemcpyHostToDevice) != cudaSuccess)
      return fail("cudaMemcpy vt");
  }
  std::vector<double> hloc;
  hloc.insert(hloc.end(), ctx->hx.begin(), ctx->hx.end());
  hloc.insert(hloc.end(), ctx->hy.begin(), ctx->hy.end());
  hloc.insert(hloc.end(), ctx->hz.begin() + z0, ctx->hz.begin() + z1);
  if (cudaMalloc(&ctx->d_h, sizeof(double) * hloc.size()) != cudaSuccess) return fail("cudaMalloc h");
  if (cudaMemcpy(ctx->d_h, hloc.data(), sizeof(double) * hloc.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return fail("cudaMemcpy h");
  g.hx = ctx->d_h; g.hy = ctx->d_h + nx; g.hz = ctx->d_h + nx + ny;
  g.tab = ctx->d_tab;
  g.dinv = nullptr;
  if (uniform) {
    double h1 = ctx->hx[0], h2 = ctx->hy[0], h3 = ctx->hz[0];
    double s = h1 * h2 * h3 * 0.125;
    double d[4] = {s * prm->lambda, s * 4.0 / (h1 * h1), s * 4.0 / (h2 * h2), s * 4.0 / (h3 * h3)};
    for (int q = 0; q < 4; ++q) g.d_uni[q] = d[q];
    std::vector<double> dinv((size_t)ni * ni * ni);
    for (int k = 0; k < ni; ++k)
      for (int j = 0; j < ni; ++j)
        for (int i = 0; i < ni; ++i) {
          double D = d[0] + d[1] * B.lam[i] + d[2] * B.lam[j] + d[3] * B.lam[k];
          if (!(D > 0)) { ctx->err = "non-positive D entry"; sc_destroy(ctx); return SC_EINVAL; }
          dinv[i + ni * (j + (size_t)ni * k)] = 1.0 / D;
        }
    if (cudaMalloc(&ctx->d_dinv, sizeof(double) * dinv.size()) != cudaSuccess) return fail("cudaMalloc dinv");
    if (cudaMemcpy(ctx->d_dinv, dinv.data(), sizeof(double) * dinv.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail("cudaMemcpy dinv");
    g.dinv = ctx->d_dinv;
  }
  // ---- operator kernel selection: p = 2 row-warp, p = 3, 4 row-warp with staging,
  // 5 <= p <= 8 tile-column v3 (uniform geometry), 9 <= p <= 32 colour element v4 (any geometry),
  // v1 for tiny grids and non-uniform p <= 8
  {
    // tiny grids (the launch-bound cfg1 / cfg2 sizes): the one-launch v1 kernel beats the
    // tile-column march and the 8 colour launches (cfg2: 23 vs 41 us per application);
    // SC_SMALL_V1=0 disables the switch (the parity tests use it to exercise the fast kernels)
    const char* sv = getenv("SC_SMALL_V1");
    const long long ne_local = (long long)nx * ny * nz;
    // thresholds measured at n_e = 512 (profiles/variants_r2.json): v1 0.028 / 0.036 / 0.045 /
    // 0.059 ms vs the colour launches 0.085 / 0.069 / 0.073 / 0.086 ms at p = 10 / 12 / 14 / 16
    const bool small_v1 = !(sv && sv[0] == '0') && ne_local <= (p <= 8 ? 2048 : (p <= 16 ? 512 : 256));
    const char* env0 = getenv("SC_APPLY_V1");
    const char* env = small_v1 ? "1" : env0;
    bool sig_ok = true;
    for (int m = 0; m < ni; ++m) sig_ok &= (B.sigma[m] == ((m & 1) ? -1 : 1));
    const char* np2 = getenv("SC_NO_P2");
    const char* nrw = getenv("SC_NO_RW");
    // SC_OP selects the p <= 8 operator family: "v6" (halo-recompute tile columns, kernels_v6.cu),
    // "v3" (tile columns with look-back, kernels_col.cu), "rw" (p = 3, 4 row-warp kernels); default:
    // the measured fastest per p
    const char* opsel = getenv("SC_OP");
    const std::string op = opsel ? opsel : "";
    // measured (tools/op_time.py, r2 runs): on one rank v7 (two passes) is fastest for every p = 3..16
    // (cfg5 5.16 ms vs v3 7.89 / v6 7.96; cfg3 p = 12 0.93 vs v4 1.57 ms), on any number of
    // ranks; without the memory for v7's two face-part vectors: v6 for p = 5, 6, 7, v3 for p = 8, the
    // row-warp kernels for p = 3, 4, v4 above
    const bool want_v6 = op == "v6" || (op.empty() && ni >= 4 && ni <= 6);
    const bool want_v7 = op == "v7" || (op.empty() && ni <= 15);
    bool v7_ok = v7_supported(ni) && uniform && sig_ok && want_v7 && !(env && env[0] == '1');
    std::vector<double> dinv;
    const size_t nu = 2 * (size_t)g.n_total;   // U0 | U1, then the D^{-1} table (n_I^3)
    if (v7_ok) {
      v7_make_coef(ni, g.d_uni, B.a0, B.ap, B.lam, B.K00, B.K0p, B.w0, ctx->v7_coef, dinv);
      const char* nm = getenv("SC_TEST_V7_NOMEM");   // tests: behave as if the allocation failed
      if ((nm && nm[0] == '1') || cudaMalloc(&ctx->d_u7, sizeof(double) * (nu + dinv.size())) != cudaSuccess) {
        (void)cudaGetLastError();   // out of memory for U0 / U1: fall back to a one-pass family
        ctx->d_u7 = nullptr;
        if (op == "v7") return fail("cudaMalloc u7 (SC_OP=v7)");
        v7_ok = false;
      }
    }
    if (v7_ok) {
      if (cudaMemset(ctx->d_u7, 0, sizeof(double) * nu) != cudaSuccess) return fail("memset u7");
      if (cudaMemcpy(ctx->d_u7 + nu, dinv.data(), sizeof(double) * dinv.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return fail("copy dinv");
      v7_set_dinv(ctx->v7_coef, ctx->d_u7 + nu);
      if (cudaMalloc(&ctx->d_dotp, sizeof(double) * (size_t)v7_dot_parts(g)) != cudaSuccess) return fail("cudaMalloc dotp");
      const char* fd = getenv("SC_FUSED_DOT");
      ctx->fused_dot = !(fd && fd[0] == '0');
      ctx->use_v7 = true;
    } else if (v6_supported(ni) && uniform && sig_ok && want_v6 && !(env && env[0] == '1')) {
      const char* hs = getenv("SC_V6_H");
      ctx->v6_h = (hs && atoi(hs) == 8) ? 8 : ((hs && atoi(hs) == 4) ? 4 : 4);
      v6_make_coef(ni, g.d_uni, B.a0, B.lam, B.K00, B.K0p, B.w0, ctx->v6_coef);
      v6_tiles(nx, ny, ctx->v6_h, &ctx->v6_ntx, &ctx->v6_nty);
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      const char* zs = getenv("SC_ZSEG");
      if (zs && atoi(zs) > 0) {
        const int s = atoi(zs) > nz ? nz : atoi(zs);
        ctx->v6_zseg = (nz + s - 1) / s;
        ctx->v6_nseg = (nz + ctx->v6_zseg - 1) / ctx->v6_zseg;
      } else {
        v6_segments(ctx->v6_ntx * ctx->v6_nty, nz, (ctx->v6_h == 4 ? 2 : 1) * nsm, &ctx->v6_nseg, &ctx->v6_zseg);
      }
      const size_t nitems = (size_t)ctx->v6_ntx * ctx->v6_nty * ctx->v6_nseg;
      if (cudaMalloc(&ctx->d_dotp, sizeof(double) * nitems) != cudaSuccess) return fail("cudaMalloc dotp");
      const char* fd = getenv("SC_FUSED_DOT");
      ctx->fused_dot = !(fd && fd[0] == '0');
      ctx->use_v6 = true;
    } else if (ni == 1 && uniform && sig_ok && !(env && env[0] == '1') && !(np2 && np2[0] == '1')) {
      // one rank: the owner-computes stencil (every free node's elements are all local); z-slab
      // ranks keep the colour-scheduled kernel, whose interface planes hold local partial sums.
      // SC_P2_COLOUR=1 forces the colour-scheduled kernel.
      const char* pc = getenv("SC_P2_COLOUR");
      std::string perr;
      if (prm->nranks == 1 && !(pc && pc[0] == '1') &&
          p2s_make_coef(g.d_uni, B.lam[0], B.a0[0], B.ap[0], B.K00, B.K0p, B.w0, ctx->p2s_coef, perr)) {
        ctx->use_p2s = true;
      } else {
        big_make_coef(ni, g.d_uni, B.a0, B.lam, B.K00, B.K0p, B.w0, ctx->big_coef);
        ctx->use_p2 = true;
      }
    } else if (rw_supported(ni) && uniform && sig_ok && !(env && env[0] == '1') && !(nrw && nrw[0] == '1') &&
               op != "v3") {
      big_make_coef(ni, g.d_uni, B.a0, B.lam, B.K00, B.K0p, B.w0, ctx->big_coef);
      ctx->use_rw = true;
    } else if (col_supported(ni) && uniform && sig_ok && !(env && env[0] == '1')) {
      col_make_coef(ni, g.d_uni, B.a0, B.lam, B.K00, B.K0p, B.w0, ctx->col_coef);
      int tx, ty, pend;
      col_tile(ni, &tx, &ty, &pend);
      ctx->col_ntx = (nx + tx - 1) / tx;
      ctx->col_nty = (ny + ty - 1) / ty;
      {
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        col_choose_segments(ctx->col_ntx * ctx->col_nty, nz, nsm, &ctx->col_nseg, &ctx->col_zseg);
      }
      const size_t nitems = (size_t)ctx->col_ntx * ctx->col_nty * ctx->col_nseg;
      size_t nflags = nitems * 2;   // one 64-bit progress word per item (kernels_col.cu)
      size_t ncorner = (size_t)(ctx->col_ntx + 1) * (ctx->col_nty + 1) * (nz + 1) * 3 * (ni + 1);
      if (cudaMalloc(&ctx->d_colstate, 64) != cudaSuccess) return fail("cudaMalloc colstate");
      if (cudaMalloc(&ctx->d_flags, sizeof(int) * nflags) != cudaSuccess) return fail("cudaMalloc flags");
      if (cudaMalloc(&ctx->d_corner, sizeof(double) * ncorner) != cudaSuccess) return fail("cudaMalloc corner");
      size_t npend = nitems * col_slots() * pend;   // look-back distance + 1 step slots (kernels_col.cu)
      if (cudaMalloc(&ctx->d_pending, sizeof(double) * npend) != cudaSuccess) return fail("cudaMalloc pending");
      if (cudaMalloc(&ctx->d_dotp, sizeof(double) * nitems) != cudaSuccess)
        return fail("cudaMalloc dotp");
      const char* fd = getenv("SC_FUSED_DOT");
      ctx->fused_dot = !(fd && fd[0] == '0');
      if (cudaMemset(ctx->d_colstate, 0, 64) != cudaSuccess) return fail("memset colstate");
      if (cudaMemset(ctx->d_flags, 0, sizeof(int) * nflags) != cudaSuccess) return fail("memset flags");
      if (cudaMemset(ctx->d_corner, 0, sizeof(double) * ncorner) != cudaSuccess) return fail("memset corner");
      ctx->use_col = true;
    }
    // v4 also runs non-uniform grids: each CTA derives its element's coefficients from d_e
    if (!ctx->use_v6 && !ctx->use_v7 && !ctx->use_col && !ctx->use_p2 && !ctx->use_p2s && !ctx->use_rw && big_supported(ni) && sig_ok && !(env && env[0] == '1')) {
      const double d_one[4] = {1.0, 1.0, 1.0, 1.0};
      big_make_coef(ni, uniform ? g.d_uni : d_one, B.a0, B.lam, B.K00, B.K0p, B.w0, ctx->big_coef);
      ctx->use_big = true;
    }
  }
  // ---- interface planes (z-face plane, x-edges, y-edges, vertices at fz = 0 / nz)
  long long lens[4] = {(long long)nx * ny * n2, (long long)nx * (ny + 1) * ni, (long long)(nx + 1) * ny * ni,
                       (long long)(nx + 1) * (ny + 1)};
  for (int side = 0; side < 2; ++side) {
    long long fz = side == 0 ? 0 : nz;
    ctx->seg_off[side][0] = g.off_f[2] + fz * lens[0];
    ctx->seg_off[side][1] = g.off_e[0] + fz * lens[1];
    ctx->seg_off[side][2] = g.off_e[1] + fz * lens[2];
    ctx->seg_off[side][3] = g.off_v + fz * lens[3];
  }
  ctx->plane_len = 0;
  for (int q = 0; q < 4; ++q) { ctx->seg_len[q] = lens[q]; ctx->plane_len += lens[q]; }
  memset(&ctx->own, 0, sizeof(ctx->own));
  if (r > 0) {
    ctx->own.n = 4;
    for (int q = 0; q < 4; ++q) { ctx->own.lo[q] = ctx->seg_off[0][q]; ctx->own.hi[q] = ctx->seg_off[0][q] + lens[q]; }
  }
  if (R > 1 && is_loop_comm(prm->nccl_comm)) {
    ctx->loop = (LoopComm*)prm->nccl_comm;
    if (ctx->loop->rank != r || ctx->loop->grp->nranks != R) { sc_destroy(ctx); return SC_EINVAL; }
  } else if (R > 1) {
    if (!load_nccl()) { ctx->err = "libnccl.so.2 not loadable"; sc_destroy(ctx); return SC_ENCCL; }
    ctx->comm = (ncclComm_t)prm->nccl_comm;
  }
  *out = ctx;
  return SC_OK;
}

extern "C" sc_status sc_destroy(sc_ctx* ctx) {
  if (!ctx) return SC_OK;
  if (ctx->d_tab) cudaFree(ctx->d_tab);
  if (ctx->d_h) cudaFree(ctx->d_h);
  if (ctx->d_dinv) cudaFree(ctx->d_dinv);
  if (ctx->d_colstate) cudaFree(ctx->d_colstate);
  if (ctx->d_flags) cudaFree(ctx->d_flags);
  if (ctx->d_corner) cudaFree(ctx->d_corner);
  if (ctx->d_pending) cudaFree(ctx->d_pending);
  if (ctx->d_dotp) cudaFree(ctx->d_dotp);
  if (ctx->d_u7) cudaFree(ctx->d_u7);
  if (ctx->d_vt) cudaFree(ctx->d_vt);
  cublas_destroy(ctx->cublas);
  if (ctx->pcg_graph) cudaGraphExecDestroy(ctx->pcg_graph);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  for (cudaEvent_t e : ctx->prof_ev) cudaEventDestroy(e);
  delete ctx;
  return SC_OK;
}

extern "C" sc_status sc_layout(const sc_ctx* ctx, sc_layout_info* out) {
  if (!ctx || !out) return SC_EINVAL;
  *out = ctx->L;
  return SC_OK;
}

static const long long kScratchCtas = 296;

extern "C" size_t sc_workspace_bytes(const sc_ctx* ctx) {
  if (!ctx) return 0;
  long long n = ctx->g.n_total;
  long long n3 = (long long)(ctx->g.p + 1) * (ctx->g.p + 1) * (ctx->g.p + 1);
  const long long ntab = 3LL * ctx->g.ni * ctx->g.ni + 3LL * ctx->g.ni + 1;
  long long tot = 6 * n + align_up(SCAL_COUNT) + align_up(4 * SC_RED_BLOCKS) + 4 * align_up(ctx->plane_len) +
                  align_up(ntab) + kScratchCtas * 2 * n3;
  return (size_t)tot * sizeof(double);
}

static sc_status halo_sum(sc_ctx* ctx, double* y, cudaStream_t st);

extern "C" sc_status sc_bind_workspace(sc_ctx* ctx, void* d_ws, size_t bytes) {
  if (!ctx || !d_ws) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (bytes < sc_workspace_bytes(ctx)) return SC_ENOMEM;
  if (((uintptr_t)d_ws) % 256 != 0) return SC_EINVAL;
  double* w = (double*)d_ws;
  long long n = ctx->g.n_total;
  // the cached PCG graph bakes in the previous workspace's buffers (pv, q, r, scal, partials,
  // Pinv table): a new binding invalidates it
  if (ctx->pcg_graph) { cudaGraphExecDestroy(ctx->pcg_graph); ctx->pcg_graph = nullptr; }
  ctx->pcg_graph_x = nullptr;
  ctx->pcg_seen_x = nullptr;
  ctx->x_cur = nullptr;
  ctx->ws = w; ctx->ws_bytes = bytes;
  ctx->pinv = w; w += n;
  ctx->r = w; w += n;
  ctx->pv = w; w += n;
  ctx->q = w; w += n;
  ctx->bdev = w; w += n;
  ctx->xdev = w; w += n;
  ctx->scal = w; w += align_up(SCAL_COUNT);
  ctx->partials = w; w += align_up(4 * SC_RED_BLOCKS);
  ctx->halo = w; w += 4 * align_up(ctx->plane_len);
  double* const ptab = w;
  w += align_up(3LL * ctx->g.ni * ctx->g.ni + 3LL * ctx->g.ni + 1);
  ctx->scratch = w;
  long long n3 = (long long)(ctx->g.p + 1) * (ctx->g.p + 1) * (ctx->g.p + 1);
  ctx->scratch_elems = kScratchCtas * 2 * n3;
  CK(cudaSetDevice(ctx->prm.device));
  cudaStream_t st = 0;
  CK(cudaMemsetAsync(ctx->scal, 0, sizeof(double) * SCAL_COUNT, st));
  // BT preconditioner: Pinv = 1 / diag(Rhat Htilde Rhat^T)
  LAUNCH(launch_diag(ctx->g, ctx->pinv, st, &nl_));
  sc_status s = halo_sum(ctx, ctx->pinv, st);
  if (s != SC_OK) return s;
  LAUNCH(launch_invert_diag(ctx->g, ctx->pinv, st, &nl_));
  // uniform geometry: Pinv per (entity class, index in the entity) from one non-Dirichlet
  // representative of each class (all of them share the value; classes without one are all
  // Dirichlet, where r = 0)
  ctx->use_ptab = false;
  const char* pv_env = getenv("SC_PINV_VECTOR");
  // Multi-rank: the representative is a slab-interior z-plane (1..nz-1) on every rank, so all
  // ranks hold bitwise the same table (an interface plane's halo-summed value is rounded in a
  // different order than an interior plane's) and the replicated interface entries of z and p
  // stay identical across ranks; that needs every slab >= 2 element layers thick.
  const bool multi = ctx->prm.nranks > 1;
  if (ctx->g.uniform && !(pv_env && pv_env[0] == '1') && (!multi || ctx->prm.ne[2] / ctx->prm.nranks >= 2)) {
    const Geom& g = ctx->g;
    const int ni = g.ni, n2 = ni * ni, nx = g.nx, ny = g.ny, nz = g.nz;
    int fzf = -1;                                   // a non-Dirichlet z-plane, slab-interior first
    for (int fz = 1; fz < nz && fzf < 0; ++fz) fzf = fz;
    for (int fz = 0; fz <= nz && fzf < 0 && !multi; ++fz)
      if (!((fz == 0 && g.dir_bot) || (fz == nz && g.dir_top))) fzf = fz;
    const bool ix = nx >= 2, iy = ny >= 2;
    PinvTab& T = ctx->ptab;
    const long long ent[7] = {
        ix ? g.off_f[0] + (1LL) * n2 : -1,                                                        // x-face (1, 0, 0)
        iy ? g.off_f[1] + ((long long)nx * 1) * n2 : -1,                                          // y-face (0, 1, 0)
        fzf >= 0 ? g.off_f[2] + ((long long)nx * ny * fzf) * n2 : -1,                            // z-face (0, 0, fzf)
        (iy && fzf >= 0) ? g.off_e[0] + ((long long)nx * (1 + (long long)(ny + 1) * fzf)) * ni : -1,   // x-edge
        (ix && fzf >= 0) ? g.off_e[1] + (1 + (long long)(nx + 1) * ny * fzf) * ni : -1,            // y-edge
        (ix && iy) ? g.off_e[2] + (1 + (long long)(nx + 1) * 1) * ni : -1,                        // z-edge (1, 1, 0)
        (ix && iy && fzf >= 0) ? g.off_v + 1 + (long long)(nx + 1) * (1 + (long long)(ny + 1) * fzf) : -1};
    const long long lens[7] = {g.n_f[0] * n2, g.n_f[1] * n2, g.n_f[2] * n2, g.n_e[0] * ni, g.n_e[1] * ni,
                               g.n_e[2] * ni, g.n_v};
    const long long offs[7] = {g.off_f[0], g.off_f[1], g.off_f[2], g.off_e[0], g.off_e[1], g.off_e[2], g.off_v};
    const int per[7] = {n2, n2, n2, ni, ni, ni, 1};
    int base = 0;
    for (int c = 0; c < 7; ++c) {
      T.off[c] = offs[c]; T.len[c] = lens[c]; T.n[c] = per[c]; T.base[c] = base;
      if (ent[c] >= 0)
        CK(cudaMemcpyAsync(ptab + base, ctx->pinv + ent[c], sizeof(double) * per[c], cudaMemcpyDeviceToDevice, st));
      else
        CK(cudaMemsetAsync(ptab + base, 0, sizeof(double) * per[c], st));
      base += per[c];
    }
    T.tab = ptab;
    ctx->use_ptab = true;
  }
  CK(cudaStreamSynchronize(st));
  return SC_OK;
}

extern "C" sc_status sc_basis_1d(const sc_ctx* ctx, double* lam, double* a0, double* ap, double* S, double* w,
                                 double* kt) {
  if (!ctx) return SC_EINVAL;
  const Basis1D& B = ctx->B;
  int ni = B.ni;
  for (int m = 0; m < ni; ++m) {
    if (lam) lam[m] = B.lam[m];
    if (a0) a0[m] = B.a0[m];
    if (ap) ap[m] = B.ap[m];
    if (S)
      for (int i = 0; i < ni; ++i) S[m * ni + i] = B.S[m * ni + i];
  }
  if (w)
    for (int i = 0; i <= B.p; ++i) w[i] = B.w[i];
  if (kt) { kt[0] = B.K00; kt[1] = B.K0p; kt[2] = B.w0; kt[3] = B.parity_err; }
  return SC_OK;
}

extern "C" sc_status sc_basis_1d_host(int p, double* lam, double* a0, double* ap, double* S, double* w,
                                      double* kt) {
  if (p < 2 || p > SC_PMAX) return SC_EINVAL;
  sc_ctx tmp;
  std::string err;
  if (!build_basis_1d(p, tmp.B, err)) return SC_EINVAL;
  return sc_basis_1d(&tmp, lam, a0, ap, S, w, kt);
}

// Interface-plane halo: after every rank has its partial sums on its bottom / top plane,
// exchange them with the z-neighbours and add (P:107-109 gather across the slab cut).
static sc_status halo_sum(sc_ctx* ctx, double* y, cudaStream_t st) {
  const int R = ctx->prm.nranks, r = ctx->prm.rank;
  if (R == 1 || (!ctx->comm && !ctx->loop)) return SC_OK;   // SC_TEST_LOCAL_SLAB: local partials
  if (!ctx->halo) { ctx->err = "workspace not bound (needed for the halo exchange)"; return SC_ESTATE; }
  const long long pl = align_up(ctx->plane_len);
  double* recv_lo = ctx->halo;
  double* recv_hi = ctx->halo + pl;
  if (ctx->loop) {
    // loopback: publish this rank's plane segments, copy the neighbours' once every rank's
    // partials are complete, and add only after every rank has copied.
    LoopGroup* G = ctx->loop->grp;
    CK(cudaStreamSynchronize(st));
    for (int side = 0; side < 2; ++side)
      for (int q = 0; q < 4; ++q) G->seg[(r * 2 + side) * 4 + q] = y + ctx->seg_off[side][q];
    if (!G->barrier()) { ctx->err = "loopback barrier timed out"; return SC_ESTATE; }
    for (int side = 0; side < 2; ++side) {
      int peer = side == 0 ? r - 1 : r + 1;
      if (peer < 0 || peer >= R) continue;
      double* rb = side == 0 ? recv_lo : recv_hi;
      long long o = 0;
      for (int q = 0; q < 4; ++q) {
        CK(cudaMemcpyAsync(rb + o, G->seg[(peer * 2 + (1 - side)) * 4 + q], sizeof(double) * ctx->seg_len[q],
                           cudaMemcpyDefault, st));
        o += ctx->seg_len[q];
      }
    }
    CK(cudaStreamSynchronize(st));
    if (!G->barrier()) { ctx->err = "loopback barrier timed out"; return SC_ESTATE; }
  } else {
  NK(g_nccl.GroupStart());
  for (int side = 0; side < 2; ++side) {
    int peer = side == 0 ? r - 1 : r + 1;
    if (peer < 0 || peer >= R) continue;
    double* rb = side == 0 ? recv_lo : recv_hi;
    long long o = 0;
    for (int q = 0; q < 4; ++q) {
      NK(g_nccl.Send(y + ctx->seg_off[side][q], (size_t)ctx->seg_len[q], ncclDouble, peer, ctx->comm, st));
      NK(g_nccl.Recv(rb + o, (size_t)ctx->seg_len[q], ncclDouble, peer, ctx->comm, st));
      o += ctx->seg_len[q];
    }
  }
  NK(g_nccl.GroupEnd());
  }
  if (r > 0) LAUNCH(launch_add_segments(y, recv_lo, ctx->seg_off[0], ctx->seg_len, 4, st, &nl_));
  if (r < R - 1) LAUNCH(launch_add_segments(y, recv_hi, ctx->seg_off[1], ctx->seg_len, 4, st, &nl_));
  return SC_OK;
}

static sc_status allreduce_scal(sc_ctx* ctx, int slot, int n, cudaStream_t st) {
  if (ctx->prm.nranks == 1 || (!ctx->comm && !ctx->loop)) return SC_OK;
  if (ctx->loop) {
    // loopback: every rank sums the published values in rank order (identical on all ranks)
    LoopGroup* G = ctx->loop->grp;
    const int R = ctx->prm.nranks;
    double sum[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tmp[8];
    if (n > 8) return SC_EINVAL;
    CK(cudaStreamSynchronize(st));
    G->val[ctx->prm.rank] = ctx->scal + slot;
    if (!G->barrier()) { ctx->err = "loopback barrier timed out"; return SC_ESTATE; }
    for (int q = 0; q < R; ++q) {
      CK(cudaMemcpy(tmp, G->val[q], sizeof(double) * n, cudaMemcpyDefault));
      for (int i = 0; i < n; ++i) sum[i] += tmp[i];
    }
    if (!G->barrier()) { ctx->err = "loopback barrier timed out"; return SC_ESTATE; }
    CK(cudaMemcpyAsync(ctx->scal + slot, sum, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return SC_OK;
  }
  NK(g_nccl.AllReduce(ctx->scal + slot, ctx->scal + slot, (size_t)n, ncclDouble, ncclSum, ctx->comm, st));
  return SC_OK;
}

// y = A x.  dotp != nullptr (single GPU, tile-column operator): the kernel also leaves the
// per-tile partials of x . y over the final entries in dotp (fused PCG p . q).
static sc_status apply_impl(sc_ctx* ctx, const double* x, double* y, const double* done, cudaStream_t st,
                            double* dotp = nullptr) {
  const bool rec = ctx->prof_on && ctx->prof_n < (int)ctx->prof_ev.size() / 2;
  cudaEvent_t* ev = rec ? &ctx->prof_ev[2 * ctx->prof_n] : nullptr;
  if (ctx->use_v7)
    LAUNCH(launch_apply_v7(ctx->g, x, y, ctx->d_u7, ctx->d_u7 + ctx->g.n_total, done, ctx->v7_coef.data(), dotp, st,
                           &nl_, ev));
  else if (ctx->use_v6)
    LAUNCH(launch_apply_v6(ctx->g, x, y, done, ctx->v6_ntx, ctx->v6_nty, ctx->v6_nseg, ctx->v6_zseg,
                           ctx->v6_coef.data(), dotp, st, &nl_, ev, ctx->v6_h));
  else if (ctx->use_col)
    LAUNCH(launch_apply_col_raw(ctx->g, x, y, done, ctx->d_colstate, ctx->d_flags, ctx->d_corner, ctx->d_pending,
                                ctx->col_ntx, ctx->col_nty, ctx->col_nseg, ctx->col_zseg, ctx->col_coef.data(), dotp,
                                st, &nl_, ev));
  else if (ctx->use_p2s)
    LAUNCH(launch_apply_p2s(ctx->g, x, y, done, ctx->p2s_coef.data(), st, &nl_, ev));
  else if (ctx->use_p2)
    LAUNCH(launch_apply_p2(ctx->g, x, y, done, ctx->big_coef.data(), st, &nl_, ev));
  else if (ctx->use_rw)
    LAUNCH(launch_apply_rw(ctx->g, x, y, done, ctx->big_coef.data(), st, &nl_, ev));
  else if (ctx->use_big)
    LAUNCH(launch_apply_big(ctx->g, x, y, done, ctx->big_coef.data(), st, &nl_, ev));
  else
    LAUNCH(launch_apply(ctx->g, x, y, done, st, &nl_, ev));
  if (rec) ctx->prof_n++;
  return halo_sum(ctx, y, st);
}

extern "C" sc_status sc_apply_condensed(sc_ctx* ctx, const double* d_x, double* d_y, void* stream) {
  if (!ctx || !d_x || !d_y || d_x == d_y) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  return apply_impl(ctx, d_x, d_y, nullptr, (cudaStream_t)stream);
}

static sc_status pcg_start_impl(sc_ctx* ctx, const double* b, double* x, double rtol, int maxit, cudaStream_t st) {
  const long long n = ctx->g.n_total;
  ctx->tol2 = rtol > 0 ? rtol * rtol : -1.0;
  ctx->x_cur = x;
  LAUNCH(launch_pcg_init(b, ctx->pinv, x, ctx->r, ctx->pv, n, ctx->own, ctx->partials, st, &nl_));
  LAUNCH(launch_reduce2(ctx->partials, ctx->scal, SCAL_RED0, 2, nullptr, st, &nl_));
  sc_status s = allreduce_scal(ctx, SCAL_RED0, 2, st);
  if (s) return s;
  LAUNCH(launch_pcg_init_finalize(ctx->scal, ctx->partials, ctx->tol2, maxit, st, &nl_));
  return SC_OK;
}

// One BT-PCG iteration (rows a3-a10): q = A p; alpha = rz / p.q; x += alpha p; r -= alpha q;
// z = Pinv r; beta = r.z / rz_old; p = z + beta p.  Scalars stay on the device.
static sc_status pcg_iteration(sc_ctx* ctx, cudaStream_t st) {
  const long long n = ctx->g.n_total;
  double* done = ctx->scal + SCAL_DONE;
  double* x = ctx->x_cur;
  // p . q fused into the tile-column operator (single GPU): each tile accumulates x . y over the
  // entries it finalizes, one fixed-order sum follows.  At cfg5 12.47 -> 11.74 ms per iteration
  // against the separate dot kernel (which streams p and q once more); SC_FUSED_DOT=0 disables it.
  // (Early in round 1, with a slower operator, it measured slower: 10.67 vs 9.55 + 0.9 ms.)
  // v6 returns per-CTA partials of x . A x over its owned entities / elements, which sum to p . q on
  // any number of ranks (each rank's partial interface-plane sums included): fused there on every rank.
  const bool fused = ((ctx->use_col && ctx->prm.nranks == 1) || ctx->use_v6 || ctx->use_v7) && ctx->fused_dot;
  const int nparts = ctx->use_v7 ? (int)v7_dot_parts(ctx->g)
                     : ctx->use_v6 ? ctx->v6_ntx * ctx->v6_nty * ctx->v6_nseg : ctx->col_ntx * ctx->col_nty * ctx->col_nseg;
  sc_status s = apply_impl(ctx, ctx->pv, ctx->q, done, st, fused ? ctx->d_dotp : nullptr);
  if (s) return s;
  if (fused) {
    LAUNCH(launch_sum_ordered(ctx->d_dotp, nparts, ctx->scal, SCAL_RED0, done, st, &nl_));
  } else {
    LAUNCH(launch_dot_partial(ctx->pv, ctx->q, n, ctx->own, ctx->partials, done, st, &nl_));
    LAUNCH(launch_reduce2(ctx->partials, ctx->scal, SCAL_RED0, 1, done, st, &nl_));
  }
  if ((s = allreduce_scal(ctx, SCAL_RED0, 1, st))) return s;
  LAUNCH(launch_pcg_alpha(ctx->scal, st, &nl_));
  if (ctx->use_ptab)
    LAUNCH(launch_pcg_update_tab(ctx->r, ctx->q, ctx->ptab, ctx->own, ctx->scal, ctx->partials, st, &nl_));
  else
    LAUNCH(launch_pcg_update(ctx->r, ctx->q, ctx->pinv, n, ctx->own, ctx->scal, ctx->partials, st, &nl_));
  LAUNCH(launch_reduce2(ctx->partials, ctx->scal, SCAL_RED0, 2, done, st, &nl_));
  if ((s = allreduce_scal(ctx, SCAL_RED0, 2, st))) return s;
  LAUNCH(launch_pcg_beta(ctx->scal, st, &nl_));
  if (ctx->use_ptab)
    LAUNCH(launch_pcg_direction_tab(x, ctx->pv, ctx->r, ctx->ptab, ctx->scal, st, &nl_));
  else
    LAUNCH(launch_pcg_direction(x, ctx->pv, ctx->r, ctx->pinv, n, ctx->scal, st, &nl_));
  return SC_OK;
}

static sc_status pcg_report_impl(sc_ctx* ctx, sc_pcg_report* rep, cudaStream_t st, double t_s) {
  double sc[SCAL_COUNT];
  CK(cudaMemcpyAsync(sc, ctx->scal, sizeof(sc), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (rep) {
    rep->iters = (int)sc[SCAL_ITERS];
    rep->r0norm = std::sqrt(sc[SCAL_RR0]);
    rep->relres = sc[SCAL_RR0] > 0 ? std::sqrt(sc[SCAL_RR] / sc[SCAL_RR0]) : 0.0;
    rep->converged = (sc[SCAL_RR0] == 0.0) || (ctx->tol2 > 0 && sc[SCAL_RR] <= ctx->tol2 * sc[SCAL_RR0]);
    rep->t_solve_s = t_s;
  }
  if (sc[SCAL_BREAK] != 0.0) { ctx->err = "PCG breakdown: p^T A p <= 0"; return SC_EBREAKDOWN; }
  return SC_OK;
}

// kPcgChunk iterations, replayed from a CUDA graph when possible: every iteration's kernels take
// only device-resident scalars and fixed buffers, so the chunk is captured once per iterate x and
// replayed (one launch instead of ~8 per iteration; the launch-bound small configurations gain
// most).  Multi-GPU (NCCL in the chunk) and kernel profiling run the plain launches.
static constexpr int kPcgChunk = 8;
static sc_status pcg_chunk(sc_ctx* ctx, cudaStream_t st) {
  const char* ng = getenv("SC_NO_GRAPH");
  const bool graph_ok = ctx->prm.nranks == 1 && !ctx->prof_on && !(ng && ng[0] == '1');
  if (graph_ok && ctx->pcg_graph && ctx->pcg_graph_x == ctx->x_cur) {
    CK(cudaGraphLaunch(ctx->pcg_graph, st));
    ctx->nlaunch += ctx->pcg_graph_launches;
    return SC_OK;
  }
  if (graph_ok && ctx->pcg_seen_x == ctx->x_cur) {
    // second chunk with this iterate: capture on a private stream (capture is not allowed on the
    // legacy default stream; the exec is then launched on the caller's stream).  The first chunk
    // ran eagerly, so every lazily set kernel attribute is in place before the capture.
    if (ctx->pcg_graph) { cudaGraphExecDestroy(ctx->pcg_graph); ctx->pcg_graph = nullptr; }
    if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    const long long nl0 = ctx->nlaunch;
    CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    sc_status s = SC_OK;
    for (int k = 0; k < kPcgChunk && s == SC_OK; ++k) s = pcg_iteration(ctx, ctx->cap_stream);
    cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &graph);
    ctx->pcg_graph_launches = (int)(ctx->nlaunch - nl0);
    ctx->nlaunch = nl0;
    if (s) { if (graph) cudaGraphDestroy(graph); return s; }
    CK(ce);
    ce = cudaGraphInstantiate(&ctx->pcg_graph, graph, 0);
    cudaGraphDestroy(graph);
    CK(ce);
    ctx->pcg_graph_x = ctx->x_cur;
    CK(cudaGraphLaunch(ctx->pcg_graph, st));
    ctx->nlaunch += ctx->pcg_graph_launches;
    return SC_OK;
  }
  ctx->pcg_seen_x = ctx->x_cur;
  for (int k = 0; k < kPcgChunk; ++k) {
    sc_status s = pcg_iteration(ctx, st);
    if (s) return s;
  }
  return SC_OK;
}

static sc_status pcg_impl(sc_ctx* ctx, const double* b, double* x, double rtol, int maxit, sc_pcg_report* rep,
                          cudaStream_t st) {
  auto t0 = std::chrono::steady_clock::now();
  double* done = ctx->scal + SCAL_DONE;
  sc_status s = pcg_start_impl(ctx, b, x, rtol, maxit, st);
  if (s) return s;
  const int check_every = rtol > 0 ? kPcgChunk : 0;
  int it = 0;
  bool stop = false;
  auto poll = [&]() -> sc_status {
    double dflag = 0;
    CK(cudaMemcpyAsync(&dflag, done, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    stop = dflag != 0.0;
    return SC_OK;
  };
  for (; it + kPcgChunk <= maxit && !stop; it += kPcgChunk) {
    if ((s = pcg_chunk(ctx, st))) return s;
    if (check_every && (s = poll())) return s;
  }
  for (; it < maxit && !stop; ++it) {
    if ((s = pcg_iteration(ctx, st))) return s;
    if (check_every && (it + 1) % check_every == 0 && (s = poll())) return s;
  }
  CK(cudaStreamSynchronize(st));
  auto t1 = std::chrono::steady_clock::now();
  return pcg_report_impl(ctx, rep, st, std::chrono::duration<double>(t1 - t0).count());
}

extern "C" sc_status sc_pcg_start(sc_ctx* ctx, const double* d_b, double* d_x, double rtol, int maxit, void* stream) {
  if (!ctx || !d_b || !d_x || d_b == d_x || maxit < 0 || !std::isfinite(rtol)) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (!ctx->ws) { ctx->err = "workspace not bound"; return SC_ESTATE; }
  return pcg_start_impl(ctx, d_b, d_x, rtol, maxit, (cudaStream_t)stream);
}

extern "C" sc_status sc_pcg_iterate(sc_ctx* ctx, int niter, void* stream) {
  if (!ctx || niter < 0) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (!ctx->x_cur) { ctx->err = "sc_pcg_start not called"; return SC_ESTATE; }
  for (int it = 0; it < niter; ++it) {
    sc_status s = pcg_iteration(ctx, (cudaStream_t)stream);
    if (s) return s;
  }
  return SC_OK;
}

extern "C" sc_status sc_pcg_status(sc_ctx* ctx, sc_pcg_report* rep, void* stream) {
  if (!ctx || !rep) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (!ctx->x_cur) { ctx->err = "sc_pcg_start not called"; return SC_ESTATE; }
  return pcg_report_impl(ctx, rep, (cudaStream_t)stream, 0.0);
}

extern "C" sc_status sc_profile_enable(sc_ctx* ctx, int on) {
  if (!ctx) return SC_EINVAL;
  if (on && ctx->prof_ev.empty()) {
    ctx->prof_ev.resize(2 * 8192);
    for (auto& e : ctx->prof_ev) CK(cudaEventCreate(&e));
  }
  ctx->prof_on = on != 0;
  ctx->prof_n = 0;
  return SC_OK;
}

extern "C" sc_status sc_profile_read(sc_ctx* ctx, double* h_total_ms, long long* h_count) {
  if (!ctx || !h_total_ms || !h_count) return SC_EINVAL;
  double tot = 0.0;
  for (int i = 0; i < ctx->prof_n; ++i) {
    CK(cudaEventSynchronize(ctx->prof_ev[2 * i + 1]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->prof_ev[2 * i], ctx->prof_ev[2 * i + 1]));
    tot += ms;
  }
  *h_total_ms = tot;
  *h_count = ctx->prof_n;
  ctx->prof_n = 0;
  return SC_OK;
}

extern "C" sc_status sc_pcg_solve(sc_ctx* ctx, const double* d_b, double* d_x, double rtol, int maxit,
                                  sc_pcg_report* rep, void* stream) {
  if (!ctx || !d_b || !d_x || d_b == d_x || maxit < 0 || !std::isfinite(rtol)) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (!ctx->ws) { ctx->err = "workspace not bound"; return SC_ESTATE; }
  return pcg_impl(ctx, d_b, d_x, rtol, maxit, rep, (cudaStream_t)stream);
}

extern "C" sc_status sc_pcg_solve_host(sc_ctx* ctx, const double* h_b, double* h_x, double rtol, int maxit,
                                       sc_pcg_report* rep, void* stream) {
  if (!ctx || !h_b || !h_x || maxit < 0 || !std::isfinite(rtol)) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (!ctx->ws) { ctx->err = "workspace not bound"; return SC_ESTATE; }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t bytes = sizeof(double) * ctx->g.n_total;
  CK(cudaMemcpyAsync(ctx->bdev, h_b, bytes, cudaMemcpyHostToDevice, st));
  sc_status s = pcg_impl(ctx, ctx->bdev, ctx->xdev, rtol, maxit, rep, st);
  if (s != SC_OK && s != SC_EBREAKDOWN) return s;
  CK(cudaMemcpyAsync(h_x, ctx->xdev, bytes, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return s;
}

extern "C" sc_status sc_condense_rhs(sc_ctx* ctx, const double* d_f, double* d_b, void* stream) {
  if (!ctx || !d_f || !d_b) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (!ctx->ws) { ctx->err = "workspace not bound"; return SC_ESTATE; }
  cudaStream_t st = (cudaStream_t)stream;
  LAUNCH(launch_condense(ctx->g, d_f, d_b, ctx->scratch, ctx->scratch_elems, st, &nl_));
  return halo_sum(ctx, d_b, st);
}

extern "C" sc_status sc_recover(sc_ctx* ctx, const double* d_f, const double* d_x, double* d_u, void* stream) {
  if (!ctx || !d_f || !d_x || !d_u) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (!ctx->ws) { ctx->err = "workspace not bound"; return SC_ESTATE; }
  LAUNCH(launch_recover(ctx->g, d_f, d_x, d_u, ctx->scratch, ctx->scratch_elems, (cudaStream_t)stream, &nl_));
  return SC_OK;
}

// Inhomogeneous Dirichlet data (the paper's solver benchmark E3: u = u_ex on the
// boundary of (0, 2 pi)^3).  With the data g on the Dirichlet skeleton entities D and the free ones F,
// the condensed system is  A_FF x_F = b_F - A_FD g_D  (reading R17).  In the transformed
// basis the lifting vector is g~ = Shat^{-T} g on D (every skeleton entity is either entirely in D
// or entirely in F, and Shat acts inside entities), and A_FD g~_D is one operator application with
// the Dirichlet columns kept (one-CTA-per-element kernel, any geometry).  Uses the PCG buffers of
// the workspace as scratch: not to be called between sc_pcg_start and sc_pcg_status.
extern "C" sc_status sc_condense_rhs_dirichlet(sc_ctx* ctx, const double* d_f, const double* d_g, double* d_b,
                                               void* stream) {
  if (!ctx || !d_f || !d_g || !d_b) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (!ctx->ws) { ctx->err = "workspace not bound"; return SC_ESTATE; }
  cudaStream_t st = (cudaStream_t)stream;
  LAUNCH(launch_condense(ctx->g, d_f, d_b, ctx->scratch, ctx->scratch_elems, st, &nl_));
  sc_status s = halo_sum(ctx, d_b, st);
  if (s) return s;
  Geom gn = ctx->g;
  gn.nodir = 1;
  LAUNCH(launch_convert(gn, d_g, ctx->pv, 1, MAT_SM, st, &nl_));       // Shat^{-T} g at every entity
  LAUNCH(launch_dir_split(ctx->g, ctx->pv, nullptr, 0, st, &nl_));    // keep D only: g~_D
  LAUNCH(launch_apply(gn, ctx->pv, ctx->q, nullptr, st, &nl_));       // A (., D) g~_D
  if ((s = halo_sum(ctx, ctx->q, st))) return s;
  LAUNCH(launch_dir_split(ctx->g, d_b, ctx->q, 1, st, &nl_));         // b_F -= (A g~_D)_F, b_D = 0
  return SC_OK;
}

// Alg. 4 post with the Dirichlet data: the skeleton solution is x~ on F and g~ on D; interiors by
// u~_I = D^{-1}(F~_I - Htilde_IB u~_B), lattice values u = (S(x)S(x)S)^T u~ (boundary nodes = g).
extern "C" sc_status sc_recover_dirichlet(sc_ctx* ctx, const double* d_f, const double* d_g, const double* d_x,
                                          double* d_u, void* stream) {
  if (!ctx || !d_f || !d_g || !d_x || !d_u) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (!ctx->ws) { ctx->err = "workspace not bound"; return SC_ESTATE; }
  cudaStream_t st = (cudaStream_t)stream;
  Geom gn = ctx->g;
  gn.nodir = 1;
  LAUNCH(launch_convert(gn, d_g, ctx->pv, 1, MAT_SM, st, &nl_));
  CK(cudaMemcpyAsync(ctx->q, d_x, sizeof(double) * ctx->g.n_total, cudaMemcpyDeviceToDevice, st));
  LAUNCH(launch_dir_split(ctx->g, ctx->q, ctx->pv, 2, st, &nl_));     // x~ on F, g~ on D
  LAUNCH(launch_recover(gn, d_f, ctx->q, d_u, ctx->scratch, ctx->scratch_elems, st, &nl_));
  return SC_OK;
}

static int to_mat(int mode, bool to) {
  if (mode == SC_PERM) return MAT_I;
  if (mode == SC_PRIMAL) return to ? MAT_SM : MAT_ST;
  return to ? MAT_S : MAT_MST;
}

extern "C" sc_status sc_to_transformed(sc_ctx* ctx, const double* d_lattice, double* d_skel, int mode, void* stream) {
  if (!ctx || !d_lattice || !d_skel || mode < 0 || mode > 2) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  LAUNCH(launch_convert(ctx->g, d_lattice, d_skel, 1, to_mat(mode, true), stream, &nl_));
  return SC_OK;
}

extern "C" sc_status sc_from_transformed(sc_ctx* ctx, const double* d_skel, double* d_lattice, int mode, void* stream) {
  if (!ctx || !d_lattice || !d_skel || mode < 0 || mode > 2) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  LAUNCH(launch_convert(ctx->g, d_skel, d_lattice, 0, to_mat(mode, false), stream, &nl_));
  return SC_OK;
}

extern "C" sc_status sc_fill_random(sc_ctx* ctx, uint64_t seed, double* d_skel, void* stream) {
  if (!ctx || !d_skel) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  LAUNCH(launch_fill_random(ctx->g, seed, d_skel, stream, &nl_));
  return SC_OK;
}

extern "C" sc_status sc_dot(sc_ctx* ctx, const double* d_a, const double* d_b, double* h_out, void* stream) {
  if (!ctx || !d_a || !d_b || !h_out) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (!ctx->ws) { ctx->err = "workspace not bound"; return SC_ESTATE; }
  cudaStream_t st = (cudaStream_t)stream;
  double* part = ctx->partials + 2 * SC_RED_BLOCKS;   // keep PCG partials untouched
  LAUNCH(launch_dot_partial(d_a, d_b, ctx->g.n_total, ctx->own, part, nullptr, st, &nl_));
  // use partial slots [2R, 3R) -> reduce into scal[RED2]
  LAUNCH(launch_reduce2(part, ctx->scal, SCAL_RED2, 1, nullptr, st, &nl_));
  sc_status s = allreduce_scal(ctx, SCAL_RED2, 1, st);
  if (s) return s;
  CK(cudaMemcpyAsync(h_out, ctx->scal + SCAL_RED2, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return SC_OK;
}

extern "C" sc_status sc_preconditioner(sc_ctx* ctx, double* d_pinv, void* stream) {
  if (!ctx || !d_pinv) return SC_EINVAL;
  if (!ctx->ws) { ctx->err = "workspace not bound"; return SC_ESTATE; }
  CK(cudaMemcpyAsync(d_pinv, ctx->pinv, sizeof(double) * ctx->g.n_total, cudaMemcpyDeviceToDevice,
                     (cudaStream_t)stream));
  return SC_OK;
}

extern "C" sc_status sc_nccl_unique_id(unsigned char h_id[128]) {
  if (!h_id) return SC_EINVAL;
  if (!load_nccl()) return SC_ENCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return SC_ENCCL;
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(h_id, &id, 128);
  return SC_OK;
}

extern "C" sc_status sc_nccl_comm_init(const unsigned char h_id[128], int nranks, int rank, int device, void** comm_out) {
  if (!h_id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return SC_EINVAL;
  if (!load_nccl()) return SC_ENCCL;
  if (cudaSetDevice(device) != cudaSuccess) return SC_ECUDA;
  ncclUniqueId id;
  memcpy(&id, h_id, 128);
  ncclComm_t c;
  if (g_nccl.CommInitRank(&c, nranks, id, rank) != ncclSuccess) return SC_ENCCL;
  *comm_out = (void*)c;
  return SC_OK;
}

extern "C" sc_status sc_nccl_comm_destroy(void* comm) {
  if (!comm) return SC_OK;
  if (!load_nccl()) return SC_ENCCL;
  return g_nccl.CommDestroy((ncclComm_t)comm) == ncclSuccess ? SC_OK : SC_ENCCL;
}

extern "C" sc_status sc_loopback_comms_create(int nranks, void** comms_out) {
  if (nranks < 1 || !comms_out) return SC_EINVAL;
  LoopGroup* G = new LoopGroup;
  G->nranks = nranks;
  G->seg.assign((size_t)nranks * 8, nullptr);
  G->val.assign((size_t)nranks, nullptr);
  std::lock_guard<std::mutex> lk(g_loop_mu);
  for (int r = 0; r < nranks; ++r) {
    LoopComm* c = new LoopComm{G, r};
    g_loop_comms.insert(c);
    comms_out[r] = c;
  }
  return SC_OK;
}

extern "C" sc_status sc_loopback_comms_destroy(void** comms, int nranks) {
  if (!comms || nranks < 1) return SC_EINVAL;
  std::lock_guard<std::mutex> lk(g_loop_mu);
  LoopGroup* G = nullptr;
  for (int r = 0; r < nranks; ++r) {
    if (!comms[r] || !g_loop_comms.count(comms[r])) return SC_EINVAL;
    LoopComm* c = (LoopComm*)comms[r];
    G = c->grp;
    g_loop_comms.erase(c);
    delete c;
  }
  delete G;
  return SC_OK;
}

// ---------------------------------------------------------------- PAPER.md §7 operator variants
extern "C" sc_status sc_apply_tpc(sc_ctx* ctx, const double* d_x, double* d_y, void* stream) {
  if (!ctx || !d_x || !d_y || d_x == d_y) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  cudaStream_t st = (cudaStream_t)stream;
  const bool rec = ctx->prof_on && ctx->prof_n < (int)ctx->prof_ev.size() / 2;
  cudaEvent_t* ev = rec ? &ctx->prof_ev[2 * ctx->prof_n] : nullptr;
  LAUNCH(launch_apply_tpc(ctx->g, ctx->d_vt, d_x, d_y, st, &nl_, ev));
  if (rec) ctx->prof_n++;
  return halo_sum(ctx, d_y, st);
}

static int mmc_shell(const sc_ctx* ctx) {
  const long long ni = ctx->g.ni;
  return (int)(6 * ni * ni + 12 * ni + 8);
}

static long long mmc_ngeom(const sc_ctx* ctx) {
  return ctx->g.uniform ? 1 : (long long)ctx->g.nx * ctx->g.ny * ctx->g.nz;
}

extern "C" size_t sc_mmc_bytes(const sc_ctx* ctx) {
  if (!ctx) return 0;
  const long long nB = mmc_shell(ctx), ne = (long long)ctx->g.nx * ctx->g.ny * ctx->g.nz;
  const long long mat = align_up(nB * nB * mmc_ngeom(ctx));
  return sizeof(double) * (size_t)(mat + 2 * align_up(nB * ne));
}

extern "C" sc_status sc_mmc_bind(sc_ctx* ctx, void* d_buf, size_t bytes, void* stream) {
  if (!ctx || !d_buf) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (bytes < sc_mmc_bytes(ctx)) {
    ctx->err = "MMC buffer too small: need " + std::to_string(sc_mmc_bytes(ctx)) + " bytes (sc_mmc_bytes)";
    return SC_ENOMEM;
  }
  if (!load_cublas()) { ctx->err = "libcublas.so.12 not loadable"; return SC_ECUDA; }
  if (!ctx->cublas && g_cublas.Create(&ctx->cublas) != 0) { ctx->err = "cublasCreate failed"; return SC_ECUDA; }
  cudaStream_t st = (cudaStream_t)stream;
  const long long nB = mmc_shell(ctx), ne = (long long)ctx->g.nx * ctx->g.ny * ctx->g.nz;
  const long long ng = mmc_ngeom(ctx);
  ctx->mmc_nB = (int)nB;
  ctx->mmc_ngeom = ng;
  ctx->mmc_H = (double*)d_buf;
  ctx->mmc_X = ctx->mmc_H + align_up(nB * nB * ng);   // matrices packed with stride nB^2
  ctx->mmc_Y = ctx->mmc_X + align_up(nB * ne);
  // precomputation, O(n_I^5) per geometry (Table 3): Hhat_e column by column
  LAUNCH(launch_mmc_columns(ctx->g, ctx->d_vt, ctx->mmc_H, (int)nB, ng, st, &nl_));
  CK(cudaStreamSynchronize(st));
  return SC_OK;
}

extern "C" sc_status sc_apply_mmc(sc_ctx* ctx, const double* d_x, double* d_y, void* stream) {
  if (!ctx || !d_x || !d_y || d_x == d_y) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (!ctx->mmc_H) { ctx->err = "sc_mmc_bind not called"; return SC_ESTATE; }
  cudaStream_t st = (cudaStream_t)stream;
  const int nB = ctx->mmc_nB;
  const long long ne = (long long)ctx->g.nx * ctx->g.ny * ctx->g.nz;
  const bool rec = ctx->prof_on && ctx->prof_n < (int)ctx->prof_ev.size() / 2;
  cudaEvent_t* ev = rec ? &ctx->prof_ev[2 * ctx->prof_n] : nullptr;
  if (ev) CK(cudaEventRecord(ev[0], st));
  LAUNCH(launch_mmc_gather(ctx->g, d_x, ctx->mmc_X, nB, st, &nl_));
  if (ne > 0) {
    if (g_cublas.SetStream(ctx->cublas, st) != 0) { ctx->err = "cublasSetStream failed"; return SC_ECUDA; }
    const double one = 1.0, zero = 0.0;
    int rc;
    if (ctx->mmc_ngeom == 1) {   // Y (nB x ne) = Hhat (nB x nB) X (nB x ne), column-major, one DGEMM
      rc = g_cublas.Dgemm(ctx->cublas, 0, 0, nB, (int)ne, nB, &one, ctx->mmc_H, nB, ctx->mmc_X, nB, &zero,
                          ctx->mmc_Y, nB);
    } else {                     // one matrix per element: a strided batch of GEMVs
      rc = g_cublas.DgemmStridedBatched(ctx->cublas, 0, 0, nB, 1, nB, &one, ctx->mmc_H, nB, (long long)nB * nB,
                                        ctx->mmc_X, nB, nB, &zero, ctx->mmc_Y, nB, nB, (int)ne);
    }
    if (rc != 0) { ctx->err = "cublasDgemm failed (" + std::to_string(rc) + ")"; ctx->broken = true; return SC_ECUDA; }
    ctx->nlaunch++;
  }
  LAUNCH(launch_mmc_assemble(ctx->g, ctx->mmc_Y, d_y, nB, st, &nl_));
  if (ev) { CK(cudaEventRecord(ev[1], st)); ctx->prof_n++; }
  return halo_sum(ctx, d_y, st);
}

// Solvers UC / DC / BC of PAPER.md §8 (Table 4) on the NODAL condensed system with the
// TPC (or MMC) operator.  Hestenes-Stiefel PCG as in BT; stopping rule ||r_k||_2 <= rtol ||r_0||_2 on the
// recursively updated NODAL residual (DESIGN reading R18).  Workspace use: q, pv, r as in BT; bdev = z,
// xdev = the UC mask / DC inverse diagonal; the BT diagonal ctx->pinv is BC's transformed-block inverse.
static sc_status nodal_apply(sc_ctx* ctx, int op, const double* x, double* y, cudaStream_t st) {
  return op == SC_OP_MMC ? sc_apply_mmc(ctx, x, y, st) : sc_apply_tpc(ctx, x, y, st);
}

extern "C" sc_status sc_pcg_solve_nodal(sc_ctx* ctx, int op, int prec, const double* d_b, double* d_x, double rtol,
                                        int maxit, sc_pcg_report* rep, void* stream) {
  if (!ctx || !d_b || !d_x || d_b == d_x) return SC_EINVAL;
  if ((op != SC_OP_TPC && op != SC_OP_MMC) || prec < SC_PREC_NONE || prec > SC_PREC_BLOCK) return SC_EINVAL;
  if (ctx->broken) return SC_ESTATE;
  if (!ctx->ws) { ctx->err = "workspace not bound"; return SC_ESTATE; }
  if (op == SC_OP_MMC && !ctx->mmc_H) { ctx->err = "sc_mmc_bind not called"; return SC_ESTATE; }
  cudaStream_t st = (cudaStream_t)stream;
  auto t0 = std::chrono::steady_clock::now();
  const long long n = ctx->g.n_total;
  double* z = ctx->bdev;
  double* m = ctx->xdev;
  const double* mask = ctx->pinv;     // nonzero exactly on the free entries
  ctx->tol2 = rtol > 0 ? rtol * rtol : -1.0;
  if (prec == SC_PREC_DIAG) {
    LAUNCH(launch_var_diag(ctx->g, ctx->d_vt, m, st, &nl_));
    sc_status s = halo_sum(ctx, m, st);
    if (s) return s;
    LAUNCH(launch_invert_diag(ctx->g, m, st, &nl_));
  }
  if (prec == SC_PREC_NONE) LAUNCH(launch_unit_mask(mask, m, n, st, &nl_));   // m = 1 on free entries
  const double* pm = prec == SC_PREC_BLOCK ? ctx->pinv : m;
  CK(cudaMemsetAsync(z, 0, sizeof(double) * n, st));
  LAUNCH(launch_var_init(d_b, mask, ctx->r, d_x, n, st, &nl_));
  LAUNCH(launch_var_prec(ctx->g, prec, pm, ctx->r, z, st, &nl_));
  LAUNCH(launch_var_direction(d_x, ctx->pv, z, n, ctx->scal, 1, st, &nl_));
  LAUNCH(launch_dot_partial(ctx->r, z, n, ctx->own, ctx->partials, nullptr, st, &nl_));
  LAUNCH(launch_dot_partial(ctx->r, ctx->r, n, ctx->own, ctx->partials + SC_RED_BLOCKS, nullptr, st, &nl_));
  LAUNCH(launch_reduce2(ctx->partials, ctx->scal, SCAL_RED0, 2, nullptr, st, &nl_));
  sc_status s = allreduce_scal(ctx, SCAL_RED0, 2, st);
  if (s) return s;
  LAUNCH(launch_pcg_init_finalize(ctx->scal, ctx->partials, ctx->tol2, maxit, st, &nl_));
  double* done = ctx->scal + SCAL_DONE;
  bool stop = false;
  for (int it = 0; it < maxit && !stop; ++it) {
    if ((s = nodal_apply(ctx, op, ctx->pv, ctx->q, st))) return s;
    LAUNCH(launch_dot_partial(ctx->pv, ctx->q, n, ctx->own, ctx->partials, done, st, &nl_));
    LAUNCH(launch_reduce2(ctx->partials, ctx->scal, SCAL_RED0, 1, done, st, &nl_));
    if ((s = allreduce_scal(ctx, SCAL_RED0, 1, st))) return s;
    LAUNCH(launch_pcg_alpha(ctx->scal, st, &nl_));
    LAUNCH(launch_var_update(ctx->r, ctx->q, n, ctx->scal, st, &nl_));
    LAUNCH(launch_var_prec(ctx->g, prec, pm, ctx->r, z, st, &nl_));
    LAUNCH(launch_dot_partial(ctx->r, z, n, ctx->own, ctx->partials, done, st, &nl_));
    LAUNCH(launch_dot_partial(ctx->r, ctx->r, n, ctx->own, ctx->partials + SC_RED_BLOCKS, done, st, &nl_));
    LAUNCH(launch_reduce2(ctx->partials, ctx->scal, SCAL_RED0, 2, done, st, &nl_));
    if ((s = allreduce_scal(ctx, SCAL_RED0, 2, st))) return s;
    LAUNCH(launch_pcg_beta(ctx->scal, st, &nl_));
    LAUNCH(launch_var_direction(d_x, ctx->pv, z, n, ctx->scal, 0, st, &nl_));
    if (rtol > 0 && (it + 1) % kPcgChunk == 0) {
      double dflag = 0;
      CK(cudaMemcpyAsync(&dflag, done, sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      stop = dflag != 0.0;
    }
  }
  CK(cudaStreamSynchronize(st));
  auto t1 = std::chrono::steady_clock::now();
  return pcg_report_impl(ctx, rep, st, std::chrono::duration<double>(t1 - t0).count());
}

extern "C" long long sc_launch_count(const sc_ctx* ctx) { return ctx ? ctx->nlaunch : 0; }

extern "C" const char* sc_operator_kernel(const sc_ctx* ctx) {
  if (!ctx) return "";
  if (ctx->use_v7) return "v7";
  if (ctx->use_v6) return ctx->v6_h == 8 ? "v6h8" : "v6";
  if (ctx->use_col) return "v3";
  if (ctx->use_p2s) return "p2s";
  if (ctx->use_p2) return "p2";
  if (ctx->use_rw) return "rw";
  if (ctx->use_big) return "v4";
  return "v1";
}

extern "C" const char* sc_last_error(const sc_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

extern "C" const char* sc_version(void) {
  return "sc 0.1 (sm_100a, fp64, TPT condensed operator v1, BT-PCG)";
}
