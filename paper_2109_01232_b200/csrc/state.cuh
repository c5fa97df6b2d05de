// Typed views of the caller-allocated cycle state and reduction workspace,
// plus the host-side launcher declarations shared by the translation units.
#pragma once

#include "common.cuh"

namespace mpg {

// ------------------------------------------------------------------ state
struct StateLayout {
  int64_t implicit, H, R, cs, sn, g, c1, c2, d, red, total;
};

inline __host__ __device__ int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

inline __host__ __device__ StateLayout state_layout(int prec, int m) {
  const int64_t s = prec == MPG_FP64 ? 8 : 4;
  StateLayout L;
  int64_t off = align_up((int64_t)sizeof(mpg_state_header), 64);
  L.implicit = off; off = align_up(off + 8 * (int64_t)m, 64);
  L.H = off; off = align_up(off + s * (int64_t)(m + 1) * m, 64);
  L.R = off; off = align_up(off + s * (int64_t)(m + 1) * m, 64);
  L.cs = off; off = align_up(off + s * m, 64);
  L.sn = off; off = align_up(off + s * m, 64);
  L.g = off; off = align_up(off + s * (m + 1), 64);
  L.c1 = off; off = align_up(off + s * (m + 1), 64);
  L.c2 = off; off = align_up(off + s * (m + 1), 64);
  L.d = off; off = align_up(off + s * (m + 1), 64);
  L.red = off; off = align_up(off + s * (m + 8), 64);   // raw per-rank sums (distributed mode)
  L.total = off;
  return L;
}

template <typename T>
struct StateView {
  mpg_state_header* h;
  double* implicit;
  T *H, *R, *cs, *sn, *g, *c1, *c2, *d, *red;
  int m;
  int dist;   // 1: kernels publish raw local sums to red[] for a cross-rank allreduce
  __device__ __forceinline__ T& Hc(int col, int row) const { return H[(size_t)col * (m + 1) + row]; }
  __device__ __forceinline__ T& Rc(int col, int row) const { return R[(size_t)col * (m + 1) + row]; }
};

template <typename T>
inline StateView<T> make_state(void* base, int m) {
  const int prec = sizeof(T) == 8 ? MPG_FP64 : MPG_FP32;
  StateLayout L = state_layout(prec, m);
  char* b = static_cast<char*>(base);
  StateView<T> s;
  s.h = reinterpret_cast<mpg_state_header*>(b);
  s.implicit = reinterpret_cast<double*>(b + L.implicit);
  s.H = reinterpret_cast<T*>(b + L.H);
  s.R = reinterpret_cast<T*>(b + L.R);
  s.cs = reinterpret_cast<T*>(b + L.cs);
  s.sn = reinterpret_cast<T*>(b + L.sn);
  s.g = reinterpret_cast<T*>(b + L.g);
  s.c1 = reinterpret_cast<T*>(b + L.c1);
  s.c2 = reinterpret_cast<T*>(b + L.c2);
  s.d = reinterpret_cast<T*>(b + L.d);
  s.red = reinterpret_cast<T*>(b + L.red);
  s.m = m;
  s.dist = 0;
  return s;
}

// -------------------------------------------------------------- workspace
constexpr int kMaxM = 512;                       // largest restart length supported
constexpr int kMaxParts = 148 * 8;               // partial rows (CTAs) per reduction
constexpr int64_t kWsCounterBytes = 256;
// two-level grid reductions (grid_reduce_cols): CTAs are grouped by kRedGroup
constexpr int kRedGroup = 32;
constexpr int kRedGroups = (kMaxParts + kRedGroup - 1) / kRedGroup;   // 37
constexpr int64_t kPartBytes = (int64_t)kMaxParts * (kMaxM + 8) * 8;
constexpr int64_t kGPartBytes = (int64_t)64 * (kMaxM + 8) * 8;
constexpr int64_t kWsBytes = kWsCounterBytes + kPartBytes + kGPartBytes + 4096;

struct WsView {
  unsigned int* counter;   // one election counter (kernels on a stream are serial)
  int64_t* scratch_i64;    // small integer scratch (overflow index etc.)
  void* part;              // partials, [parts][stride] of T (column-major [c][kMaxParts] for grid_reduce_cols)
  void* gpart;             // group partials [c][64] (grid_reduce_cols)
  unsigned int* gcount;    // per-group arrival counters [64] (grid_reduce_cols)
};
inline WsView make_ws(void* base) {
  WsView w;
  char* b = static_cast<char*>(base);
  w.counter = reinterpret_cast<unsigned int*>(b);
  w.scratch_i64 = reinterpret_cast<int64_t*>(b + 128);
  w.part = b + kWsCounterBytes;
  w.gpart = b + kWsCounterBytes + kPartBytes;
  w.gcount = reinterpret_cast<unsigned int*>(b + kWsCounterBytes + kPartBytes + kGPartBytes);
  return w;
}

// ------------------------------------------------------------- launchers
void count_launch(int n = 1);

// matrix views (defined in spmv.cuh): CSR and the stencil (DIA) storage
template <typename T> struct CsrView;
template <typename T> struct StencilView;

// spmv family (spmv_kernels.cu); M = CsrView<T> or StencilView<T>
template <typename T, typename M>
cudaError_t launch_spmv(const M& A, const T* x, T* y, WsView ws, cudaStream_t st,
                        const mpg_state_header* kt = nullptr);
template <typename T, typename M>
cudaError_t launch_residual(const M& A, const T* b, const T* x, T* r, double* norm_out,
                            mpg_state_header* hdr, WsView ws, cudaStream_t st, int raw = 0,
                            const mpg_state_header* kt = nullptr, int kcat = KC_SPMV);
template <typename T, typename M>
cudaError_t launch_spmv_dot1(const M& A, const T* x, T* w, const T* V, long long ldv, int k,
                             StateView<T> sv, WsView ws, cudaStream_t st);
template <typename T, typename M>
cudaError_t launch_poly_op(const M& A, const mpg_poly_op& op, const T* x, T* y, T* t0, T* t1,
                           T* t2, const mpg_state_header* gate, long long n, WsView ws,
                           cudaStream_t st, const mpg_state_header* kt = nullptr);
template <typename T>
cudaError_t launch_stencil_pack(int dims, int nx, long long row0, long long n, const int32_t* rp,
                                const int32_t* ci, const T* v, T* out, long long ldv, int* bad,
                                cudaStream_t st);

// arnoldi family (arnoldi_kernels.cu)
template <typename T>
cudaError_t launch_dot1_w(const T* w, long long n, const T* V, long long ldv, int k,
                          StateView<T> sv, WsView ws, cudaStream_t st);
template <typename T>
cudaError_t launch_dot1_wo(const T* w, long long n, const T* V, long long ldv, int k,
                           StateView<T> sv, WsView ws, cudaStream_t st);
bool split_spmv_dot1();
template <typename T>
cudaError_t launch_update_dot(const T* V, long long ldv, long long n, int k, T* w,
                              StateView<T> sv, WsView ws, cudaStream_t st);
template <typename T>
cudaError_t launch_update_norm(const T* V, long long ldv, long long n, int j, T* w,
                               StateView<T> sv, WsView ws, int m_limit, cudaStream_t st);
// K_C + K_S in one cooperative launch (grid barrier); falls back to the pair
template <typename T>
cudaError_t launch_update_norm_scale(const T* V, long long ldv, long long n, int j, T* w,
                                     StateView<T> sv, WsView ws, int m_limit, cudaStream_t st);
bool fuse_update_norm_scale();
template <typename T>
cudaError_t launch_step_scale(const T* w, T* vnext, long long n, int j, StateView<T> sv,
                              cudaStream_t st);
// start of a cycle: gamma = ||src|| (IR: src = fp32(r64 / rho), written to r_in)
template <typename T>
cudaError_t launch_start(const T* r0, long long n, StateView<T> sv, double rtol,
                         const double* b_norm_src, double breakdown_tol, WsView ws,
                         cudaStream_t st);
cudaError_t launch_start_ir(const double* r64, float* r32, long long n, StateView<float> sv,
                            double rtol, double breakdown_tol, WsView ws, cudaStream_t st);
template <typename T>
cudaError_t launch_start_scale(const T* r0, T* v0, long long n, StateView<T> sv, cudaStream_t st);
template <typename T>
cudaError_t launch_lsq(StateView<T> sv, cudaStream_t st);

// distributed peer-memory halo: scale + remote halo stores + flag release; flag wait
template <typename T>
cudaError_t launch_step_scale_peer(const T* w, T* vn, long long n, long long halo, int j, StateView<T> sv,
                                   T* prev_row, T* next_row, uint32_t* prev_flag, uint32_t* next_flag,
                                   WsView ws, cudaStream_t st);
cudaError_t launch_halo_wait(mpg_state_header* h, const uint32_t* flags, int has_prev, int has_next,
                             cudaStream_t st);

// ---------------------------------------------------------- exchange box
// One rank's mailbox for the distributed persistent step (MPG_PH_STEP): for
// each of the step's three cross-rank sums p (pass-1 dots + ||w||^2 + flag,
// pass-2 dots, ||w''||^2), rank r's local column sums land in vals[p][r][:]
// (written by rank r through its peer mapping) and rank r then release-stores
// the step's sequence number into seq[p][r].  Sums are read back in rank
// order, so every rank gets the same bits.  `step` counts this rank's step
// kernels (identical on every rank).
constexpr int kXMaxRanks = 8;
constexpr int kXCols = 72;                                   // >= kMegaMaxCols
constexpr int64_t kXValsBytes = (int64_t)3 * kXMaxRanks * kXCols * 8;
constexpr int64_t kXSeqOff = kXValsBytes;                     // uint32 seq[3][kXMaxRanks]
constexpr int64_t kXStepOff = kXSeqOff + 3 * kXMaxRanks * 4;  // uint32 step
constexpr int64_t kXBoxBytes = kXStepOff + 256;
template <typename T>
__device__ __forceinline__ T* xbox_vals(void* box, int p, int r) {
  return reinterpret_cast<T*>(static_cast<char*>(box)) + ((size_t)p * kXMaxRanks + r) * kXCols;
}
__device__ __forceinline__ uint32_t* xbox_seq(void* box, int p, int r) {
  return reinterpret_cast<uint32_t*>(static_cast<char*>(box) + kXSeqOff) + p * kXMaxRanks + r;
}
__device__ __forceinline__ uint32_t* xbox_step(void* box) {
  return reinterpret_cast<uint32_t*>(static_cast<char*>(box) + kXStepOff);
}

// The distributed persistent step's view of the peers (DIST instantiation).
template <typename T>
struct MegaX {
  void* box[kXMaxRanks];   // every rank's exchange box as mapped here
  int world, rank;
  long long halo;          // rows of one halo plane
  T* prev_V;               // prev rank's basis (row 0 at its owned offset) or null
  long long prev_ld, prev_off;
  T* next_V;
  long long next_ld, next_off;
  uint32_t* hflags;        // this rank's halo flags ([0] from prev, [1] from next)
  uint32_t* prev_flag;     // where we release into prev's / next's flags
  uint32_t* next_flag;
};

// persistent per-step kernel (step_kernel.cu), stencil storage, single GPU;
// steps with k > kMegaMaxK basis vectors use the four-launch step
constexpr int kMegaMaxK = 56;
// jdiag / zout: Jacobi(1) right preconditioning -- the kernel also writes the
// next step's operator input z = V[:, j+1] / diag (x is then z_j, not V[:, j])
template <typename T>
cudaError_t launch_step_mega(const StencilView<T>& S, const T* x, T* V, long long ldv, long long n, int j,
                             T* w, StateView<T> sv, WsView ws, int m_limit, cudaStream_t st,
                             const T* jdiag = nullptr, T* zout = nullptr, const MegaX<T>* xd = nullptr);
int mega_env();   // MPG_MEGA: 1 / 0 forces the persistent / four-launch step, -1 unset

// distributed-mode post phases (k_dist_post)
enum DistPostPhase {
  DP_POST_START = 0,
  DP_POST_DOT1 = 1,
  DP_POST_DOT2 = 2,
  DP_POST_NORM = 3,
  DP_POST_RESID = 4,
  DP_POST_BNORM = 5,
};
template <typename T>
cudaError_t launch_dist_post(int phase, StateView<T> sv, int j, int m_limit, double rtol,
                             double btol, int flag, cudaStream_t st);

enum CombineMode {
  CMB_STORE = 0,    // u = V d
  CMB_ADD = 1,      // x += V d
  CMB_IR = 2,       // x64 += rho * fp64(V d)
  CMB_J1_ADD = 3,   // x += (V d) / diag
  CMB_J1_IR = 4,    // x64 += rho * fp64((V d) / diag)
  CMB_J1_CAST = 5,  // x64 += fp64(fp32(V d) / diag32)
};
template <typename T>
cudaError_t launch_combine(const T* V, long long ldv, long long n, StateView<T> sv, int mode,
                           void* x, const void* diag, T* u, cudaStream_t st);

// misc (misc_kernels.cu)
template <typename T>
cudaError_t launch_norm2(const T* x, long long n, double* out, WsView ws, cudaStream_t st,
                         int raw = 0);
template <typename T>
cudaError_t launch_gemv_t(const T* A, long long lda, long long rows, int cols, const T* x, T* y,
                          T alpha, T beta, WsView ws, cudaStream_t st);
template <typename T>
cudaError_t launch_gemv_n(const T* A, long long lda, long long rows, int cols, const T* x, T* y,
                          T alpha, T beta, cudaStream_t st);
cudaError_t launch_convert(int sp, int dp, long long n, const void* x, void* y, int64_t* ovf,
                           cudaStream_t st);
template <typename T>
cudaError_t launch_scale_div(const T* x, const double* s, T* y, long long n, cudaStream_t st);
cudaError_t launch_ir_correct(double* x, const float* u, const double* rho, long long n,
                              const mpg_state_header* gate, cudaStream_t st);
template <typename T, typename TX>
cudaError_t launch_finish_add(TX* x, const T* z, long long n, const mpg_state_header* gate,
                              int ir, cudaStream_t st);
template <typename T>
cudaError_t launch_poly_elem(int op, T a, const T* src, T* dst, T* y, long long n,
                             const mpg_state_header* gate, cudaStream_t st);
template <typename T>
cudaError_t launch_jacobi(long long n, int k, const T* lu, const int64_t* piv, const T* x, T* y,
                          const mpg_state_header* gate, cudaStream_t st);
template <typename T>
cudaError_t launch_jacobi_build(long long n, int k, const int32_t* rp, const int32_t* ci,
                                const T* v, T* lu, int64_t* piv, int64_t* bad, cudaStream_t st);
template <typename TS, typename TD>
cudaError_t launch_cast_gated(const TS* x, TD* y, long long n, const mpg_state_header* gate,
                              int64_t* ovf, cudaStream_t st);
long long host_nnz_before(int kind, long long nx, long long r);
cudaError_t launch_generate(int kind, long long nx, double conv, double stretch, long long r0,
                            long long r1, int32_t* rp, int32_t* ci, double* v, cudaStream_t st);

}  // namespace mpg
