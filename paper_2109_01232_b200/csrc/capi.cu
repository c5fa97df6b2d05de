// extern "C" entry points of libmpgmres_b200.so (declared in
// include/mpgmres_b200.h).  Thin argument checks, then the launchers.
#include <atomic>

#include "spmv.cuh"
#include "state.cuh"

namespace mpg {
static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace mpg

using namespace mpg;

static inline cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }
static inline int rc(cudaError_t e) { return (int)e; }

extern "C" {

const char* mpg_version(void) { return "mpgmres_b200 0.1.0 sm_100a"; }
int64_t mpg_workspace_bytes(void) { return kWsBytes; }
int64_t mpg_solver_desc_bytes(void) { return (int64_t)sizeof(mpg_solver_desc); }
int64_t mpg_xbox_bytes(void) { return kXBoxBytes; }
int mpg_enable_peer(int32_t peer) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return (int)cudaGetLastError();
  if (peer == dev) return MPG_OK;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, dev, peer) != cudaSuccess || !can) {
    cudaGetLastError();
    return MPG_EUNSUPPORTED;
  }
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return MPG_OK;
  }
  return (int)e;
}
int64_t mpg_launch_count(void) { return g_launches.load(); }

int mpg_spmv(int prec, int64_t n, const int32_t* rp, const int32_t* ci, const void* v,
             const void* x, void* y, void* ws, void* stream) {
  if (n < 0 || !rp || !ws) return MPG_EARG;
  if (n == 0) return MPG_OK;
  WsView w = make_ws(ws);
  if (prec == MPG_FP64)
    return rc(launch_spmv<double>(CsrView<double>{rp, ci, (const double*)v, n}, (const double*)x,
                                  (double*)y, w, S(stream)));
  if (prec == MPG_FP32)
    return rc(launch_spmv<float>(CsrView<float>{rp, ci, (const float*)v, n}, (const float*)x,
                                 (float*)y, w, S(stream)));
  return MPG_EARG;
}

int mpg_residual(int prec, int64_t n, const int32_t* rp, const int32_t* ci, const void* v,
                 const void* b, const void* x, void* r, double* out, void* ws, void* stream) {
  if (n < 1 || !rp || !ws) return MPG_EARG;
  WsView w = make_ws(ws);
  if (prec == MPG_FP64)
    return rc(launch_residual<double>(CsrView<double>{rp, ci, (const double*)v, n}, (const double*)b,
                                      (const double*)x, (double*)r, out, nullptr, w, S(stream)));
  if (prec == MPG_FP32)
    return rc(launch_residual<float>(CsrView<float>{rp, ci, (const float*)v, n}, (const float*)b,
                                     (const float*)x, (float*)r, out, nullptr, w, S(stream)));
  return MPG_EARG;
}

int mpg_norm2(int prec, int64_t n, const void* x, double* out, void* ws, void* stream) {
  if (n < 1 || !ws || !out) return MPG_EARG;
  WsView w = make_ws(ws);
  if (prec == MPG_FP64) return rc(launch_norm2<double>((const double*)x, n, out, w, S(stream)));
  if (prec == MPG_FP32) return rc(launch_norm2<float>((const float*)x, n, out, w, S(stream)));
  return MPG_EARG;
}

int mpg_gemv(int prec, int trans, int64_t rows, int64_t cols, const void* A, int64_t lda,
             const void* x, void* y, double alpha, double beta, void* ws, void* stream) {
  if (rows < 1 || cols < 1 || lda < rows || !ws) return MPG_EARG;
  if (trans && cols > kMaxM + 8) return MPG_EUNSUPPORTED;
  WsView w = make_ws(ws);
  if (prec == MPG_FP64) {
    if (trans)
      return rc(launch_gemv_t<double>((const double*)A, lda, rows, (int)cols, (const double*)x,
                                      (double*)y, alpha, beta, w, S(stream)));
    return rc(launch_gemv_n<double>((const double*)A, lda, rows, (int)cols, (const double*)x,
                                    (double*)y, alpha, beta, S(stream)));
  }
  if (prec == MPG_FP32) {
    if (trans)
      return rc(launch_gemv_t<float>((const float*)A, lda, rows, (int)cols, (const float*)x,
                                     (float*)y, (float)alpha, (float)beta, w, S(stream)));
    return rc(launch_gemv_n<float>((const float*)A, lda, rows, (int)cols, (const float*)x,
                                   (float*)y, (float)alpha, (float)beta, S(stream)));
  }
  return MPG_EARG;
}

int mpg_convert(int sp, int dp, int64_t n, const void* x, void* y, int64_t* ovf, void* stream) {
  if (n < 0 || (sp != MPG_FP32 && sp != MPG_FP64) || (dp != MPG_FP32 && dp != MPG_FP64))
    return MPG_EARG;
  if (n == 0) return MPG_OK;
  return rc(launch_convert(sp, dp, n, x, y, ovf, S(stream)));
}

int mpg_scale_div(int prec, int64_t n, const void* x, const double* s, void* y, void* stream) {
  if (n < 0) return MPG_EARG;
  if (n == 0) return MPG_OK;
  if (prec == MPG_FP64) return rc(launch_scale_div<double>((const double*)x, s, (double*)y, n, S(stream)));
  if (prec == MPG_FP32) return rc(launch_scale_div<float>((const float*)x, s, (float*)y, n, S(stream)));
  return MPG_EARG;
}

int mpg_ir_correct(int64_t n, double* x64, const float* u32, const double* rho, void* stream) {
  if (n < 0 || !rho) return MPG_EARG;
  if (n == 0) return MPG_OK;
  return rc(launch_ir_correct(x64, u32, rho, n, nullptr, S(stream)));
}

// ------------------------------------------------------------------ stencils
static int kind_ok(int kind) { return kind >= MPG_LAPLACE2D && kind <= MPG_RECIRC2D; }

int mpg_stencil_counts(int kind, int64_t nx, int64_t* n, int64_t* nnz) {
  if (!kind_ok(kind) || nx < 2 || !n || !nnz) return MPG_EARG;
  const long long N = kind == MPG_LAPLACE3D ? nx * nx * nx : nx * nx;
  *n = N;
  *nnz = host_nnz_before(kind, nx, N);
  return MPG_OK;
}

int64_t mpg_stencil_nnz_before(int kind, int64_t nx, int64_t row) {
  if (!kind_ok(kind) || nx < 2 || row < 0) return -1;
  return host_nnz_before(kind, nx, row);
}

int mpg_generate_stencil(int kind, int64_t nx, double conv, double stretch, int64_t r0, int64_t r1,
                         int32_t* rp, int32_t* ci, double* v, void* stream) {
  if (!kind_ok(kind) || nx < 2 || r0 < 0 || r1 < r0 || !rp) return MPG_EARG;
  const long long N = kind == MPG_LAPLACE3D ? nx * nx * nx : nx * nx;
  if (r1 > N) return MPG_EARG;
  if (host_nnz_before(kind, nx, r1) - host_nnz_before(kind, nx, r0) >= (1LL << 31)) return MPG_EUNSUPPORTED;
  return rc(launch_generate(kind, nx, conv, stretch, r0, r1, rp, ci, v, S(stream)));
}

static int stencil_shape_ok(int dims, int64_t nx, int64_t n) {
  if ((dims != 2 && dims != 3) || nx < 2) return 0;
  return n == (dims == 3 ? nx * nx * nx : nx * nx) && n < (1LL << 32);
}

int mpg_stencil_pack_rows(int prec, int dims, int64_t nx, int64_t row0, int64_t nrows,
                          const int32_t* rp, const int32_t* ci, const void* v, void* dia,
                          int64_t ldv, int32_t* bad, void* stream) {
  const int64_t N = dims == 3 ? nx * nx * nx : nx * nx;
  if (!stencil_shape_ok(dims, nx, N) || row0 < 0 || nrows < 1 || row0 + nrows > N || ldv < nrows ||
      !rp || !dia || !bad)
    return MPG_EARG;
  if (prec == MPG_FP64)
    return rc(launch_stencil_pack<double>(dims, (int)nx, row0, nrows, rp, ci, (const double*)v,
                                          (double*)dia, ldv, bad, S(stream)));
  if (prec == MPG_FP32)
    return rc(launch_stencil_pack<float>(dims, (int)nx, row0, nrows, rp, ci, (const float*)v,
                                         (float*)dia, ldv, bad, S(stream)));
  return MPG_EARG;
}

int mpg_stencil_pack(int prec, int dims, int64_t nx, int64_t n, const int32_t* rp,
                     const int32_t* ci, const void* v, void* dia, int64_t ldv, int32_t* bad,
                     void* stream) {
  if (!stencil_shape_ok(dims, nx, n)) return MPG_EARG;
  return mpg_stencil_pack_rows(prec, dims, nx, 0, n, rp, ci, v, dia, ldv, bad, stream);
}

int mpg_spmv_dia(int prec, int dims, int64_t nx, int64_t n, const void* dia, int64_t ldv,
                 const void* x, void* y, void* ws, void* stream) {
  if (!stencil_shape_ok(dims, nx, n) || ldv < n || !dia || !ws) return MPG_EARG;
  WsView w = make_ws(ws);
  if (prec == MPG_FP64)
    return rc(launch_spmv<double>(StencilView<double>{(const double*)dia, ldv, n, (int)nx, dims, 0},
                                  (const double*)x, (double*)y, w, S(stream)));
  if (prec == MPG_FP32)
    return rc(launch_spmv<float>(StencilView<float>{(const float*)dia, ldv, n, (int)nx, dims, 0},
                                 (const float*)x, (float*)y, w, S(stream)));
  return MPG_EARG;
}

// ------------------------------------------------------------ preconditioners
int mpg_jacobi_apply(int prec, int64_t n, int32_t k, const void* lu, const int64_t* piv,
                     const void* x, void* y, void* stream) {
  if (n < 0 || k < 1 || !lu || (k > 1 && !piv)) return MPG_EARG;
  if (n == 0) return MPG_OK;
  if (prec == MPG_FP64)
    return rc(launch_jacobi<double>(n, k, (const double*)lu, piv, (const double*)x, (double*)y, nullptr, S(stream)));
  if (prec == MPG_FP32)
    return rc(launch_jacobi<float>(n, k, (const float*)lu, piv, (const float*)x, (float*)y, nullptr, S(stream)));
  return MPG_EARG;
}

int mpg_jacobi_build(int prec, int64_t n, int32_t k, const int32_t* rp, const int32_t* ci,
                     const void* v, void* lu, int64_t* piv, int64_t* bad, void* stream) {
  if (n < 1 || k < 1 || !rp || !lu || !piv || !bad) return MPG_EARG;
  if (prec == MPG_FP64)
    return rc(launch_jacobi_build<double>(n, k, rp, ci, (const double*)v, (double*)lu, piv, bad, S(stream)));
  if (prec == MPG_FP32)
    return rc(launch_jacobi_build<float>(n, k, rp, ci, (const float*)v, (float*)lu, piv, bad, S(stream)));
  return MPG_EARG;
}

int mpg_poly_apply(int prec, int64_t n, const int32_t* rp, const int32_t* ci, const void* v,
                   const mpg_poly_op* ops, int32_t nops, const void* x, void* y, void* t0,
                   void* t1, void* t2, void* ws, void* stream) {
  if (n < 1 || !ops || nops < 1 || !ws) return MPG_EARG;
  WsView w = make_ws(ws);
  for (int i = 0; i < nops; ++i) {
    const mpg_poly_op& op = ops[i];
    if (op.src < 0 || op.src > 4 || op.dst < 0 || op.dst > 4 || op.x2 < 0 || op.x2 > 4) return MPG_EARG;
    cudaError_t e;
    if (prec == MPG_FP64) {
      double* b[5] = {(double*)x, (double*)y, (double*)t0, (double*)t1, (double*)t2};
      if (op.op == MPG_POLY_SCALE || op.op == MPG_POLY_ACC || op.op == MPG_POLY_ZERO)
        e = launch_poly_elem<double>(op.op, op.a, b[op.src], b[op.dst], b[1], n, nullptr, S(stream));
      else
        e = launch_poly_op<double>(CsrView<double>{rp, ci, (const double*)v, n}, op, b[0], b[1], b[2],
                                   b[3], b[4], nullptr, n, w, S(stream));
    } else if (prec == MPG_FP32) {
      float* b[5] = {(float*)x, (float*)y, (float*)t0, (float*)t1, (float*)t2};
      if (op.op == MPG_POLY_SCALE || op.op == MPG_POLY_ACC || op.op == MPG_POLY_ZERO)
        e = launch_poly_elem<float>(op.op, (float)op.a, b[op.src], b[op.dst], b[1], n, nullptr, S(stream));
      else
        e = launch_poly_op<float>(CsrView<float>{rp, ci, (const float*)v, n}, op, b[0], b[1], b[2], b[3],
                                  b[4], nullptr, n, w, S(stream));
    } else {
      return MPG_EARG;
    }
    if (e) return rc(e);
  }
  return MPG_OK;
}

// ------------------------------------------------------------ Krylov layer
int64_t mpg_state_bytes(int prec, int32_t m) {
  if (m < 1 || m > kMaxM) return -1;
  return state_layout(prec, m).total;
}

int64_t mpg_state_offset(int prec, int32_t m, int32_t which) {
  StateLayout L = state_layout(prec, m);
  const int64_t offs[10] = {L.H, L.R, L.cs, L.sn, L.g, L.c1, L.c2, L.d, L.implicit, L.red};
  if (which < 0 || which > 9) return -1;
  return offs[which];
}

int mpg_cycle_start(int prec, int64_t n, int64_t ldv, int32_t m, const void* r0, void* V,
                    void* state, double rtol, double b_norm, double btol, int32_t m_limit,
                    void* ws, void* stream) {
  if (n < 1 || ldv < n || m < 1 || m > kMaxM || !ws || !state) return MPG_EARG;
  (void)m_limit;
  WsView w = make_ws(ws);
  mpg_state_header* h = static_cast<mpg_state_header*>(state);
  // b_norm < 0: use gamma; else stash it in the header slot the kernel reads
  const double* bsrc = nullptr;
  if (b_norm >= 0) {
    cudaError_t e = cudaMemcpyAsync(&h->outer_b_norm, &b_norm, sizeof(double), cudaMemcpyHostToDevice, S(stream));
    if (e) return rc(e);
    cudaError_t e2 = cudaStreamSynchronize(S(stream));  // b_norm lives on this host stack
    if (e2) return rc(e2);
    bsrc = &h->outer_b_norm;
  }
  if (prec == MPG_FP64) {
    StateView<double> sv = make_state<double>(state, m);
    cudaError_t e = launch_start<double>((const double*)r0, n, sv, rtol, bsrc, btol, w, S(stream));
    if (e) return rc(e);
    return rc(launch_start_scale<double>((const double*)r0, (double*)V, n, sv, S(stream)));
  }
  if (prec == MPG_FP32) {
    StateView<float> sv = make_state<float>(state, m);
    cudaError_t e = launch_start<float>((const float*)r0, n, sv, rtol, bsrc, btol, w, S(stream));
    if (e) return rc(e);
    return rc(launch_start_scale<float>((const float*)r0, (float*)V, n, sv, S(stream)));
  }
  return MPG_EARG;
}

// Generic-operator Arnoldi step: w = op(V[:,j]) already computed by the
// caller (krylov.py:128).  Pass-1 dots + w0 + finite check, then the fused
// K_B / K_C / K_S kernels.
}  // extern "C"

template <typename T>
static int arnoldi_step_t(int64_t n, int64_t ldv, int32_t m, int32_t j, int32_t m_limit, void* Vp,
                          void* wp, void* state, void* ws, cudaStream_t st) {
  StateView<T> sv = make_state<T>(state, m);
  WsView w = make_ws(ws);
  T* V = static_cast<T*>(Vp);
  T* wv = static_cast<T*>(wp);
  cudaError_t e = launch_dot1_wo<T>(wv, n, V, ldv, j + 1, sv, w, st);
  if (!e) e = launch_update_dot<T>(V, ldv, n, j + 1, wv, sv, w, st);
  if (!e) e = launch_update_norm<T>(V, ldv, n, j, wv, sv, w, m_limit, st);
  if (!e) e = launch_step_scale<T>(wv, V + (size_t)(j + 1) * ldv, n, j, sv, st);
  return rc(e);
}

extern "C" {

int mpg_arnoldi_step(int prec, int64_t n, int64_t ldv, int32_t m, int32_t j, int32_t m_limit,
                     void* V, void* w, void* state, void* ws, void* stream) {
  if (n < 1 || ldv < n || m < 1 || m > kMaxM || j < 0 || j >= m || !V || !w || !state || !ws)
    return MPG_EARG;
  if (prec == MPG_FP64) return arnoldi_step_t<double>(n, ldv, m, j, m_limit, V, w, state, ws, S(stream));
  if (prec == MPG_FP32) return arnoldi_step_t<float>(n, ldv, m, j, m_limit, V, w, state, ws, S(stream));
  return MPG_EARG;
}

int mpg_cycle_finish(int prec, int64_t n, int64_t ldv, int32_t m, const void* V, void* state,
                     void* u, void* stream) {
  if (n < 1 || ldv < n || m < 1 || m > kMaxM || !V || !state || !u) return MPG_EARG;
  cudaError_t e;
  if (prec == MPG_FP64) {
    StateView<double> sv = make_state<double>(state, m);
    e = launch_lsq<double>(sv, S(stream));
    if (!e) e = launch_combine<double>((const double*)V, ldv, n, sv, CMB_STORE, nullptr, nullptr, (double*)u, S(stream));
  } else if (prec == MPG_FP32) {
    StateView<float> sv = make_state<float>(state, m);
    e = launch_lsq<float>(sv, S(stream));
    if (!e) e = launch_combine<float>((const float*)V, ldv, n, sv, CMB_STORE, nullptr, nullptr, (float*)u, S(stream));
  } else {
    return MPG_EARG;
  }
  return rc(e);
}

}  // extern "C"
