// Vector kernels (norm, multivector gemv, casts), block-Jacobi apply/build,
// and the on-device stencil generator.
#include <algorithm>

#include "spmv.cuh"
#include "state.cuh"

namespace mpg {

static unsigned grid_for_rows(long long n, int per_sm = 8, int rows_per_thread = 1) {
  long long g = (n + (long long)kThreads * rows_per_thread - 1) / ((long long)kThreads * rows_per_thread);
  const long long cap = (long long)num_sms() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

__device__ __forceinline__ bool gate_done(const mpg_state_header* h) {
  return h && *(volatile const int*)&h->done != 0;
}

// ============================================================ norm2 (core.py:341-354)
template <typename T>
__global__ void __launch_bounds__(kThreads) k_norm2(const T* __restrict__ x, long long n,
                                                    double* out, WsView ws, int raw) {
  __shared__ T red[32];
  T ss = T(0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const T v = __ldg(x + i);
    ss = fma_rn(v, v, ss);
  }
  const T t = block_sum(ss, red);
  T* part = static_cast<T*>(ws.part);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
  if (last_cta(ws.counter)) {
    T s = T(0);
    for (int p = threadIdx.x; p < (int)gridDim.x; p += blockDim.x) s += __ldcg(part + p);
    s = block_sum(s, red);
    if (threadIdx.x == 0) *out = raw ? (double)s : (double)sqrt_rn(s);   // raw: distributed sum
  }
}

// ======================================================= gemv (core.py:295-338)
// trans: y[c] = alpha * sum_r A[c*lda + r] x[r] + beta * y[c]
template <typename T>
__global__ void __launch_bounds__(kThreads) k_gemv_t(const T* __restrict__ A, long long lda,
                                                     long long rows, int cols,
                                                     const T* __restrict__ x, T* y, T alpha,
                                                     T beta, WsView ws) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long R0, R1;
  cta_rows(rows, R0, R1);
  T* part = static_cast<T*>(ws.part);
  for (int c = warp; c < cols; c += kWarps) {
    T p = T(0);
    for (long long r = R0 + lane; r < R1; r += 32) p = fma_rn(__ldg(A + (size_t)c * lda + r), __ldg(x + r), p);
    p = warp_sum(p);
    if (lane == 0) part[(size_t)blockIdx.x * cols + c] = p;
  }
  if (last_cta(ws.counter)) {
    finalize_columns(part, gridDim.x, cols, cols, [&](int c, T s) {
      T v = mul_rn(alpha, s);
      if (beta != T(0)) v = add_rn(v, mul_rn(beta, y[c]));
      y[c] = v;
    });
  }
}

// no-trans: y[r] = alpha * sum_c A[c*lda + r] x[c] + beta * y[r]
template <typename T>
__global__ void __launch_bounds__(kThreads) k_gemv_n(const T* __restrict__ A, long long lda,
                                                     long long rows, int cols,
                                                     const T* __restrict__ x, T* y, T alpha,
                                                     T beta) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int c = 0; c < cols; ++c) acc = fma_rn(__ldg(A + (size_t)c * lda + r), __ldg(x + c), acc);
    T v = mul_rn(alpha, acc);
    if (beta != T(0)) v = add_rn(v, mul_rn(beta, y[r]));
    y[r] = v;
  }
}

// ==================================================== casts (core.py:252-289)
template <typename TS, typename TD>
__global__ void __launch_bounds__(kThreads) k_convert(const TS* __restrict__ x, TD* __restrict__ y,
                                                      long long n, int64_t* ovf,
                                                      const mpg_state_header* gate) {
  if (gate_done(gate)) return;
  kt_mark(gate, KC_OTHER);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const TS v = x[i];
    const TD o = (TD)v;   // round to nearest even (cvt.rn)
    if (sizeof(TD) < sizeof(TS) && ovf && isinf((double)o) && isfinite((double)v))
      atomicMin(reinterpret_cast<unsigned long long*>(ovf), (unsigned long long)i);
    y[i] = o;
  }
}

// y = x / s with s a device double holding a working-precision value
template <typename T>
__global__ void __launch_bounds__(kThreads) k_scale_div(const T* __restrict__ x,
                                                        const double* s, T* __restrict__ y,
                                                        long long n) {
  const T d = (T)*s;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = div_rn(x[i], d);
}

// x64 += rho * fp64(u32)   (solvers.py:357)
__global__ void __launch_bounds__(kThreads) k_ir_correct(double* x, const float* __restrict__ u,
                                                         const double* rho, long long n,
                                                         const mpg_state_header* gate) {
  if (gate && gate->steps == 0) return;
  const double r = gate ? gate->rho : *rho;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = __dadd_rn(x[i], __dmul_rn(r, (double)u[i]));
}

// end-of-cycle update after a separately applied preconditioner:
// ir 0: x += z   ir 1: x64 += rho * fp64(z)   ir 2: x64 += fp64(z32)
template <typename T, typename TX>
__global__ void __launch_bounds__(kThreads) k_finish_add(TX* x, const T* __restrict__ z,
                                                         long long n, const mpg_state_header* gate,
                                                         int ir) {
  if (gate->steps == 0) return;
  kt_mark(gate, KC_OTHER);
  if (gate->flags & (MPG_FLAG_NONFINITE_OP | MPG_FLAG_NONFINITE_GAMMA | MPG_FLAG_OVERFLOW |
                     MPG_FLAG_SINGULAR))
    return;
  const double rho = gate->rho;
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const T v = z[i];
    if (ir == 1) {
      bad |= !isfinite(v);
      x[i] = (TX)__dadd_rn((double)x[i], __dmul_rn(rho, (double)v));
    } else if (ir == 2) {
      x[i] = (TX)__dadd_rn((double)x[i], (double)v);
    } else {
      x[i] = add_rn(x[i], (TX)v);
    }
  }
  if (bad) atomicOr(const_cast<int*>(&gate->flags), MPG_FLAG_NONFINITE_X);
}

// elementwise polynomial ops (precond.py:286-305): SCALE dst = a*src,
// ACC y = y + a*src, ZERO y = 0
template <typename T>
__global__ void __launch_bounds__(kThreads) k_poly_elem(int op, T a, const T* __restrict__ src,
                                                        T* dst, T* y, long long n,
                                                        const mpg_state_header* gate) {
  if (gate_done(gate)) return;
  kt_mark(gate, KC_OTHER);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (op == MPG_POLY_SCALE) dst[i] = mul_rn(a, src[i]);
    else if (op == MPG_POLY_ACC) y[i] = add_rn(y[i], mul_rn(a, src[i]));
    else y[i] = T(0);
  }
}

// ========================================== block Jacobi (precond.py:326-390)
constexpr int kMaxJacobiBlock = 32;

template <typename T>
__global__ void __launch_bounds__(kThreads) k_jacobi1(const T* __restrict__ d, const T* __restrict__ x,
                                                      T* __restrict__ y, long long n,
                                                      const mpg_state_header* gate) {
  if (gate_done(gate)) return;
  kt_mark(gate, KC_OTHER);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = div_rn(x[i], d[i]);   // xb[:, 0] /= lu[:, 0, 0]
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_jacobi_blocks(const T* __restrict__ lu,
                                                            const int64_t* __restrict__ piv,
                                                            const T* __restrict__ x, T* y,
                                                            long long n, int k,
                                                            const mpg_state_header* gate) {
  if (gate_done(gate)) return;
  kt_mark(gate, KC_OTHER);
  const long long nb = (n + k - 1) / k;
  T xb[kMaxJacobiBlock];
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb;
       b += (long long)gridDim.x * blockDim.x) {
    const T* L = lu + (size_t)b * k * k;
    for (int i = 0; i < k; ++i) {
      const long long r = b * k + i;
      xb[i] = r < n ? x[r] : T(0);
    }
    for (int i = 0; i < k; ++i) {  // row interchanges in factorisation order
      const int j = (int)piv[(size_t)b * k + i];
      const T t = xb[i];
      xb[i] = xb[j];
      xb[j] = t;
    }
    for (int i = 1; i < k; ++i) {  // unit lower forward substitution
      T s = T(0);
      for (int t = 0; t < i; ++t) s = add_rn(s, mul_rn(L[i * k + t], xb[t]));
      xb[i] = sub_rn(xb[i], s);
    }
    for (int i = k - 1; i >= 0; --i) {  // upper backward substitution
      if (i < k - 1) {
        T s = T(0);
        for (int t = i + 1; t < k; ++t) s = add_rn(s, mul_rn(L[i * k + t], xb[t]));
        xb[i] = sub_rn(xb[i], s);
      }
      xb[i] = div_rn(xb[i], L[i * k + i]);
    }
    for (int i = 0; i < k; ++i) {
      const long long r = b * k + i;
      if (r < n) y[r] = xb[i];
    }
  }
}

// Diagonal-block extraction + partially pivoted LU, one thread per block.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_jacobi_build(long long n, int k, const int32_t* rp,
                                                           const int32_t* ci, const T* v, T* lu,
                                                           int64_t* piv, int64_t* bad) {
  const long long nb = (n + k - 1) / k;
  T a[kMaxJacobiBlock * kMaxJacobiBlock];
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb;
       b += (long long)gridDim.x * blockDim.x) {
    const long long base = b * k;
    for (int i = 0; i < k * k; ++i) a[i] = T(0);
    for (int i = 0; i < k; ++i) {
      const long long r = base + i;
      if (r >= n) { a[i * k + i] = T(1); continue; }   // identity padding (precond.py:348-349)
      for (int p = rp[r]; p < rp[r + 1]; ++p) {
        const long long c = ci[p];
        if (c >= base && c < base + k && c < n) a[i * k + (c - base)] = v[p];
      }
    }
    bool singular = false;
    for (int j = 0; j < k; ++j) {
      int p = j;
      T best = fabs(a[j * k + j]);
      for (int i = j + 1; i < k; ++i) {
        const T t = fabs(a[i * k + j]);
        if (t > best) { best = t; p = i; }
      }
      piv[(size_t)b * k + j] = p;
      if (p != j)
        for (int t = 0; t < k; ++t) { const T s = a[j * k + t]; a[j * k + t] = a[p * k + t]; a[p * k + t] = s; }
      const T d = a[j * k + j];
      if (d == T(0) || !isfinite(d)) { singular = true; continue; }
      for (int i = j + 1; i < k; ++i) {
        const T l = div_rn(a[i * k + j], d);
        a[i * k + j] = l;
        for (int t = j + 1; t < k; ++t) a[i * k + t] = sub_rn(a[i * k + t], mul_rn(l, a[j * k + t]));
      }
    }
    if (singular) atomicMin(reinterpret_cast<unsigned long long*>(bad), (unsigned long long)b);
    for (int i = 0; i < k * k; ++i) lu[(size_t)b * k * k + i] = a[i];
  }
}

// ============================================ stencil generator (gen.py:129-202)
struct Off { int dx, dy, dz; };
// offsets in ascending column order for each kind
__constant__ Off c_offs[7][13] = {
    /* laplace2d */ {{0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}},
    /* laplace3d */ {{0, 0, -1}, {0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
    /* convdiff  */ {{0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}},
    /* stretched */ {{0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}},
    /* biharm    */ {{0, -2, 0}, {-1, -1, 0}, {0, -1, 0}, {1, -1, 0}, {-2, 0, 0}, {-1, 0, 0}, {0, 0, 0},
                     {1, 0, 0}, {2, 0, 0}, {-1, 1, 0}, {0, 1, 0}, {1, 1, 0}, {0, 2, 0}},
    /* star2d    */ {{-1, -1, 0}, {0, -1, 0}, {1, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {-1, 1, 0},
                     {0, 1, 0}, {1, 1, 0}},
    /* recirc    */ {{0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}},
};
__constant__ int c_noffs[7] = {5, 7, 5, 5, 13, 9, 5};

__host__ __device__ inline long long clampi(long long v) { return v < 0 ? 0 : v; }
// #{t in [0, T) : 0 <= t + d < nx}
__host__ __device__ inline long long valid_count(long long T, long long d, long long nx) {
  const long long lo = d < 0 ? -d : 0;
  const long long hi = (nx - d < T) ? nx - d : T;
  return clampi(hi - lo);
}
__host__ __device__ inline bool in_grid(long long t, long long d, long long nx) {
  return t + d >= 0 && t + d < nx;
}

// stored entries of offset (dx,dy,dz) over rows [0, r)
__host__ __device__ inline long long off_before(long long r, long long nx, int dx, int dy, int dz,
                                                bool three_d) {
  const long long X = r % nx;
  const long long Y = three_d ? (r / nx) % nx : r / nx;
  const long long Z = three_d ? r / (nx * nx) : 0;
  const long long wx = nx - (dx < 0 ? -dx : dx);
  const long long wy = nx - (dy < 0 ? -dy : dy);
  if (wx <= 0 || wy <= 0) return 0;
  long long cnt = 0;
  if (three_d) {
    cnt += valid_count(Z, dz, nx) * wx * wy;
    if (!in_grid(Z, dz, nx)) return cnt;
  }
  cnt += valid_count(Y, dy, nx) * wx;
  if (!in_grid(Y, dy, nx)) return cnt;
  cnt += valid_count(X, dx, nx);
  return cnt;
}

__device__ double gen_value(int kind, int o, long long ix, long long iy, long long nx,
                            double conv, double stretch) {
  const Off f = c_offs[kind][o];
  const bool center = f.dx == 0 && f.dy == 0 && f.dz == 0;
  switch (kind) {
    case MPG_LAPLACE2D: return center ? 4.0 : -1.0;
    case MPG_LAPLACE3D: return center ? 6.0 : -1.0;
    case MPG_STAR2D: return center ? 8.0 : -1.0;
    case MPG_BIHARMONIC2D: {
      const int ad = abs(f.dx) + abs(f.dy);
      if (center) return 20.0;
      if (abs(f.dx) == 2 || abs(f.dy) == 2) return 1.0;
      return ad == 1 ? -8.0 : 2.0;
    }
    case MPG_STRETCHED2D:
      if (center) return __dadd_rn(2.0, __dmul_rn(2.0, stretch));
      return f.dy != 0 ? -stretch : -1.0;
    default: {  // convdiff2d / recirc2d, coefficients at the row node
      if (center) return 4.0;
      const double h = __ddiv_rn(1.0, (double)(nx + 1));
      const double xh = __dsub_rn(__dmul_rn(2.0 * (double)(ix + 1), h), 1.0);
      const double yh = __dsub_rn(__dmul_rn(2.0 * (double)(iy + 1), h), 1.0);
      double cx, cy;
      if (kind == MPG_CONVDIFF2D) {
        cx = conv;
        cy = 0.0;
      } else {
        cx = __dmul_rn(__dmul_rn(conv * 2.0, yh), __dsub_rn(1.0, __dmul_rn(xh, xh)));
        cy = __dmul_rn(__dmul_rn(-conv * 2.0, xh), __dsub_rn(1.0, __dmul_rn(yh, yh)));
      }
      const double h2 = h / 2.0;
      const double ddx = __dmul_rn(cx, h2), ddy = __dmul_rn(cy, h2);
      if (f.dx == -1) return __dsub_rn(-1.0, ddx);
      if (f.dx == 1) return __dadd_rn(-1.0, ddx);
      if (f.dy == -1) return __dsub_rn(-1.0, ddy);
      return __dadd_rn(-1.0, ddy);
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_generate(int kind, long long nx, double conv,
                                                       double stretch, long long r0, long long r1,
                                                       int32_t* rp, int32_t* ci, double* v) {
  const bool three = kind == MPG_LAPLACE3D;
  const int no = c_noffs[kind];
  long long base0 = 0;
  for (int o = 0; o < no; ++o)
    base0 += off_before(r0, nx, c_offs[kind][o].dx, c_offs[kind][o].dy, c_offs[kind][o].dz, three);
  for (long long r = r0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; r <= r1;
       r += (long long)gridDim.x * blockDim.x) {
    long long pos = -base0;
    for (int o = 0; o < no; ++o)
      pos += off_before(r, nx, c_offs[kind][o].dx, c_offs[kind][o].dy, c_offs[kind][o].dz, three);
    rp[r - r0] = (int32_t)pos;
    if (r == r1) continue;
    const long long ix = r % nx;
    const long long iy = three ? (r / nx) % nx : r / nx;
    const long long iz = three ? r / (nx * nx) : 0;
    for (int o = 0; o < no; ++o) {
      const Off f = c_offs[kind][o];
      if (!in_grid(ix, f.dx, nx) || !in_grid(iy, f.dy, nx) || (three && !in_grid(iz, f.dz, nx)))
        continue;
      ci[pos] = (int32_t)(r + ((long long)f.dz * nx + f.dy) * nx + f.dx);
      v[pos] = gen_value(kind, o, ix, iy, nx, conv, stretch);
      ++pos;
    }
  }
}

// ================================================================= launchers

template <typename T>
cudaError_t launch_norm2(const T* x, long long n, double* out, WsView ws, cudaStream_t st, int raw) {
  count_launch();
  k_norm2<T><<<grid_for_rows(n, 4), kThreads, 0, st>>>(x, n, out, ws, raw);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_gemv_t(const T* A, long long lda, long long rows, int cols, const T* x, T* y,
                          T alpha, T beta, WsView ws, cudaStream_t st) {
  unsigned G = grid_for_rows(rows, 4, 8);
  if ((long long)G * cols > (long long)kMaxParts * (kMaxM + 8)) G = std::max(1, (int)(((long long)kMaxParts * (kMaxM + 8)) / cols));
  count_launch();
  k_gemv_t<T><<<G, kThreads, 0, st>>>(A, lda, rows, cols, x, y, alpha, beta, ws);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_gemv_n(const T* A, long long lda, long long rows, int cols, const T* x, T* y,
                          T alpha, T beta, cudaStream_t st) {
  count_launch();
  k_gemv_n<T><<<grid_for_rows(rows), kThreads, 0, st>>>(A, lda, rows, cols, x, y, alpha, beta);
  return cudaGetLastError();
}

cudaError_t launch_convert(int sp, int dp, long long n, const void* x, void* y, int64_t* ovf,
                           cudaStream_t st) {
  const unsigned G = grid_for_rows(n);
  count_launch();
  if (sp == MPG_FP64 && dp == MPG_FP32)
    k_convert<double, float><<<G, kThreads, 0, st>>>((const double*)x, (float*)y, n, ovf, nullptr);
  else if (sp == MPG_FP32 && dp == MPG_FP64)
    k_convert<float, double><<<G, kThreads, 0, st>>>((const float*)x, (double*)y, n, ovf, nullptr);
  else if (sp == MPG_FP32)
    k_convert<float, float><<<G, kThreads, 0, st>>>((const float*)x, (float*)y, n, ovf, nullptr);
  else
    k_convert<double, double><<<G, kThreads, 0, st>>>((const double*)x, (double*)y, n, ovf, nullptr);
  return cudaGetLastError();
}

template <typename TS, typename TD>
cudaError_t launch_cast_gated(const TS* x, TD* y, long long n, const mpg_state_header* gate,
                              int64_t* ovf, cudaStream_t st) {
  count_launch();
  k_convert<TS, TD><<<grid_for_rows(n), kThreads, 0, st>>>(x, y, n, ovf, gate);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_scale_div(const T* x, const double* s, T* y, long long n, cudaStream_t st) {
  count_launch();
  k_scale_div<T><<<grid_for_rows(n), kThreads, 0, st>>>(x, s, y, n);
  return cudaGetLastError();
}

cudaError_t launch_ir_correct(double* x, const float* u, const double* rho, long long n,
                              const mpg_state_header* gate, cudaStream_t st) {
  count_launch();
  k_ir_correct<<<grid_for_rows(n), kThreads, 0, st>>>(x, u, rho, n, gate);
  return cudaGetLastError();
}

template <typename T, typename TX>
cudaError_t launch_finish_add(TX* x, const T* z, long long n, const mpg_state_header* gate,
                              int ir, cudaStream_t st) {
  count_launch();
  k_finish_add<T, TX><<<grid_for_rows(n), kThreads, 0, st>>>(x, z, n, gate, ir);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_poly_elem(int op, T a, const T* src, T* dst, T* y, long long n,
                             const mpg_state_header* gate, cudaStream_t st) {
  count_launch();
  k_poly_elem<T><<<grid_for_rows(n), kThreads, 0, st>>>(op, a, src, dst, y, n, gate);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_jacobi(long long n, int k, const T* lu, const int64_t* piv, const T* x, T* y,
                          const mpg_state_header* gate, cudaStream_t st) {
  count_launch();
  if (k == 1) {
    k_jacobi1<T><<<grid_for_rows(n), kThreads, 0, st>>>(lu, x, y, n, gate);
  } else {
    if (k > kMaxJacobiBlock) return cudaErrorInvalidValue;
    k_jacobi_blocks<T><<<grid_for_rows((n + k - 1) / k), kThreads, 0, st>>>(lu, piv, x, y, n, k, gate);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_jacobi_build(long long n, int k, const int32_t* rp, const int32_t* ci,
                                const T* v, T* lu, int64_t* piv, int64_t* bad, cudaStream_t st) {
  if (k > kMaxJacobiBlock) return cudaErrorInvalidValue;
  count_launch();
  k_jacobi_build<T><<<grid_for_rows((n + k - 1) / k), kThreads, 0, st>>>(n, k, rp, ci, v, lu, piv, bad);
  return cudaGetLastError();
}

cudaError_t launch_generate(int kind, long long nx, double conv, double stretch, long long r0,
                            long long r1, int32_t* rp, int32_t* ci, double* v, cudaStream_t st) {
  count_launch();
  k_generate<<<grid_for_rows(r1 - r0 + 1), kThreads, 0, st>>>(kind, nx, conv, stretch, r0, r1, rp, ci, v);
  return cudaGetLastError();
}

// host-side counts (gen.py:111-126) — same closed forms as the device
long long host_nnz_before(int kind, long long nx, long long r) {
  static const int offs[7][13][3] = {
      {{0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}},
      {{0, 0, -1}, {0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
      {{0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}},
      {{0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}},
      {{0, -2, 0}, {-1, -1, 0}, {0, -1, 0}, {1, -1, 0}, {-2, 0, 0}, {-1, 0, 0}, {0, 0, 0},
       {1, 0, 0}, {2, 0, 0}, {-1, 1, 0}, {0, 1, 0}, {1, 1, 0}, {0, 2, 0}},
      {{-1, -1, 0}, {0, -1, 0}, {1, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {-1, 1, 0},
       {0, 1, 0}, {1, 1, 0}},
      {{0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}},
  };
  static const int noffs[7] = {5, 7, 5, 5, 13, 9, 5};
  long long s = 0;
  for (int o = 0; o < noffs[kind]; ++o)
    s += off_before(r, nx, offs[kind][o][0], offs[kind][o][1], offs[kind][o][2], kind == MPG_LAPLACE3D);
  return s;
}

#define INST(T)                                                                                  \
  template cudaError_t launch_norm2<T>(const T*, long long, double*, WsView, cudaStream_t, int); \
  template cudaError_t launch_gemv_t<T>(const T*, long long, long long, int, const T*, T*, T, T, \
                                        WsView, cudaStream_t);                                 \
  template cudaError_t launch_gemv_n<T>(const T*, long long, long long, int, const T*, T*, T, T, \
                                        cudaStream_t);                                         \
  template cudaError_t launch_scale_div<T>(const T*, const double*, T*, long long, cudaStream_t); \
  template cudaError_t launch_poly_elem<T>(int, T, const T*, T*, T*, long long,                   \
                                           const mpg_state_header*, cudaStream_t);             \
  template cudaError_t launch_jacobi<T>(long long, int, const T*, const int64_t*, const T*, T*,  \
                                        const mpg_state_header*, cudaStream_t);                \
  template cudaError_t launch_jacobi_build<T>(long long, int, const int32_t*, const int32_t*,   \
                                              const T*, T*, int64_t*, int64_t*, cudaStream_t);
INST(float)
INST(double)
#undef INST
template cudaError_t launch_finish_add<float, float>(float*, const float*, long long,
                                                     const mpg_state_header*, int, cudaStream_t);
template cudaError_t launch_finish_add<double, double>(double*, const double*, long long,
                                                       const mpg_state_header*, int, cudaStream_t);
template cudaError_t launch_finish_add<float, double>(double*, const float*, long long,
                                                      const mpg_state_header*, int, cudaStream_t);
template cudaError_t launch_cast_gated<double, float>(const double*, float*, long long,
                                                      const mpg_state_header*, int64_t*, cudaStream_t);
template cudaError_t launch_cast_gated<float, double>(const float*, double*, long long,
                                                      const mpg_state_header*, int64_t*, cudaStream_t);

}  // namespace mpg
