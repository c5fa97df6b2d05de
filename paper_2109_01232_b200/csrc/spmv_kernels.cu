// SpMV-family kernels: plain SpMV, explicit residual, the fused
// SpMV + first CGS pass (K_A), and the polynomial-preconditioner steps.
// All share spmv_pipeline (spmv.cuh); they differ only in the epilogue.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "spmv.cuh"
#include "state.cuh"

namespace mpg {

// MPG_CSR_TMA=1 selects the TMA-ring CSR kernel for every epilogue (A/B)
static bool csr_warp_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MPG_CSR_TMA");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

// Consumer-only last-CTA election (the producer warp has exited).
__device__ __forceinline__ bool consumers_last_cta(unsigned int* counter, bool* flag) {
  __threadfence();
  consumer_sync();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(counter, 1u);
    *flag = (t == gridDim.x - 1);
  }
  consumer_sync();
  const bool last = *flag;
  if (last) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0u;
  }
  return last;
}

// Sum columns of partials, consumer warps only.
template <typename T, typename OutF>
__device__ __forceinline__ void consumers_finalize(const T* part, int nparts, int stride,
                                                   int ncols, OutF out) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int c = w; c < ncols; c += kSpConsumerWarps) {
    T s = T(0);
    for (int p = l; p < nparts; p += 32) s += __ldcg(part + (size_t)p * stride + c);
    s = warp_sum(s);
    if (l == 0) out(c, s);
  }
}

// ---------------------------------------------------------------- epilogues

template <typename T>
struct EpiPlain {
  static constexpr bool kPdl = true;   // the Arnoldi-step SpMV (split K_A)
  static constexpr bool kOrderFree = true;
  const mpg_state_header* kt = nullptr;   // kernel-time stamp target (null: untimed)
  int kcat = KC_SPMV;
  __device__ void mark() const { kt_mark(kt, kcat); }
  T* y;
  __device__ bool skip() const { return false; }
  __device__ void init(EpiShared<T>&, unsigned char*) {}
  __device__ T on_row(long long r, T v) { y[r] = v; return v; }
  static constexpr bool kVecRows = true;
  __device__ void on_rows(long long r0, T (&v)[Vec<T>::n], int cnt, T*) {
    if (cnt == Vec<T>::n) vstore(y + r0, v);
    else for (int e = 0; e < cnt; ++e) y[r0 + e] = v[e];
  }
  __device__ void on_tile(long long, int, const T*) {}
  __device__ void on_end() {}
};

// explicit_residual (solvers.py:443-453): r = b - A x, ||r||
template <typename T>
struct EpiResid {
  static constexpr bool kPdl = false;
  const mpg_state_header* kt = nullptr;   // kernel-time stamp target (null: untimed)
  int kcat = KC_SPMV;
  __device__ void mark() const { kt_mark(kt, kcat); }
  const T* b;
  T* r;
  double* out;
  mpg_state_header* hdr;
  T* part;
  unsigned int* counter;
  int raw;
  T ss;
  EpiShared<T>* sm;
  __device__ bool skip() const { return false; }
  __device__ void init(EpiShared<T>& s, unsigned char*) { sm = &s; ss = T(0); }
  __device__ T on_row(long long i, T y) {
    const T v = sub_rn(__ldg(b + i), y);
    r[i] = v;
    ss = fma_rn(v, v, ss);
    return v;
  }
  __device__ void on_tile(long long, int, const T*) {}
  __device__ void on_end() {
    T t = consumer_block_sum(ss, sm->red);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
    __shared__ bool flag;
    if (consumers_last_cta(counter, &flag)) {
      consumers_finalize(part, gridDim.x, 1, 1, [&](int, T s) {
        if (raw) {                  // distributed: local sum of squares, finished after the allreduce
          hdr->reserved[0] = (double)s;
          return;
        }
        const double nr = (double)sqrt_rn(s);
        if (out) *out = nr;
        if (hdr) hdr->rnorm = nr;
      });
    }
  }
};

// K_A: w = A x; w0 = ||w||; finite check; c1 = V[:, :k]^T w  (krylov.py:128-139)
template <typename T>
struct EpiDot1 {
  static constexpr bool kPdl = false;
  const mpg_state_header* kt = nullptr;   // kernel-time stamp target (null: untimed)
  int kcat = KC_SPMV;
  __device__ void mark() const { kt_mark(kt, kcat); }
  static constexpr bool kNeedsTiles = true;
  T* w;
  const T* V;
  long long ldv;
  int k;
  StateView<T> sv;
  T* part;
  unsigned int* counter;
  T ss;
  int bad;
  T* acc;
  EpiShared<T>* sm;
  __device__ bool skip() const { return *(volatile int*)&sv.h->done != 0; }
  __device__ void init(EpiShared<T>& s, unsigned char* extra) {
    sm = &s;
    acc = reinterpret_cast<T*>(extra);
    for (int i = threadIdx.x; i < k; i += blockDim.x) acc[i] = T(0);
    ss = T(0);
    bad = 0;
  }
  __device__ T on_row(long long i, T y) {
    w[i] = y;
    ss = fma_rn(y, y, ss);
    bad |= !isfinite(y);
    return y;
  }
  __device__ void on_tile(long long a, int nr, const T* ys) {
    auto vrow = [&](int i) { return V + (size_t)i * ldv + a; };
    tile_dots<T, kLoadStream>(k, nr, vrow, ys, acc, sm->acc);
  }
  __device__ void on_end() {
    T t = consumer_block_sum(ss, sm->red);
    const int stride = k + 2;
    // publish partials: acc[0..k), ||w||^2, non-finite count
    consumer_sync();
    for (int i = threadIdx.x; i < k; i += kSpConsumers) part[(size_t)blockIdx.x * stride + i] = acc[i];
    const int anybad = __any_sync(0xffffffffu, bad);
    __shared__ int badw[kSpConsumerWarps];
    if ((threadIdx.x & 31) == 0) badw[threadIdx.x >> 5] = anybad;
    consumer_sync();
    if (threadIdx.x == 0) {
      int b = 0;
      for (int i = 0; i < kSpConsumerWarps; ++i) b |= badw[i];
      part[(size_t)blockIdx.x * stride + k] = t;
      part[(size_t)blockIdx.x * stride + k + 1] = b ? T(1) : T(0);
    }
    __shared__ bool flag;
    if (consumers_last_cta(counter, &flag)) {
      consumers_finalize(part, gridDim.x, stride, k + 2, [&](int c, T s) {
        if (sv.dist) {
          sv.red[c] = s;
        } else if (c < k) {
          sv.c1[c] = s;
        } else if (c == k) {
          sv.h->w0 = (double)sqrt_rn(s);
        } else if (s != T(0)) {
          sv.h->flags |= MPG_FLAG_NONFINITE_OP;
          sv.h->done = 1;
        }
      });
    }
  }
};

// K_A, warp-owned-vector variant (k <= 8*KV): consumer warp w owns basis
// vectors i = w + 8q.  After a tile's w is in shared memory, each lane streams
// one 16-byte slice per owned vector per 32*VN-row group (a warp-wide load
// = 512 contiguous bytes of one vector) into KV per-lane accumulators.
template <typename T, int KV>
struct EpiDot1Warp {
  static constexpr bool kPdl = false;
  const mpg_state_header* kt = nullptr;   // kernel-time stamp target (null: untimed)
  int kcat = KC_SPMV;
  __device__ void mark() const { kt_mark(kt, kcat); }
  static constexpr bool kNeedsTiles = true;
  static constexpr int VN = 16 / (int)sizeof(T);
  static constexpr int RB = 32 * VN;
  T* w;
  const T* V;
  long long ldv;
  int k;
  StateView<T> sv;
  T* part;
  unsigned int* counter;
  T ss;
  int bad;
  T acc[KV];
  EpiShared<T>* sm;
  __device__ bool skip() const { return *(volatile int*)&sv.h->done != 0; }
  __device__ void init(EpiShared<T>& s, unsigned char*) {
    sm = &s;
#pragma unroll
    for (int q = 0; q < KV; ++q) acc[q] = T(0);
    ss = T(0);
    bad = 0;
  }
  __device__ T on_row(long long r, T y) {
    w[r] = y;
    ss = fma_rn(y, y, ss);
    bad |= !isfinite(y);
    return y;
  }
  // one 16-byte row group (vectorised stencil loop)
  static constexpr bool kVecRows = true;
  __device__ void on_rows(long long r0, T (&y)[VN], int cnt, T* ysp) {
    if (cnt == VN) {
      vstore(w + r0, y);
      vstore(ysp, y);
#pragma unroll
      for (int e = 0; e < VN; ++e) {
        ss = fma_rn(y[e], y[e], ss);
        bad |= !isfinite(y[e]);
      }
    } else {
      for (int e = 0; e < cnt; ++e) ysp[e] = on_row(r0 + e, y[e]);
    }
  }
  __device__ void on_tile(long long a, int nr, const T* ys) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int g = 0; g < kStTileMax / RB; ++g) {
      const int r0 = g * RB + lane * VN;
      if (r0 + VN <= nr) {
        T y[VN];
        vload_smem(ys + r0, y);
#pragma unroll
        for (int q = 0; q < KV; ++q) {
          const int i = warp + kSpConsumerWarps * q;
          if (i < k) {
            T v[VN];
            vload_cs(V + (size_t)i * ldv + a + r0, v);
            T s = acc[q];
#pragma unroll
            for (int e = 0; e < VN; ++e) s = fma_rn(v[e], y[e], s);
            acc[q] = s;
          }
        }
      } else if (r0 < nr) {
        for (int e = 0; r0 + e < nr; ++e) {
          const T ye = ys[r0 + e];
#pragma unroll
          for (int q = 0; q < KV; ++q) {
            const int i = warp + kSpConsumerWarps * q;
            if (i < k) acc[q] = fma_rn(__ldcs(V + (size_t)i * ldv + a + r0 + e), ye, acc[q]);
          }
        }
      }
    }
  }
  __device__ void on_end() {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T t = consumer_block_sum(ss, sm->red);
    const int stride = k + 2;
#pragma unroll
    for (int q = 0; q < KV; ++q) {
      const int i = warp + kSpConsumerWarps * q;
      const T v = warp_sum(acc[q]);
      if (lane == 0 && i < k) part[(size_t)blockIdx.x * stride + i] = v;
    }
    const int anybad = __any_sync(0xffffffffu, bad);
    __shared__ int badw[kSpConsumerWarps];
    if (lane == 0) badw[warp] = anybad;
    consumer_sync();
    if (threadIdx.x == 0) {
      int b = 0;
      for (int i = 0; i < kSpConsumerWarps; ++i) b |= badw[i];
      part[(size_t)blockIdx.x * stride + k] = t;
      part[(size_t)blockIdx.x * stride + k + 1] = b ? T(1) : T(0);
    }
    __shared__ bool flag;
    if (consumers_last_cta(counter, &flag)) {
      consumers_finalize(part, gridDim.x, stride, k + 2, [&](int c, T s) {
        if (sv.dist) {              // raw local sums; k_dist_post finishes after the allreduce
          sv.red[c] = s;
        } else if (c < k) {
          sv.c1[c] = s;
        } else if (c == k) {
          sv.h->w0 = (double)sqrt_rn(s);
        } else if (s != T(0)) {
          sv.h->flags |= MPG_FLAG_NONFINITE_OP;
          sv.h->done = 1;
        }
      });
    }
  }
};

// polynomial preconditioner steps (precond.py:272-319); the SpMV input is
// `x` of the pipeline; other operands are own-row elementwise.
template <typename T>
struct EpiPoly {
  static constexpr bool kPdl = false;
  static constexpr bool kOrderFree = true;
  const mpg_state_header* kt = nullptr;   // kernel-time stamp target (null: untimed)
  int kcat = KC_SPMV;
  __device__ void mark() const { kt_mark(kt, kcat); }
  int op;
  T a, b;
  const T* src;   // SpMV input (also own-row operand)
  const T* x2;    // second operand (x for HORNER, p for PAIR2)
  T* dst;
  T* y;           // accumulator (NEWTON_REAL, PAIR1)
  const mpg_state_header* gate;
  __device__ bool skip() const { return gate && *(volatile const int*)&gate->done != 0; }
  __device__ void init(EpiShared<T>&, unsigned char*) {}
  __device__ T on_row(long long i, T v) {
    switch (op) {
      case MPG_POLY_HORNER: {  // y = spmv(A, y); y += c[i] * x
        const T o = add_rn(v, mul_rn(a, x2[i]));
        dst[i] = o;
        return o;
      }
      case MPG_POLY_NEWTON_REAL: {  // y += inv * prod ; prod = prod - inv * A prod
        const T p = src[i];
        y[i] = add_rn(y[i], mul_rn(a, p));
        const T o = sub_rn(p, mul_rn(a, v));
        dst[i] = o;
        return o;
      }
      case MPG_POLY_PAIR1: {  // ap = A prod ; y += a*prod - b*ap
        const T p = src[i];
        y[i] = add_rn(y[i], sub_rn(mul_rn(a, p), mul_rn(b, v)));
        dst[i] = v;
        return v;
      }
      case MPG_POLY_PAIR2: {  // prod = prod - a*ap + b*(A ap)
        const T o = add_rn(sub_rn(x2[i], mul_rn(a, src[i])), mul_rn(b, v));
        dst[i] = o;
        return o;
      }
      default:
        dst[i] = v;
        return v;
    }
  }
  // one 16-byte row group (vectorised stencil loop): the same per-row
  // arithmetic with 16-byte loads/stores of the own-row operands
  static constexpr int VN = Vec<T>::n;
  static constexpr bool kVecRows = true;
  __device__ void on_rows(long long r0, T (&v)[VN], int cnt, T*) {
    if (cnt != VN) {
      for (int e = 0; e < cnt; ++e) on_row(r0 + e, v[e]);
      return;
    }
    T o[VN];
    switch (op) {
      case MPG_POLY_HORNER: {
        T xx[VN];
        vload(x2 + r0, xx);
#pragma unroll
        for (int e = 0; e < VN; ++e) o[e] = add_rn(v[e], mul_rn(a, xx[e]));
        break;
      }
      case MPG_POLY_NEWTON_REAL: {
        T p[VN], yy[VN];
        vload(src + r0, p);
        vload_smem(y + r0, yy);   // plain load: y is read and written by this thread only
#pragma unroll
        for (int e = 0; e < VN; ++e) {
          yy[e] = add_rn(yy[e], mul_rn(a, p[e]));
          o[e] = sub_rn(p[e], mul_rn(a, v[e]));
        }
        vstore(y + r0, yy);
        break;
      }
      case MPG_POLY_PAIR1: {
        T p[VN], yy[VN];
        vload(src + r0, p);
        vload_smem(y + r0, yy);
#pragma unroll
        for (int e = 0; e < VN; ++e) {
          yy[e] = add_rn(yy[e], sub_rn(mul_rn(a, p[e]), mul_rn(b, v[e])));
          o[e] = v[e];
        }
        vstore(y + r0, yy);
        break;
      }
      case MPG_POLY_PAIR2: {
        T p[VN], xx[VN];
        vload(src + r0, p);
        vload(x2 + r0, xx);
#pragma unroll
        for (int e = 0; e < VN; ++e) o[e] = add_rn(sub_rn(xx[e], mul_rn(a, p[e])), mul_rn(b, v[e]));
        break;
      }
      default:
#pragma unroll
        for (int e = 0; e < VN; ++e) o[e] = v[e];
    }
    vstore(dst + r0, o);
  }
  __device__ void on_tile(long long, int, const T*) {}
  __device__ void on_end() {}
};

template <typename T, typename E>
__global__ void __launch_bounds__(kSpThreads) k_spmv(CsrView<T> A, const T* __restrict__ x, E epi) {
  extern __shared__ __align__(128) unsigned char smraw[];
  pdl_wait();
  pdl_trigger();
  if (epi.skip()) return;
  epi.mark();
  SpSmem<T>& sm = *reinterpret_cast<SpSmem<T>*>(smraw);
  epi.init(sm.es, smraw + sizeof(SpSmem<T>));
  spmv_pipeline(A, x, epi, sm);
}

// stencil kernels: CTAs per SM the register budget must allow.  fp32 streaming
// epilogues (SpMV, residual, polynomial steps): 4 (<= 64 registers; measured
// at 400^3: SpMV 189 -> 134 us, cfg4 IR + poly(25) 0.207 -> 0.165 s); fp64: 2
// (<= 128 registers, no spills); the fused-dot epilogues keep the compiler's
// choice.  MPG_ST_MINB32 / MPG_ST_MINB64 override (A/B).
#ifndef MPG_ST_MINB32
#define MPG_ST_MINB32 4
#endif
#ifndef MPG_ST_MINB64
#define MPG_ST_MINB64 2
#endif
template <typename T, typename E>
constexpr int st_minb() {
  return needs_tiles<E>::value ? 1 : (sizeof(T) == 4 ? MPG_ST_MINB32 : MPG_ST_MINB64);
}
template <typename T, typename E, bool ALN>
__global__ void __launch_bounds__(kSpConsumers, st_minb<T, E>()) k_stencil(StencilView<T> S, const T* __restrict__ x,
                                                          E epi) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ EpiShared<T> es;
  pdl_wait();
  pdl_trigger();
  if (epi.skip()) return;
  epi.mark();
  epi.init(es, smraw);
  stencil_pipeline<T, E, ALN>(S, x, epi, es);
}

// ------------------------------------------------------------------------
// CSR SpMV, warp-chunk design (the default for epilogues without a per-tile
// hook): each warp owns chunks of 32 consecutive rows dealt round-robin over
// every warp of the grid.  The chunk's nonzeros are one contiguous range of
// col_idx / values, which the warp copies into its own shared-memory slice
// with per-lane cp.async (LDGSTS, no register staging); lane l then reduces
// row l from shared memory in the reference's add.reduceat order, gathering
// x through the read-only path -- rows of <= 8 entries issue all their x
// gathers at once.  Software pipeline, per warp: while chunk c is reduced,
// chunk c+1's nonzeros are in flight into the other slice and chunk c+2's
// row_ptr entries are in registers, so the dependent chain row_ptr -> values
// -> x costs one exposed latency per chunk instead of three.  A chunk with
// more than csr_cap() nonzeros (long rows) is reduced straight from global
// memory.  No CTA-wide barrier, no producer warp.
constexpr int kCsrThreads = 256;
constexpr int kCsrWarps = kCsrThreads / 32;
#ifndef MPG_CSR_CAP
#define MPG_CSR_CAP 256
#endif
#ifndef MPG_CSR_MINB
#define MPG_CSR_MINB 4
#endif
#ifndef MPG_CSR_SHORT
#define MPG_CSR_SHORT 1   // A/B: 0 = one dependent gather per product
#endif
// rows per lane: a warp chunk is 32 * RPL consecutive rows (lane l owns rows
// l, l + 32, ...), so the per-chunk bookkeeping (row_ptr shuffles, staging
// loop, loop control) is amortised over RPL rows and every lane has RPL rows'
// x gathers in flight
#ifndef MPG_CSR_RPL32
#define MPG_CSR_RPL32 1
#endif
#ifndef MPG_CSR_RPL64
#define MPG_CSR_RPL64 1
#endif
template <typename T>
constexpr int csr_rpl() { return sizeof(T) == 8 ? MPG_CSR_RPL64 : MPG_CSR_RPL32; }
constexpr int kCsrShort = 8;           // rows up to this length gather all of x before summing
// slices per warp = pipeline depth (chunks in flight + the one being reduced).
// 2 (measured: 3 slices in fp32 / fp64 ran 2-3 % / 25 % slower -- the extra
// slice costs occupancy and the chain is bound by the x gathers, not staging;
// issuing the next chunk's x gathers a whole iteration ahead was 4 % slower)
constexpr int kCsrBufs = 2;
template <typename T>
constexpr int csr_cap() { return MPG_CSR_CAP * csr_rpl<T>(); }   // staged nonzeros per chunk and slice
// staging engine: per-warp TMA bulk copies (one cp.async.bulk per array and
// chunk, completion on a per-slice mbarrier) or per-lane cp.async (LDGSTS)
#ifndef MPG_CSR_BULK
#define MPG_CSR_BULK 1
#endif
// slice length: the bulk copies move the 16-byte-aligned superset of the
// chunk's range (at most 3 extra elements at each end)
template <typename T>
constexpr int csr_slice() { return csr_cap<T>() + (MPG_CSR_BULK ? 8 : 0); }
template <typename T>
constexpr size_t csr_smem_bytes() { return (size_t)kCsrBufs * kCsrWarps * csr_slice<T>() * (sizeof(T) + 4); }

template <int R>
struct CsrChunk {
  int lo[R], hi[R];   // this lane's row ranges
  int s, e;           // the chunk's nonzero range (warp-uniform)
};
// row_ptr entries of chunk c, as loaded (rows past n clamp to row_ptr[n]: an
// empty chunk).  csr_chunk() shuffles them into the lane's row ranges only
// when the chunk is staged, one iteration later, so the loads are a real
// prefetch.
template <int R>
struct CsrRaw {
  int q[R], qe;
};
template <int R>
__device__ __forceinline__ CsrRaw<R> csr_load(const int32_t* __restrict__ rp, long long n, long long c,
                                              int lane) {
  const long long r0 = c * 32 * R;
  CsrRaw<R> w;
#pragma unroll
  for (int j = 0; j < R; ++j) w.q[j] = __ldg(rp + min(r0 + 32 * j + lane, n));
  w.qe = __ldg(rp + min(r0 + 32 * R, n));
  return w;
}
template <int R>
__device__ __forceinline__ CsrChunk<R> csr_chunk(const CsrRaw<R>& w, int lane) {
  CsrChunk<R> k;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int nxt = __shfl_down_sync(0xffffffffu, w.q[j], 1);
    const int first_next = j + 1 < R ? __shfl_sync(0xffffffffu, w.q[j + 1 < R ? j + 1 : j], 0) : w.qe;
    k.lo[j] = w.q[j];
    k.hi[j] = lane < 31 ? nxt : first_next;
  }
  k.s = __shfl_sync(0xffffffffu, w.q[0], 0);
  k.e = w.qe;
  return k;
}

template <typename T, int R>
__device__ __forceinline__ void csr_stage(const CsrView<T>& A, const CsrChunk<R>& k, T* v_s, int32_t* ci_s,
                                          int lane, uint64_t* bar) {
  constexpr int cap = csr_cap<T>();
  const int cnt = k.e - k.s;
  if constexpr (MPG_CSR_BULK) {
    // lane 0: two bulk copies of the aligned supersets (the C ABI guarantees
    // 16-byte-aligned arrays with 16 readable bytes past their end)
    if (lane == 0) {
      if (cnt > 0 && cnt <= cap) {
        constexpr int VE = 16 / (int)sizeof(T);
        const int s4 = k.s & ~3, e4 = (k.e + 3) & ~3;
        const int sv = k.s & ~(VE - 1), ev = (k.e + VE - 1) & ~(VE - 1);
        const uint32_t bc = (uint32_t)(e4 - s4) * 4u, bv = (uint32_t)(ev - sv) * (uint32_t)sizeof(T);
        fence_proxy_async();   // this warp's generic reads of the slice precede the async writes
        mbar_expect_tx(bar, bc + bv);
        bulk_g2s(ci_s, A.ci + s4, bc, bar);
        bulk_g2s(v_s, A.v + sv, bv, bar);
      } else {
        mbar_arrive(bar);      // nothing to stage: complete the phase
      }
    }
  } else {
    if (cnt <= cap) {
#pragma unroll
      for (int it = 0; it < cap / 32; ++it) {
        const int i = lane + 32 * it;
        if (i < cnt) {
          cp_async_ca<4>(ci_s + i, A.ci + k.s + i);
          cp_async_ca<(int)sizeof(T)>(v_s + i, A.v + k.s + i);
        }
      }
    }
    cp_async_commit();   // one group per chunk, empty for long-row or past-the-end chunks
  }
}

template <typename T, typename E>
__global__ void __launch_bounds__(kCsrThreads, MPG_CSR_MINB) k_csr_warp(CsrView<T> A, const T* __restrict__ x, E epi) {
  constexpr int R = csr_rpl<T>();
  constexpr int cap = csr_cap<T>();
  extern __shared__ __align__(16) unsigned char csr_smem[];   // [bufs][warps][cap] T, then int32
  __shared__ EpiShared<T> es;
  pdl_wait();
  pdl_trigger();
  if (epi.skip()) return;
  epi.mark();
  epi.init(es, nullptr);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long n = A.n;
  const long long nchunks = (n + 32 * R - 1) / (32 * R);
  const long long gw = (long long)blockIdx.x * kCsrWarps + warp;
  const long long nw = (long long)gridDim.x * kCsrWarps;
  constexpr int SL = csr_slice<T>();
  T* vbase = reinterpret_cast<T*>(csr_smem);
  int32_t* cbase = reinterpret_cast<int32_t*>(csr_smem + sizeof(T) * kCsrBufs * kCsrWarps * SL);
  auto vslice = [&](int b) { return vbase + ((size_t)b * kCsrWarps + warp) * SL; };
  auto cslice = [&](int b) { return cbase + ((size_t)b * kCsrWarps + warp) * SL; };
  __shared__ uint64_t bars[kCsrWarps][kCsrBufs];
  if (MPG_CSR_BULK && lane == 0) {
    mbar_init(&bars[warp][0], 1);
    mbar_init(&bars[warp][1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  // where element i of the chunk's range landed in a slice
  constexpr int VE = MPG_CSR_BULK ? 16 / (int)sizeof(T) : 1;
  constexpr int CE = MPG_CSR_BULK ? 4 : 1;
  if (gw < nchunks) {
    // cur: chunk c (in flight); nxt: chunk c + nw (staged at the top of the
    // iteration); raw: row_ptr loads of chunk c + 2 nw
    CsrChunk<R> cur = csr_chunk<R>(csr_load<R>(A.rp, n, gw, lane), lane);
    csr_stage<T, R>(A, cur, vslice(0), cslice(0), lane, &bars[warp][0]);
    CsrRaw<R> raw = csr_load<R>(A.rp, n, gw + nw, lane);
    int buf = 0;
    uint32_t ph = 0;   // bit b: parity of slice b's next completion
    for (long long c = gw; c < nchunks; c += nw) {
      __syncwarp();   // every lane is done reading the other slice (chunk c - nw)
      const CsrChunk<R> nxt = csr_chunk<R>(raw, lane);
      csr_stage<T, R>(A, nxt, vslice(buf ^ 1), cslice(buf ^ 1), lane, &bars[warp][buf ^ 1]);
      raw = csr_load<R>(A.rp, n, c + 2 * nw, lane);
      if constexpr (MPG_CSR_BULK) {
        mbar_wait(&bars[warp][buf], (ph >> buf) & 1u);   // chunk c's copies landed
        ph ^= 1u << buf;
      } else {
        cp_async_wait<1>();   // chunk c's group; chunk c + nw's may still fly
        __syncwarp();
      }
      const bool staged = cur.e - cur.s <= cap;
      const int cofs = cur.s & ~(CE - 1), vofs = cur.s & ~(VE - 1);
      T y[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int len = cur.hi[j] - cur.lo[j];
        if (staged && MPG_CSR_SHORT && len <= kCsrShort) {
          // all of the row's x gathers in flight at once (predicated), then the
          // reference's order p0 + (((p1 + p2) + p3) ...) (row_reduce, len <= 8)
          const int32_t* cs = cslice(buf) + (cur.lo[j] - cofs);
          const T* vs = vslice(buf) + (cur.lo[j] - vofs);
          T p[kCsrShort];
#pragma unroll
          for (int i = 0; i < kCsrShort; ++i) p[i] = i < len ? mul_rn(vs[i], __ldg(x + cs[i])) : T(0);
          y[j] = row_sum_short<T, kCsrShort>(p, len);
        } else if (staged) {
          const int32_t* cs = cslice(buf) + (cur.lo[j] - cofs);
          const T* vs = vslice(buf) + (cur.lo[j] - vofs);
          auto get = [&](int i) -> T { return mul_rn(vs[i], __ldg(x + cs[i])); };
          y[j] = row_reduce<T>(get, len);
        } else {
          const int32_t* cg = A.ci + cur.lo[j];
          const T* vg = A.v + cur.lo[j];
          auto get = [&](int i) -> T { return mul_rn(__ldg(vg + i), __ldg(x + __ldg(cg + i))); };
          y[j] = row_reduce<T>(get, len);
        }
      }
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const long long r = c * 32 * R + 32 * j + lane;
        if (r < n) epi.on_row(r, y[j]);
      }
      cur = nxt;
      buf ^= 1;
    }
    if constexpr (MPG_CSR_BULK) {
      mbar_wait(&bars[warp][buf], (ph >> buf) & 1u);   // the last (empty) stage before exit
    } else {
      cp_async_wait<0>();
    }
  }
  epi.on_end();
}

// DIA packing + pattern check: one thread per row.  *bad != 0 when the CSR
// pattern is not exactly the Dirichlet 5/7-point stencil of the grid.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_stencil_pack(int dims, int nx, long long row0, long long n,
                                                           const int32_t* __restrict__ rp,
                                                           const int32_t* __restrict__ ci,
                                                           const T* __restrict__ v, T* out,
                                                           long long ldv, int* bad) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
       r += (long long)gridDim.x * blockDim.x) {
    const long long rg = r + row0;   // global row (row_ptr local, col_idx global)
    const unsigned unx = (unsigned)nx, ur = (unsigned)rg;
    const unsigned ix = ur % unx, q = ur / unx;
    bool pres[7];
    long long off[7];
    int S;
    if (dims == 3) {
      const unsigned iy = q % unx, iz = q / unx;
      const long long p2 = (long long)nx * nx;
      S = 7;
      pres[0] = iz > 0; off[0] = -p2;
      pres[1] = iy > 0; off[1] = -(long long)nx;
      pres[2] = ix > 0; off[2] = -1;
      pres[3] = true; off[3] = 0;
      pres[4] = ix + 1 < unx; off[4] = 1;
      pres[5] = iy + 1 < unx; off[5] = nx;
      pres[6] = iz + 1 < unx; off[6] = p2;
    } else {
      S = 5;
      pres[0] = q > 0; off[0] = -(long long)nx;
      pres[1] = ix > 0; off[1] = -1;
      pres[2] = true; off[2] = 0;
      pres[3] = ix + 1 < unx; off[3] = 1;
      pres[4] = q + 1 < unx; off[4] = nx;
    }
    int p = rp[r];
    const int e = rp[r + 1];
    int ok = 1;
    for (int sl = 0; sl < S; ++sl) {
      T val = absent_value<T>();   // sentinel for neighbours outside the grid
      if (pres[sl]) {
        if (p < e && (long long)ci[p] == rg + off[sl]) val = v[p++];
        else ok = 0;
      }
      out[(size_t)sl * ldv + r] = val;
    }
    if (p != e) ok = 0;
    if (!ok) atomicOr(bad, 1);
  }
}

// ----------------------------------------------------------------- launches

template <typename T, typename E>
static cudaError_t launch_matrix(const CsrView<T>& A, const T* x, const E& epi, size_t extra,
                                 cudaStream_t st) {
  if constexpr (!needs_tiles<E>::value) {
    if (csr_warp_enabled()) {
      static std::once_flag once_w;
      static int occ_w = 1;
      constexpr size_t dsm = csr_smem_bytes<T>();
      std::call_once(once_w, [&] {
        cudaFuncSetAttribute(k_csr_warp<T, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_w, k_csr_warp<T, E>, kCsrThreads, dsm);
        cudaGetLastError();
        if (occ_w < 1) occ_w = 1;
      });
      long long G = (A.n + 32LL * kCsrWarps - 1) / (32LL * kCsrWarps);
      const long long cap = std::min<long long>((long long)num_sms() * occ_w, kMaxParts);
      if (G > cap) G = cap;
      if (G < 1) G = 1;
      count_launch();
      return launch_k(E::kPdl, false, k_csr_warp<T, E>, dim3((unsigned)G), dim3(kCsrThreads), dsm, st, A, x, epi);
    }
  }
  const size_t smem = sizeof(SpSmem<T>) + extra;
  static std::once_flag once;
  static int occ = 1;
  std::call_once(once, [&] {
    cudaFuncSetAttribute(k_spmv<T, E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(SpSmem<T>) + (size_t)(kMaxM + 8) * sizeof(T)));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmv<T, E>, kSpThreads, smem);
    cudaGetLastError();
    if (occ < 1) occ = 1;
  });
  long long tiles = (A.n + kSpTile - 1) / kSpTile;
  long long G = (long long)num_sms() * occ;
  if (tiles < G) G = tiles;
  if (G < 1) G = 1;
  count_launch();
  return launch_k(E::kPdl, false, k_spmv<T, E>, dim3((unsigned)G), dim3(kSpThreads), smem, st, A, x, epi);
}

template <typename T, typename E, bool ALN>
static cudaError_t launch_stencil_k(const StencilView<T>& S, const T* x, const E& epi, size_t extra,
                                    cudaStream_t st) {
  static std::once_flag once;
  static int occ = 1;
  std::call_once(once, [&] {
    cudaFuncSetAttribute(k_stencil<T, E, ALN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((size_t)(kMaxM + 8) * sizeof(T) * 8));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stencil<T, E, ALN>, kSpConsumers, extra);
    cudaGetLastError();
    if (occ < 1) occ = 1;
  });
  // the padded (branchless) path deals tiles of one 16-byte row group per thread
  const long long tile_rows = S.padded ? (long long)kSpConsumers * Vec<T>::n : kSpTile;
  long long tiles = (S.n + tile_rows - 1) / tile_rows;
  long long G = (long long)num_sms() * occ;
  if (tiles < G) G = tiles;
  if (G > kMaxParts) G = kMaxParts;
  if (G < 1) G = 1;
  count_launch();
  return launch_k(E::kPdl, false, k_stencil<T, E, ALN>, dim3((unsigned)G), dim3(kSpConsumers), extra, st, S, x, epi);
}

// Aligned instantiation when every neighbour window is 16-byte aligned
// (nx % VN == 0: no misaligned-window code in the loop) for the streaming
// epilogues; the tile (fused-dot) epilogues keep the general one.
template <typename T, typename E>
static cudaError_t launch_matrix(const StencilView<T>& S, const T* x, const E& epi, size_t extra,
                                 cudaStream_t st) {
  if constexpr (!needs_tiles<E>::value) {
    if (S.padded && S.nx % Vec<T>::n == 0) return launch_stencil_k<T, E, true>(S, x, epi, extra, st);
  }
  return launch_stencil_k<T, E, false>(S, x, epi, extra, st);
}

template <typename T, typename M>
cudaError_t launch_spmv(const M& A, const T* x, T* y, WsView, cudaStream_t st,
                        const mpg_state_header* kt) {
  EpiPlain<T> e{};
  e.y = y;
  e.kt = kt;
  return launch_matrix(A, x, e, 0, st);
}

template <typename T, typename M>
cudaError_t launch_residual(const M& A, const T* b, const T* x, T* r, double* norm_out,
                            mpg_state_header* hdr, WsView ws, cudaStream_t st, int raw,
                            const mpg_state_header* kt, int kcat) {
  EpiResid<T> e{};
  e.b = b; e.r = r; e.out = norm_out; e.hdr = hdr; e.raw = raw;
  e.kt = kt; e.kcat = kcat;
  e.part = static_cast<T*>(ws.part);
  e.counter = ws.counter;
  return launch_matrix(A, x, e, 0, st);
}

template <typename T, typename M>
cudaError_t launch_spmv_dot1(const M& A, const T* x, T* w, const T* V, long long ldv, int k,
                             StateView<T> sv, WsView ws, cudaStream_t st) {
  auto reg = [&](auto tag) {
    constexpr int KV = decltype(tag)::value;
    EpiDot1Warp<T, KV> e{};
    e.w = w; e.V = V; e.ldv = ldv; e.k = k; e.sv = sv;
    e.kt = sv.h;
    e.part = static_cast<T*>(ws.part);
    e.counter = ws.counter;
    return launch_matrix(A, x, e, 0, st);
  };
  switch ((k + kSpConsumerWarps - 1) / kSpConsumerWarps) {
    case 1: return reg(std::integral_constant<int, 1>{});
    case 2: return reg(std::integral_constant<int, 2>{});
    case 3: return reg(std::integral_constant<int, 3>{});
    case 4: return reg(std::integral_constant<int, 4>{});
    case 5: return reg(std::integral_constant<int, 5>{});
    case 6: return reg(std::integral_constant<int, 6>{});
    case 7: return reg(std::integral_constant<int, 7>{});
    case 8: return reg(std::integral_constant<int, 8>{});
    default: break;
  }
  EpiDot1<T> e{};
  e.w = w; e.V = V; e.ldv = ldv; e.k = k; e.sv = sv;
  e.kt = sv.h;
  e.part = static_cast<T*>(ws.part);
  e.counter = ws.counter;
  return launch_matrix(A, x, e, (size_t)(k + 8) * sizeof(T), st);
}

template <typename T, typename M>
cudaError_t launch_poly_op(const M& A, const mpg_poly_op& op, const T* x, T* y, T* t0, T* t1,
                           T* t2, const mpg_state_header* gate, long long n, WsView ws,
                           cudaStream_t st, const mpg_state_header* kt) {
  T* bufs[5] = {const_cast<T*>(x), y, t0, t1, t2};
  EpiPoly<T> e{};
  e.op = op.op;
  e.a = (T)op.a;
  e.b = (T)op.b;
  e.src = bufs[op.src];
  e.dst = bufs[op.dst];
  e.x2 = bufs[op.x2];
  e.y = y;
  e.gate = gate;
  e.kt = kt;
  return launch_matrix(A, e.src, e, 0, st);
}

// Constant-coefficient scan of packed values: per slot, the min and max bit
// pattern over the present entries (u64 atomics into the tail scratch).
template <typename T>
__global__ void __launch_bounds__(kThreads) k_stencil_const_scan(int S, const T* __restrict__ dia, long long ldv,
                                                                 long long n, unsigned long long* mm) {
  unsigned long long lo[7], hi[7];
#pragma unroll
  for (int s = 0; s < 7; ++s) { lo[s] = ~0ull; hi[s] = 0ull; }
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
       r += (long long)gridDim.x * blockDim.x) {
#pragma unroll
    for (int s = 0; s < 7; ++s) {
      if (s < S) {
        const T v = dia[(size_t)s * ldv + r];
        if (present(v)) {
          unsigned long long b;
          if constexpr (sizeof(T) == 8) b = (unsigned long long)__double_as_longlong(v);
          else b = (unsigned long long)__float_as_uint(v);
          lo[s] = b < lo[s] ? b : lo[s];
          hi[s] = b > hi[s] ? b : hi[s];
        }
      }
    }
  }
#pragma unroll
  for (int s = 0; s < 7; ++s) {
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo[s], o);
      const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi[s], o);
      lo[s] = l2 < lo[s] ? l2 : lo[s];
      hi[s] = h2 > hi[s] ? h2 : hi[s];
    }
    if ((threadIdx.x & 31) == 0 && s < S) {
      atomicMin(mm + s, lo[s]);
      atomicMax(mm + 7 + s, hi[s]);
    }
  }
}

template <typename T>
__global__ void k_stencil_const_header(int S, T* h, const unsigned long long* mm, int enable) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  bool on = enable != 0;
  for (int s = 0; s < S; ++s) on = on && (mm[s] == mm[7 + s] || mm[s] == ~0ull);   // one value, or never present
  h[0] = on ? T(1) : T(0);
  for (int s = 0; s < S; ++s) {
    const unsigned long long b = mm[s] == ~0ull ? 0ull : mm[s];
    T v;
    if constexpr (sizeof(T) == 8) v = __longlong_as_double((long long)b);
    else v = __uint_as_float((unsigned)b);
    h[1 + s] = on ? v : T(0);
  }
}

// MPG_STENCIL_CONST=0 keeps the header off (A/B of the coefficient-stream path)
static int stencil_const_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MPG_STENCIL_CONST");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v;
}

template <typename T>
cudaError_t launch_stencil_pack(int dims, int nx, long long row0, long long n, const int32_t* rp,
                                const int32_t* ci, const T* v, T* out, long long ldv, int* bad,
                                cudaStream_t st) {
  long long G = (n + kThreads - 1) / kThreads;
  if (G > (long long)num_sms() * 8) G = (long long)num_sms() * 8;
  if (G < 1) G = 1;
  count_launch();
  k_stencil_pack<T><<<(unsigned)G, kThreads, 0, st>>>(dims, nx, row0, n, rp, ci, v, out, ldv, bad);
  // constant-coefficient header in the tail (the caller allocates S*ldv + kDiaTail)
  const int S = dims == 3 ? 7 : 5;
  T* h = out + (size_t)S * ldv;
  unsigned long long* mm = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(h) + 64);
  cudaError_t e = cudaMemsetAsync(mm, 0xff, 7 * sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(mm + 7, 0, 7 * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  count_launch();
  k_stencil_const_scan<T><<<(unsigned)G, kThreads, 0, st>>>(S, out, ldv, n, mm);
  count_launch();
  k_stencil_const_header<T><<<1, 32, 0, st>>>(S, h, mm, stencil_const_env());
  return cudaGetLastError();
}

#define INST_M(T, M)                                                                            \
  template cudaError_t launch_spmv<T, M>(const M&, const T*, T*, WsView, cudaStream_t,          \
                                         const mpg_state_header*);                              \
  template cudaError_t launch_residual<T, M>(const M&, const T*, const T*, T*, double*,         \
                                             mpg_state_header*, WsView, cudaStream_t, int,     \
                                             const mpg_state_header*, int);                    \
  template cudaError_t launch_spmv_dot1<T, M>(const M&, const T*, T*, const T*, long long, int, \
                                              StateView<T>, WsView, cudaStream_t);             \
  template cudaError_t launch_poly_op<T, M>(const M&, const mpg_poly_op&, const T*, T*, T*, T*, \
                                            T*, const mpg_state_header*, long long, WsView,    \
                                            cudaStream_t, const mpg_state_header*);
INST_M(float, CsrView<float>)
INST_M(double, CsrView<double>)
INST_M(float, StencilView<float>)
INST_M(double, StencilView<double>)
#undef INST_M
template cudaError_t launch_stencil_pack<float>(int, int, long long, long long, const int32_t*,
                                                const int32_t*, const float*, float*, long long, int*,
                                                cudaStream_t);
template cudaError_t launch_stencil_pack<double>(int, int, long long, long long, const int32_t*,
                                                 const int32_t*, const double*, double*, long long,
                                                 int*, cudaStream_t);

}  // namespace mpg
