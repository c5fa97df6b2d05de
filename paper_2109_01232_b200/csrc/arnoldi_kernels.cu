// CGS2 Arnoldi kernels (krylov.py:112-202, solvers.py:122-174).
//
// The four-launch Arnoldi step j (k = j + 1 basis vectors):
//   K_A1 SpMV          w = A z                                (spmv_kernels.cu)
//   K_A2 dot1          ||w||, finite check, c1 = V^T w        (k_dot1_wo / k_dot1_small)
//   K_B  update_dot    w <- w - V c1 ; c2 = V^T w ; H[:,j] = c1 + c2
//                      (k_update_dot_w / k_update_dot_small; TMA-staged k_update_dot for k > 64)
//   K_CS update_norm   w <- w - V c2 ; h_sub = ||w|| ; breakdown ; Givens rotation ;
//        + scale       implicit residual ; done flag ; V[:, j+1] = w / h_sub
//                      (cooperative k_update_norm_scale; k_update_norm + k_step_scale in
//                      distributed mode, where an allreduce sits between them)
// so the basis is swept three times per step (the reference's BLAS sequence
// sweeps it four times).  step_kernel.cu fuses the whole step into one
// persistent launch for small vectors.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "arnoldi_common.cuh"
#include "spmv.cuh"
#include "state.cuh"

namespace mpg {


// ============================================================== K_B update_dot
// TMA-staged: a producer warp bulk-copies the tile slices V[0..k)[tile] and
// w[tile] into an S-stage shared ring; consumers form w' = w - V c1 from the
// staged copy, then c2 partials = V^T w' from the same copy, so V is read
// from HBM exactly once for both halves.

constexpr int kUdConsumers = 256;
constexpr int kUdThreads = kUdConsumers + 32;

template <typename T>
__global__ void __launch_bounds__(kUdThreads) k_update_dot(const T* __restrict__ V, long long ldv,
                                                           long long n, int k, T* __restrict__ w,
                                                           StateView<T> sv, WsView ws, int TB,
                                                           int S) {
  if (gated(sv.h)) return;
  kt_mark(sv.h, KC_GEMV_TN);
  extern __shared__ __align__(128) unsigned char smraw[];
  const size_t stage_elems = (size_t)(k + 1) * TB;
  T* stages = reinterpret_cast<T*>(smraw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + (size_t)S * stage_elems * sizeof(T));
  uint64_t* empty = full + S;
  T* c1s = reinterpret_cast<T*>(empty + S);
  T* acc = c1s + k;
  T* pw = acc + k;     // 8
  T* red = pw + 8;     // 32
  __shared__ bool lastflag;

  long long R0, R1;
  cta_rows(n, R0, R1);
  const int nt = (int)((R1 - R0 + TB - 1) / TB);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kUdConsumers / 32);
    }
    fence_mbar_init();
  }
  for (int i = tid; i < k; i += blockDim.x) {
    c1s[i] = sv.c1[i];
    acc[i] = T(0);
  }
  __syncthreads();

  if (warp == kUdConsumers / 32) {
    if (lane == 0) {
      for (int t = 0; t < nt; ++t) {
        const int s = t % S;
        if (t >= S) mbar_wait(&empty[s], ((t / S) - 1) & 1);
        const long long a = R0 + (long long)t * TB;
        const long long nr = min((long long)TB, R1 - a);
        const uint32_t bytes = (uint32_t)round16(nr * (long long)sizeof(T));
        T* dst = stages + (size_t)s * stage_elems;
        fence_proxy_async();
        mbar_expect_tx(&full[s], bytes * (uint32_t)(k + 1));
        for (int i = 0; i < k; ++i) bulk_g2s(dst + (size_t)i * TB, V + (size_t)i * ldv + a, bytes, &full[s]);
        bulk_g2s(dst + (size_t)k * TB, w + a, bytes, &full[s]);
      }
    }
    return;
  }

  for (int t = 0; t < nt; ++t) {
    const int s = t % S;
    const long long a = R0 + (long long)t * TB;
    const int nr = (int)min((long long)TB, R1 - a);
    mbar_wait(&full[s], (t / S) & 1);
    T* vs = stages + (size_t)s * stage_elems;
    T* wsm = vs + (size_t)k * TB;
    // phase 1: w' = w - V c1 (the second half of CGS pass 1, krylov.py:140)
    for (int rr = tid; rr < nr; rr += kUdConsumers) {
      T u = T(0);
      int i = 0;
      for (; i + 4 <= k; i += 4) {
        u = fma_rn(vs[(size_t)(i + 0) * TB + rr], c1s[i + 0], u);
        u = fma_rn(vs[(size_t)(i + 1) * TB + rr], c1s[i + 1], u);
        u = fma_rn(vs[(size_t)(i + 2) * TB + rr], c1s[i + 2], u);
        u = fma_rn(vs[(size_t)(i + 3) * TB + rr], c1s[i + 3], u);
      }
      for (; i < k; ++i) u = fma_rn(vs[(size_t)i * TB + rr], c1s[i], u);
      const T wv = sub_rn(wsm[rr], u);
      wsm[rr] = wv;
      w[a + rr] = wv;
    }
    consumer_sync();
    // phase 2: c2 partials = V^T w' (CGS pass 2 dot, krylov.py:139)
    auto vrow = [&](int i) { return (const T*)(vs + (size_t)i * TB); };
    tile_dots<T, kLoadShared>(k, nr, vrow, wsm, acc, pw);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
  }
  consumer_sync();
  T* part = static_cast<T*>(ws.part);
  for (int i = tid; i < k; i += kUdConsumers) part[(size_t)blockIdx.x * k + i] = acc[i];
  (void)red;
  __threadfence();
  consumer_sync();
  if (tid == 0) lastflag = (atomicAdd(ws.counter, 1u) == gridDim.x - 1);
  consumer_sync();
  if (lastflag) {
    __threadfence();
    if (tid == 0) *ws.counter = 0u;
    const int j = k - 1;
    for (int c = warp; c < k; c += kUdConsumers / 32) {
      T s2 = T(0);
      for (int p = lane; p < (int)gridDim.x; p += 32) s2 += __ldcg(part + (size_t)p * k + c);
      s2 = warp_sum(s2);
      if (lane == 0) {
        if (sv.dist) { sv.red[c] = s2; continue; }   // raw local sum (distributed)
        sv.c2[c] = s2;
        // h = 0; h += c1; h += c2  (krylov.py:137-141)
        sv.Hc(j, c) = add_rn(add_rn(T(0), c1s[c]), s2);
      }
    }
  }
}

// ========================= K_B, warp-owned-vector variant (k <= 8*KV <= 64)
// Warp w owns basis vectors i = w + 8q (q < KV).  Per block of RB = 32*VN
// rows each lane loads one 16-byte slice of each owned vector (a warp-wide
// load = 512 contiguous bytes of one vector), forms its warp's partial
// u_w = sum_q V_i c1_i, and the 8 partials are summed in a fixed order
// through a double-buffered shared array (one barrier per block).  Then
// w' = w - u and the lane's KV pass-2 accumulators.  V is read once; per
// lane registers hold KV slices and KV accumulators.
template <typename T, int KV>
#ifndef MPG_KB_MINB
#define MPG_KB_MINB 4   // measured: 4 CTAs/SM (<= 64 regs) beats the unbounded 74-reg build
#endif
#ifndef MPG_KA2_MINB
#define MPG_KA2_MINB 1
#endif
#ifndef MPG_KCS_MINB
#define MPG_KCS_MINB 1
#endif
// basis loads in flight per thread in K_CS: fp32 4 (2 / 4 / 8: 3.52 / 3.47 /
// 3.52 ms per cycle), fp64 8 (cfg2 fp64 cycle: 6.92 -> 6.20 ms)
#ifndef MPG_KCS_BATCH32
#define MPG_KCS_BATCH32 4
#endif
#ifndef MPG_KCS_BATCH64
#define MPG_KCS_BATCH64 8
#endif
__global__ void __launch_bounds__(kThreads, MPG_KB_MINB) k_update_dot_w(const T* __restrict__ V, long long ldv,
                                                           long long n, int k, T* __restrict__ w,
                                                           StateView<T> sv, WsView ws) {
  pdl_wait();
  pdl_trigger();
  if (gated(sv.h)) return;
  kt_mark(sv.h, KC_GEMV_TN);
  constexpr int VN = Vec<T>::n;
  constexpr int RB = 32 * VN;
  constexpr int RPW = RB / kWarps;   // rows each warp reduces per block
  // U blocks per barrier pair: more loads in flight for small KV
  constexpr int U = KV <= 2 ? 4 : (KV <= 4 ? 2 : 1);
  // single-buffered: a warp writes upart (xs) of group it+1 only after the
  // barrier every warp reaches once done reading upart (xs) of group it
  __shared__ __align__(16) T upart[U][kWarps][RB];
  __shared__ __align__(16) T xs[U][RB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  T c1q[KV], acc[KV];
#pragma unroll
  for (int q = 0; q < KV; ++q) {
    const int i = warp + kWarps * q;
    c1q[q] = i < k ? sv.c1[i] : T(0);
    acc[q] = T(0);
  }
  // grid-stride over blocks of U * RB rows (one compact window of V streams at a time)
  const long long R1 = n;
  for (long long rg = (long long)blockIdx.x * U * RB; rg < R1; rg += (long long)gridDim.x * U * RB) {
    T v[U][KV][VN];
#pragma unroll
    for (int b = 0; b < U; ++b) {
      const long long r = rg + (long long)b * RB + (long long)lane * VN;
      const bool full = r + VN <= R1;
#pragma unroll
      for (int q = 0; q < KV; ++q) {
        const int i = warp + kWarps * q;
        if (i < k && full) {
          vload_cs(V + (size_t)i * ldv + r, v[b][q]);
        } else {
#pragma unroll
          for (int e = 0; e < VN; ++e)
            v[b][q][e] = (i < k && r + e < R1) ? __ldcs(V + (size_t)i * ldv + r + e) : T(0);
        }
      }
    }
    // reducer lane: row rrow of each block (warp w owns RPW rows of it)
    const int rrow = warp * RPW + lane;
    T wv[U];
#pragma unroll
    for (int b = 0; b < U; ++b) {
      const long long rr = rg + (long long)b * RB + rrow;
      wv[b] = (lane < RPW && rr < R1) ? w[rr] : T(0);
    }
#pragma unroll
    for (int b = 0; b < U; ++b) {
      T u[VN];
#pragma unroll
      for (int e = 0; e < VN; ++e) u[e] = T(0);
#pragma unroll
      for (int q = 0; q < KV; ++q)
#pragma unroll
        for (int e = 0; e < VN; ++e) u[e] = fma_rn(v[b][q][e], c1q[q], u[e]);
      vstore(upart[b][warp] + lane * VN, u);
    }
    __syncthreads();
    // the 8 warp partials of each row are summed in warp order by one lane
    if (lane < RPW) {
#pragma unroll
      for (int b = 0; b < U; ++b) {
        const long long rr = rg + (long long)b * RB + rrow;
        T xr = T(0);
        if (rr < R1) {
          T s = T(0);
#pragma unroll
          for (int ww = 0; ww < kWarps; ++ww) s += upart[b][ww][rrow];
          xr = sub_rn(wv[b], s);
          w[rr] = xr;
        }
        xs[b][rrow] = xr;
      }
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < U; ++b) {
      T x[VN];
      vload_smem(xs[b] + lane * VN, x);
#pragma unroll
      for (int q = 0; q < KV; ++q)
#pragma unroll
        for (int e = 0; e < VN; ++e) acc[q] = fma_rn(v[b][q][e], x[e], acc[q]);
    }
  }
  T* part = static_cast<T*>(ws.part);
#pragma unroll
  for (int q = 0; q < KV; ++q) {
    const int i = warp + kWarps * q;
    const T a = warp_sum(acc[q]);
    if (lane == 0 && i < k) part[(size_t)i * kMaxParts + blockIdx.x] = a;
  }
  const int jj = k - 1;
  grid_reduce_cols<kRedGroup>(part, kMaxParts, static_cast<T*>(ws.gpart), ws.gcount, k,
                              [&](int c, T s2) {
    if (sv.dist) { sv.red[c] = s2; return; }   // raw local sum (distributed)
    sv.c2[c] = s2;
    sv.Hc(jj, c) = add_rn(add_rn(T(0), sv.c1[c]), s2);   // h = 0; h += c1; h += c2
  });
}

// ================================== generic-operator pass-1 dots (no SpMV)
// c1 = V[:, :k]^T w, w0 = ||w||, finite check (krylov.py:133-139) for a w
// produced by an arbitrary operator.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_dot1_w(const T* __restrict__ w, long long n,
                                                     const T* __restrict__ V, long long ldv, int k,
                                                     StateView<T> sv, WsView ws) {
  if (gated(sv.h)) return;
  kt_mark(sv.h, KC_GEMV_T);
  constexpr int VN = Vec<T>::n;
  __shared__ T red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long R0, R1;
  cta_rows(n, R0, R1);
  const int stride = k + 2;
  T* part = static_cast<T*>(ws.part);
  const long long nv = (R1 - R0) / VN;
  for (int i = warp; i < k; i += kWarps) {
    const T* v = V + (size_t)i * ldv;
    T p = T(0);
    for (long long g = lane; g < nv; g += 32) {
      T a[VN], b[VN];
      vload_cs(v + R0 + g * VN, a);
      vload(w + R0 + g * VN, b);
#pragma unroll
      for (int e = 0; e < VN; ++e) p = fma_rn(a[e], b[e], p);
    }
    for (long long r = R0 + nv * VN + lane; r < R1; r += 32) p = fma_rn(v[r], w[r], p);
    p = warp_sum(p);
    if (lane == 0) part[(size_t)blockIdx.x * stride + i] = p;
  }
  T ss = T(0);
  int bad = 0;
  for (long long r = R0 + threadIdx.x; r < R1; r += kThreads) {
    const T y = w[r];
    ss = fma_rn(y, y, ss);
    bad |= !isfinite(y);
  }
  const T t = block_sum(ss, red);
  const int anybad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    part[(size_t)blockIdx.x * stride + k] = t;
    part[(size_t)blockIdx.x * stride + k + 1] = anybad ? T(1) : T(0);
  }
  if (last_cta(ws.counter)) {
    finalize_columns(part, gridDim.x, stride, k + 2, [&](int c, T s) {
      if (c < k) sv.c1[c] = s;
      else if (c == k) sv.h->w0 = (double)sqrt_rn(s);
      else if (s != T(0)) { sv.h->flags |= MPG_FLAG_NONFINITE_OP; sv.h->done = 1; }
    });
  }
}

// ============================= pass-1 dots on a stored w (split K_A, A/B path)
// c1 = V[:, :k]^T w, w0 = ||w||, finite check (krylov.py:133-139) when the
// SpMV has already written w (L2-resident at the bench sizes).  Warp w owns
// basis vectors i = w + 8q (q < KV); blocks of U * 32 * VN rows are dealt
// round-robin over the grid; warp 0 also accumulates ||w||^2 and the finite
// flag.  One deterministic CTA reduction + fixed-order last-CTA finalisation.
template <typename T, int KV, int U>
__global__ void __launch_bounds__(kThreads, MPG_KA2_MINB) k_dot1_wo(const T* __restrict__ w, long long n,
                                                      const T* __restrict__ V, long long ldv, int k,
                                                      StateView<T> sv, WsView ws) {
  pdl_wait();
  pdl_trigger();
  if (gated(sv.h)) return;
  kt_mark(sv.h, KC_GEMV_T);
  constexpr int VN = Vec<T>::n;
  constexpr int RB = 32 * VN;
  __shared__ T red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T acc[KV];
#pragma unroll
  for (int q = 0; q < KV; ++q) acc[q] = T(0);
  T ss = T(0);
  int bad = 0;
  for (long long base = (long long)blockIdx.x * U * RB; base < n; base += (long long)gridDim.x * U * RB) {
    T wv[U][VN], v[U][KV][VN];
#pragma unroll
    for (int b = 0; b < U; ++b) {
      const long long r = base + (long long)b * RB + (long long)lane * VN;
      const bool in = r < n;   // rows in [n, ldv) are zero padding
      if (in) vload(w + r, wv[b]);
      else {
#pragma unroll
        for (int e = 0; e < VN; ++e) wv[b][e] = T(0);
      }
#pragma unroll
      for (int q = 0; q < KV; ++q) {
        const int i = warp + kWarps * q;
        if (in && i < k) vload_cs(V + (size_t)i * ldv + r, v[b][q]);
        else {
#pragma unroll
          for (int e = 0; e < VN; ++e) v[b][q][e] = T(0);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < U; ++b) {
#pragma unroll
      for (int q = 0; q < KV; ++q)
#pragma unroll
        for (int e = 0; e < VN; ++e) acc[q] = fma_rn(v[b][q][e], wv[b][e], acc[q]);
      if (warp == 0) {
#pragma unroll
        for (int e = 0; e < VN; ++e) {
          ss = fma_rn(wv[b][e], wv[b][e], ss);
          bad |= !isfinite(wv[b][e]);
        }
      }
    }
  }
  // column-major partials (c1[0..k), ||w||^2, non-finite), two-level reduction
  T* part = static_cast<T*>(ws.part);
#pragma unroll
  for (int q = 0; q < KV; ++q) {
    const int i = warp + kWarps * q;
    const T a = warp_sum(acc[q]);
    if (lane == 0 && i < k) part[(size_t)i * kMaxParts + blockIdx.x] = a;
  }
  if (warp == 0) {
    const T t = warp_sum(ss);
    const int anybad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      part[(size_t)k * kMaxParts + blockIdx.x] = t;
      part[(size_t)(k + 1) * kMaxParts + blockIdx.x] = anybad ? T(1) : T(0);
    }
  }
  grid_reduce_cols<kRedGroup>(part, kMaxParts, static_cast<T*>(ws.gpart), ws.gcount, k + 2,
                              [&](int c, T s) {
    if (sv.dist) sv.red[c] = s;
    else if (c < k) sv.c1[c] = s;
    else if (c == k) sv.h->w0 = (double)sqrt_rn(s);
    else if (s != T(0)) { sv.h->flags |= MPG_FLAG_NONFINITE_OP; sv.h->done = 1; }
  });
  (void)red;
}

// ============================ small-k variants (k <= KT <= 8): thread-owned rows
// With k < 8 the warp-owned kernels leave most warps without a basis vector,
// so few loads are in flight (measured ~20-30 us per launch at k = 1..8 for
// ~27-150 MB).  Here every thread owns 16-byte row groups (grid-stride) and
// all k vectors of them: KT accumulators per thread, one CTA reduction of
// the k columns (warp trees, then the 8 warps in order), then the same
// two-level grid reduction.
template <typename T, int KT>
__device__ __forceinline__ void cta_columns_to_part(T (&acc)[KT], int ncols, T* part, T* red8) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < KT; ++q) {
    const T a = warp_sum(acc[q]);
    if (lane == 0) red8[q * kWarps + warp] = a;
  }
  __syncthreads();
  if ((int)threadIdx.x < ncols) {
    T t = T(0);
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) t += red8[threadIdx.x * kWarps + ww];
    part[(size_t)threadIdx.x * kMaxParts + blockIdx.x] = t;
  }
}

// pass-1 dots (+ ||w||^2 + finite flag) for k <= KT - 2 ... KT columns = k + 2
template <typename T, int KT>
__global__ void __launch_bounds__(kThreads) k_dot1_small(const T* __restrict__ w, long long n,
                                                         const T* __restrict__ V, long long ldv, int k,
                                                         StateView<T> sv, WsView ws) {
  pdl_wait();
  pdl_trigger();
  if (gated(sv.h)) return;
  kt_mark(sv.h, KC_GEMV_T);
  constexpr int VN = Vec<T>::n;
  __shared__ T red8[(KT + 2) * kWarps];
  T acc[KT + 2];
#pragma unroll
  for (int q = 0; q < KT + 2; ++q) acc[q] = T(0);
  int bad = 0;
  const long long ng = (n + VN - 1) / VN;
  for (long long g = blockIdx.x * (long long)kThreads + threadIdx.x; g < ng; g += (long long)gridDim.x * kThreads) {
    const long long r = g * VN;
    T wv[VN], v[KT][VN];
    vload(w + r, wv);   // rows in [n, ldv) are zero padding
#pragma unroll
    for (int q = 0; q < KT; ++q)
      if (q < k) vload_cs(V + (size_t)q * ldv + r, v[q]);
#pragma unroll
    for (int q = 0; q < KT; ++q)
      if (q < k) {
#pragma unroll
        for (int e = 0; e < VN; ++e) acc[q] = fma_rn(v[q][e], wv[e], acc[q]);
      }
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      acc[KT] = fma_rn(wv[e], wv[e], acc[KT]);
      bad |= !isfinite(wv[e]);
    }
  }
  acc[KT + 1] = __syncthreads_or(bad) ? T(1) : T(0);
  // compact to k + 2 columns: c1[0..k), ||w||^2, flag
  T cols[KT + 2];
#pragma unroll
  for (int q = 0; q < KT + 2; ++q) cols[q] = T(0);
#pragma unroll
  for (int q = 0; q < KT; ++q) if (q < k) cols[q] = acc[q];
#pragma unroll
  for (int q = 0; q < KT + 2; ++q) {
    if (q == k) cols[q] = acc[KT];
    if (q == k + 1) cols[q] = (threadIdx.x == 0) ? acc[KT + 1] : T(0);   // flag counted once per CTA
  }
  T* part = static_cast<T*>(ws.part);
  cta_columns_to_part<T, KT + 2>(cols, k + 2, part, red8);
  grid_reduce_cols<kRedGroup>(part, kMaxParts, static_cast<T*>(ws.gpart), ws.gcount, k + 2,
                              [&](int c, T s) {
    if (sv.dist) sv.red[c] = s;
    else if (c < k) sv.c1[c] = s;
    else if (c == k) sv.h->w0 = (double)sqrt_rn(s);
    else if (s != T(0)) { sv.h->flags |= MPG_FLAG_NONFINITE_OP; sv.h->done = 1; }
  });
}

// K_B for k <= KT: w' = w - V c1 ; c2 = V^T w' ; H[:, j] = c1 + c2
template <typename T, int KT>
__global__ void __launch_bounds__(kThreads) k_update_dot_small(const T* __restrict__ V, long long ldv,
                                                               long long n, int k, T* __restrict__ w,
                                                               StateView<T> sv, WsView ws) {
  pdl_wait();
  pdl_trigger();
  if (gated(sv.h)) return;
  kt_mark(sv.h, KC_GEMV_TN);
  constexpr int VN = Vec<T>::n;
  __shared__ T red8[KT * kWarps];
  T c1q[KT], acc[KT];
#pragma unroll
  for (int q = 0; q < KT; ++q) {
    c1q[q] = q < k ? sv.c1[q] : T(0);
    acc[q] = T(0);
  }
  const long long ng = (n + VN - 1) / VN;
  for (long long g = blockIdx.x * (long long)kThreads + threadIdx.x; g < ng; g += (long long)gridDim.x * kThreads) {
    const long long r = g * VN;
    T wv[VN], v[KT][VN], u[VN];
    vload(w + r, wv);
#pragma unroll
    for (int q = 0; q < KT; ++q)
      if (q < k) vload_cs(V + (size_t)q * ldv + r, v[q]);
#pragma unroll
    for (int e = 0; e < VN; ++e) u[e] = T(0);
#pragma unroll
    for (int q = 0; q < KT; ++q)
      if (q < k) {
#pragma unroll
        for (int e = 0; e < VN; ++e) u[e] = fma_rn(v[q][e], c1q[q], u[e]);
      }
#pragma unroll
    for (int e = 0; e < VN; ++e) wv[e] = r + e < n ? sub_rn(wv[e], u[e]) : T(0);
    vstore(w + r, wv);
#pragma unroll
    for (int q = 0; q < KT; ++q)
      if (q < k) {
#pragma unroll
        for (int e = 0; e < VN; ++e) acc[q] = fma_rn(v[q][e], wv[e], acc[q]);
      }
  }
  T* part = static_cast<T*>(ws.part);
  cta_columns_to_part<T, KT>(acc, k, part, red8);
  const int jj = k - 1;
  grid_reduce_cols<kRedGroup>(part, kMaxParts, static_cast<T*>(ws.gpart), ws.gcount, k,
                              [&](int c, T s2) {
    if (sv.dist) { sv.red[c] = s2; return; }
    sv.c2[c] = s2;
    sv.Hc(jj, c) = add_rn(add_rn(T(0), sv.c1[c]), s2);   // h = 0; h += c1; h += c2
  });
}

// ================================================= K_C update_norm + Givens

template <typename T>
__global__ void __launch_bounds__(kThreads) k_update_norm(const T* __restrict__ V, long long ldv,
                                                          long long n, int j, T* __restrict__ w,
                                                          StateView<T> sv, WsView ws, int m_limit) {
  if (gated(sv.h)) return;
  kt_mark(sv.h, KC_GEMV_N);
  constexpr int VN = Vec<T>::n;
  const int k = j + 1;
  extern __shared__ __align__(128) unsigned char smraw[];
  T* c2s = reinterpret_cast<T*>(smraw);
  __shared__ T red[32];
  for (int i = threadIdx.x; i < k; i += blockDim.x) c2s[i] = sv.c2[i];
  __syncthreads();
  // grid-stride 16-byte row groups, the same order as k_update_norm_scale (launched
  // on the same grid, so the distributed phases are bitwise the fused kernel)
  const long long ng = (n + VN - 1) / VN;
  const long long stride = (long long)gridDim.x * kThreads;
  T ss = T(0);
  for (long long g = blockIdx.x * (long long)kThreads + threadIdx.x; g < ng; g += stride) {
    const long long r = g * VN;
    T wv[VN], u[VN];
    vload(w + r, wv);
#pragma unroll
    for (int e = 0; e < VN; ++e) u[e] = T(0);
    int i = 0;
    for (; i + 4 <= k; i += 4) {
      T v0[VN], v1[VN], v2[VN], v3[VN];
      vload_cs(V + (size_t)(i + 0) * ldv + r, v0);
      vload_cs(V + (size_t)(i + 1) * ldv + r, v1);
      vload_cs(V + (size_t)(i + 2) * ldv + r, v2);
      vload_cs(V + (size_t)(i + 3) * ldv + r, v3);
#pragma unroll
      for (int e = 0; e < VN; ++e) {
        u[e] = fma_rn(v0[e], c2s[i + 0], u[e]);
        u[e] = fma_rn(v1[e], c2s[i + 1], u[e]);
        u[e] = fma_rn(v2[e], c2s[i + 2], u[e]);
        u[e] = fma_rn(v3[e], c2s[i + 3], u[e]);
      }
    }
    for (; i < k; ++i) {
      T v0[VN];
      vload_cs(V + (size_t)i * ldv + r, v0);
#pragma unroll
      for (int e = 0; e < VN; ++e) u[e] = fma_rn(v0[e], c2s[i], u[e]);
    }
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      wv[e] = r + e < n ? sub_rn(wv[e], u[e]) : T(0);
      ss = fma_rn(wv[e], wv[e], ss);
    }
    vstore(w + r, wv);
  }
  const T t = block_sum(ss, red);
  T* part = static_cast<T*>(ws.part);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
  if (last_cta(ws.counter)) {
    T s = T(0);
    for (int p = threadIdx.x; p < (int)gridDim.x; p += blockDim.x) s += __ldcg(part + p);
    s = block_sum(s, red);
    if (threadIdx.x == 0) {
      if (sv.dist) { sv.red[0] = s; return; }   // raw local sum (distributed)
      const T hs = sqrt_rn(s);
      sv.Hc(j, j + 1) = hs;
      sv.h->h_sub = (double)hs;
      // krylov.py:146: breakdown when h_sub <= tol * w0 (Python floats)
      const bool brk = (double)hs <= sv.h->breakdown_tol * sv.h->w0;
      givens_column(sv, j, sv.h->threshold, brk, m_limit);
    }
  }
}

// K_S: V[:, j+1] = w / h_sub (krylov.py:148; IEEE division, no reciprocal)
template <typename T>
__global__ void __launch_bounds__(kThreads) k_step_scale(const T* __restrict__ w, T* __restrict__ vn,
                                                         long long n, int j, StateView<T> sv) {
  if (gated(sv.h)) return;
  kt_mark(sv.h, KC_OTHER);
  constexpr int VN = Vec<T>::n;
  const T hs = sv.Hc(j, j + 1);
  const long long nv = n / VN;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < nv;
       g += (long long)gridDim.x * blockDim.x) {
    T a[VN];
    vload(w + g * VN, a);
#pragma unroll
    for (int e = 0; e < VN; ++e) a[e] = div_rn(a[e], hs);
    vstore(vn + g * VN, a);
  }
  for (long long r = nv * VN + blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
       r += (long long)gridDim.x * blockDim.x)
    vn[r] = div_rn(w[r], hs);
}

// ============================================ K_CS update_norm + scale, fused
// K_C and K_S in one cooperative launch (every CTA co-resident):
//   phase 1  w' = w - V c2 for the CTA's rows, kept in shared memory (CACHE)
//            or written back (L2-resident re-read); per-CTA ||w'||^2 partial
//   barrier  one grid-wide barrier
//   phase 2  every CTA sums the partials in the same fixed order as k_update_norm's
//            last CTA (bitwise the same h_sub), CTA 0 does the Givens rotation, and
//            every CTA writes V[:, j+1] = w' / h_sub for its rows (krylov.py:148)
// This drops K_S's launch and its 2 n s bytes (read w, write v) for n s (write v).
// Shared arrival counter + generation word in the workspace; the last arriver
// resets the counter before releasing, so the slot is reusable.
template <typename T, bool CACHE>
__global__ void __launch_bounds__(kThreads, MPG_KCS_MINB) k_update_norm_scale(const T* __restrict__ V, long long ldv,
                                                                long long n, int j, T* __restrict__ w,
                                                                StateView<T> sv, WsView ws, int m_limit,
                                                                int kpad) {
  pdl_wait();
  pdl_trigger();
  if (gated(sv.h)) return;
  kt_mark(sv.h, KC_GEMV_N);
  constexpr int VN = Vec<T>::n;
  const int k = j + 1;
  extern __shared__ __align__(128) unsigned char smraw[];
  T* c2s = reinterpret_cast<T*>(smraw);
  T* wsm = c2s + kpad;   // CACHE: this CTA's groups of w', slot it * kThreads + tid
  __shared__ T red[32];
  for (int i = threadIdx.x; i < k; i += blockDim.x) c2s[i] = sv.c2[i];
  __syncthreads();
  // grid-stride over 16-byte row groups: at any moment the whole grid streams one
  // compact window of every basis vector (measured faster than per-CTA slices);
  // rows in [n, ldv) are zero padding and are masked out of w'
  const long long ng = (n + VN - 1) / VN;
  const long long stride = (long long)gridDim.x * kThreads;
  T ss = T(0);
  int it = 0;
  for (long long g = blockIdx.x * (long long)kThreads + threadIdx.x; g < ng; g += stride, ++it) {
    const long long r = g * VN;
    T wv[VN], u[VN];
    vload(w + r, wv);
#pragma unroll
    for (int e = 0; e < VN; ++e) u[e] = T(0);
    int i = 0;
    // B basis loads in flight per thread; u accumulates in i order either way
    constexpr int B = sizeof(T) == 8 ? MPG_KCS_BATCH64 : MPG_KCS_BATCH32;
    for (; i + B <= k; i += B) {
      T vb[B][VN];
#pragma unroll
      for (int b = 0; b < B; ++b) vload_cs(V + (size_t)(i + b) * ldv + r, vb[b]);
#pragma unroll
      for (int e = 0; e < VN; ++e)
#pragma unroll
        for (int b = 0; b < B; ++b) u[e] = fma_rn(vb[b][e], c2s[i + b], u[e]);
    }
    for (; i < k; ++i) {
      T v0[VN];
      vload_cs(V + (size_t)i * ldv + r, v0);
#pragma unroll
      for (int e = 0; e < VN; ++e) u[e] = fma_rn(v0[e], c2s[i], u[e]);
    }
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      wv[e] = r + e < n ? sub_rn(wv[e], u[e]) : T(0);
      ss = fma_rn(wv[e], wv[e], ss);
    }
    if (CACHE) vstore(wsm + ((size_t)it * kThreads + threadIdx.x) * VN, wv);
    else vstore(w + r, wv);
  }
  const T t = block_sum(ss, red);
  T* part = static_cast<T*>(ws.part);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
  if (blockIdx.x == 0 && threadIdx.x == 0) kt_stamp(sv.h, KC_NORM);   // barrier + norm tail
  grid_barrier(ws.counter, ws.counter + 1);
  // the same fixed-order sum in every CTA (identical to k_update_norm's last CTA)
  T s = T(0);
  for (int p = threadIdx.x; p < (int)gridDim.x; p += blockDim.x) s += __ldcg(part + p);
  s = block_sum(s, red);
  const T hs = sqrt_rn(s);
  if (blockIdx.x == 0 && threadIdx.x == 0) kt_stamp(sv.h, KC_OTHER);  // Givens + v = w / h
  const bool brk = (double)hs <= sv.h->breakdown_tol * sv.h->w0;   // krylov.py:146
  if (blockIdx.x == 0 && threadIdx.x < 32) {   // c2s (>= 3m + 2 elements) is free after the barrier
    if (threadIdx.x == 0) {
      sv.Hc(j, j + 1) = hs;
      sv.h->h_sub = (double)hs;
    }
    __syncwarp();
    givens_column_warp(sv, j, sv.h->threshold, brk, m_limit, c2s);
  }
  if (brk) return;   // no new basis vector on breakdown
  T* vn = const_cast<T*>(V) + (size_t)(j + 1) * ldv;
  it = 0;
  for (long long g = blockIdx.x * (long long)kThreads + threadIdx.x; g < ng; g += stride, ++it) {
    T a[VN];
    if (CACHE) vload_smem(wsm + ((size_t)it * kThreads + threadIdx.x) * VN, a);
    else vload_cg(w + g * VN, a);   // written by this thread in this launch: L2 path
#pragma unroll
    for (int e = 0; e < VN; ++e) a[e] = div_rn(a[e], hs);   // padding stays 0
    vstore(vn + g * VN, a);
  }
}

// ======================================= distributed: peer-memory halo (dist)
// V[:, j+1] = w / h_sub (krylov.py:148) for this rank's rows, and the rows a
// neighbour needs for its next SpMV written straight into its halo through
// the peer mapping: our first `halo` rows go to prev's upper halo, our last
// `halo` rows to next's lower halo.  After every CTA's stores are fenced
// system-wide, the last CTA bumps this rank's halo sequence number (header
// reserved1) and release-stores it into both neighbours' flags.

template <typename T>
__global__ void __launch_bounds__(kThreads) k_step_scale_peer(const T* __restrict__ w, T* __restrict__ vn,
                                                              long long n, long long halo, int j,
                                                              StateView<T> sv, T* prev_row, T* next_row,
                                                              uint32_t* prev_flag, uint32_t* next_flag,
                                                              unsigned int* counter) {
  if (gated(sv.h)) return;
  kt_mark(sv.h, KC_OTHER);
  const T hs = sv.Hc(j, j + 1);
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
       r += (long long)gridDim.x * blockDim.x) {
    const T v = div_rn(w[r], hs);
    vn[r] = v;
    if (prev_row && r < halo) prev_row[r] = v;
    if (next_row && r >= n - halo) next_row[r - (n - halo)] = v;
  }
  __threadfence_system();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    *counter = 0u;
    __threadfence_system();
    volatile int32_t* seqp = &sv.h->reserved1;
    const uint32_t seq = (uint32_t)(*seqp) + 1u;
    *seqp = (int32_t)seq;
    if (prev_flag) st_release_sys_u32(prev_flag, seq);
    if (next_flag) st_release_sys_u32(next_flag, seq);
  }
}

// Before the SpMV of step j >= 1: wait until both neighbours have released the
// halo rows of V[:, j] (their sequence number caught up with ours).
// Bounded: after ~20 s without the flag the cycle is stopped with
// MPG_FLAG_HALO_TIMEOUT (raised on the host) instead of hanging the GPU.
__global__ void k_halo_wait(mpg_state_header* h, const uint32_t* flags, int has_prev, int has_next) {
  if (gated(h) || threadIdx.x != 0) return;
  const uint32_t seq = (uint32_t)(*(volatile const int32_t*)&h->reserved1);
  const unsigned long long t0 = clock64(), limit = 40ull * 1000 * 1000 * 1000;   // ~20 s at 2 GHz
  for (int side = 0; side < 2; ++side) {
    if (side == 0 ? !has_prev : !has_next) continue;
    while ((int32_t)(ld_acquire_sys_u32(flags + side) - seq) < 0) {
      if (clock64() - t0 > limit) {
        h->flags |= MPG_FLAG_HALO_TIMEOUT;
        h->done = 1;
        __threadfence_system();
        return;
      }
      __nanosleep(64);
    }
  }
  __threadfence_system();
}

template <typename T>
cudaError_t launch_step_scale_peer(const T* w, T* vn, long long n, long long halo, int j, StateView<T> sv,
                                   T* prev_row, T* next_row, uint32_t* prev_flag, uint32_t* next_flag,
                                   WsView ws, cudaStream_t st) {
  count_launch();
  long long G = (n + kThreads - 1) / kThreads;
  const long long cap = (long long)num_sms() * 8;
  if (G > cap) G = cap;
  if (G < 1) G = 1;
  k_step_scale_peer<T><<<(unsigned)G, kThreads, 0, st>>>(w, vn, n, halo, j, sv, prev_row, next_row, prev_flag,
                                                         next_flag, ws.counter);
  return cudaGetLastError();
}

cudaError_t launch_halo_wait(mpg_state_header* h, const uint32_t* flags, int has_prev, int has_next,
                             cudaStream_t st) {
  count_launch();
  k_halo_wait<<<1, 32, 0, st>>>(h, flags, has_prev, has_next);
  return cudaGetLastError();
}

// ===================================================================== start

// Reset the cycle state (krylov.py:62-68, 96-100) — whole CTA.
template <typename T>
__device__ void init_state(const StateView<T>& sv, T gamma, double b_norm, double rtol,
                           double btol, int extra_flags) {
  const int m = sv.m;
  const size_t hm = (size_t)(m + 1) * m;
  for (size_t i = threadIdx.x; i < hm; i += blockDim.x) { sv.H[i] = T(0); sv.R[i] = T(0); }
  for (int i = threadIdx.x; i < m + 1; i += blockDim.x) {
    sv.g[i] = T(0); sv.c1[i] = T(0); sv.c2[i] = T(0); sv.d[i] = T(0);
    if (i < m) { sv.cs[i] = T(0); sv.sn[i] = T(0); sv.implicit[i] = 0.0; }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    sv.g[0] = gamma;
    mpg_state_header* h = sv.h;
    int flags = extra_flags;
    int done = 0;
    if (!isfinite(gamma)) { flags |= MPG_FLAG_NONFINITE_GAMMA; done = 1; }
    if (gamma == T(0)) done = 1;                 // solvers.py:150-151
    if (extra_flags) done = 1;
    h->flags = flags;
    h->steps = 0;
    h->done = done;
    h->breakdown = 0;
    h->m = m;
    h->prec = sizeof(T) == 8 ? MPG_FP64 : MPG_FP32;
    h->gamma = (double)gamma;
    h->b_norm = b_norm < 0 ? (double)gamma : b_norm;
    h->threshold = rtol * h->b_norm;            // solvers.py:158
    h->rtol = rtol;
    h->breakdown_tol = btol;
    h->w0 = 0.0;
    h->h_sub = 0.0;
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_start(const T* __restrict__ r0, long long n,
                                                    StateView<T> sv, double rtol,
                                                    const double* b_norm_src, double btol,
                                                    WsView ws) {
  kt_mark(sv.h, KC_NORM);
  __shared__ T red[32];
  T ss = T(0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const T v = r0[i];
    ss = fma_rn(v, v, ss);
  }
  const T t = block_sum(ss, red);
  T* part = static_cast<T*>(ws.part);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
  if (last_cta(ws.counter)) {
    T s = T(0);
    for (int p = threadIdx.x; p < (int)gridDim.x; p += blockDim.x) s += __ldcg(part + p);
    s = block_sum(s, red);
    const T gamma = sqrt_rn(s);
    // restarted cycles threshold on the outer ||b|| (solvers.py:186,198);
    // a null source means "use gamma" (gmres_cycle with b_norm=None, r0=b)
    const double bn = b_norm_src ? *b_norm_src : -1.0;
    if (sv.dist) {                   // raw local sum; k_dist_post initialises
      if (threadIdx.x == 0) sv.red[0] = s;
      return;
    }
    init_state(sv, gamma, bn, rtol, btol, 0);
  }
}

// IR inner right-hand side: r32 = fp32(r64 / rho) with rho = ||r64||
// (solvers.py:339-341), overflow check (core.py:264-271), gamma = ||r32||.
__global__ void __launch_bounds__(kThreads) k_start_ir(const double* __restrict__ r64,
                                                       float* __restrict__ r32, long long n,
                                                       StateView<float> sv, double rtol,
                                                       double btol, WsView ws) {
  kt_mark(sv.h, KC_OTHER);
  __shared__ float red[32];
  __shared__ int ovf_s;
  const double rho = sv.h->rnorm;
  if (threadIdx.x == 0) ovf_s = 0;
  __syncthreads();
  float ss = 0.f;
  int ovf = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double q = __ddiv_rn(r64[i], rho);
    const float v = __double2float_rn(q);
    ovf |= (isinf(v) && isfinite(q));
    r32[i] = v;
    ss = fma_rn(v, v, ss);
  }
  if (ovf) atomicOr(&ovf_s, 1);
  const float t = block_sum(ss, red);
  float* part = static_cast<float*>(ws.part);
  if (threadIdx.x == 0) part[(size_t)blockIdx.x * 2] = t, part[(size_t)blockIdx.x * 2 + 1] = ovf_s ? 1.f : 0.f;
  if (last_cta(ws.counter)) {
    float s = 0.f, o = 0.f;
    for (int p = threadIdx.x; p < (int)gridDim.x; p += blockDim.x) {
      s += __ldcg(part + (size_t)p * 2);
      o += __ldcg(part + (size_t)p * 2 + 1);
    }
    s = block_sum(s, red);
    o = block_sum(o, red);
    const float gamma = sqrt_rn(s);
    // the inner cycle's b_norm is ||r32|| itself (solvers.py:146 with b = r32)
    if (threadIdx.x == 0) sv.h->rho = rho;
    if (sv.dist) {                   // raw local sums; k_dist_post initialises
      if (threadIdx.x == 0) { sv.red[0] = s; sv.red[1] = o; }
      return;
    }
    init_state(sv, gamma, -1.0, rtol, btol, o > 0.f ? MPG_FLAG_OVERFLOW : 0);
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_start_scale(const T* __restrict__ r0, T* __restrict__ v0,
                                                          long long n, StateView<T> sv) {
  if (gated(sv.h)) return;
  kt_mark(sv.h, KC_OTHER);
  const T gamma = sv.g[0];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v0[i] = div_rn(r0[i], gamma);
}

// ======================================================= distributed: post
// After the allreduce of a phase's raw local sums (red[] or reserved[0]),
// one CTA finishes the phase exactly as the single-GPU last CTA would: the
// derived scalars, the Hessenberg column and the Givens rotation are computed
// from bitwise-identical inputs on every rank, so the replicated small state
// stays identical across ranks.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_dist_post(int phase, StateView<T> sv, int j,
                                                        int m_limit, double rtol, double btol,
                                                        int flag) {
  mpg_state_header* h = sv.h;
  switch (phase) {
    case DP_POST_START: {   // flag: 1 = IR (b_norm = gamma, overflow flag in red[1])
      const T gamma = sqrt_rn(sv.red[0]);
      const int f = (flag && sv.red[1] > T(0)) ? MPG_FLAG_OVERFLOW : 0;
      init_state(sv, gamma, flag ? -1.0 : h->outer_b_norm, rtol, btol, f);
      return;
    }
    case DP_POST_DOT1: {
      if (gated(h)) return;
      const int k = j + 1;
      for (int c = threadIdx.x; c < k; c += blockDim.x) sv.c1[c] = sv.red[c];
      if (threadIdx.x == 0) {
        h->w0 = (double)sqrt_rn(sv.red[k]);
        if (sv.red[k + 1] != T(0)) {
          h->flags |= MPG_FLAG_NONFINITE_OP;
          h->done = 1;
        }
      }
      return;
    }
    case DP_POST_DOT2: {
      if (gated(h)) return;
      const int k = j + 1;
      for (int c = threadIdx.x; c < k; c += blockDim.x) {
        sv.c2[c] = sv.red[c];
        sv.Hc(j, c) = add_rn(add_rn(T(0), sv.c1[c]), sv.red[c]);   // h = 0; h += c1; h += c2
      }
      return;
    }
    case DP_POST_NORM: {
      if (gated(h)) return;
      // one warp, the rotation staged in shared memory (givens_column_warp):
      // on the critical path of every distributed Arnoldi step
      __shared__ T gsm[3 * kMaxM + 2];
      if (threadIdx.x < 32) {
        const T hs = sqrt_rn(sv.red[0]);
        const bool brk = (double)hs <= h->breakdown_tol * h->w0;
        if (threadIdx.x == 0) {
          sv.Hc(j, j + 1) = hs;
          h->h_sub = (double)hs;
        }
        __syncwarp();
        givens_column_warp(sv, j, h->threshold, brk, m_limit, gsm);
      }
      return;
    }
    case DP_POST_RESID:     // flag: 1 = the outer precision is fp64
      if (threadIdx.x == 0)
        h->rnorm = flag ? __dsqrt_rn(h->reserved[0]) : (double)__fsqrt_rn((float)h->reserved[0]);
      return;
    case DP_POST_BNORM:
      if (threadIdx.x == 0)
        h->outer_b_norm = flag ? __dsqrt_rn(h->reserved[0]) : (double)__fsqrt_rn((float)h->reserved[0]);
      return;
    default:
      return;
  }
}

template <typename T>
cudaError_t launch_dist_post(int phase, StateView<T> sv, int j, int m_limit, double rtol,
                             double btol, int flag, cudaStream_t st) {
  count_launch();
  k_dist_post<T><<<1, kThreads, 0, st>>>(phase, sv, j, m_limit, rtol, btol, flag);
  return cudaGetLastError();
}
template cudaError_t launch_dist_post<float>(int, StateView<float>, int, int, double, double, int, cudaStream_t);
template cudaError_t launch_dist_post<double>(int, StateView<double>, int, int, double, double, int, cudaStream_t);

// ======================================================================= lsq
// Back-substitution R[:k,:k] d = g[:k] (krylov.py:190-202; LAPACK xTRSV 'U','N'
// column order).  One warp.
template <typename T>
__global__ void k_lsq(StateView<T> sv) {
  kt_mark(sv.h, KC_OTHER);
  const int k = sv.h->steps;
  const int lane = threadIdx.x;
  if (k == 0 || (sv.h->flags & (MPG_FLAG_NONFINITE_OP | MPG_FLAG_NONFINITE_GAMMA | MPG_FLAG_OVERFLOW)))
    return;
  int bad = 0;
  for (int i = lane; i < k; i += 32) {
    const T r = sv.Rc(i, i);
    bad |= (r == T(0)) || !isfinite(r);
    sv.d[i] = sv.g[i];
  }
  bad = __any_sync(0xffffffffu, bad);
  if (bad) {
    if (lane == 0) atomicOr(&sv.h->flags, MPG_FLAG_SINGULAR);
    return;
  }
  __syncwarp();
  for (int jj = k - 1; jj >= 0; --jj) {
    if (lane == 0 && sv.d[jj] != T(0)) sv.d[jj] = div_rn(sv.d[jj], sv.Rc(jj, jj));
    __syncwarp();
    const T temp = sv.d[jj];
    if (temp != T(0))
      for (int i = lane; i < jj; i += 32) sv.d[i] = fma_rn(-temp, sv.Rc(jj, i), sv.d[i]);
    __syncwarp();
  }
}

// ================================================================== combine
// u = V[:, :k] d (solvers.py:171) fused with the update of the iterate.
template <typename T, typename TX, int MODE>
__global__ void __launch_bounds__(kThreads) k_combine(const T* __restrict__ V, long long ldv,
                                                      long long n, StateView<T> sv, TX* x,
                                                      const void* diag, T* u) {
  kt_mark(sv.h, KC_GEMV_N);
  const int k = sv.h->steps;
  if (k == 0 || (sv.h->flags & (MPG_FLAG_NONFINITE_OP | MPG_FLAG_NONFINITE_GAMMA |
                                 MPG_FLAG_OVERFLOW | MPG_FLAG_SINGULAR)))
    return;
  extern __shared__ __align__(128) unsigned char smraw[];
  T* ds = reinterpret_cast<T*>(smraw);
  for (int i = threadIdx.x; i < k; i += blockDim.x) ds[i] = sv.d[i];
  __syncthreads();
  const double rho = sv.h->rho;
  int bad = 0;
  // 16-byte vector loads over VN consecutive rows (k independent loads in flight)
  constexpr int VN = Vec<T>::n;
  const long long nv = n / VN;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < nv + (n - nv * VN); g += stride) {
    T accv[VN];
    long long r0;
    int cnt;
    if (g < nv) {
      r0 = g * VN;
      cnt = VN;
#pragma unroll
      for (int e = 0; e < VN; ++e) accv[e] = T(0);
      int i = 0;
      for (; i + 2 <= k; i += 2) {
        T a[VN], b[VN];
        vload_cs(V + (size_t)i * ldv + r0, a);
        vload_cs(V + (size_t)(i + 1) * ldv + r0, b);
#pragma unroll
        for (int e = 0; e < VN; ++e) accv[e] = fma_rn(b[e], ds[i + 1], fma_rn(a[e], ds[i], accv[e]));
      }
      for (; i < k; ++i) {
        T a[VN];
        vload_cs(V + (size_t)i * ldv + r0, a);
#pragma unroll
        for (int e = 0; e < VN; ++e) accv[e] = fma_rn(a[e], ds[i], accv[e]);
      }
    } else {
      r0 = nv * VN + (g - nv);
      cnt = 1;
      accv[0] = T(0);
      for (int i = 0; i < k; ++i) accv[0] = fma_rn(__ldcs(V + (size_t)i * ldv + r0), ds[i], accv[0]);
    }
    for (int e = 0; e < cnt; ++e) {
    const long long r = r0 + e;
    const T acc = accv[e];
    if constexpr (MODE == CMB_STORE) {
      u[r] = acc;
    } else if constexpr (MODE == CMB_ADD) {
      x[r] = add_rn(x[r], (TX)acc);
    } else if constexpr (MODE == CMB_IR) {
      bad |= !isfinite(acc);
      x[r] = __dadd_rn(x[r], __dmul_rn(rho, (double)acc));
    } else if constexpr (MODE == CMB_J1_ADD) {
      const T y = div_rn(acc, static_cast<const T*>(diag)[r]);
      x[r] = add_rn(x[r], (TX)y);
    } else if constexpr (MODE == CMB_J1_IR) {
      const T y = div_rn(acc, static_cast<const T*>(diag)[r]);
      bad |= !isfinite(y);
      x[r] = __dadd_rn(x[r], __dmul_rn(rho, (double)y));
    } else if constexpr (MODE == CMB_J1_CAST) {
      const float a32 = __double2float_rn((double)acc);
      const float y = __fdiv_rn(a32, static_cast<const float*>(diag)[r]);
      x[r] = __dadd_rn((double)x[r], (double)y);
    }
    }
  }
  if (bad) atomicOr(&sv.h->flags, MPG_FLAG_NONFINITE_X);
}

// ================================================================= launchers

// MPG_FUSE_CS=0 selects the separate K_C + K_S launches (A/B measurement)
// Off by default: measured no change on the graph-replayed cfg2 solve
// (0.513 s vs 0.515 s); MPG_PDL=1 enables it for A/B runs.
bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MPG_PDL");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// PDL on the cooperative K_CS launch (MPG_KCS_PDL=0 to disable)
static bool kcs_pdl() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MPG_KCS_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

bool fuse_update_norm_scale() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MPG_FUSE_CS");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static int g_sms = 0;
int num_sms() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

static unsigned grid_stream(long long n, int per_sm = 8) {
  long long g = (n + kThreads - 1) / kThreads;
  const long long cap = (long long)num_sms() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

template <typename T>
cudaError_t launch_dot1_w(const T* w, long long n, const T* V, long long ldv, int k,
                          StateView<T> sv, WsView ws, cudaStream_t st) {
  long long G = (n + 2047) / 2048;
  const long long cap = (long long)num_sms() * 4;
  if (G > cap) G = cap;
  if (G < 1) G = 1;
  count_launch();
  k_dot1_w<T><<<(unsigned)G, kThreads, 0, st>>>(w, n, V, ldv, k, sv, ws);
  return cudaGetLastError();
}

template <typename T, int KV, int U>
static cudaError_t launch_dot1_wo_k(const T* w, long long n, const T* V, long long ldv, int k,
                                    StateView<T> sv, WsView ws, cudaStream_t st) {
  static std::once_flag once;
  static int occ = 1;
  std::call_once(once, [] {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dot1_wo<T, KV, U>, kThreads, 0);
    cudaGetLastError();
    if (occ < 1) occ = 1;
  });
  const long long blk = (long long)U * 32 * Vec<T>::n;
  long long G = (n + blk - 1) / blk;
  const long long cap = std::min<long long>((long long)num_sms() * occ, kMaxParts);
  if (G > cap) G = cap;
  if (G < 1) G = 1;
  count_launch();
  return launch_k(true, false, k_dot1_wo<T, KV, U>, dim3((unsigned)G), dim3(kThreads), 0, st, w, n, V, ldv,
                  k, sv, ws);
}

// k <= 8: thread-owned small-k kernels (MPG_SMALLK=0 keeps the warp-owned ones)
static bool smallk_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MPG_SMALLK");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <typename K>
static long long small_grid(K kernel, long long n, int vn) {
  static std::once_flag once;
  static int occ = 1;
  std::call_once(once, [&] {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, 0);
    cudaGetLastError();
    if (occ < 1) occ = 1;
  });
  long long G = (n + (long long)kThreads * vn - 1) / ((long long)kThreads * vn);
  const long long cap = std::min<long long>((long long)num_sms() * occ, kMaxParts);
  if (G > cap) G = cap;
  if (G < 1) G = 1;
  return G;
}

template <typename T, int KT>
static cudaError_t launch_dot1_small(const T* w, long long n, const T* V, long long ldv, int k,
                                     StateView<T> sv, WsView ws, cudaStream_t st) {
  const long long G = small_grid(k_dot1_small<T, KT>, n, Vec<T>::n);
  count_launch();
  return launch_k(true, false, k_dot1_small<T, KT>, dim3((unsigned)G), dim3(kThreads), 0, st, w, n, V, ldv, k,
                  sv, ws);
}

template <typename T, int KT>
static cudaError_t launch_update_dot_small(const T* V, long long ldv, long long n, int k, T* w,
                                           StateView<T> sv, WsView ws, cudaStream_t st) {
  const long long G = small_grid(k_update_dot_small<T, KT>, n, Vec<T>::n);
  count_launch();
  return launch_k(true, false, k_update_dot_small<T, KT>, dim3((unsigned)G), dim3(kThreads), 0, st, V, ldv, n,
                  k, w, sv, ws);
}

template <typename T>
cudaError_t launch_dot1_wo(const T* w, long long n, const T* V, long long ldv, int k,
                           StateView<T> sv, WsView ws, cudaStream_t st) {
  if (smallk_enabled() && k <= 8) {
    if (k <= 2) return launch_dot1_small<T, 2>(w, n, V, ldv, k, sv, ws, st);
    if (k <= 4) return launch_dot1_small<T, 4>(w, n, V, ldv, k, sv, ws, st);
    return launch_dot1_small<T, 8>(w, n, V, ldv, k, sv, ws, st);
  }
  switch ((k + kWarps - 1) / kWarps) {
    case 1: return launch_dot1_wo_k<T, 1, 4>(w, n, V, ldv, k, sv, ws, st);
    case 2: return launch_dot1_wo_k<T, 2, 4>(w, n, V, ldv, k, sv, ws, st);
    case 3: return launch_dot1_wo_k<T, 3, 2>(w, n, V, ldv, k, sv, ws, st);
    case 4: return launch_dot1_wo_k<T, 4, 2>(w, n, V, ldv, k, sv, ws, st);
    case 5: return launch_dot1_wo_k<T, 5, 2>(w, n, V, ldv, k, sv, ws, st);
    case 6: return launch_dot1_wo_k<T, 6, 1>(w, n, V, ldv, k, sv, ws, st);
    case 7: return launch_dot1_wo_k<T, 7, 1>(w, n, V, ldv, k, sv, ws, st);
    case 8: return launch_dot1_wo_k<T, 8, 1>(w, n, V, ldv, k, sv, ws, st);
    default: return launch_dot1_w<T>(w, n, V, ldv, k, sv, ws, st);
  }
}

// K_A as two launches, SpMV (w written, L2-resident) + k_dot1_wo, is the
// default: measured on B200 (cfg2, 50-step cycle) 4.80 ms vs 5.53 ms fused in
// fp32 and 8.93 vs 12.29 ms in fp64 -- the fused kernel's SpMV phase and dot
// phase serialise inside each CTA and its registers cap occupancy at 3 CTAs/SM.
// MPG_SPLIT_KA=0 selects the fused kernel (A/B measurement).
bool split_spmv_dot1() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MPG_SPLIT_KA");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <typename T>
cudaError_t launch_update_dot_tma(const T* V, long long ldv, long long n, int k, T* w,
                                  StateView<T> sv, WsView ws, cudaStream_t st);

template <typename T, int KV>
static cudaError_t launch_update_dot_w(const T* V, long long ldv, long long n, int k, T* w,
                                       StateView<T> sv, WsView ws, cudaStream_t st) {
  static std::once_flag once;
  static int occ = 1;
  std::call_once(once, [] {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_update_dot_w<T, KV>, kThreads, 0);
    cudaGetLastError();
    if (occ < 1) occ = 1;
  });
  constexpr long long RB = 32 * Vec<T>::n;
  long long G = (n + RB - 1) / RB;
  const long long cap = (long long)num_sms() * occ;
  if (G > cap) G = cap;
  if (G < 1) G = 1;
  count_launch();
  return launch_k(true, false, k_update_dot_w<T, KV>, dim3((unsigned)G), dim3(kThreads), 0, st, V, ldv, n,
                  k, w, sv, ws);
}

template <typename T>
cudaError_t launch_update_dot(const T* V, long long ldv, long long n, int k, T* w,
                              StateView<T> sv, WsView ws, cudaStream_t st) {
  if (smallk_enabled() && k <= 8) {
    if (k <= 2) return launch_update_dot_small<T, 2>(V, ldv, n, k, w, sv, ws, st);
    if (k <= 4) return launch_update_dot_small<T, 4>(V, ldv, n, k, w, sv, ws, st);
    return launch_update_dot_small<T, 8>(V, ldv, n, k, w, sv, ws, st);
  }
  switch ((k + kWarps - 1) / kWarps) {
    case 1: return launch_update_dot_w<T, 1>(V, ldv, n, k, w, sv, ws, st);
    case 2: return launch_update_dot_w<T, 2>(V, ldv, n, k, w, sv, ws, st);
    case 3: return launch_update_dot_w<T, 3>(V, ldv, n, k, w, sv, ws, st);
    case 4: return launch_update_dot_w<T, 4>(V, ldv, n, k, w, sv, ws, st);
    case 5: return launch_update_dot_w<T, 5>(V, ldv, n, k, w, sv, ws, st);
    case 6: return launch_update_dot_w<T, 6>(V, ldv, n, k, w, sv, ws, st);
    case 7: return launch_update_dot_w<T, 7>(V, ldv, n, k, w, sv, ws, st);
    case 8: return launch_update_dot_w<T, 8>(V, ldv, n, k, w, sv, ws, st);
    default: return launch_update_dot_tma<T>(V, ldv, n, k, w, sv, ws, st);
  }
}

template <typename T>
cudaError_t launch_update_dot_tma(const T* V, long long ldv, long long n, int k, T* w,
                                  StateView<T> sv, WsView ws, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(k_update_dot<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaGetLastError();
  });
  const size_t sz = sizeof(T);
  const size_t budget = 200 * 1024;
  const size_t tail = 16 * 8 + (size_t)(2 * k + 8 + 32) * sz + 64;
  // tile rows: grow while a stage stays <= 48 KB; shrink while 2 stages do not fit
  int TB = 256;
  while (TB < 2048 && (size_t)(k + 1) * (TB * 2) * sz <= 48 * 1024) TB *= 2;
  while (TB > 32 && 2 * (size_t)(k + 1) * TB * sz + tail > budget) TB /= 2;
  if (2 * (size_t)(k + 1) * TB * sz + tail > budget) return cudaErrorInvalidConfiguration;
  const size_t stage = (size_t)(k + 1) * TB * sz;
  int S = (int)std::min<size_t>(4, (budget - tail) / stage);
  if (S < 2) S = 2;
  const size_t smem = (size_t)S * stage + tail;
  int occ = (int)((228 * 1024) / (smem + 1024));
  if (occ < 1) occ = 1;
  if (occ > 4) occ = 4;
  long long tiles = (n + TB - 1) / TB;
  long long G = (long long)num_sms() * occ;
  if (tiles < G) G = tiles;
  if (G > kMaxParts) G = kMaxParts;
  if (G < 1) G = 1;
  count_launch();
  k_update_dot<T><<<(unsigned)G, kUdThreads, smem, st>>>(V, ldv, n, k, w, sv, ws, TB, S);
  return cudaGetLastError();
}

// K_CS grid: the largest co-resident grid (<= 6 CTAs/SM, K_C's occupancy) for
// which the CTA's row slice of w' fits in shared memory; else the uncached
// variant at full occupancy.  Returns 0 when no cooperative grid is possible.
template <typename T>
struct UnsPlan { unsigned grid = 0; size_t smem = 0; bool cache = false; };
// leading shared-memory region of K_CS: the c2 coefficients during phase 1,
// then the warp-staged Givens scratch (>= 3m + 2 elements)
static inline int kcs_kpad(int m) { return std::max((m + 16) & ~7, (3 * m + 2 + 7) & ~7); }

template <typename T>
static UnsPlan<T> plan_update_norm_scale(long long n, int m) {
  static std::once_flag once;
  static int dev_smem_optin = 0;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&dev_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(k_update_norm_scale<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         dev_smem_optin - 1024);
    cudaFuncSetAttribute(k_update_norm_scale<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kcs_kpad(kMaxM) * (int)sizeof(T));
    cudaGetLastError();
  });
  UnsPlan<T> p;
  constexpr int VN = Vec<T>::n;
  const int kpad = kcs_kpad(m);
  const size_t base = (size_t)kpad * sizeof(T);
  long long tiles = (n + (long long)kThreads * VN - 1) / ((long long)kThreads * VN);
  if (tiles < 1) tiles = 1;
  for (int occ = 6; occ >= 1; --occ) {
    long long G = std::min<long long>((long long)num_sms() * occ, tiles);
    // grid-stride groups: each CTA caches ceil(groups / (G * kThreads)) * kThreads groups
    const long long groups = (n + VN - 1) / VN;
    const long long rows = (groups + G * kThreads - 1) / (G * kThreads) * kThreads * VN;
    const size_t smem = base + (size_t)rows * sizeof(T);
    if (smem > (size_t)(dev_smem_optin - 1024)) continue;
    int got = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&got, k_update_norm_scale<T, true>, kThreads, smem) !=
        cudaSuccess) { cudaGetLastError(); continue; }
    if ((long long)got * num_sms() >= G) { p.grid = (unsigned)G; p.smem = smem; p.cache = true; return p; }
  }
  int got = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&got, k_update_norm_scale<T, false>, kThreads, base) ==
          cudaSuccess && got >= 1) {
    p.grid = (unsigned)std::min<long long>((long long)num_sms() * std::min(got, 6), tiles);
    p.smem = base;
    p.cache = false;
  }
  cudaGetLastError();
  return p;
}

template <typename T>
cudaError_t launch_update_norm(const T* V, long long ldv, long long n, int j, T* w,
                               StateView<T> sv, WsView ws, int m_limit, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(k_update_norm<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (kMaxM + 8) * (int)sizeof(T));
  });
  constexpr int VN = Vec<T>::n;
  long long G = (n + (long long)kThreads * VN - 1) / ((long long)kThreads * VN);
  const long long cap = (long long)num_sms() * 6;
  if (G > cap) G = cap;
  if (G < 1) G = 1;
  // the fused K_CS grid when there is one: identical partials and norm
  const unsigned pg = plan_update_norm_scale<T>(n, sv.m).grid;
  if (pg) G = pg;
  count_launch();
  k_update_norm<T><<<(unsigned)G, kThreads, (size_t)(j + 9) * sizeof(T), st>>>(V, ldv, n, j, w, sv, ws,
                                                                                 m_limit);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_update_norm_scale(const T* V, long long ldv, long long n, int j, T* w,
                                     StateView<T> sv, WsView ws, int m_limit, cudaStream_t st) {
  if (j + 1 > sv.m) return cudaErrorInvalidValue;
  const UnsPlan<T> p = plan_update_norm_scale<T>(n, sv.m);
  if (!p.grid) {   // no co-resident grid: separate K_C + K_S
    const cudaError_t e = launch_update_norm<T>(V, ldv, n, j, w, sv, ws, m_limit, st);
    if (e != cudaSuccess) return e;
    return launch_step_scale<T>(w, const_cast<T*>(V) + (size_t)(j + 1) * ldv, n, j, sv, st);
  }
  const int kpad = kcs_kpad(sv.m);
  count_launch();
  const bool pdl = kcs_pdl();
  if (p.cache)
    return launch_k(pdl, true, k_update_norm_scale<T, true>, dim3(p.grid), dim3(kThreads), p.smem, st, V, ldv,
                    n, j, w, sv, ws, m_limit, kpad);
  return launch_k(pdl, true, k_update_norm_scale<T, false>, dim3(p.grid), dim3(kThreads), p.smem, st, V, ldv,
                  n, j, w, sv, ws, m_limit, kpad);
}

template <typename T>
cudaError_t launch_step_scale(const T* w, T* vnext, long long n, int j, StateView<T> sv,
                              cudaStream_t st) {
  count_launch();
  k_step_scale<T><<<grid_stream((n + Vec<T>::n - 1) / Vec<T>::n), kThreads, 0, st>>>(w, vnext, n, j, sv);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_start(const T* r0, long long n, StateView<T> sv, double rtol,
                         const double* b_norm_src, double btol, WsView ws, cudaStream_t st) {
  count_launch();
  k_start<T><<<grid_stream(n, 4), kThreads, 0, st>>>(r0, n, sv, rtol, b_norm_src, btol, ws);
  return cudaGetLastError();
}

cudaError_t launch_start_ir(const double* r64, float* r32, long long n, StateView<float> sv,
                            double rtol, double btol, WsView ws, cudaStream_t st) {
  count_launch();
  k_start_ir<<<grid_stream(n, 4), kThreads, 0, st>>>(r64, r32, n, sv, rtol, btol, ws);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_start_scale(const T* r0, T* v0, long long n, StateView<T> sv, cudaStream_t st) {
  count_launch();
  k_start_scale<T><<<grid_stream(n), kThreads, 0, st>>>(r0, v0, n, sv);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_lsq(StateView<T> sv, cudaStream_t st) {
  count_launch();
  k_lsq<T><<<1, 32, 0, st>>>(sv);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_combine(const T* V, long long ldv, long long n, StateView<T> sv, int mode,
                           void* x, const void* diag, T* u, cudaStream_t st) {
  const unsigned G = grid_stream((n + Vec<T>::n - 1) / Vec<T>::n, 6);
  const size_t smem = (size_t)(sv.m + 1) * sizeof(T);
  count_launch();
  switch (mode) {
    case CMB_STORE:
      k_combine<T, T, CMB_STORE><<<G, kThreads, smem, st>>>(V, ldv, n, sv, (T*)x, diag, u);
      break;
    case CMB_ADD:
      k_combine<T, T, CMB_ADD><<<G, kThreads, smem, st>>>(V, ldv, n, sv, (T*)x, diag, u);
      break;
    case CMB_J1_ADD:
      k_combine<T, T, CMB_J1_ADD><<<G, kThreads, smem, st>>>(V, ldv, n, sv, (T*)x, diag, u);
      break;
    case CMB_IR:
      if constexpr (sizeof(T) == 4)
        k_combine<T, double, CMB_IR><<<G, kThreads, smem, st>>>(V, ldv, n, sv, (double*)x, diag, u);
      else
        return cudaErrorInvalidValue;
      break;
    case CMB_J1_IR:
      if constexpr (sizeof(T) == 4)
        k_combine<T, double, CMB_J1_IR><<<G, kThreads, smem, st>>>(V, ldv, n, sv, (double*)x, diag, u);
      else
        return cudaErrorInvalidValue;
      break;
    case CMB_J1_CAST:
      if constexpr (sizeof(T) == 8)
        k_combine<T, double, CMB_J1_CAST><<<G, kThreads, smem, st>>>(V, ldv, n, sv, (double*)x, diag, u);
      else
        return cudaErrorInvalidValue;
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

#define INST(T)                                                                                  \
  template cudaError_t launch_dot1_w<T>(const T*, long long, const T*, long long, int,          \
                                        StateView<T>, WsView, cudaStream_t);                   \
  template cudaError_t launch_update_dot<T>(const T*, long long, long long, int, T*,            \
                                            StateView<T>, WsView, cudaStream_t);               \
  template cudaError_t launch_dot1_wo<T>(const T*, long long, const T*, long long, int,         \
                                         StateView<T>, WsView, cudaStream_t);                  \
  template cudaError_t launch_update_norm<T>(const T*, long long, long long, int, T*,           \
                                             StateView<T>, WsView, int, cudaStream_t);         \
  template cudaError_t launch_step_scale<T>(const T*, T*, long long, int, StateView<T>,         \
                                            cudaStream_t);                                     \
  template cudaError_t launch_update_norm_scale<T>(const T*, long long, long long, int, T*,     \
                                                   StateView<T>, WsView, int, cudaStream_t);   \
  template cudaError_t launch_step_scale_peer<T>(const T*, T*, long long, long long, int,       \
                                                 StateView<T>, T*, T*, uint32_t*, uint32_t*,   \
                                                 WsView, cudaStream_t);                        \
  template cudaError_t launch_start<T>(const T*, long long, StateView<T>, double, const double*, \
                                       double, WsView, cudaStream_t);                          \
  template cudaError_t launch_start_scale<T>(const T*, T*, long long, StateView<T>,             \
                                             cudaStream_t);                                    \
  template cudaError_t launch_lsq<T>(StateView<T>, cudaStream_t);                               \
  template cudaError_t launch_combine<T>(const T*, long long, long long, StateView<T>, int,     \
                                         void*, const void*, T*, cudaStream_t);
INST(float)
INST(double)
#undef INST

}  // namespace mpg
