// Shared device helpers for the B200 mixed-precision GMRES kernels (sm_100a).
//
// Conventions
//  * T is float (fp32 working precision) or double (fp64).
//  * Every vector the library owns is padded to `ld` elements (a multiple of
//    64), so 16-byte vector loads and TMA bulk copies never run past an
//    allocation.  CSR arrays are 16-byte aligned with >= 16 bytes of
//    readable padding (the Python layer guarantees both).
//  * Reductions are deterministic: per-CTA partials in a fixed order, then a
//    fixed-order grid finalisation by the last CTA to arrive (no float
//    atomics), so repeated runs are bitwise identical.
//  * Parity-critical arithmetic (SpMV products/sums, Givens scalars, the IR
//    correction, preconditioner epilogues) uses explicit _rn intrinsics so
//    nvcc never contracts a multiply and an add into an FMA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mpgmres_b200.h"

namespace mpg {

constexpr int kThreads = 256;           // threads per CTA for streaming kernels
constexpr int kWarps = kThreads / 32;
constexpr int kRowAlign = 32;           // CTA row ranges start on 32-row boundaries

// ---------------------------------------------------------------------------
// exact-rounding scalar ops (no FMA contraction)
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

template <typename T> struct Vec;           // 16-byte vector of T
template <> struct Vec<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec<double> { using type = double2; static constexpr int n = 2; };

template <typename T>
__device__ __forceinline__ void vload(const T* p, T (&v)[Vec<T>::n]) {
  auto q = __ldg(reinterpret_cast<const typename Vec<T>::type*>(p));
  if constexpr (Vec<T>::n == 4) { v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w; }
  else { v[0] = q.x; v[1] = q.y; }
}
// streaming (evict-first) load: for data read exactly once per kernel
template <typename T>
__device__ __forceinline__ void vload_cs(const T* p, T (&v)[Vec<T>::n]) {
#ifdef MPG_BASIS_LDG
  auto q = __ldg(reinterpret_cast<const typename Vec<T>::type*>(p));   // A/B: keep the basis in L2
#else
  auto q = __ldcs(reinterpret_cast<const typename Vec<T>::type*>(p));
#endif
  if constexpr (Vec<T>::n == 4) { v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w; }
  else { v[0] = q.x; v[1] = q.y; }
}
// L2 (coherent) load: for data written earlier in the same launch
template <typename T>
__device__ __forceinline__ void vload_cg(const T* p, T (&v)[Vec<T>::n]) {
  auto q = __ldcg(reinterpret_cast<const typename Vec<T>::type*>(p));
  if constexpr (Vec<T>::n == 4) { v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w; }
  else { v[0] = q.x; v[1] = q.y; }
}
template <typename T>
__device__ __forceinline__ void vload_smem(const T* p, T (&v)[Vec<T>::n]) {
  auto q = *reinterpret_cast<const typename Vec<T>::type*>(p);
  if constexpr (Vec<T>::n == 4) { v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w; }
  else { v[0] = q.x; v[1] = q.y; }
}
template <typename T>
__device__ __forceinline__ void vstore(T* p, const T (&v)[Vec<T>::n]) {
  typename Vec<T>::type q;
  if constexpr (Vec<T>::n == 4) { q.x = v[0]; q.y = v[1]; q.z = v[2]; q.w = v[3]; }
  else { q.x = v[0]; q.y = v[1]; }
  *reinterpret_cast<typename Vec<T>::type*>(p) = q;
}

// ---------------------------------------------------------------------------
// deterministic reductions

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-tree block sum; result valid in every thread.  `red` needs kWarps slots.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  T t = (l < (int)(blockDim.x >> 5)) ? red[l] : T(0);
  t = warp_sum(t);
  return t;
}

// Last-CTA election after each CTA has published its partials.
// Returns true in every thread of the last CTA to arrive.  The counter is
// reset by the elected CTA so the slot can be reused by the next kernel on
// the same stream.
#ifndef MPG_RED_ACQREL
#define MPG_RED_ACQREL 1
#endif
__device__ __forceinline__ unsigned atom_add_acqrel_u32(unsigned* p) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}
__device__ __forceinline__ bool last_cta(unsigned int* counter) {
  __shared__ bool is_last;
#if MPG_RED_ACQREL
  // acq_rel election: bar.sync + thread 0's cumulative release publish the
  // CTA's stores; the elected CTA's acquire + bar.sync order its loads after
  // every CTA's stores (no SC fences on the tail's critical path)
  __syncthreads();
  if (threadIdx.x == 0) is_last = atom_add_acqrel_u32(counter) == gridDim.x - 1;
  __syncthreads();
  if (is_last && threadIdx.x == 0) *counter = 0u;
#else
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0u;
  }
#endif
  return is_last;
}

// Sum `ncols` columns of a [nparts][stride] partial array in a fixed order.
// Executed by one whole CTA; column c's total lands in out[c] (any writer).
// Warp w handles columns c = w, w + kWarps, ...; lanes stride over parts.
template <typename T, typename OutF>
__device__ __forceinline__ void finalize_columns(const T* part, int nparts, int stride,
                                                 int ncols, OutF out) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int c = w; c < ncols; c += (int)(blockDim.x >> 5)) {
    T s = T(0);
    for (int p = l; p < nparts; p += 32) s += __ldcg(part + (size_t)p * stride + c);
    s = warp_sum(s);
    if (l == 0) out(c, s);
  }
}

// Two-level deterministic grid reduction of `ncols` per-CTA partials, in
// place of a single last CTA summing every partial (measured ~11 us of
// serialised L2 latency per launch at 592 CTAs x 30 columns on B200).
// part is column-major, part[c * ldp + blockIdx.x], written by each CTA before
// the call.  CTAs form groups of GS consecutive blocks; the last CTA to
// arrive in a group sums the group's partials (one lane per CTA, fixed tree)
// into gpart[c * 64 + group]; the last group to finish sums the group
// partials in the same fixed way and calls out(c, total).  The order depends
// only on gridDim.x, so results are reproducible.  gcount[0..ngroups] must be
// zero on entry and are left zero.  Returns true in the CTA that called out.
// columns per warp with loads in flight together in grid_reduce_cols' two
// stages.  fp32: 8 (cfg2 IR four-launch 0.478 -> 0.470 s with the acq_rel
// elections); fp64: 1 (the batch costs the register-capped K_B spills: cfg2
// fp64 0.911 at 8 vs 0.908 s at 1; profiles/r2_ab_grid_reduce.log)
#ifndef MPG_RED_CB32
#define MPG_RED_CB32 8
#endif
#ifndef MPG_RED_CB64
#define MPG_RED_CB64 1
#endif
template <int GS, typename T, typename OutF>
__device__ __forceinline__ bool grid_reduce_cols(const T* part, int ldp, T* gpart,
                                                 unsigned int* gcount, int ncols, OutF out) {
  __shared__ bool s_last;
  const int G = gridDim.x, b = blockIdx.x;
  const int g = b / GS, ng = (G + GS - 1) / GS;
  const int gsz = min(GS, G - g * GS);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
#if MPG_RED_ACQREL
  // elections by acq_rel atomics: bar.sync orders the CTA's partial stores
  // before thread 0's (cumulative) release; its acquire + bar.sync orders the
  // elected CTA's loads after every group member's stores -- no SC fences
  __syncthreads();
  if (threadIdx.x == 0) s_last = atom_add_acqrel_u32(&gcount[1 + g]) == (unsigned)(gsz - 1);
  __syncthreads();
  if (!s_last) return false;
#else
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&gcount[1 + g], 1u) == (unsigned)(gsz - 1);
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
#endif
  // stage 1: this group's gsz <= 32 partials, one lane each, warp per column
  // (columns c, c + nw, ... of a warp: kRedCB of them with their loads in
  // flight together, then the same per-column shuffle trees)
  constexpr int kRedCB = sizeof(T) == 8 ? MPG_RED_CB64 : MPG_RED_CB32;
  for (int c0 = w; c0 < ncols; c0 += nw * kRedCB) {
    T v[kRedCB];
#pragma unroll
    for (int i = 0; i < kRedCB; ++i) {
      const int c = c0 + i * nw;
      v[i] = (c < ncols && l < gsz) ? __ldcg(part + (size_t)c * ldp + g * GS + l) : T(0);
    }
#pragma unroll
    for (int i = 0; i < kRedCB; ++i) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
      if (l == 0 && c0 + i * nw < ncols) gpart[(size_t)(c0 + i * nw) * 64 + g] = v[i];
    }
  }
#if MPG_RED_ACQREL
  __syncthreads();
  if (threadIdx.x == 0) {
    gcount[1 + g] = 0u;
    s_last = atom_add_acqrel_u32(&gcount[0]) == (unsigned)(ng - 1);
  }
  __syncthreads();
  if (!s_last) return false;
#else
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    gcount[1 + g] = 0u;
    s_last = atomicAdd(&gcount[0], 1u) == (unsigned)(ng - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
#endif
  // stage 2: ng <= 64 group partials, two per lane in a fixed order
  for (int c0 = w; c0 < ncols; c0 += nw * kRedCB) {
    T a[kRedCB], b2[kRedCB];
#pragma unroll
    for (int i = 0; i < kRedCB; ++i) {
      const T* gp = gpart + (size_t)(c0 + i * nw) * 64;
      const bool in = c0 + i * nw < ncols;
      a[i] = in && l < ng ? __ldcg(gp + l) : T(0);
      b2[i] = in && l + 32 < ng ? __ldcg(gp + l + 32) : T(0);
    }
#pragma unroll
    for (int i = 0; i < kRedCB; ++i) {
      T v = a[i];
      if (l + 32 < ng) v += b2[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (l == 0 && c0 + i * nw < ncols) out(c0 + i * nw, v);
    }
  }
  if (threadIdx.x == 0) gcount[0] = 0u;
  return true;
}

// Contiguous, 32-row aligned partition of [0, n) over gridDim.x CTAs.
__device__ __forceinline__ void cta_rows(long long n, long long& r0, long long& r1) {
  const long long G = gridDim.x, c = blockIdx.x;
  r0 = (c * n / G) & ~(long long)(kRowAlign - 1);
  r1 = (c + 1 == G) ? n : (((c + 1) * n / G) & ~(long long)(kRowAlign - 1));
  if (r1 < r0) r1 = r0;
}

// ---------------------------------------------------------------------------
// Per-thread asynchronous global -> shared copies (cp.async, SASS LDGSTS):
// no register staging, so a warp keeps a whole chunk's loads in flight.
template <int B>
__device__ __forceinline__ void cp_async_ca(void* smem, const void* g) {
  static_assert(B == 4 || B == 8 || B == 16, "cp.async sizes");
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(g), "n"(B)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---------------------------------------------------------------------------
// mbarrier + TMA bulk copy (cp.async.bulk, SASS UBLKCP) helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 1-D bulk global->shared copy; dst/src 16-byte aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// numpy add.reduceat row order (spmv.py:63-70): y = p0 + pairwise(p1..p_{L-1})
// where pairwise is numpy's pairwise_sum: sequential from -0.0 below 8 terms,
// 8 interleaved accumulators up to 128, recursive halving above.

// 8 <= n <= 128: eight interleaved accumulators, tree, sequential remainder
template <typename T, typename Get>
__device__ __forceinline__ T pairwise_block(const Get& get, int i0, int n) {
  T r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = get(i0 + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = add_rn(r[j], get(i0 + i + j));
  }
  T res = add_rn(add_rn(add_rn(r[0], r[1]), add_rn(r[2], r[3])),
                 add_rn(add_rn(r[4], r[5]), add_rn(r[6], r[7])));
  for (; i < n; ++i) res = add_rn(res, get(i0 + i));
  return res;
}

// numpy's recursive halving (n2 = n/2 rounded down to a multiple of 8) for
// n > 128, evaluated post-order with an explicit stack: no device-side call,
// so the common short-row path keeps every register.
template <typename T, typename Get>
__device__ __forceinline__ T pairwise_split(const Get& get, int i0, int n) {
  int si[32], sn[32], ss[32];
  T sv[32];
  int sp = 0;
  si[0] = i0; sn[0] = n; ss[0] = 0;
  T ret = T(0);
  while (sp >= 0) {
    const int cn = sn[sp];
    if (cn <= 128) {
      ret = pairwise_block<T>(get, si[sp], cn);
      --sp;
      continue;
    }
    const int n2 = cn / 2 - (cn / 2) % 8;
    if (ss[sp] == 0) {
      ss[sp] = 1;
      si[sp + 1] = si[sp]; sn[sp + 1] = n2; ss[sp + 1] = 0;
      ++sp;
    } else if (ss[sp] == 1) {
      sv[sp] = ret;
      ss[sp] = 2;
      si[sp + 1] = si[sp] + n2; sn[sp + 1] = cn - n2; ss[sp + 1] = 0;
      ++sp;
    } else {
      ret = add_rn(sv[sp], ret);
      --sp;
    }
  }
  return ret;
}

template <typename T, typename Get>
__device__ __forceinline__ T pairwise(const Get& get, int i0, int n) {
  if (n < 8) {
    T r = T(-0.0);
    for (int i = 0; i < n; ++i) r = add_rn(r, get(i0 + i));
    return r;
  }
  if (n <= 128) return pairwise_block<T>(get, i0, n);
  return pairwise_split<T>(get, i0, n);
}

// row_reduce over precomputed products p[0..len), len <= N <= 8: the same
// association (p0 + sequential sum of p1.. from -0.0, numpy's n < 8 path)
template <typename T, int N>
__device__ __forceinline__ T row_sum_short(const T (&p)[N], int len) {
  static_assert(N <= 8, "pairwise's sequential branch covers fewer than 8 terms after p0");
  if (len <= 0) return T(0);
  if (len == 1) return p[0];
  T r = T(-0.0);
#pragma unroll
  for (int i = 1; i < N; ++i)
    if (i < len) r = add_rn(r, p[i]);
  return add_rn(p[0], r);
}

template <typename T, typename Get>
__device__ __forceinline__ T row_reduce(const Get& get, int len) {
  if (len <= 0) return T(0);
  T p0 = get(0);
  if (len == 1) return p0;
  return add_rn(p0, pairwise<T>(get, 1, len - 1));
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  Kernels of the Arnoldi step are
// launched with programmatic stream serialisation: a kernel may be scheduled
// while its predecessor drains, runs until pdl_wait() (griddepcontrol.wait:
// returns once the predecessor grid has completed and its writes are
// visible; a no-op for a normal launch), and lets its own successor launch
// early with pdl_trigger().  Every kernel launched with launch_k(pdl = true)
// calls pdl_wait() before it reads anything a predecessor wrote.
// System-scope release / acquire (peer-memory flags across GPUs / processes).
__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin until *p >= want (wrap-safe), bounded: ~20 s of SM clock, then false.
__device__ __forceinline__ bool wait_seq_sys(const uint32_t* p, uint32_t want) {
  const unsigned long long t0 = clock64(), limit = 40ull * 1000 * 1000 * 1000;
  int spins = 0;
  while ((int32_t)(ld_acquire_sys_u32(p) - want) < 0) {
    if (clock64() - t0 > limit) return false;
    if (++spins > 64) __nanosleep(32);   // tight spin first: the wait is usually short
  }
  return true;
}

// Prefetch the 128-byte line holding p into L2 (no register, no scoreboard).
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// Bulk (TMA-engine) prefetch of `bytes` (multiple of 16, 16-byte aligned) into L2.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------------------
// Device kernel-time attribution (the reference's KernelTimer categories,
// timing.py:17-23; header fields ktime_ns / kt_mark / kt_cat).  CTA 0 thread 0
// of each kernel of a cycle stamps %globaltimer once at entry; the interval
// since the previous stamp is charged to the category that stamp opened.
// Kernels on a stream run in order, so one thread per kernel suffices and no
// atomics are needed.  KC_OTHER is not stored (host: total - sum).
enum KtCat { KC_SPMV = 0, KC_GEMV_T = 1, KC_NORM = 2, KC_GEMV_N = 3, KC_OTHER = 4,
             KC_GEMV_TN = 5 /* fused update + dots: half GemvNoTrans, half GemvTrans */ };
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Unconditional stamp (the caller picks the thread).
__device__ __forceinline__ void kt_stamp(const mpg_state_header* hc, int cat) {
  mpg_state_header* h = const_cast<mpg_state_header*>(hc);
  const unsigned long long now = gtimer_ns();
  const int prev = h->kt_cat;
  const unsigned long long d = now - h->kt_mark;
  if (h->kt_mark == 0) {
    // first stamp since the reset (mpg_solver_begin / a zeroed state): opens only
  } else if (prev >= 0 && prev < 4) {
    h->ktime_ns[prev] += d;
  } else if (prev == KC_GEMV_TN) {
    h->ktime_ns[KC_GEMV_N] += d / 2;
    h->ktime_ns[KC_GEMV_T] += d - d / 2;
  }
  h->kt_mark = now;
  h->kt_cat = cat;
}
// Kernel-entry stamp: CTA 0, thread 0; null header = untimed launch.
__device__ __forceinline__ void kt_mark(const mpg_state_header* h, int cat) {
  if (h != nullptr && blockIdx.x == 0 && threadIdx.x == 0) kt_stamp(h, cat);
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------------------
// launch helpers (host)
int num_sms();
int grid_for(long long rows, int rows_per_tile, int ctas_per_sm);
bool pdl_enabled();   // MPG_PDL=0 disables programmatic dependent launches

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(bool pdl, bool coop, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                            size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl && pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (coop) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace mpg
