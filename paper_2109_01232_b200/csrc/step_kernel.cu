// Persistent per-step Arnoldi kernel for stencil storage (single GPU).
//
// One cooperative launch runs a whole CGS2 Arnoldi step (krylov.py:112-151 +
// givens_update :154-187) on 148 CTAs of 1024 threads (one per SM).  Each CTA
// owns a fixed set of 32*VN-row blocks (dealt round-robin over the grid) for
// every phase, so the new vector w = A v_j never leaves shared memory:
//
//   P1   w = A v_j for the CTA's rows (stencil_group, bit-exact SpMV);
//        ||w||^2 and the finite flag; w kept in shared memory
//   P1b  pass-1 dots c1 = V^T w: four row groups of 8 warps, warp owns
//        basis vectors gw + 8q (16-byte lane slices, KV accumulators)
//   B1   grid barrier; every CTA sums the 148 CTA partials of each column in
//        the same fixed order (warp per column) -> c1, w0, flag
//   P2   w' = w - V c1 (8 warp partials of u summed per row in warp order
//        through shared memory) and pass-2 dots c2 = V^T w' from the same
//        registers: the basis is read once for both halves
//   B2   grid barrier; c2; CTA 0 writes c1, c2 and the Hessenberg column
//   P3   w'' = w' - V c2, ||w''||^2
//   B3   grid barrier; h_sub; breakdown test; CTA 0 rotates the column
//        (givens_column) and sets the done flag
//   P4   V[:, j+1] = w'' / h_sub for the CTA's rows (IEEE division)
//
// Against the four-launch step (K_A1, K_A2, K_B, K_CS) this removes three
// kernel boundaries and their reduction tails, and w's global write and its
// three re-reads.  When a CTA's rows do not fit in shared memory (n >~ 13M
// rows fp32 / 6.5M fp64) the CACHE = false variant keeps w in global memory.
// The basis is swept three times per step, as in the four-launch path.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "arnoldi_common.cuh"
#include "spmv.cuh"
#include "state.cuh"

namespace mpg {

constexpr int kMegaThreads = 1024;
constexpr int kMegaWarps = kMegaThreads / 32;
constexpr int kMegaGroups = kMegaWarps / 8;   // row groups of 8 warps
constexpr int kMegaMaxCols = 72;              // k + 2 <= kMegaMaxCols (m <= 64)
// column blocks of the (column-major) partial array, one per barrier, so a fast
// CTA never overwrites partials a slow CTA is still summing
constexpr int kColDot1 = 0;
constexpr int kColDot2 = kMegaMaxCols;
constexpr int kColNorm = 2 * kMegaMaxCols;
// L2 bulk prefetch of basis blocks ahead of the barrier-paced phases (A/B: -DMPG_MEGA_PF=0)
#ifndef MPG_MEGA_PF
#define MPG_MEGA_PF 1
#endif

#ifdef MPG_MEGA_TIMING
// A/B instrumentation (tools/mega_phases.py): per-CTA globaltimer stamps at the
// phase boundaries of step MPG_MEGA_TIMING
__device__ unsigned long long g_mega_t[148 * 2][10];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define MEGA_STAMP(i) \
  if (j == MPG_MEGA_TIMING && threadIdx.x == 0 && blockIdx.x < 296) g_mega_t[blockIdx.x][i] = gtimer();
extern "C" int mpg_debug_mega_times(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_mega_t, sizeof(g_mega_t));
}
#else
#define MEGA_STAMP(i)
#endif

// P2 blocks per barrier pair: 2 while the doubled basis registers fit the
// 64-register budget of 1024-thread CTAs (fp32 KV <= 4, fp64 KV <= 3: no or
// few-byte spills).  Measured at cfg2 IR: P2 64.5 -> 62.3 us at k = 27, solve
// 0.500 -> 0.4925 s; bitwise identical iterates.  A/B: -DMPG_MEGA_U2_KV=0.
#ifndef MPG_MEGA_U2_KV
#define MPG_MEGA_U2_KV 4
#endif
template <typename T, int KV>
struct MegaU {
  static constexpr int u = KV <= (sizeof(T) == 8 ? (MPG_MEGA_U2_KV < 3 ? MPG_MEGA_U2_KV : 3) : MPG_MEGA_U2_KV) ? 2 : 1;
};

__device__ __forceinline__ void group_sync(int grp) {
  asm volatile("bar.sync %0, 256;" ::"r"(grp + 1) : "memory");
}

// Sum column `col` of the CTA partials in a fixed order (warp-level), all lanes
// get it: lane l adds partials l, l + 32, ... in turn, then the warp tree.  The
// (up to 5 per lane at G <= 160) loads are issued together before the adds, so
// the sums after a grid barrier cost one L2 round trip instead of two (the
// compiler's remainder-then-unroll-by-4 loop serialised them).
template <typename T>
__device__ __forceinline__ T sum_column(const T* part, int col, int G) {
  const int lane = threadIdx.x & 31;
  const T* pc = part + (size_t)col * kMaxParts;
  constexpr int NL = 5;
  T v[NL];
#pragma unroll
  for (int i = 0; i < NL; ++i) v[i] = lane + 32 * i < G ? __ldcg(pc + lane + 32 * i) : T(0);
  T s = T(0);
#pragma unroll
  for (int i = 0; i < NL; ++i)
    if (lane + 32 * i < G) s += v[i];
  for (int p = lane + 32 * NL; p < G; p += 32) s += __ldcg(pc + p);
  return warp_sum(s);
}

// Two columns per warp (col0 and col1 when has1), all loads in flight together;
// each column summed exactly as sum_column sums it.
template <typename T>
__device__ __forceinline__ void sum_column2(const T* part, int col0, int col1, bool has1, int G, T& s0, T& s1) {
  const int lane = threadIdx.x & 31;
  const T* p0 = part + (size_t)col0 * kMaxParts;
  const T* p1 = part + (size_t)col1 * kMaxParts;
  constexpr int NL = 5;
  T v0[NL], v1[NL];
#pragma unroll
  for (int i = 0; i < NL; ++i) {
    const bool in = lane + 32 * i < G;
    v0[i] = in ? __ldcg(p0 + lane + 32 * i) : T(0);
    v1[i] = in && has1 ? __ldcg(p1 + lane + 32 * i) : T(0);
  }
  T a = T(0), b = T(0);
#pragma unroll
  for (int i = 0; i < NL; ++i)
    if (lane + 32 * i < G) {
      a += v0[i];
      b += v1[i];
    }
  for (int p = lane + 32 * NL; p < G; p += 32) {
    a += __ldcg(p0 + p);
    if (has1) b += __ldcg(p1 + p);
  }
  s0 = warp_sum(a);
  s1 = warp_sum(b);
}

// Grid barrier on a monotonic 64-bit arrival counter (the step kernel's own
// word in the workspace, zero at creation; every launch passes its barriers
// uniformly, so the counter is a multiple of G at each launch's start): each
// CTA's arrival is one acq_rel atomic add, whose old value names the barrier's
// target; the CTAs poll the counter itself.  Against the count + generation
// barrier (arnoldi_common.cuh) this drops the generation read before the
// arrival and the last arriver's reset + release after it: two L2 round trips
// off each barrier's critical path.
#ifndef MPG_MEGA_MONO
#define MPG_MEGA_MONO 1
#endif
#ifndef MPG_MONO_SLEEP
#define MPG_MONO_SLEEP 0
#endif
__device__ __forceinline__ void grid_barrier_mono(unsigned long long* cnt) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long old;
    asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(cnt) : "memory");
    const unsigned long long G = gridDim.x;
    const unsigned long long target = old - old % G + G;
    if (old + 1 != target) {
      unsigned long long v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
        if ((long long)(v - target) >= 0) break;
        if (MPG_MONO_SLEEP > 0) __nanosleep(MPG_MONO_SLEEP);   // A/B: back off the counter's L2 line
      }
    }
  }
  __syncthreads();
}
// The counter word (bytes 64 / 72 of the workspace for fp32 / fp64) belongs to
// the step kernel of one solver, whose row count and precision -- hence G --
// are fixed for the workspace's lifetime (solvers.py: one workspace per
// NativeSolve / distributed solver).
template <typename T>
__device__ __forceinline__ void mega_barrier(const WsView& ws) {
  if (MPG_MEGA_MONO) grid_barrier_mono(reinterpret_cast<unsigned long long*>(ws.counter + (sizeof(T) == 8 ? 18 : 16)));
  else grid_barrier(ws.counter, ws.counter + 1);
}

// Distributed persistent step (DIST, MPG_PH_STEP): the same kernel on one
// rank's rows, with each of the three reductions finished across ranks inside
// the kernel: after the local grid barrier CTA 0 pushes this rank's column
// sums into every rank's exchange box (peer stores) and release-stores the
// step's sequence number; every CTA acquire-waits for all ranks' entries in
// its own box and sums them in rank order (identical bits on every rank, and
// bitwise the single-GPU step at one rank).  The halo planes of V[:, j+1] are
// stored straight into the neighbours' basis rows in P4; the next step's
// kernel releases them at entry and waits for its own.
template <typename T>
__device__ __forceinline__ void mega_xsum(const MegaX<T>& X, int p, int ncols, uint32_t seqv, T* col,
                                          mpg_state_header* h) {
  const int tid = threadIdx.x;
  void* self = X.box[X.rank];
  if (blockIdx.x == 0) {   // col[] holds this rank's sums (all CTAs computed them; CTA 0 sends)
    for (int idx = tid; idx < X.world * ncols; idx += blockDim.x) {
      const int r = idx / ncols, c = idx - r * ncols;
      xbox_vals<T>(X.box[r], p, X.rank)[c] = col[c];
    }
    // bar.sync orders the CTA's value stores before the (cumulative) system-
    // scope release of the sequence number: no separate fence.sc.sys
    __syncthreads();
    if (tid < X.world) st_release_sys_u32(xbox_seq(X.box[tid], p, X.rank), seqv);
  }
  if (tid < X.world && !wait_seq_sys(xbox_seq(self, p, tid), seqv)) {
    atomicOr(&h->flags, MPG_FLAG_HALO_TIMEOUT);   // a rank never arrived: finish flagged, no hang
    h->done = 1;
  }
  __syncthreads();
  if (tid < ncols) {
    T s = __ldcg(xbox_vals<T>(self, p, 0) + tid);
    for (int r = 1; r < X.world; ++r) s += __ldcg(xbox_vals<T>(self, p, r) + tid);
    col[tid] = s;
  }
  __syncthreads();
}

template <typename T, int S, int KV, bool CACHE, bool KONST, bool DIST>
__global__ void __launch_bounds__(kMegaThreads, 1)
k_step_mega(StencilView<T> SV, const T* __restrict__ x, T* V, long long ldv, long long n, int j,
            T* wg, StateView<T> sv, WsView ws, int m_limit, const T* __restrict__ jdiag, T* zout, MegaX<T> X) {
  if (gated(sv.h)) return;
  uint32_t seqv = 0;
  if constexpr (DIST) {
    seqv = *(volatile const uint32_t*)xbox_step(X.box[X.rank]) + 1u;
    if (j >= 1 && (X.prev_V || X.next_V)) {
      // our previous step kernel stored the halo rows of V[:, j] into the
      // neighbours (kernel boundary: complete); release them, then wait for ours
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        __threadfence_system();
        if (X.prev_V) st_release_sys_u32(X.prev_flag, seqv);
        if (X.next_V) st_release_sys_u32(X.next_flag, seqv);
      }
      if (threadIdx.x == 0) {
        const bool ok = (!X.prev_V || wait_seq_sys(X.hflags + 0, seqv)) &&
                        (!X.next_V || wait_seq_sys(X.hflags + 1, seqv));
        if (!ok) {
          atomicOr(&sv.h->flags, MPG_FLAG_HALO_TIMEOUT);
          sv.h->done = 1;
        }
      }
      __syncthreads();
    }
  }
  // kernel-time categories (timing.py): CTA 0 stamps at its own phase ends and
  // after each grid barrier, so each interval ends when the grid has finished
  // the phase (B1..B3) or, for the SpMV, when CTA 0 has
  const bool kt0 = blockIdx.x == 0 && threadIdx.x == 0;
  if (kt0) kt_stamp(sv.h, KC_SPMV);
  MEGA_STAMP(0)
  constexpr int VN = Vec<T>::n;
  constexpr int RB = 32 * VN;
  constexpr int RPW = RB / 8;
  const int k = j + 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = warp >> 3, gw = warp & 7;
  const int G = gridDim.x;
  const long long nblk = (n + RB - 1) / RB;
  const int nb = (long long)blockIdx.x < nblk ? (int)((nblk - 1 - blockIdx.x) / G + 1) : 0;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* wsm = reinterpret_cast<T*>(smraw);
  constexpr int U = MegaU<T, KV>::u;
  __shared__ __align__(16) T upart[kMegaGroups][8][U * RB];
  __shared__ __align__(16) T xs[kMegaGroups][U * RB];
  __shared__ T cred[kMegaGroups][kMegaMaxCols];
  __shared__ T c1v[kMegaMaxCols];
  __shared__ T c2v[kMegaMaxCols];
  __shared__ T red[kMegaWarps];
  __shared__ int badw[kMegaWarps];
  T* part = static_cast<T*>(ws.part);
  auto bstart = [&](int t) -> long long { return ((long long)blockIdx.x + (long long)t * G) * RB; };
  auto wptr = [&](int t) -> T* { return CACHE ? wsm + (size_t)t * RB : wg + bstart(t); };

  // P1 streams x alone (latency-bound, HBM mostly idle): stage the first
  // MPG_MEGA_PF1 blocks of each group's pass-1 dot sweep into L2 meanwhile
#ifndef MPG_MEGA_PF1
#define MPG_MEGA_PF1 8
#endif
  if (MPG_MEGA_PF1 > 0) {
    for (int idx = lane; idx < KV * MPG_MEGA_PF1; idx += 32) {
      const int q = idx % KV, d = idx / KV;
      const int t = grp + d * kMegaGroups;
      const long long b0 = bstart(t);
      if (gw + 8 * q < k && t < nb && b0 + RB <= n)
        prefetch_l2_bulk(V + (size_t)(gw + 8 * q) * ldv + b0, RB * sizeof(T));
    }
  }

  // ---------------------------------------------------------------- P1 SpMV
  long long off[S];
  {
    const long long nx = SV.nx, p2 = nx * nx;
    if constexpr (S == 7) {
      const long long o[7] = {-p2, -nx, -1, 0, 1, nx, p2};
#pragma unroll
      for (int s = 0; s < 7; ++s) off[s] = o[s];
    } else {
      const long long o[5] = {-nx, -1, 0, 1, nx};
#pragma unroll
      for (int s = 0; s < 5; ++s) off[s] = o[s];
    }
  }
  int mis[S];
  stencil_mis<T, S>(off, mis);
  // KONST: the host read the constant-coefficient header at create, so only
  // the coefficient-stream SpMV is compiled in (and only the packed-values one
  // otherwise): the 64-register budget holds one path, not both
  StencilConst<T, S> K = stencil_const<T, S>(SV);
  K.on = KONST;
  T ss = T(0);
  int bad = 0;
  // one row group's SpMV result -> w (smem or global), ||w||^2, finite flag
  auto p1_emit = [&](int L, long long r0, T (&y)[VN]) {
#pragma unroll
    for (int e = 0; e < VN; ++e) y[e] = r0 + e < n ? y[e] : T(0);
    if (CACHE || r0 < n) vstore(wptr(L >> 5) + (L & 31) * VN, y);   // global w ends at ldv
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      ss = fma_rn(y[e], y[e], ss);
      bad |= !isfinite(y[e]);
    }
  };
  auto p1_r0 = [&](int L) { return bstart(L >> 5) + (long long)(L & 31) * VN; };
  // (two row groups' x loads in flight per thread measured slower: P1 13.4 ->
  // 18.4 us at k = 27, cfg2 fp32 -- the phase is not bound by loads in flight)
  {
    for (int L = tid; L < nb * 32; L += kMegaThreads) {
      const long long r0 = p1_r0(L);
      T y[VN];
      if (r0 < n) stencil_group<T, S>(SV, x, r0, off, mis, K, y);
      else {
#pragma unroll
        for (int e = 0; e < VN; ++e) y[e] = T(0);
      }
      p1_emit(L, r0, y);
    }
  }
  __syncthreads();
  if (kt0) kt_stamp(sv.h, KC_GEMV_T);                    // pass-1 dots up to B1's sums
  MEGA_STAMP(1)

  // --------------------------------------------------------- P1b c1 = V^T w
  {
    T acc[KV];
#pragma unroll
    for (int q = 0; q < KV; ++q) acc[q] = T(0);
    for (int t = grp; t < nb; t += kMegaGroups) {
      const long long r = bstart(t) + (long long)lane * VN;
      const bool in = r < n;
      T wv[VN], v[KV][VN];
      if (CACHE || in) vload_smem(wptr(t) + lane * VN, wv);
      else {
#pragma unroll
        for (int e = 0; e < VN; ++e) wv[e] = T(0);
      }
#pragma unroll
      for (int q = 0; q < KV; ++q) {
        const int i = gw + 8 * q;
        if (in && i < k) vload_cs(V + (size_t)i * ldv + r, v[q]);
        else {
#pragma unroll
          for (int e = 0; e < VN; ++e) v[q][e] = T(0);
        }
      }
#pragma unroll
      for (int q = 0; q < KV; ++q)
#pragma unroll
        for (int e = 0; e < VN; ++e) acc[q] = fma_rn(v[q][e], wv[e], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < KV; ++q) {
      const int i = gw + 8 * q;
      const T a = warp_sum(acc[q]);
      if (lane == 0 && i < k) cred[grp][i] = a;
    }
  }
  {
    const T sw = warp_sum(ss);
    const int bw = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      red[warp] = sw;
      badw[warp] = bw;
    }
  }
  __syncthreads();
  if (tid < k) {
    T t = T(0);
#pragma unroll
    for (int g = 0; g < kMegaGroups; ++g) t += cred[g][tid];
    part[(size_t)(kColDot1 + tid) * kMaxParts + blockIdx.x] = t;
  } else if (tid == k) {
    T t = T(0);
    for (int w = 0; w < kMegaWarps; ++w) t += red[w];
    part[(size_t)(kColDot1 + k) * kMaxParts + blockIdx.x] = t;
  } else if (tid == k + 1) {
    int b = 0;
    for (int w = 0; w < kMegaWarps; ++w) b |= badw[w];
    part[(size_t)(kColDot1 + k + 1) * kMaxParts + blockIdx.x] = b ? T(1) : T(0);
  }
  // the basis blocks P2 starts with do not depend on c1: stage them into L2
  // while the grid waits at B1
#ifndef MPG_MEGA_PFB
#define MPG_MEGA_PFB 1
#endif
  if (MPG_MEGA_PF && lane < KV && gw + 8 * lane < k) {
#pragma unroll
    for (int d = 0; d < MPG_MEGA_PFB; ++d) {
      const long long b0 = bstart(grp + d * kMegaGroups);
      if (grp + d * kMegaGroups < nb && b0 + RB <= n)
        prefetch_l2_bulk(V + (size_t)(gw + 8 * lane) * ldv + b0, RB * sizeof(T));
    }
  }
  MEGA_STAMP(2)
  mega_barrier<T>(ws);                                       // B1
  MEGA_STAMP(3)
  for (int c = warp; c < k + 2; c += 2 * kMegaWarps) {   // k + 2 <= 2 * 32 columns: one round trip
    const int c2 = c + kMegaWarps;
    T s0, s1;
    sum_column2(part, kColDot1 + c, kColDot1 + c2, c2 < k + 2, G, s0, s1);
    if (lane == 0) {
      c1v[c] = s0;
      if (c2 < k + 2) c1v[c2] = s1;
    }
  }
  __syncthreads();
  if constexpr (DIST) {
    mega_xsum<T>(X, 0, k + 2, seqv, c1v, sv.h);
    // every CTA has read the step counter (at entry, before B1): advance it
    if (blockIdx.x == 0 && tid == 0) *(volatile uint32_t*)xbox_step(X.box[X.rank]) = seqv;
  }
  if (c1v[k + 1] != T(0)) {   // non-finite operator output (krylov.py:131-133): every CTA agrees
    if (blockIdx.x == 0 && tid == 0) {
      sv.h->flags |= MPG_FLAG_NONFINITE_OP;
      sv.h->done = 1;
    }
    return;
  }
  const double w0 = (double)sqrt_rn(c1v[k]);
  if (kt0) kt_stamp(sv.h, KC_GEMV_TN);                   // P2: update + pass-2 dots, to B2
  if (blockIdx.x == 0) {
    if (tid < k) sv.c1[tid] = c1v[tid];
    if (tid == 0) sv.h->w0 = w0;
  }

  // ------------------------------------ P2 w' = w - V c1 ; c2 = V^T w'
  // U blocks of the group per barrier pair (blocks t and t + 4 when U = 2:
  // twice the loads in flight between barriers; the per-row sums and the
  // accumulation order over blocks are unchanged, so results are bitwise the
  // same as with U = 1)
  {
    T acc[KV];
#pragma unroll
    for (int q = 0; q < KV; ++q) acc[q] = T(0);
    constexpr int RL = (U * RPW <= 32) ? U * RPW : 32;   // reducing lanes
    const int ub_r = lane / RPW, rrow = gw * RPW + lane % RPW;
    for (int t = grp; t < nb; t += kMegaGroups * U) {
      // the barriers below keep the group's warps in lock step, so the basis
      // loads of the next block(s) are staged into L2 ahead of time
      if (MPG_MEGA_PF && lane < KV && gw + 8 * lane < k) {
#pragma unroll
        for (int ub = 0; ub < U; ++ub) {
          const long long bn = bstart(t + (U + ub) * kMegaGroups);
          if (t + (U + ub) * kMegaGroups < nb && bn + RB <= n)
            prefetch_l2_bulk(V + (size_t)(gw + 8 * lane) * ldv + bn, RB * sizeof(T));
        }
      }
      T v[U][KV][VN], u[U][VN];
#pragma unroll
      for (int ub = 0; ub < U; ++ub) {
        const long long r = bstart(t + ub * kMegaGroups) + (long long)lane * VN;
        const bool in = t + ub * kMegaGroups < nb && r < n;
#pragma unroll
        for (int q = 0; q < KV; ++q) {
          const int i = gw + 8 * q;
          if (in && i < k) vload_cs(V + (size_t)i * ldv + r, v[ub][q]);
          else {
#pragma unroll
            for (int e = 0; e < VN; ++e) v[ub][q][e] = T(0);
          }
        }
      }
#pragma unroll
      for (int ub = 0; ub < U; ++ub) {
#pragma unroll
        for (int e = 0; e < VN; ++e) u[ub][e] = T(0);
#pragma unroll
        for (int q = 0; q < KV; ++q) {
          const int i = gw + 8 * q;
          const T c = i < k ? c1v[i] : T(0);
#pragma unroll
          for (int e = 0; e < VN; ++e) u[ub][e] = fma_rn(v[ub][q][e], c, u[ub][e]);
        }
        vstore(upart[grp][gw] + ub * RB + lane * VN, u[ub]);
      }
      group_sync(grp);
      if (lane < RL) {
        const int tb = t + ub_r * kMegaGroups;
        const long long b0 = bstart(tb);
        T s = T(0);
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) s += upart[grp][ww][ub_r * RB + rrow];
        const bool rin = tb < nb && b0 + rrow < n;
        T xr = T(0);
        if (tb < nb) {
          T* wr = wptr(tb) + rrow;
          if (rin) xr = sub_rn(*wr, s);
          if (CACHE || rin) *wr = xr;
        }
        xs[grp][ub_r * RB + rrow] = xr;
      }
      group_sync(grp);
#pragma unroll
      for (int ub = 0; ub < U; ++ub) {
        T xv[VN];
        vload_smem(xs[grp] + ub * RB + lane * VN, xv);
#pragma unroll
        for (int q = 0; q < KV; ++q)
#pragma unroll
          for (int e = 0; e < VN; ++e) acc[q] = fma_rn(v[ub][q][e], xv[e], acc[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < KV; ++q) {
      const int i = gw + 8 * q;
      const T a = warp_sum(acc[q]);
      if (lane == 0 && i < k) cred[grp][i] = a;
    }
  }
  __syncthreads();
  if (tid < k) {
    T t = T(0);
#pragma unroll
    for (int g = 0; g < kMegaGroups; ++g) t += cred[g][tid];
    part[(size_t)(kColDot2 + tid) * kMaxParts + blockIdx.x] = t;
  }
  if (MPG_MEGA_PF && lane < k) {   // P3's first block(s) per warp, likewise
#pragma unroll
    for (int d = 0; d < MPG_MEGA_PFB; ++d) {
      const long long b0 = bstart(warp + d * kMegaWarps);
      if (warp + d * kMegaWarps < nb && b0 + RB <= n) prefetch_l2_bulk(V + (size_t)lane * ldv + b0, RB * sizeof(T));
    }
  }
  MEGA_STAMP(4)
  mega_barrier<T>(ws);                                       // B2
  MEGA_STAMP(5)
  for (int c = warp; c < k; c += 2 * kMegaWarps) {
    const int c2 = c + kMegaWarps;
    T s0, s1;
    sum_column2(part, kColDot2 + c, kColDot2 + c2, c2 < k, G, s0, s1);
    if (lane == 0) {
      c2v[c] = s0;
      if (c2 < k) c2v[c2] = s1;
    }
  }
  __syncthreads();
  if constexpr (DIST) mega_xsum<T>(X, 1, k, seqv, c2v, sv.h);
  if (kt0) kt_stamp(sv.h, KC_GEMV_N);                    // P3: w'' = w' - V c2
  if (blockIdx.x == 0 && tid < k) {
    sv.c2[tid] = c2v[tid];
    sv.Hc(j, tid) = add_rn(add_rn(T(0), c1v[tid]), c2v[tid]);   // h = 0; h += c1; h += c2
  }

  // ----------------------------------------------- P3 w'' = w' - V c2, norm
  T ss2 = T(0);
  for (int L = tid; L < nb * 32; L += kMegaThreads) {
    const int t = L >> 5, l = L & 31;
    const long long r = bstart(t) + (long long)l * VN;
    if (!CACHE && r >= n) continue;   // global w ends at ldv (nothing to add to ss2)
    T* wp = wptr(t) + l * VN;
    T wv[VN], u[VN];
    vload_smem(wp, wv);
#pragma unroll
    for (int e = 0; e < VN; ++e) u[e] = T(0);
    if (r < n) {
      int i = 0;
      for (; i + 4 <= k; i += 4) {
        T v0[VN], v1[VN], v2[VN], v3[VN];
        vload_cs(V + (size_t)(i + 0) * ldv + r, v0);
        vload_cs(V + (size_t)(i + 1) * ldv + r, v1);
        vload_cs(V + (size_t)(i + 2) * ldv + r, v2);
        vload_cs(V + (size_t)(i + 3) * ldv + r, v3);
#pragma unroll
        for (int e = 0; e < VN; ++e) {
          u[e] = fma_rn(v0[e], c2v[i + 0], u[e]);
          u[e] = fma_rn(v1[e], c2v[i + 1], u[e]);
          u[e] = fma_rn(v2[e], c2v[i + 2], u[e]);
          u[e] = fma_rn(v3[e], c2v[i + 3], u[e]);
        }
      }
      for (; i < k; ++i) {
        T v0[VN];
        vload_cs(V + (size_t)i * ldv + r, v0);
#pragma unroll
        for (int e = 0; e < VN; ++e) u[e] = fma_rn(v0[e], c2v[i], u[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      wv[e] = r + e < n ? sub_rn(wv[e], u[e]) : T(0);
      ss2 = fma_rn(wv[e], wv[e], ss2);
    }
    vstore(wp, wv);
  }
  {
    const T sw = warp_sum(ss2);
    if (lane == 0) red[warp] = sw;
  }
  __syncthreads();
  if (tid == 0) {
    T t = T(0);
    for (int w = 0; w < kMegaWarps; ++w) t += red[w];
    part[(size_t)kColNorm * kMaxParts + blockIdx.x] = t;
    if (kt0) kt_stamp(sv.h, KC_NORM);                    // B3 + the norm's column sum
  }
  MEGA_STAMP(6)
  mega_barrier<T>(ws);                                       // B3
  MEGA_STAMP(7)
  if (warp == 0) {
    const T s = sum_column(part, kColNorm, G);
    if (lane == 0) red[0] = s;
  }
  __syncthreads();
  if constexpr (DIST) mega_xsum<T>(X, 2, 1, seqv, red, sv.h);
  const T hs = sqrt_rn(red[0]);
  if (kt0) kt_stamp(sv.h, KC_OTHER);                     // Givens + V[:, j+1] = w'' / h
  const bool brk = (double)hs <= sv.h->breakdown_tol * w0;   // krylov.py:146
  if (blockIdx.x == 0 && warp == 0) {   // the rotation runs in warp 0 while warps 1.. start P4
    if (lane == 0) {
      sv.Hc(j, j + 1) = hs;
      sv.h->h_sub = (double)hs;
    }
    __syncwarp();
    givens_column_warp(sv, j, sv.h->threshold, brk, m_limit, &cred[0][0]);   // cred is free after B2
  }
  if (brk) return;   // no new basis vector on breakdown

  // ------------------------------------------------- P4 V[:, j+1] = w'' / h
  T* vn = V + (size_t)(j + 1) * ldv;
  for (int L = tid; L < nb * 32; L += kMegaThreads) {
    const int t = L >> 5, l = L & 31;
    const long long r = bstart(t) + (long long)l * VN;
    if (r >= n) continue;
    T a[VN];
    vload_smem(wptr(t) + l * VN, a);
#pragma unroll
    for (int e = 0; e < VN; ++e) a[e] = div_rn(a[e], hs);   // rows >= n stay 0
    vstore(vn + r, a);
    if constexpr (DIST) {   // the halo planes of V[:, j+1], straight into the neighbours' rows
      if (X.prev_V && r < X.halo) {
        T* d = X.prev_V + (size_t)(j + 1) * X.prev_ld + X.prev_off;
#pragma unroll
        for (int e = 0; e < VN; ++e)
          if (r + e < X.halo) d[r + e] = a[e];
      }
      if (X.next_V && r + VN > n - X.halo) {
        T* d = X.next_V + (size_t)(j + 1) * X.next_ld + X.next_off - (n - X.halo);
#pragma unroll
        for (int e = 0; e < VN; ++e)
          if (r + e >= n - X.halo && r + e < n) d[r + e] = a[e];
      }
    }
    if (jdiag) {   // Jacobi(1): the next step's operator input z = v / diag (precond.py:384-390)
      if (r + VN <= n) {
        T dv[VN];
        vload(jdiag + r, dv);
#pragma unroll
        for (int e = 0; e < VN; ++e) a[e] = div_rn(a[e], dv[e]);
        vstore(zout + r, a);
      } else {
        for (int e = 0; r + e < n; ++e) zout[r + e] = div_rn(a[e], __ldg(jdiag + r + e));
      }
    }
  }
  if constexpr (DIST) {   // this CTA's peer halo stores are system-visible before the kernel ends
    if (X.prev_V || X.next_V) __threadfence_system();
  }
  __syncthreads();
  MEGA_STAMP(8)
}

// ------------------------------------------------------------------ launch

// MPG_MEGA=1 / 0 forces the persistent / four-launch step for every solver
// (A/B runs); unset (-1) leaves the choice to the descriptor (step_kernel).
// Measured on B200 (IR solves, Laplace3D): the persistent step wins while the
// launch and reduction-tail costs are a large share of a step -- nx 60: 15.1 vs
// 19.2 ms, nx 75: 32.3 vs 39.5 ms, nx 100: 89 vs 100 ms, nx 126: 241 vs 247 ms
// (fp64 nx 126: 453 vs 472 ms) -- ties at cfg2 fp32 (0.501 vs 0.503 s) and loses
// at cfg2 fp64 (1.123 vs 0.999 s: 64-register cap at 1024 threads spills, one
// CTA per SM).  Hence the 20 MB vector-size rule in solver.cu.
int mega_env() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("MPG_MEGA");
    v = e ? (e[0] == '1' ? 1 : 0) : -1;
  }
  return v;
}

template <typename T, int S, int KV, bool CACHE, bool KONST, bool DIST>
static cudaError_t launch_mega_k(const StencilView<T>& SV, const T* x, T* V, long long ldv, long long n,
                                 int j, T* w, StateView<T> sv, WsView ws, int m_limit, cudaStream_t st,
                                 unsigned grid, size_t smem, const T* jdiag, T* zout, const MegaX<T>& X) {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(k_step_mega<T, S, KV, CACHE, KONST, DIST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         optin - (int)sizeof(T) * (kMegaGroups * 9 * MegaU<T, KV>::u * 32 * Vec<T>::n + 3 * kMegaMaxCols * 2) - 2048);
    cudaGetLastError();
  });
  count_launch();
  return launch_k(false, true, k_step_mega<T, S, KV, CACHE, KONST, DIST>, dim3(grid), dim3(kMegaThreads), smem, st,
                  SV, x, V, ldv, n, j, w, sv, ws, m_limit, jdiag, zout, X);
}

template <typename T, int S, int KV, bool DIST>
static cudaError_t launch_mega_kv(const StencilView<T>& SV, const T* x, T* V, long long ldv, long long n,
                                  int j, T* w, StateView<T> sv, WsView ws, int m_limit, cudaStream_t st,
                                  const T* jdiag, T* zout, const MegaX<T>& X) {
  constexpr int RB = 32 * Vec<T>::n;
  const long long nblk = (n + RB - 1) / RB;
  const long long G = std::min<long long>(num_sms(), nblk);
  const size_t cache = (size_t)((nblk + G - 1) / G) * RB * sizeof(T);
  static int optin = -1;
  if (optin < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  // static shared memory of the kernel (upart, xs, column scratch) + headroom
  const size_t stat = sizeof(T) * (kMegaGroups * 9 * MegaU<T, KV>::u * RB + 3 * kMegaMaxCols * 2) + 2048;
  if (cache + stat <= (size_t)optin) {
    if (SV.konst == 2)
      return launch_mega_k<T, S, KV, true, true, DIST>(SV, x, V, ldv, n, j, w, sv, ws, m_limit, st, (unsigned)G,
                                                       cache, jdiag, zout, X);
    return launch_mega_k<T, S, KV, true, false, DIST>(SV, x, V, ldv, n, j, w, sv, ws, m_limit, st, (unsigned)G,
                                                      cache, jdiag, zout, X);
  }
  return launch_mega_k<T, S, KV, false, false, DIST>(SV, x, V, ldv, n, j, w, sv, ws, m_limit, st, (unsigned)G, 0,
                                                     jdiag, zout, X);
}

template <typename T>
cudaError_t launch_step_mega(const StencilView<T>& SV, const T* x, T* V, long long ldv, long long n, int j,
                             T* w, StateView<T> sv, WsView ws, int m_limit, cudaStream_t st, const T* jdiag,
                             T* zout, const MegaX<T>* xd) {
  const int k = j + 1;
  if (k > kMegaMaxK || k + 2 > kMegaMaxCols || !SV.padded) return cudaErrorInvalidValue;
  if (xd && (xd->world < 1 || xd->world > kXMaxRanks || jdiag)) return cudaErrorInvalidValue;
  const int kv = (k + 7) / 8;
  const MegaX<T> X = xd ? *xd : MegaX<T>{};
#define MEGA_CASE(KVV)                                                                            \
  case KVV:                                                                                       \
    if (xd)                                                                                       \
      return SV.dims == 3                                                                         \
                 ? launch_mega_kv<T, 7, KVV, true>(SV, x, V, ldv, n, j, w, sv, ws, m_limit, st, jdiag, zout, X) \
                 : launch_mega_kv<T, 5, KVV, true>(SV, x, V, ldv, n, j, w, sv, ws, m_limit, st, jdiag, zout, X); \
    return SV.dims == 3                                                                           \
               ? launch_mega_kv<T, 7, KVV, false>(SV, x, V, ldv, n, j, w, sv, ws, m_limit, st, jdiag, zout, X) \
               : launch_mega_kv<T, 5, KVV, false>(SV, x, V, ldv, n, j, w, sv, ws, m_limit, st, jdiag, zout, X);
  switch (kv) {
    MEGA_CASE(1)
    MEGA_CASE(2)
    MEGA_CASE(3)
    MEGA_CASE(4)
    MEGA_CASE(5)
    MEGA_CASE(6)
    MEGA_CASE(7)
    default:
      return cudaErrorInvalidValue;
  }
#undef MEGA_CASE
}

template cudaError_t launch_step_mega<float>(const StencilView<float>&, const float*, float*, long long,
                                             long long, int, float*, StateView<float>, WsView, int,
                                             cudaStream_t, const float*, float*, const MegaX<float>*);
template cudaError_t launch_step_mega<double>(const StencilView<double>&, const double*, double*, long long,
                                              long long, int, double*, StateView<double>, WsView, int,
                                              cudaStream_t, const double*, double*, const MegaX<double>*);

}  // namespace mpg
