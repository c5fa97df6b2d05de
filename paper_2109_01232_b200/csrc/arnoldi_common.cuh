// Device pieces shared by the Arnoldi kernels (arnoldi_kernels.cu) and the
// persistent per-step kernel (step_kernel.cu): the done-flag gate, the
// reference-faithful Givens rotation (krylov.py:154-187) and the grid barrier
// of the cooperative kernels.
#pragma once

#include "state.cuh"

namespace mpg {

__device__ __forceinline__ bool gated(const mpg_state_header* h) {
  return *(volatile const int*)&h->done != 0;
}

// glibc-style hypot for the fp64 rotation (np.hypot -> libm hypot);
// fp32 follows glibc hypotf: correctly rounded double evaluation.
__device__ __forceinline__ float hypot_ref(float a, float b) {
  const double x = (double)a, y = (double)b;
  return (float)__dsqrt_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
}
__device__ inline double hypot_kernel(double ax, double ay) {
  // ax >= ay > 0, both well inside the exponent range (Borges 2019, as glibc)
  double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= 2.0 * ay) {
    const double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    const double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}
__device__ __forceinline__ double hypot_ref(double a, double b) {
  double ax = fabs(a), ay = fabs(b);
  if (isinf(ax) || isinf(ay)) return __longlong_as_double(0x7ff0000000000000LL);
  if (isnan(ax) || isnan(ay)) return ax + ay;
  if (ax < ay) { const double t = ax; ax = ay; ay = t; }
  if (ay == 0.0) return ax;
  if (ax > 0x1p+511) {
    if (ay <= ax * 0x1p-54) return ax + ay;
    return hypot_kernel(ax * 0x1p-600, ay * 0x1p-600) * 0x1p+600;
  }
  if (ay < 0x1p-511) {
    if (ax >= ay * 0x1p+54) return ax + ay;
    return hypot_kernel(ax * 0x1p+600, ay * 0x1p+600) * 0x1p-600;
  }
  if (ay <= ax * 0x1p-54) return ax + ay;
  return hypot_kernel(ax, ay);
}

// Rotate column j into the triangular factor (krylov.py:154-187).  One thread.
template <typename T>
__device__ void givens_column(const StateView<T>& sv, int j, double threshold, bool brk,
                              int m_limit) {
  T* col = &sv.Rc(j, 0);
  for (int i = 0; i <= j + 1; ++i) col[i] = sv.Hc(j, i);
  for (int i = 0; i < j; ++i) {
    const T c = sv.cs[i], s = sv.sn[i];
    const T a = col[i], b = col[i + 1];
    const T top = add_rn(mul_rn(c, a), mul_rn(s, b));
    col[i + 1] = add_rn(mul_rn(-s, a), mul_rn(c, b));
    col[i] = top;
  }
  const T a = col[j], b = col[j + 1];
  const T r = hypot_ref(a, b);
  double res;
  if (r == T(0)) {
    sv.cs[j] = T(1);
    sv.sn[j] = T(0);
    res = (double)fabs(sv.g[j]);
  } else {
    const T c = div_rn(a, r), s = div_rn(b, r);
    sv.cs[j] = c;
    sv.sn[j] = s;
    col[j] = add_rn(mul_rn(c, a), mul_rn(s, b));
    col[j + 1] = T(0);
    const T gj = sv.g[j], gj1 = sv.g[j + 1];
    const T top = add_rn(mul_rn(c, gj), mul_rn(s, gj1));
    sv.g[j + 1] = add_rn(mul_rn(-s, gj), mul_rn(c, gj1));
    sv.g[j] = top;
    res = (double)fabs(sv.g[j + 1]);
  }
  sv.implicit[j] = res;
  sv.h->steps = j + 1;
  sv.h->breakdown = brk ? 1 : 0;
  // solvers.py:160-168: stop on breakdown, on the implicit threshold, or when
  // the cycle's step budget is exhausted
  if (brk || res <= threshold || j + 1 >= m_limit) sv.h->done = 1;
}


// givens_column by one whole warp: the column, cos and sin are staged in shared
// memory `sm` (>= 3 * j + 2 elements) by all lanes, lane 0 runs the same
// rotation sequence on the staged values (identical arithmetic and order), and
// the lanes write the rotated column back.  Replaces j dependent global
// load/store round trips of the one-thread version with shared-memory ones.
template <typename T>
__device__ void givens_column_warp(const StateView<T>& sv, int j, double threshold, bool brk, int m_limit,
                                   T* sm) {
  const int lane = threadIdx.x & 31;
  T* col = sm;            // j + 2
  T* cc = sm + j + 2;     // j
  T* ss = cc + j;         // j
  for (int i = lane; i <= j + 1; i += 32) col[i] = sv.Hc(j, i);
  for (int i = lane; i < j; i += 32) {
    cc[i] = sv.cs[i];
    ss[i] = sv.sn[i];
  }
  __syncwarp();
  if (lane == 0) {
    for (int i = 0; i < j; ++i) {
      const T c = cc[i], s = ss[i];
      const T a = col[i], b = col[i + 1];
      const T top = add_rn(mul_rn(c, a), mul_rn(s, b));
      col[i + 1] = add_rn(mul_rn(-s, a), mul_rn(c, b));
      col[i] = top;
    }
    const T a = col[j], b = col[j + 1];
    const T r = hypot_ref(a, b);
    double res;
    if (r == T(0)) {
      sv.cs[j] = T(1);
      sv.sn[j] = T(0);
      res = (double)fabs(sv.g[j]);
    } else {
      const T c = div_rn(a, r), s = div_rn(b, r);
      sv.cs[j] = c;
      sv.sn[j] = s;
      col[j] = add_rn(mul_rn(c, a), mul_rn(s, b));
      col[j + 1] = T(0);
      const T gj = sv.g[j], gj1 = sv.g[j + 1];
      const T top = add_rn(mul_rn(c, gj), mul_rn(s, gj1));
      sv.g[j + 1] = add_rn(mul_rn(-s, gj), mul_rn(c, gj1));
      sv.g[j] = top;
      res = (double)fabs(sv.g[j + 1]);
    }
    sv.implicit[j] = res;
    sv.h->steps = j + 1;
    sv.h->breakdown = brk ? 1 : 0;
    if (brk || res <= threshold || j + 1 >= m_limit) sv.h->done = 1;
  }
  __syncwarp();
  for (int i = lane; i <= j + 1; i += 32) sv.Rc(j, i) = col[i];
}

// Grid barrier for cooperative launches (every CTA co-resident): shared
// arrival counter + generation word in the workspace; the last arriver resets
// the counter before releasing, so the slot is reusable.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// A/B: -DMPG_BAR_SC=1 restores the sequentially consistent fences
// (__threadfence) around the arrival; the default uses acquire/release
// ordering: arrival atom.acq_rel, release red.release, poll ld.acquire.
#ifndef MPG_BAR_SC
#define MPG_BAR_SC 0
#endif
// default: the count + generation pair as one 64-bit word (MPG_BAR_WORD=0:
// separate words, the generation read before arriving)
#ifndef MPG_BAR_WORD
#define MPG_BAR_WORD 1
#endif
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
#if MPG_BAR_SC
    const unsigned g0 = ld_acquire_u32(gen);
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      atomicExch(count, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (ld_acquire_u32(gen) == g0) __nanosleep(20);
    }
    __threadfence();
#elif MPG_BAR_WORD
    // count (low) and generation (high) read as one 64-bit word, so the
    // generation comes back with the arrival instead of a load before it; the
    // last arriver zeroes the count and bumps the generation in one add
    (void)gen;   // == count + 1 (the workspace's counter pair)
    unsigned long long* wd = reinterpret_cast<unsigned long long*>(count);
    unsigned long long old;
    asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(wd) : "memory");
    if ((unsigned)old == gridDim.x - 1) {
      asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(wd), "l"((1ull << 32) - gridDim.x) : "memory");
    } else {
      const unsigned gw = (unsigned)(old >> 32);
      unsigned long long v;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(wd) : "memory");
      } while ((unsigned)(v >> 32) == gw);
    }
#else
    const unsigned g0 = ld_acquire_u32(gen);
    unsigned old;
    // release: this CTA's writes (ordered before by bar.sync) precede the
    // arrival; acquire: the last arriver sees every CTA's writes
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(count) : "memory");
    if (old == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(count) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gen) : "memory");
    } else {
      while (ld_acquire_u32(gen) == g0) __nanosleep(20);
    }
#endif
  }
  __syncthreads();
}


}  // namespace mpg
