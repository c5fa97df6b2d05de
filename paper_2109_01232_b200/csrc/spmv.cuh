// CSR SpMV tile pipeline for sm_100a.
//
// Each persistent CTA walks tiles of kSpTile rows dealt round-robin over the
// grid (tile = blockIdx.x + i * gridDim.x).  One producer warp streams each tile's
// row_ptr slice, col_idx range and values range into shared memory with 1-D
// TMA bulk copies (cp.async.bulk -> UBLKCP) into a 2-stage ring guarded by
// full/empty mbarriers; eight consumer warps compute one row per thread with
// the reference's exact summation order (common.cuh: row_reduce), gathering
// x through the read-only path.  A tile whose nnz range does not fit the
// stage falls back to direct global loads (long-row matrices).
//
// Epilogue policy (template parameter E):
//   T   on_row(long long r, T y)              per row, by the computing thread
//   void on_tile(long long a, int nrows, const T* ys)   all consumers, after a
//                                              consumer barrier (ys complete)
//   void on_end()                              all consumers, after the last tile
//
// Reference: spmv.py:48-72 (products rounded, rows reduced by add.reduceat).
#pragma once

#include "common.cuh"

namespace mpg {

constexpr int kSpTile = 512;                   // rows per tile
constexpr int kSpCap = 8 * kSpTile + 32;       // staged entries per stage
constexpr int kSpStages = 2;
constexpr int kSpConsumers = 256;
constexpr int kSpConsumerWarps = kSpConsumers / 32;
constexpr int kSpThreads = kSpConsumers + 32;  // + 1 producer warp

template <typename T>
struct CsrView {
  const int32_t* rp;
  const int32_t* ci;
  const T* v;
  long long n;
};

// largest tile any pipeline hands to an epilogue (the vectorised stencil loop:
// kSpConsumers threads x one 16-byte row group)
constexpr int kStTileMax = kSpConsumers * 4;

// shared memory the epilogues use (tile of SpMV results + reduction scratch)
template <typename T>
struct alignas(16) EpiShared {
  alignas(16) T ys[2][kStTileMax];
  T red[32];
  T acc[8];
};

// Epilogues with a per-tile hook (on_tile reads the tile's results from shared
// memory: the fused K_A dots) declare kNeedsTiles; the others skip the
// per-tile barrier.
template <typename E, typename = void> struct needs_tiles { static constexpr bool value = false; };
template <typename E> struct needs_tiles<E, decltype((void)E::kNeedsTiles)> {
  static constexpr bool value = E::kNeedsTiles;
};

template <typename T>
struct alignas(128) SpSmem {
  alignas(16) int32_t rp[kSpStages][kSpTile + 8];
  alignas(16) int32_t ci[kSpStages][kSpCap];
  alignas(16) T v[kSpStages][kSpCap];
  uint64_t full[kSpStages];
  uint64_t empty[kSpStages];
  int32_t meta[kSpStages][4];  // base, off_ci, off_v, staged
  EpiShared<T> es;
};

__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kSpConsumers) : "memory");
}

template <typename T>
__device__ __forceinline__ T consumer_block_sum(T v, T* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  consumer_sync();
  if (l == 0) red[w] = v;
  consumer_sync();
  T t = (l < kSpConsumerWarps) ? red[l] : T(0);
  return warp_sum(t);
}

__device__ __forceinline__ long long round16(long long b) { return (b + 15) & ~15LL; }

// Accumulate acc[i] += sum_r V_i[r] * y[r] over one tile for i < k, with a
// deterministic (tile-independent) combination order.  V_i(i) returns the
// tile start of basis vector i; y is the tile in shared memory.
enum { kLoadLdg = 0, kLoadStream = 1, kLoadShared = 2 };

template <typename T, int kLoad, typename VRow>
__device__ __forceinline__ void tile_dots(int k, int nr, const VRow& vrow, const T* y, T* acc,
                                          T* pw) {
  constexpr int VN = Vec<T>::n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ng = nr / VN;
  auto range_dot = [&](const T* v, int g0, int g1, bool tail) -> T {
    T p = T(0);
#pragma unroll 4
    for (int g = g0 + lane; g < g1; g += 32) {
      T a[VN], b[VN];
      if (kLoad == kLoadStream) vload_cs(v + (size_t)g * VN, a);
      else if (kLoad == kLoadLdg) vload(v + (size_t)g * VN, a);
      else vload_smem(v + (size_t)g * VN, a);
      const T* yy = y + g * VN;
#pragma unroll
      for (int e = 0; e < VN; ++e) b[e] = yy[e];
#pragma unroll
      for (int e = 0; e < VN; ++e) p = fma_rn(a[e], b[e], p);
    }
    if (tail) {
      const int r = ng * VN + lane;
      if (r < nr) p = fma_rn(kLoad == kLoadStream ? __ldcs(v + r) : (kLoad == kLoadLdg ? __ldg(v + r) : v[r]), y[r], p);
    }
    return warp_sum(p);
  };
  if (k >= kSpConsumerWarps) {
    for (int i = warp; i < k; i += kSpConsumerWarps) {
      T p = range_dot(vrow(i), 0, ng, true);
      if (lane == 0) acc[i] += p;
    }
  } else {
    const int nc = kSpConsumerWarps / k;
    T p = T(0);
    if (warp < k * nc) {
      const int i = warp / nc, c = warp % nc;
      const int g0 = (int)((long long)ng * c / nc), g1 = (int)((long long)ng * (c + 1) / nc);
      p = range_dot(vrow(i), g0, g1, c == nc - 1);
    }
    if (lane == 0) pw[warp] = p;
    consumer_sync();
    if ((int)threadIdx.x < k) {
      T s = T(0);
      for (int c = 0; c < nc; ++c) s += pw[threadIdx.x * nc + c];
      acc[threadIdx.x] += s;
    }
  }
}

// ---------------------------------------------------------------------------
// Stencil-specialised storage (the north star's "specialised stencil path").
// For a Dirichlet 5-point (dims 2) or 7-point (dims 3) stencil matrix the
// pattern is implied by the grid, so only the values are stored, slot-major:
// slot s of row r at vals[s * ldv + r], slots in ascending column order
// (3D: z-1, y-1, x-1, c, x+1, y+1, z+1; 2D: y-1, x-1, c, x+1, y+1).  A slot
// whose neighbour is outside the grid is absent and skipped (never added as
// a zero), so each row is reduced over exactly the CSR row's entries, in the
// same order: bit-identical to the CSR kernel and to the reference.
// Traffic per row drops from nnz_row*(s+4)+4 bytes to S*s bytes of values.
// vals/x are indexed by LOCAL row r in [0, n); grid coordinates come from the
// global row r + row0 (row-partitioned ranks).  x may be read at r + off
// outside [0, n): the halo planes a distributed caller stores around the
// owned block (csrc/solver.cu, distributed mode).
template <typename T>
struct StencilView {
  const T* vals;
  long long ldv;
  long long n;
  int nx;
  int dims;
  long long row0;
  // 1: every SpMV input has >= one grid plane of readable padding (or halo)
  // on both sides, so rows use the branchless sentinel path below
  int padded = 0;
  // 1: vals carries the constant-coefficient header (buffers packed by
  // launch_stencil_pack with the kDiaTail tail); padded path only
  int konst = 0;
};

// Absent stencil slots (neighbour outside the grid) hold this NaN payload in
// the packed values; arithmetic never produces it (generated NaNs are quiet,
// canonical), so presence can be read off the loaded value.
__host__ __device__ constexpr unsigned kAbsent32 = 0x7fa5a5a5u;
__host__ __device__ constexpr unsigned long long kAbsent64 = 0x7ff4a5a5a5a5a5a5ull;
__device__ __forceinline__ bool present(float v) { return __float_as_uint(v) != kAbsent32; }
__device__ __forceinline__ bool present(double v) {
  return (unsigned long long)__double_as_longlong(v) != kAbsent64;
}
template <typename T> __host__ __device__ inline T absent_value();
template <> __host__ __device__ inline float absent_value<float>() {
#ifdef __CUDA_ARCH__
  return __uint_as_float(kAbsent32);
#else
  float f; unsigned u = kAbsent32; __builtin_memcpy(&f, &u, 4); return f;
#endif
}
template <> __host__ __device__ inline double absent_value<double>() {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)kAbsent64);
#else
  double d; unsigned long long u = kAbsent64; __builtin_memcpy(&d, &u, 8); return d;
#endif
}

// exact q = r / nx for r < 2^32, 2 <= nx < 2^32: q = hi64(r * M) with
// M = floor((2^64 - 1) / nx) + 1 (M - 2^64/nx lies in (0, 1], so the error term
// r * (M - 2^64/nx) / 2^64 < 1/nx cannot carry into the quotient)
__device__ __forceinline__ unsigned div_nx(unsigned r, unsigned long long magic) {
  return (unsigned)__umul64hi((unsigned long long)r, magic);
}
__host__ __device__ inline unsigned long long nx_magic(unsigned nx) {
  return ~0ull / nx + 1ull;
}

template <typename T, int S>
__device__ __forceinline__ T stencil_reduce(const bool (&pr)[S], const T (&pv)[S], const T (&px)[S]) {
  // add.reduceat order for rows of <= 8 entries: p0 + (((p1 + p2) + p3) ...),
  // over the present slots only (absent neighbours are not stored entries)
  bool have = false;
  T p0 = T(0), rest = T(-0.0);
#pragma unroll
  for (int s = 0; s < S; ++s) {
    if (pr[s]) {
      const T p = mul_rn(pv[s], px[s]);
      if (!have) { p0 = p; have = true; }
      else rest = add_rn(rest, p);
    }
  }
  return add_rn(p0, rest);
}

template <typename T>
__device__ __forceinline__ T stencil_row(const StencilView<T>& S, const T* __restrict__ x, long long r) {
  const unsigned nx = (unsigned)S.nx;
  const unsigned long long mg = nx_magic(nx);
  const unsigned ur = (unsigned)(r + S.row0);
  const unsigned q = div_nx(ur, mg);
  const unsigned ix = ur - q * nx;
  const T* v = S.vals + r;
  const size_t ld = (size_t)S.ldv;
  // every load is issued up front (predicated), the reduction below is load-free
  if (S.dims == 3) {
    const unsigned iz = div_nx(q, mg);
    const unsigned iy = q - iz * nx;
    const long long p2 = (long long)nx * nx;
    const bool pr[7] = {iz > 0, iy > 0, ix > 0, true, ix + 1 < nx, iy + 1 < nx, iz + 1 < nx};
    const long long off[7] = {-p2, -(long long)nx, -1, 0, 1, (long long)nx, p2};
    T pv[7], px[7];
#pragma unroll
    for (int s = 0; s < 7; ++s) {
      pv[s] = pr[s] ? __ldg(v + s * ld) : T(0);
      px[s] = pr[s] ? __ldg(x + r + off[s]) : T(0);
    }
    return stencil_reduce<T, 7>(pr, pv, px);
  }
  const bool pr[5] = {q > 0, ix > 0, true, ix + 1 < nx, q + 1 < nx};
  const long long off[5] = {-(long long)nx, -1, 0, 1, (long long)nx};
  T pv[5], px[5];
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    pv[s] = pr[s] ? __ldg(v + s * ld) : T(0);
    px[s] = pr[s] ? __ldg(x + r + off[s]) : T(0);
  }
  return stencil_reduce<T, 5>(pr, pv, px);
}

// Constant-coefficient stencils.  Every packed dia buffer is S * ldv values
// followed by a kDiaTail-element tail whose header, written by the packing
// launch (launch_stencil_pack), reads h[0] = 1 when each slot holds one and the
// same value (bit pattern) in every row where it is present -- Laplace and
// uniform-convection stencils -- and h[1 + s] = that value.  The SpMV then
// takes the coefficients from registers and derives presence from the grid
// coordinates, so it streams x alone; the products and their summation order
// are unchanged (bit-identical results).  The values stay stored for the
// scalar / CSR paths.  Bytes 64.. of the tail are the packing scratch.
constexpr int kDiaTail = 64;
template <typename T, int S>
struct StencilConst {
  bool on;
  T kc[S];
  unsigned long long mg;   // nx_magic(nx)
};
template <typename T, int S>
__device__ __forceinline__ StencilConst<T, S> stencil_const(const StencilView<T>& SV) {
  StencilConst<T, S> c;
  const T* h = SV.vals + (size_t)S * SV.ldv;
  c.on = SV.konst && __ldg(h) != T(0);
#pragma unroll
  for (int s = 0; s < S; ++s) c.kc[s] = c.on ? __ldg(h + 1 + s) : T(0);
  c.mg = nx_magic((unsigned)SV.nx);
  return c;
}

// Tiles are dealt round-robin (tile = blockIdx.x + i * gridDim.x): the whole grid
// streams one compact window of the basis at a time, measured faster on B200
// than contiguous per-CTA slices (tools/bw_probe.cu).
template <typename T, typename E, typename RowF>
__device__ __forceinline__ void stencil_loop(long long n, E& epi, EpiShared<T>& es,
                                             const RowF& rowf) {
  const long long ntiles = (n + kSpTile - 1) / kSpTile;
  int t = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++t) {
    const long long a = tile * kSpTile;
    const int nrows = (int)min((long long)kSpTile, n - a);
    T* ys = es.ys[t & 1];
    for (int rr = threadIdx.x; rr < nrows; rr += kSpConsumers) ys[rr] = epi.on_row(a + rr, rowf(a + rr));
    if constexpr (needs_tiles<E>::value) {
      consumer_sync();
      epi.on_tile(a, nrows, ys);
    }
  }
  epi.on_end();
}

// Epilogues may take a whole 16-byte row group at once (kVecRows + on_rows);
// otherwise the group is handed over row by row.
// Epilogues whose results do not depend on which thread computes which rows
// (no reduction): they may use the z-marching loop below.
template <typename E, typename = void> struct order_free { static constexpr bool value = false; };
template <typename E> struct order_free<E, decltype((void)E::kOrderFree)> {
  static constexpr bool value = E::kOrderFree;
};

template <typename E, typename = void> struct has_vec_rows { static constexpr bool value = false; };
template <typename E> struct has_vec_rows<E, decltype((void)E::kVecRows)> {
  static constexpr bool value = E::kVecRows;
};
template <typename T, typename E>
__device__ __forceinline__ void epi_rows(E& epi, long long r0, T (&y)[Vec<T>::n], int cnt, T* ysp) {
  if constexpr (has_vec_rows<E>::value) {
    epi.on_rows(r0, y, cnt, ysp);
  } else {
    for (int e = 0; e < cnt; ++e) ysp[e] = epi.on_row(r0 + e, y[e]);
  }
}

// x[p .. p + VN) for a uniform misalignment `mis` = (p mod VN) (r0 is VN-aligned)
template <typename T>
__device__ __forceinline__ void xwindow(const T* __restrict__ p, int mis, T (&o)[Vec<T>::n]) {
  constexpr int VN = Vec<T>::n;
  if (mis == 0) {
    vload(p, o);
  } else if (VN == 4 && mis == 2) {
    const float2 a = __ldg(reinterpret_cast<const float2*>(p));
    const float2 b = __ldg(reinterpret_cast<const float2*>(p + 2));
    o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
  } else {
#pragma unroll
    for (int e = 0; e < VN; ++e) o[e] = __ldg(p + e);
  }
}

// One 16-byte group of VN consecutive rows r0.. (r0 % VN == 0) on padded
// inputs: S 16-byte value loads (slot-major storage is VN-aligned), one 16-byte
// load of x[r0..] that also feeds the +-1 neighbours (plus one scalar each),
// one window load per +-nx / +-nx^2 neighbour (16-byte when aligned);
// mis[s] = (off[s] mod VN).  The per-row reduction is branchless: every slot is
// loaded (absent neighbours read padding / the sentinel value) and add.reduceat's
// order p0 + (((p1 + p2) + p3) ...) over the present slots is applied with
// selects: bit-exact.
// The x operands of one row group (stencil_group's loads, issued together):
// px[s][e] = x[r0 + e + off[s]].
// ALN: every neighbour window is 16-byte aligned (nx % VN == 0; mis all 0)
template <typename T, int S, bool ALN = false>
__device__ __forceinline__ void stencil_xload(const T* __restrict__ x, long long r0, const long long (&off)[S],
                                              const int (&mis)[S], T (&px)[S][Vec<T>::n]) {
  constexpr int VN = Vec<T>::n;
  constexpr int C = S / 2;   // centre slot; C - 1 / C + 1 are the x -+ 1 neighbours
  vload(x + r0, px[C]);
  const T xm = __ldg(x + r0 - 1), xp = __ldg(x + r0 + VN);
#pragma unroll
  for (int s = 0; s < S; ++s)
    if (s < C - 1 || s > C + 1) {
      if (ALN) vload(x + r0 + off[s], px[s]);
      else xwindow(x + r0 + off[s], mis[s], px[s]);
    }
  px[C - 1][0] = xm;
#pragma unroll
  for (int e = 1; e < VN; ++e) px[C - 1][e] = px[C][e - 1];
#pragma unroll
  for (int e = 0; e < VN - 1; ++e) px[C + 1][e] = px[C][e + 1];
  px[C + 1][VN - 1] = xp;
}

template <typename T, int S>
__device__ __forceinline__ void stencil_const_rows(const StencilView<T>& SV, long long r0,
                                                   const StencilConst<T, S>& K, const T (&px)[S][Vec<T>::n],
                                                   T (&y)[Vec<T>::n]);

template <typename T, int S, bool ALN = false>
__device__ __forceinline__ void stencil_group(const StencilView<T>& SV, const T* __restrict__ x,
                                              long long r0, const long long (&off)[S],
                                              const int (&mis)[S], const StencilConst<T, S>& K,
                                              T (&y)[Vec<T>::n]) {
  constexpr int VN = Vec<T>::n;
  const size_t ld = (size_t)SV.ldv;
  T pv[S][VN], px[S][VN];
  if (!K.on) {
#pragma unroll
    for (int s = 0; s < S; ++s) vload(SV.vals + s * ld + r0, pv[s]);
  }
  stencil_xload<T, S, ALN>(x, r0, off, mis, px);
  if (K.on) {
    stencil_const_rows<T, S>(SV, r0, K, px, y);
    return;
  }
#pragma unroll
  for (int e = 0; e < VN; ++e) {
    bool have = false;
    T p0 = T(0), rest = T(-0.0);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const T p = mul_rn(pv[s][e], px[s][e]);
      const bool pr = present(pv[s][e]);
      const T nrest = add_rn(rest, p);
      rest = (pr && have) ? nrest : rest;
      p0 = (pr && !have) ? p : p0;
      have = have || pr;
    }
    y[e] = add_rn(p0, rest);
  }
}

// Constant-coefficient rows of one group from its loaded x operands.
// Presence comes from the grid coordinates of the group's first row (two exact
// multiply-shift divisions); the other rows' coordinates are stepped from it.
//  - interior groups (every slot present in all VN rows): p0 + (((p1 + p2) + p3) ...)
//  - x-boundary groups inside the y/z interior (first / last group of an x-line,
//    the common boundary case: ~2 groups per line): only the x-1 / x+1 slots can
//    be absent, both inside the "rest" chain, so they are skipped with one
//    select each and p0 stays the z-1 (2-D: y-1) product
//  - y/z-boundary planes and line-straddling groups: per-slot presence
// Every path sums exactly the present slots in add.reduceat's order: bit-exact.
template <typename T, int S>
__device__ __forceinline__ void stencil_const_rows(const StencilView<T>& SV, long long r0,
                                                   const StencilConst<T, S>& K, const T (&px)[S][Vec<T>::n],
                                                   T (&y)[Vec<T>::n]) {
  constexpr int VN = Vec<T>::n;
  constexpr int XM = S / 2 - 1, XP = S / 2 + 1;   // the x-1 / x+1 slots
  const unsigned nx = (unsigned)SV.nx;
  const unsigned ur0 = (unsigned)(r0 + SV.row0);
  const unsigned q0 = div_nx(ur0, K.mg);
  const unsigned ix0 = ur0 - q0 * nx;
  unsigned iy0, iz0;
  bool yz;   // every row of the group has all its y / z neighbours
  if constexpr (S == 7) {
    iz0 = div_nx(q0, K.mg);
    iy0 = q0 - iz0 * nx;
    yz = iy0 >= 1 && iy0 + 2 <= nx && iz0 >= 1 && iz0 + 2 <= nx;
  } else {
    iz0 = 0;
    iy0 = q0;
    yz = q0 >= 1 && q0 + 2 <= nx;
  }
  if (yz && ix0 + VN <= nx) {
    // the group lies in one x-line inside the y/z interior: only the x-1 / x+1
    // slots can be absent (first / last row of the line), both inside the
    // "rest" chain, so they are skipped with a predicated add and p0 stays the
    // z-1 (2-D: y-1) product.  One code path for interior and x-boundary
    // groups: no warp divergence at the ends of the x-lines.
#pragma unroll
    for (int e = 0; e < VN; ++e) {
      const unsigned ix = ix0 + (unsigned)e;
      const bool hm = ix > 0, hp = ix + 1 < nx;
      T rest;
      if constexpr (S == 7) rest = mul_rn(K.kc[1], px[1][e]);   // y-1: present
      else rest = hm ? mul_rn(K.kc[1], px[1][e]) : T(-0.0);    // x-1 is p1 in 2-D
#pragma unroll
      for (int s = 2; s < S; ++s) {
        const T nr = add_rn(rest, mul_rn(K.kc[s], px[s][e]));
        rest = s == XM ? (hm ? nr : rest) : (s == XP ? (hp ? nr : rest) : nr);
      }
      y[e] = add_rn(mul_rn(K.kc[0], px[0][e]), rest);
    }
    return;
  }
  unsigned ix = ix0, iy = iy0, iz = iz0;
#pragma unroll
  for (int e = 0; e < VN; ++e) {   // per-row presence; coordinates stepped, not divided
    if (e > 0 && ++ix == nx) {
      ix = 0;
      if (++iy == nx && S == 7) {
        iy = 0;
        ++iz;
      }
    }
    bool pr[S];
    if constexpr (S == 7) {
      pr[0] = iz > 0; pr[1] = iy > 0; pr[2] = ix > 0; pr[3] = true;
      pr[4] = ix + 1 < nx; pr[5] = iy + 1 < nx; pr[6] = iz + 1 < nx;
    } else {
      pr[0] = iy > 0; pr[1] = ix > 0; pr[2] = true; pr[3] = ix + 1 < nx; pr[4] = iy + 1 < nx;
    }
    bool have = false;
    T p0 = T(0), rest = T(-0.0);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const T p = mul_rn(K.kc[s], px[s][e]);
      const T nrest = add_rn(rest, p);
      rest = (pr[s] && have) ? nrest : rest;
      p0 = (pr[s] && !have) ? p : p0;
      have = have || pr[s];
    }
    y[e] = add_rn(p0, rest);
  }
}

template <typename T, int S>
__device__ __forceinline__ void stencil_mis(const long long (&off)[S], int (&mis)[S]) {
  constexpr int VN = Vec<T>::n;
#pragma unroll
  for (int s = 0; s < S; ++s) mis[s] = (int)(((off[s] % VN) + VN) % VN);
}

// Vectorised branchless stencil rows on padded inputs: each consumer thread
// owns one 16-byte group of VN consecutive rows per tile (stencil_group).
template <typename T, int S, typename E, bool ALN = false>
__device__ __forceinline__ void stencil_loop_vec(const StencilView<T>& SV, const T* __restrict__ x,
                                                 const long long (&off)[S], E& epi,
                                                 EpiShared<T>& es) {
  constexpr int VN = Vec<T>::n;
  constexpr int TILE = kSpConsumers * VN;
  const long long n = SV.n;
  int mis[S];
  stencil_mis<T, S>(off, mis);
  const StencilConst<T, S> K = stencil_const<T, S>(SV);
#ifndef MPG_ST_ZB
#define MPG_ST_ZB 16   // longest march; 0 disables (A/B)
#endif
  // (fp32 only: fp64 keeps its leading-edge prefetch loop, 283 vs 340 us at
  // 400^3; and from 4M rows: at 3.4M rows the march measured 15.5 -> 16.6 us)
// fp64 marches too, from 16M rows, with a one-plane-ahead L2 prefetch of the
// leading edge (400^3: 283 -> 268 us; at 3.4M rows it measured 20.9 -> 22.7 us)
#ifndef MPG_ST_ZM64
#define MPG_ST_ZM64 1
#endif
  if constexpr (S == 7 && (sizeof(T) == 4 || MPG_ST_ZM64) && order_free<E>::value && MPG_ST_ZB > 0) {
    // z-marching (3-D, constant coefficients, whole planes): each warp owns a
    // 32*VN-row chunk of a plane and marches it through ZB planes; the
    // z-1 / centre windows of plane z are the centre / z+1 windows loaded for
    // plane z-1, so a group loads 3 windows + 2 scalars instead of 5 + 2
    // (400^3 SpMV 120 -> 114 us, cfg4 IR + poly(25) 0.162 -> 0.152 s).
    // Every row is computed exactly as stencil_group computes it.
    const long long P = (long long)SV.nx * SV.nx;
    if (K.on && SV.padded && P % VN == 0 && SV.n % P == 0 && SV.n >= (sizeof(T) == 8 ? (16LL << 20) : (4LL << 20))) {
      constexpr int RB = 32 * VN;
      const long long nch = (P + RB - 1) / RB, nzl = SV.n / P;
      // march length: about one (chunk, z-range) item per resident warp (one
      // wave measured best: 200^3 IR + poly(25) 0.152 s at one wave vs 0.155 s
      // at two), between 2 and MPG_ST_ZB planes
      const long long wtot = (long long)gridDim.x * (kSpConsumers / 32);
      const long long ZB = max(2LL, min((long long)MPG_ST_ZB, (nzl * nch + wtot - 1) / wtot));
      const long long nzr = (nzl + ZB - 1) / ZB, items = nch * nzr;
      const int lane = threadIdx.x & 31;
      const long long wpc = kSpConsumers / 32;
      T* ysp = es.ys[0] + threadIdx.x * VN;   // on_row scratch, never read back
      const long long nxl = SV.nx;
      for (long long it = blockIdx.x * wpc + (threadIdx.x >> 5); it < items; it += (long long)gridDim.x * wpc) {
        const long long c = it % nch, zr = it / nch;
        const long long ofs = c * RB + lane * VN;
        if (ofs >= P) continue;
        const long long z0 = zr * ZB, z1 = min(z0 + ZB, nzl);
        long long rz = z0 * P + ofs;
        T xb[VN], xc[VN];
        vload(x + rz - P, xb);   // the guard / halo plane below plane 0
        vload(x + rz, xc);
#pragma unroll 1
        for (long long z = z0; z < z1; ++z, rz += P) {
          T px[S][VN];
          if (sizeof(T) == 8 && z + 1 < z1 && (lane & 7) == 0) prefetch_l2(x + rz + 2 * P);   // next leading edge
          vload(x + rz + P, px[6]);
          if (ALN) {
            vload(x + rz - nxl, px[1]);
            vload(x + rz + nxl, px[5]);
          } else {
            xwindow(x + rz - nxl, mis[1], px[1]);
            xwindow(x + rz + nxl, mis[5], px[5]);
          }
          const T xm = __ldg(x + rz - 1), xp = __ldg(x + rz + VN);
#pragma unroll
          for (int e = 0; e < VN; ++e) {
            px[0][e] = xb[e];
            px[3][e] = xc[e];
          }
          px[2][0] = xm;
#pragma unroll
          for (int e = 1; e < VN; ++e) px[2][e] = xc[e - 1];
#pragma unroll
          for (int e = 0; e < VN - 1; ++e) px[4][e] = xc[e + 1];
          px[4][VN - 1] = xp;
          T y[VN];
          stencil_const_rows<T, S>(SV, rz, K, px, y);
          epi_rows(epi, rz, y, VN, ysp);
#pragma unroll
          for (int e = 0; e < VN; ++e) {
            xb[e] = xc[e];
            xc[e] = px[6][e];
          }
        }
      }
      epi.on_end();
      return;
    }
  }
  if constexpr (!needs_tiles<E>::value) {
    // grid-stride over 16-byte row groups (the same rows per thread as the
    // tiled loop below: tile blockIdx.x + t * gridDim.x, group threadIdx.x)
    const long long stride = (long long)gridDim.x * TILE;
    T* ysp = es.ys[0] + threadIdx.x * VN;   // on_row scratch, never read back
    // the leading-edge window x[r0 + off[S-1]] (the +nx^2 / +nx neighbour) is the
    // only load of a group that misses L2 -- the other windows were the leading
    // edge of an earlier group -- so the thread prefetches the next iterations'
    // leading edges into L2 (MPG_ST_PF iterations ahead; 0 disables)
    // (measured at 400^3: fp64 SpMV 363 -> 287 us, residual 594 -> 526 us; fp32
    // 120 -> 124 us, so fp32 does not prefetch)
#ifndef MPG_ST_PF32
#define MPG_ST_PF32 0
#endif
#ifndef MPG_ST_PF64
#define MPG_ST_PF64 2
#endif
    constexpr int PF = sizeof(T) == 8 ? MPG_ST_PF64 : MPG_ST_PF32;
#pragma unroll 1
    for (long long r0 = ((long long)blockIdx.x * kSpConsumers + threadIdx.x) * VN; r0 < n; r0 += stride) {
      if (PF > 0) {
        const long long pf = r0 + PF * stride + off[S - 1];
        if (pf < n + off[S - 1] && (threadIdx.x & 7) == 0) prefetch_l2(x + pf);   // one lane per 128 B
      }
      T y[VN];
      stencil_group<T, S, ALN>(SV, x, r0, off, mis, K, y);
      epi_rows(epi, r0, y, (int)min((long long)VN, n - r0), ysp);
    }
    epi.on_end();
    return;
  }
  const long long ntiles = (n + TILE - 1) / TILE;
  int t = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++t) {
    const long long a = tile * TILE;
    const int nrows = (int)min((long long)TILE, n - a);
    T* ys = es.ys[t & 1];
    const int rr = threadIdx.x * VN;
    if (rr < nrows) {
      const long long r0 = a + rr;
      T y[VN];
      stencil_group<T, S>(SV, x, r0, off, mis, K, y);
      epi_rows(epi, r0, y, min(VN, nrows - rr), ys + rr);
    }
    if constexpr (needs_tiles<E>::value) {
      consumer_sync();
      epi.on_tile(a, nrows, ys);
    }
  }
  epi.on_end();
}

template <typename T, typename E, bool ALN = false>
__device__ __forceinline__ void stencil_pipeline(const StencilView<T>& S, const T* __restrict__ x,
                                                 E& epi, EpiShared<T>& es) {
  if (S.padded) {
    const long long nx = S.nx, p2 = nx * nx;
    if (S.dims == 3) {
      const long long off[7] = {-p2, -nx, -1, 0, 1, nx, p2};
      stencil_loop_vec<T, 7, E, ALN>(S, x, off, epi, es);
    } else {
      const long long off[5] = {-nx, -1, 0, 1, nx};
      stencil_loop_vec<T, 5, E, ALN>(S, x, off, epi, es);
    }
  } else {
    stencil_loop(S.n, epi, es, [&](long long r) { return stencil_row<T>(S, x, r); });
  }
}

template <typename T, typename E>
__device__ __forceinline__ void spmv_pipeline(const CsrView<T>& A, const T* __restrict__ x,
                                              E& epi, SpSmem<T>& sm) {
  // round-robin tiles, as stencil_loop: tile t of this CTA starts at row_of(t)
  const long long ntiles = (A.n + kSpTile - 1) / kSpTile;
  const int nt = blockIdx.x < ntiles ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  auto row_of = [&](int t) { return ((long long)blockIdx.x + (long long)t * gridDim.x) * kSpTile; };
  const long long R1 = A.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSpStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kSpConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kSpConsumerWarps) {
    // ------------------------------ producer warp ------------------------------
    if (lane == 0) {
      long long nb_a = row_of(0), nb_b = (nt > 0) ? min(nb_a + kSpTile, R1) : nb_a;
      int next_base = (nt > 0) ? __ldg(A.rp + nb_a) : 0;
      int next_end = (nt > 0) ? __ldg(A.rp + nb_b) : 0;
      for (int t = 0; t < nt; ++t) {
        const int s = t % kSpStages;
        const long long a = nb_a, b = nb_b;
        const int base = next_base, end = next_end;
        // prefetch the bounds of the following tile while this one streams in
        if (t + 1 < nt) {
          nb_a = row_of(t + 1);
          nb_b = min(nb_a + kSpTile, R1);
          next_base = __ldg(A.rp + nb_a);
          next_end = __ldg(A.rp + nb_b);
        }
        if (t >= kSpStages) mbar_wait(&sm.empty[s], ((t / kSpStages) - 1) & 1);
        const long long ci_lo = ((long long)base * 4) & ~15LL;
        const long long ci_hi = round16((long long)end * 4);
        const long long v_lo = ((long long)base * (long long)sizeof(T)) & ~15LL;
        const long long v_hi = round16((long long)end * (long long)sizeof(T));
        const bool staged = (ci_hi - ci_lo) <= (long long)kSpCap * 4 &&
                            (v_hi - v_lo) <= (long long)kSpCap * (long long)sizeof(T);
        sm.meta[s][0] = base;
        sm.meta[s][1] = base - (int)(ci_lo / 4);
        sm.meta[s][2] = base - (int)(v_lo / (long long)sizeof(T));
        sm.meta[s][3] = staged ? 1 : 0;
        const uint32_t rp_bytes = (uint32_t)round16((b - a + 1) * 4);
        uint32_t total = rp_bytes;
        if (staged) total += (uint32_t)(ci_hi - ci_lo) + (uint32_t)(v_hi - v_lo);
        fence_proxy_async();
        mbar_expect_tx(&sm.full[s], total);
        bulk_g2s(sm.rp[s], A.rp + a, rp_bytes, &sm.full[s]);
        if (staged) {
          if (ci_hi > ci_lo)
            bulk_g2s(sm.ci[s], reinterpret_cast<const char*>(A.ci) + ci_lo,
                     (uint32_t)(ci_hi - ci_lo), &sm.full[s]);
          if (v_hi > v_lo)
            bulk_g2s(sm.v[s], reinterpret_cast<const char*>(A.v) + v_lo,
                     (uint32_t)(v_hi - v_lo), &sm.full[s]);
        }
      }
    }
    return;
  }

  // -------------------------------- consumers --------------------------------
  const int tid = threadIdx.x;
  for (int t = 0; t < nt; ++t) {
    const int s = t % kSpStages;
    const long long a = row_of(t);
    const int nrows = (int)min((long long)kSpTile, R1 - a);
    mbar_wait(&sm.full[s], (t / kSpStages) & 1);
    const int base = sm.meta[s][0];
    const bool staged = sm.meta[s][3] != 0;
    const int32_t* rps = sm.rp[s];
    T* ys = sm.es.ys[t & 1];
    for (int rr = tid; rr < nrows; rr += kSpConsumers) {
      const int lo = rps[rr], hi = rps[rr + 1];
      T y;
      if (staged) {
        const int32_t* cs = sm.ci[s] + (lo - base + sm.meta[s][1]);
        const T* vs = sm.v[s] + (lo - base + sm.meta[s][2]);
        auto get = [&](int i) -> T { return mul_rn(vs[i], __ldg(x + cs[i])); };
        y = row_reduce<T>(get, hi - lo);
      } else {
        const int32_t* cg = A.ci + lo;
        const T* vg = A.v + lo;
        auto get = [&](int i) -> T { return mul_rn(__ldg(vg + i), __ldg(x + __ldg(cg + i))); };
        y = row_reduce<T>(get, hi - lo);
      }
      ys[rr] = epi.on_row(a + rr, y);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sm.empty[s])) : "memory");
    consumer_sync();
    epi.on_tile(a, nrows, ys);
  }
  epi.on_end();
}

}  // namespace mpg
