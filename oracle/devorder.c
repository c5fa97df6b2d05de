/* DEVICE-ORDER ORACLE — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * A plain-C restatement of the exact floating-point operation sequence of the
 * single-GPU GMRES path in paper_2109_01232_b200/csrc (the persistent
 * per-step kernel and the per-cycle kernels), for unpreconditioned solves on
 * stencil storage with steps k <= 56.  It exists to answer one question the
 * parity tests ask: when a GPU iteration count differs from the reference's,
 * is the difference entirely due to the ORDER of the floating-point
 * reductions?  The algorithm restated here is the reference's
 * (/root/reference/pkg/src/mpgmres: krylov.py:112-202 arnoldi_step /
 * givens_update / solve_least_squares, solvers.py:122-227 and :297-440); only
 * the association of each dot product, norm and basis update follows the
 * device kernels instead of single-thread OpenBLAS.  tests/test_gpu_parity_order.py
 * asserts that the GPU solve equals this restatement BIT FOR BIT, and that
 * the restatement's only difference from the reference-order oracle
 * (oracle/cpu_gmres.py, pinned to the reference) is the reduction order.
 *
 * Every function names the kernel it restates (file:function).  Products and
 * sums are rounded exactly where the device rounds them: fmaf/fma are the
 * correctly rounded C99 fused multiply-adds (the device's __fmaf_rn/__fma_rn),
 * and this file is compiled with -ffp-contract=off so no other multiply-add is
 * fused.  The geometry (SM count, grids) is a parameter: the device sizes
 * every grid from the SM count (148 on B200).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MEGA_THREADS 1024
#define MEGA_WARPS 32
#define MEGA_GROUPS 4
#define THREADS 256     /* common.cuh kThreads: streaming kernels */
#define MAX_PARTS (148 * 8)

enum { FLAG_NONFINITE_OP = 1, FLAG_NONFINITE_GAMMA = 2, FLAG_OVERFLOW = 4, FLAG_SINGULAR = 8,
       FLAG_NONFINITE_X = 16 };

static long long min_ll(long long a, long long b) { return a < b ? a : b; }

/* ---- glibc-style hypot for the fp64 rotation (arnoldi_common.cuh hypot_ref) */
static double hypot_kernel(double ax, double ay) {
  double h = sqrt(ax * ax + ay * ay);
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
static double hypot_ref_d(double a, double b) {
  double ax = fabs(a), ay = fabs(b);
  if (isinf(ax) || isinf(ay)) return INFINITY;
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
static float hypot_ref_f(float a, float b) {
  const double x = (double)a, y = (double)b;
  return (float)sqrt(x * x + y * y);
}

/* ===================================================================== *
 * One body per working precision T (float / double), instantiated below.
 * ===================================================================== */
#define DEVORDER_IMPL(T, SUF, FMA, SQRT, HYPOT, VN)                                              \
                                                                                                 \
  /* common.cuh warp_sum: xor butterfly over 32 lanes (every lane ends equal) */                 \
  static T warp_sum_##SUF(const T* v) {                                                          \
    T a[32], b[32];                                                                              \
    memcpy(a, v, sizeof a);                                                                      \
    for (int o = 16; o > 0; o >>= 1) {                                                           \
      for (int l = 0; l < 32; ++l) b[l] = a[l] + a[l ^ o];                                       \
      memcpy(a, b, sizeof a);                                                                    \
    }                                                                                            \
    return a[0];                                                                                 \
  }                                                                                              \
  /* common.cuh block_sum over 256 threads: warp sums, then one warp over 8 */                   \
  static T block_sum_##SUF(const T* v256) {                                                      \
    T w[32];                                                                                     \
    for (int q = 0; q < 32; ++q) w[q] = 0;                                                       \
    for (int q = 0; q < 8; ++q) w[q] = warp_sum_##SUF(v256 + 32 * q);                            \
    return warp_sum_##SUF(w);                                                                    \
  }                                                                                              \
  /* spmv.py:48-72 / common.cuh row_reduce: p0 + pairwise(p1..) (numpy pairwise_sum) */         \
  static T pw_block_##SUF(const T* p, int n) {                                                   \
    T r[8];                                                                                      \
    for (int j = 0; j < 8; ++j) r[j] = p[j];                                                     \
    int i = 8;                                                                                   \
    for (; i < n - (n % 8); i += 8)                                                              \
      for (int j = 0; j < 8; ++j) r[j] = r[j] + p[i + j];                                        \
    T res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));                   \
    for (; i < n; ++i) res = res + p[i];                                                         \
    return res;                                                                                  \
  }                                                                                              \
  static T pw_##SUF(const T* p, int n) {                                                         \
    if (n < 8) {                                                                                 \
      T r = (T)-0.0;                                                                             \
      for (int i = 0; i < n; ++i) r = r + p[i];                                                  \
      return r;                                                                                  \
    }                                                                                            \
    if (n <= 128) return pw_block_##SUF(p, n);                                                   \
    const int n2 = n / 2 - (n / 2) % 8;                                                          \
    const T a = pw_##SUF(p, n2);                                                                 \
    return a + pw_##SUF(p + n2, n - n2);                                                         \
  }                                                                                              \
  static void spmv_##SUF(int n, const int32_t* rp, const int32_t* ci, const T* vals, const T* x, \
                         T* y) {                                                                 \
    T buf[1024];                                                                                 \
    for (int r = 0; r < n; ++r) {                                                                \
      const int s = rp[r], L = rp[r + 1] - rp[r];                                                \
      if (L <= 0) { y[r] = 0; continue; }                                                        \
      T* p = L <= 1024 ? buf : (T*)malloc(sizeof(T) * (size_t)L);                                \
      for (int i = 0; i < L; ++i) p[i] = vals[s + i] * x[ci[s + i]];                             \
      y[r] = L == 1 ? p[0] : p[0] + pw_##SUF(p + 1, L - 1);                                      \
      if (p != buf) free(p);                                                                     \
    }                                                                                            \
  }                                                                                              \
                                                                                                 \
  /* grid-stride sum of squares over G CTAs of 256 threads, last-CTA block_sum                   \
     (misc_kernels.cu k_norm2, arnoldi_kernels.cu k_start / k_start_ir) */                       \
  static T sumsq_stream_##SUF(const T* x, long long n, long long G) {                            \
    T* part = (T*)calloc((size_t)G, sizeof(T));                                                  \
    T ss[THREADS];                                                                               \
    for (long long b = 0; b < G; ++b) {                                                          \
      for (int t = 0; t < THREADS; ++t) {                                                        \
        T s = 0;                                                                                 \
        for (long long i = b * THREADS + t; i < n; i += G * THREADS) s = FMA(x[i], x[i], s);     \
        ss[t] = s;                                                                               \
      }                                                                                          \
      part[b] = block_sum_##SUF(ss);                                                             \
    }                                                                                            \
    for (int t = 0; t < THREADS; ++t) {                                                          \
      T s = 0;                                                                                   \
      for (long long p = t; p < G; p += THREADS) s += part[p];                                   \
      ss[t] = s;                                                                                 \
    }                                                                                            \
    free(part);                                                                                  \
    return block_sum_##SUF(ss);                                                                  \
  }                                                                                              \
  static long long grid_stream_##SUF(long long n, int nsm) {                                     \
    long long g = (n + THREADS - 1) / THREADS;                                                   \
    if (g > (long long)nsm * 4) g = (long long)nsm * 4;                                          \
    return g < 1 ? 1 : g;                                                                        \
  }                                                                                              \
  /* ||x|| as k_norm2 returns it: sqrt in T, widened */                                          \
  double devorder_norm2_##SUF(const T* x, long long n, int nsm) {                                \
    return (double)SQRT(sumsq_stream_##SUF(x, n, grid_stream_##SUF(n, nsm)));                    \
  }                                                                                              \
                                                                                                 \
  /* r = b - A x and ||r|| (spmv_kernels.cu EpiResid over the padded stencil loop:               \
     tiles of 256*VN rows dealt round-robin over G CTAs, thread owns VN rows) */                 \
  double devorder_residual_##SUF(int n, const int32_t* rp, const int32_t* ci, const T* vals,     \
                                 const T* b, const T* x, T* r, long long G) {                    \
    T* y = (T*)malloc(sizeof(T) * (size_t)n);                                                    \
    spmv_##SUF(n, rp, ci, vals, x, y);                                                           \
    const long long TILE = 256LL * VN, ntiles = ((long long)n + TILE - 1) / TILE;                \
    T* part = (T*)calloc((size_t)G, sizeof(T));                                                  \
    T ss[THREADS];                                                                               \
    for (long long cb = 0; cb < G; ++cb) {                                                       \
      for (int t = 0; t < THREADS; ++t) ss[t] = 0;                                               \
      for (long long tile = cb; tile < ntiles; tile += G) {                                      \
        const long long a = tile * TILE;                                                         \
        const long long nrows = min_ll(TILE, n - a);                                             \
        for (int t = 0; t < THREADS; ++t) {                                                      \
          const long long rr = (long long)t * VN;                                                \
          if (rr >= nrows) continue;                                                             \
          const long long cnt = min_ll(VN, nrows - rr);                                          \
          for (long long e = 0; e < cnt; ++e) {                                                  \
            const long long i = a + rr + e;                                                      \
            const T v = b[i] - y[i];                                                             \
            r[i] = v;                                                                            \
            ss[t] = FMA(v, v, ss[t]);                                                            \
          }                                                                                      \
        }                                                                                        \
      }                                                                                          \
      part[cb] = block_sum_##SUF(ss);                                                            \
    }                                                                                            \
    T lanes[32];                                                                                 \
    for (int l = 0; l < 32; ++l) {                                                               \
      T s = 0;                                                                                   \
      for (long long p = l; p < G; p += 32) s += part[p];                                        \
      lanes[l] = s;                                                                              \
    }                                                                                            \
    free(part);                                                                                  \
    free(y);                                                                                     \
    return (double)SQRT(warp_sum_##SUF(lanes));                                                  \
  }                                                                                              \
                                                                                                 \
  typedef struct {                                                                               \
    int m, steps, done, brk, flags;                                                              \
    double threshold, btol, w0;                                                                  \
    T *H, *R, *cs, *sn, *g, *c1, *c2, *d;                                                        \
    double* implicit;                                                                            \
  } st_##SUF;                                                                                    \
  /* arnoldi_common.cuh givens_column(_warp) (krylov.py:154-187) */                              \
  static void givens_##SUF(st_##SUF* s, int j, int m_limit) {                                    \
    const int ld = s->m + 1;                                                                     \
    T* col = s->R + (size_t)j * ld;                                                              \
    for (int i = 0; i <= j + 1; ++i) col[i] = s->H[(size_t)j * ld + i];                          \
    for (int i = 0; i < j; ++i) {                                                                \
      const T c = s->cs[i], sn = s->sn[i];                                                       \
      const T a = col[i], b = col[i + 1];                                                        \
      const T top = c * a + sn * b;                                                              \
      col[i + 1] = -sn * a + c * b;                                                              \
      col[i] = top;                                                                              \
    }                                                                                            \
    const T a = col[j], b = col[j + 1];                                                          \
    const T r = HYPOT(a, b);                                                                     \
    double res;                                                                                  \
    if (r == (T)0) {                                                                             \
      s->cs[j] = 1;                                                                              \
      s->sn[j] = 0;                                                                              \
      res = (double)fabs(s->g[j]);                                                               \
    } else {                                                                                     \
      const T c = a / r, sn = b / r;                                                             \
      s->cs[j] = c;                                                                              \
      s->sn[j] = sn;                                                                             \
      col[j] = c * a + sn * b;                                                                   \
      col[j + 1] = 0;                                                                            \
      const T gj = s->g[j], gj1 = s->g[j + 1];                                                   \
      const T top = c * gj + sn * gj1;                                                           \
      s->g[j + 1] = -sn * gj + c * gj1;                                                          \
      s->g[j] = top;                                                                             \
      res = (double)fabs(s->g[j + 1]);                                                           \
    }                                                                                            \
    s->implicit[j] = res;                                                                        \
    s->steps = j + 1;                                                                            \
    if (s->brk || res <= s->threshold || j + 1 >= m_limit) s->done = 1;                          \
  }                                                                                              \
                                                                                                 \
  /* step_kernel.cu k_step_mega (CACHE, any storage: the SpMV is bit-exact) for step j.          \
     V: (m+1) columns of n rows (rows >= n read as the zero padding). */                         \
  static void mega_step_##SUF(int n, const int32_t* rp, const int32_t* ci, const T* vals, T* V,  \
                              int j, T* w, st_##SUF* s, int m_limit, int nsm, T* part) {         \
    const int RB = 32 * VN, RPW = RB / 8;                                                        \
    (void)RPW;                                                                                   \
    const int k = j + 1, KV = (k + 7) / 8;                                                       \
    const long long nblk = ((long long)n + RB - 1) / RB;                                         \
    const long long G = min_ll(nsm, nblk);                                                       \
    const T* x = V + (size_t)j * n;                                                              \
    spmv_##SUF(n, rp, ci, vals, x, w); /* P1: w = A v_j (rows < n) */                             \
    const int ncol = k + 2;                                                                      \
    _Static_assert(1, "");                                                                       \
    /* ---- P1 norm partial + P1b pass-1 dots, per CTA */                                        \
    for (long long b = 0; b < G; ++b) {                                                          \
      const long long nb = b < nblk ? (nblk - 1 - b) / G + 1 : 0;                                \
      T lane[32], red[MEGA_WARPS];                                                               \
      int bad = 0;                                                                               \
      for (int wp = 0; wp < MEGA_WARPS; ++wp) {                                                  \
        for (int l = 0; l < 32; ++l) {                                                           \
          T ss = 0;                                                                              \
          for (long long t = wp; t < nb; t += MEGA_WARPS) {                                      \
            const long long r0 = (b + t * G) * RB + (long long)l * VN;                           \
            for (int e = 0; e < VN; ++e) {                                                       \
              const T y = r0 + e < n ? w[r0 + e] : (T)0;                                         \
              ss = FMA(y, y, ss);                                                                \
              bad |= !isfinite(y);                                                               \
            }                                                                                    \
          }                                                                                      \
          lane[l] = ss;                                                                          \
        }                                                                                        \
        red[wp] = warp_sum_##SUF(lane);                                                          \
      }                                                                                          \
      T tn = 0;                                                                                  \
      for (int wp = 0; wp < MEGA_WARPS; ++wp) tn += red[wp];                                     \
      T cred[MEGA_GROUPS][72];                                                                   \
      for (int grp = 0; grp < MEGA_GROUPS; ++grp) {                                              \
        for (int gw = 0; gw < 8; ++gw) {                                                         \
          for (int q = 0; q < KV; ++q) {                                                         \
            const int i = gw + 8 * q;                                                            \
            for (int l = 0; l < 32; ++l) {                                                       \
              T acc = 0;                                                                         \
              for (long long t = grp; t < nb; t += MEGA_GROUPS) {                                \
                const long long r = (b + t * G) * RB + (long long)l * VN;                        \
                const int in = r < n;                                                            \
                for (int e = 0; e < VN; ++e) {                                                   \
                  const T wv = (in && r + e < n) ? w[r + e] : (T)0;                              \
                  const T v = (in && i < k && r + e < n) ? V[(size_t)i * n + r + e] : (T)0;      \
                  acc = FMA(v, wv, acc);                                                         \
                }                                                                                \
              }                                                                                  \
              lane[l] = acc;                                                                     \
            }                                                                                    \
            if (i < k) cred[grp][i] = warp_sum_##SUF(lane);                                      \
          }                                                                                      \
        }                                                                                        \
      }                                                                                          \
      for (int i = 0; i < k; ++i) {                                                              \
        T t = 0;                                                                                 \
        for (int grp = 0; grp < MEGA_GROUPS; ++grp) t += cred[grp][i];                           \
        part[(size_t)i * MAX_PARTS + b] = t;                                                     \
      }                                                                                          \
      part[(size_t)k * MAX_PARTS + b] = tn;                                                      \
      part[(size_t)(k + 1) * MAX_PARTS + b] = bad ? (T)1 : (T)0;                                 \
    }                                                                                            \
    /* ---- B1: sum_column over the G CTA partials */                                            \
    T c1v[72];                                                                                   \
    for (int c = 0; c < ncol; ++c) {                                                             \
      T lane[32];                                                                                \
      for (int l = 0; l < 32; ++l) {                                                             \
        T sm = 0;                                                                                \
        for (long long p = l; p < G; p += 32) sm += part[(size_t)c * MAX_PARTS + p];             \
        lane[l] = sm;                                                                            \
      }                                                                                          \
      c1v[c] = warp_sum_##SUF(lane);                                                             \
    }                                                                                            \
    if (c1v[k + 1] != (T)0) {                                                                    \
      s->flags |= FLAG_NONFINITE_OP;                                                             \
      s->done = 1;                                                                               \
      return;                                                                                    \
    }                                                                                            \
    const double w0 = (double)SQRT(c1v[k]);                                                      \
    for (int i = 0; i < k; ++i) s->c1[i] = c1v[i];                                               \
    s->w0 = w0;                                                                                  \
    /* ---- P2: w' = w - V c1 (8 warp partials per row, summed in warp order), pass-2 dots */    \
    for (long long b = 0; b < G; ++b) {                                                          \
      const long long nb = b < nblk ? (nblk - 1 - b) / G + 1 : 0;                                \
      T cred[MEGA_GROUPS][72];                                                                   \
      for (int grp = 0; grp < MEGA_GROUPS; ++grp) {                                              \
        T acc[8][8][32]; /* [gw][q][lane] */                                                     \
        for (int gw = 0; gw < 8; ++gw)                                                           \
          for (int q = 0; q < KV; ++q)                                                           \
            for (int l = 0; l < 32; ++l) acc[gw][q][l] = 0;                                      \
        for (long long t = grp; t < nb; t += MEGA_GROUPS) {                                      \
          const long long b0 = (b + t * G) * RB;                                                 \
          T up[8][32 * VN];                                                                      \
          for (int gw = 0; gw < 8; ++gw)                                                         \
            for (int l = 0; l < 32; ++l) {                                                       \
              const long long r = b0 + (long long)l * VN;                                        \
              const int in = r < n;                                                              \
              for (int e = 0; e < VN; ++e) {                                                     \
                T u = 0;                                                                         \
                for (int q = 0; q < KV; ++q) {                                                   \
                  const int i = gw + 8 * q;                                                      \
                  const T v = (in && i < k && r + e < n) ? V[(size_t)i * n + r + e] : (T)0;      \
                  const T c = i < k ? c1v[i] : (T)0;                                             \
                  u = FMA(v, c, u);                                                              \
                }                                                                                \
                up[gw][l * VN + e] = u;                                                          \
              }                                                                                  \
            }                                                                                    \
          for (int row = 0; row < RB; ++row) {                                                   \
            T sm = 0;                                                                            \
            for (int ww = 0; ww < 8; ++ww) sm += up[ww][row];                                    \
            if (b0 + row < n) w[b0 + row] = w[b0 + row] - sm;                                    \
          }                                                                                      \
          for (int gw = 0; gw < 8; ++gw)                                                         \
            for (int q = 0; q < KV; ++q) {                                                       \
              const int i = gw + 8 * q;                                                          \
              for (int l = 0; l < 32; ++l) {                                                     \
                const long long r = b0 + (long long)l * VN;                                      \
                const int in = r < n;                                                            \
                for (int e = 0; e < VN; ++e) {                                                   \
                  const T v = (in && i < k && r + e < n) ? V[(size_t)i * n + r + e] : (T)0;      \
                  const T xv = r + e < n ? w[r + e] : (T)0;                                      \
                  acc[gw][q][l] = FMA(v, xv, acc[gw][q][l]);                                     \
                }                                                                                \
              }                                                                                  \
            }                                                                                    \
        }                                                                                        \
        for (int gw = 0; gw < 8; ++gw)                                                           \
          for (int q = 0; q < KV; ++q) {                                                         \
            const int i = gw + 8 * q;                                                            \
            if (i < k) cred[grp][i] = warp_sum_##SUF(acc[gw][q]);                                \
          }                                                                                      \
      }                                                                                          \
      for (int i = 0; i < k; ++i) {                                                              \
        T t = 0;                                                                                 \
        for (int grp = 0; grp < MEGA_GROUPS; ++grp) t += cred[grp][i];                           \
        part[(size_t)(72 + i) * MAX_PARTS + b] = t;                                              \
      }                                                                                          \
    }                                                                                            \
    T c2v[72];                                                                                   \
    for (int c = 0; c < k; ++c) {                                                                \
      T lane[32];                                                                                \
      for (int l = 0; l < 32; ++l) {                                                             \
        T sm = 0;                                                                                \
        for (long long p = l; p < G; p += 32) sm += part[(size_t)(72 + c) * MAX_PARTS + p];      \
        lane[l] = sm;                                                                            \
      }                                                                                          \
      c2v[c] = warp_sum_##SUF(lane);                                                             \
    }                                                                                            \
    const int ld = s->m + 1;                                                                     \
    for (int i = 0; i < k; ++i) {                                                                \
      s->c2[i] = c2v[i];                                                                         \
      s->H[(size_t)j * ld + i] = ((T)0 + c1v[i]) + c2v[i];                                       \
    }                                                                                            \
    /* ---- P3: w'' = w' - V c2 (sequential over the basis per row), ||w''||^2 */                \
    for (long long b = 0; b < G; ++b) {                                                          \
      const long long nb = b < nblk ? (nblk - 1 - b) / G + 1 : 0;                                \
      T lane[32], red[MEGA_WARPS];                                                               \
      for (int wp = 0; wp < MEGA_WARPS; ++wp) {                                                  \
        for (int l = 0; l < 32; ++l) {                                                           \
          T ss = 0;                                                                              \
          for (long long t = wp; t < nb; t += MEGA_WARPS) {                                      \
            const long long r = (b + t * G) * RB + (long long)l * VN;                            \
            for (int e = 0; e < VN; ++e) {                                                       \
              T u = 0;                                                                           \
              if (r < n)                                                                         \
                for (int i = 0; i < k; ++i) {                                                    \
                  const T v = r + e < n ? V[(size_t)i * n + r + e] : (T)0;                       \
                  u = FMA(v, c2v[i], u);                                                         \
                }                                                                                \
              T wv = 0;                                                                          \
              if (r + e < n) {                                                                   \
                wv = w[r + e] - u;                                                               \
                w[r + e] = wv;                                                                   \
              }                                                                                  \
              ss = FMA(wv, wv, ss);                                                              \
            }                                                                                    \
          }                                                                                      \
          lane[l] = ss;                                                                          \
        }                                                                                        \
        red[wp] = warp_sum_##SUF(lane);                                                          \
      }                                                                                          \
      T tn = 0;                                                                                  \
      for (int wp = 0; wp < MEGA_WARPS; ++wp) tn += red[wp];                                     \
      part[(size_t)144 * MAX_PARTS + b] = tn;                                                    \
    }                                                                                            \
    T nl[32];                                                                                    \
    for (int l = 0; l < 32; ++l) {                                                               \
      T sm = 0;                                                                                  \
      for (long long p = l; p < G; p += 32) sm += part[(size_t)144 * MAX_PARTS + p];             \
      nl[l] = sm;                                                                                \
    }                                                                                            \
    const T hs = SQRT(warp_sum_##SUF(nl));                                                       \
    s->brk = (double)hs <= s->btol * w0;                                                         \
    s->H[(size_t)j * ld + j + 1] = hs;                                                           \
    givens_##SUF(s, j, m_limit);                                                                 \
    if (s->brk) return;                                                                          \
    /* ---- P4: V[:, j+1] = w'' / h */                                                           \
    T* vn = V + (size_t)(j + 1) * n;                                                             \
    for (int r = 0; r < n; ++r) vn[r] = w[r] / hs;                                               \
  }                                                                                              \
                                                                                                 \
  /* arnoldi_kernels.cu k_lsq (krylov.py:190-202, xTRSV column order) */                         \
  static void lsq_##SUF(st_##SUF* s) {                                                           \
    const int k = s->steps, ld = s->m + 1;                                                       \
    if (k == 0 || (s->flags & (FLAG_NONFINITE_OP | FLAG_NONFINITE_GAMMA | FLAG_OVERFLOW)))       \
      return;                                                                                    \
    for (int i = 0; i < k; ++i) {                                                                \
      const T r = s->R[(size_t)i * ld + i];                                                      \
      if (r == (T)0 || !isfinite(r)) {                                                           \
        s->flags |= FLAG_SINGULAR;                                                               \
        return;                                                                                  \
      }                                                                                          \
      s->d[i] = s->g[i];                                                                         \
    }                                                                                            \
    for (int jj = k - 1; jj >= 0; --jj) {                                                        \
      if (s->d[jj] != (T)0) s->d[jj] = s->d[jj] / s->R[(size_t)jj * ld + jj];                    \
      const T temp = s->d[jj];                                                                   \
      if (temp != (T)0)                                                                          \
        for (int i = 0; i < jj; ++i) s->d[i] = FMA(-temp, s->R[(size_t)jj * ld + i], s->d[i]);   \
    }                                                                                            \
  }                                                                                              \
  /* arnoldi_kernels.cu k_combine: per row, sequential fma over the basis */                     \
  static T combine_row_##SUF(const T* V, int n, int k, const T* d, int r) {                      \
    T acc = 0;                                                                                   \
    for (int i = 0; i < k; ++i) acc = FMA(V[(size_t)i * n + r], d[i], acc);                      \
    return acc;                                                                                  \
  }                                                                                              \
  static void st_init_##SUF(st_##SUF* s, int m) {                                                \
    const size_t hm = (size_t)(m + 1) * m;                                                       \
    s->m = m;                                                                                    \
    s->H = (T*)calloc(hm, sizeof(T));                                                            \
    s->R = (T*)calloc(hm, sizeof(T));                                                            \
    s->cs = (T*)calloc((size_t)m + 1, sizeof(T));                                                \
    s->sn = (T*)calloc((size_t)m + 1, sizeof(T));                                                \
    s->g = (T*)calloc((size_t)m + 1, sizeof(T));                                                 \
    s->c1 = (T*)calloc((size_t)m + 1, sizeof(T));                                                \
    s->c2 = (T*)calloc((size_t)m + 1, sizeof(T));                                                \
    s->d = (T*)calloc((size_t)m + 1, sizeof(T));                                                 \
    s->steps = s->done = s->brk = s->flags = 0;                                                  \
  }                                                                                              \
  static void st_free_##SUF(st_##SUF* s) {                                                       \
    free(s->H); free(s->R); free(s->cs); free(s->sn); free(s->g);                                \
    free(s->c1); free(s->c2); free(s->d);                                                        \
  }                                                                                              \
  /* the Arnoldi steps + least squares of one cycle from V[:, 0] (solver.cu enqueue_cycle) */    \
  static void run_steps_##SUF(int n, const int32_t* rp, const int32_t* ci, const T* vals, T* V,  \
                              st_##SUF* s, int m_limit, int nsm) {                               \
    T* w = (T*)calloc((size_t)n, sizeof(T));                                                     \
    T* part = (T*)calloc((size_t)145 * MAX_PARTS, sizeof(T));                                    \
    for (int j = 0; j < m_limit && !s->done; ++j)                                                \
      mega_step_##SUF(n, rp, ci, vals, V, j, w, s, m_limit, nsm, part);                          \
    free(part);                                                                                  \
    free(w);                                                                                     \
    lsq_##SUF(s);                                                                                \
  }

DEVORDER_IMPL(float, f32, fmaf, sqrtf, hypot_ref_f, 4)
DEVORDER_IMPL(double, f64, fma, sqrt, hypot_ref_d, 2)

/* init_state (arnoldi_kernels.cu): gamma, thresholds, done on zero/non-finite gamma */
#define INIT_STATE(s, gamma, bnorm, rtol, btol, extra)          \
  do {                                                          \
    (s)->g[0] = (gamma);                                        \
    (s)->flags = (extra);                                       \
    (s)->done = 0;                                              \
    if (!isfinite(gamma)) { (s)->flags |= FLAG_NONFINITE_GAMMA; (s)->done = 1; } \
    if ((gamma) == 0) (s)->done = 1;                            \
    if ((extra) != 0) (s)->done = 1;                                 \
    (s)->threshold = (rtol) * ((bnorm) < 0 ? (double)(gamma) : (bnorm)); \
    (s)->btol = (btol);                                         \
  } while (0)

/* Output record of one cycle: info[0] steps, [1] breakdown, [2] flags. */

/* One restarted cycle in the working precision T from the outer residual r
 * (k_start with b_norm = ||b||, k_start_scale, the steps, k_lsq, k_combine
 * CMB_ADD: x += V d).  x is updated in place. */
int devorder_cycle_f32(int n, const int32_t* rp, const int32_t* ci, const float* vals, const float* r,
                       double outer_bnorm, double rtol, double btol, int m, int m_limit, float* x,
                       double* implicit, int* info, int nsm) {
  st_f32 s;
  st_init_f32(&s, m);
  s.implicit = implicit;
  const float gamma = sqrtf(sumsq_stream_f32(r, n, grid_stream_f32(n, nsm)));
  INIT_STATE(&s, gamma, outer_bnorm, rtol, btol, 0);
  float* V = (float*)calloc((size_t)(m + 1) * n, sizeof(float));
  if (!s.done)
    for (int i = 0; i < n; ++i) V[i] = r[i] / s.g[0];
  run_steps_f32(n, rp, ci, vals, V, &s, m_limit, nsm);
  if (s.steps && !(s.flags & (FLAG_NONFINITE_OP | FLAG_NONFINITE_GAMMA | FLAG_OVERFLOW | FLAG_SINGULAR)))
    for (int i = 0; i < n; ++i) x[i] = x[i] + combine_row_f32(V, n, s.steps, s.d, i);
  info[0] = s.steps; info[1] = s.brk; info[2] = s.flags;
  free(V);
  st_free_f32(&s);
  return 0;
}

int devorder_cycle_f64(int n, const int32_t* rp, const int32_t* ci, const double* vals, const double* r,
                       double outer_bnorm, double rtol, double btol, int m, int m_limit, double* x,
                       double* implicit, int* info, int nsm) {
  st_f64 s;
  st_init_f64(&s, m);
  s.implicit = implicit;
  const double gamma = sqrt(sumsq_stream_f64(r, n, grid_stream_f64(n, nsm)));
  INIT_STATE(&s, gamma, outer_bnorm, rtol, btol, 0);
  double* V = (double*)calloc((size_t)(m + 1) * n, sizeof(double));
  if (!s.done)
    for (int i = 0; i < n; ++i) V[i] = r[i] / s.g[0];
  run_steps_f64(n, rp, ci, vals, V, &s, m_limit, nsm);
  if (s.steps && !(s.flags & (FLAG_NONFINITE_OP | FLAG_NONFINITE_GAMMA | FLAG_OVERFLOW | FLAG_SINGULAR)))
    for (int i = 0; i < n; ++i) x[i] = x[i] + combine_row_f64(V, n, s.steps, s.d, i);
  info[0] = s.steps; info[1] = s.brk; info[2] = s.flags;
  free(V);
  st_free_f64(&s);
  return 0;
}

/* One GMRES-IR inner cycle (k_start_ir: r32 = fp32(r64 / rho), gamma = ||r32||,
 * the inner b_norm is gamma; then the fp32 steps; k_combine CMB_IR:
 * x64 += rho * fp64(V d)).  x64 is updated in place. */
int devorder_cycle_ir(int n, const int32_t* rp, const int32_t* ci, const float* vals32, const double* r64,
                      double rho, double rtol, double btol, int m, int m_limit, double* x64,
                      double* implicit, int* info, int nsm) {
  st_f32 s;
  st_init_f32(&s, m);
  s.implicit = implicit;
  float* r32 = (float*)malloc(sizeof(float) * (size_t)n);
  int ovf = 0;
  for (int i = 0; i < n; ++i) {
    const double q = r64[i] / rho;
    const float v = (float)q;
    ovf |= isinf(v) && isfinite(q);
    r32[i] = v;
  }
  const float gamma = sqrtf(sumsq_stream_f32(r32, n, grid_stream_f32(n, nsm)));
  INIT_STATE(&s, gamma, -1.0, rtol, btol, ovf ? FLAG_OVERFLOW : 0);
  float* V = (float*)calloc((size_t)(m + 1) * n, sizeof(float));
  if (!s.done)
    for (int i = 0; i < n; ++i) V[i] = r32[i] / s.g[0];
  run_steps_f32(n, rp, ci, vals32, V, &s, m_limit, nsm);
  if (s.steps && !(s.flags & (FLAG_NONFINITE_OP | FLAG_NONFINITE_GAMMA | FLAG_OVERFLOW | FLAG_SINGULAR))) {
    for (int i = 0; i < n; ++i) {
      const float acc = combine_row_f32(V, n, s.steps, s.d, i);
      if (!isfinite(acc)) s.flags |= FLAG_NONFINITE_X;
      x64[i] = x64[i] + rho * (double)acc;
    }
  }
  info[0] = s.steps; info[1] = s.brk; info[2] = s.flags;
  free(V);
  free(r32);
  st_free_f32(&s);
  return 0;
}

/* the grid of the padded-stencil residual launch (spmv_kernels.cu launch_matrix)
 * for `occ` resident CTAs per SM */
long long devorder_residual_grid(long long n, int vn, int nsm, int occ) {
  const long long tile = 256LL * vn, tiles = (n + tile - 1) / tile;
  long long g = (long long)nsm * occ;
  if (tiles < g) g = tiles;
  if (g > MAX_PARTS) g = MAX_PARTS;
  return g < 1 ? 1 : g;
}

/* the SpMV alone (spmv.py:48-72 order), for the CPU pin against cpu_gmres.spmv */
void devorder_spmv_f32(int n, const int32_t* rp, const int32_t* ci, const float* v, const float* x, float* y) {
  spmv_f32(n, rp, ci, v, x, y);
}
void devorder_spmv_f64(int n, const int32_t* rp, const int32_t* ci, const double* v, const double* x, double* y) {
  spmv_f64(n, rp, ci, v, x, y);
}
