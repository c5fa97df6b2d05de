/*
 * mpgmres_b200.h — C ABI of the B200-native mixed-precision GMRES hot path.
 *
 * The reference (arXiv 2109.01232's `mpgmres` package, /root/reference/pkg)
 * is pure Python over numpy/scipy; its plug points are the Python functions
 * cited below.  This library replaces the numeric work behind each of them
 * with hand-written sm_100a kernels.  The Python package
 * `paper_2109_01232_b200` binds these symbols with ctypes and re-exposes the
 * reference's Python API on top (see INTEGRATION.md for the binding).
 *
 * Conventions (all entry points):
 *  - Plain pointers and sizes only; no torch types.  Device pointers are CUDA
 *    global-memory pointers allocated by the caller; the library never
 *    allocates or frees device memory.  `stream` is a cudaStream_t (NULL =
 *    legacy default stream).  Everything is asynchronous on `stream` unless
 *    stated otherwise.
 *  - Return value: 0 on success, a positive cudaError_t on a CUDA failure,
 *    or a negative MPG_E* code for invalid arguments.  Numerical faults
 *    (non-finite operator output, overflow on narrowing, singular triangular
 *    factor) are reported through device-side flags (MPG_FLAG_*) that the
 *    host maps onto the reference's exception types.
 *  - Precision codes: MPG_FP32 = float, MPG_FP64 = double.  Index arrays are
 *    int32 (the reference caps nnz below 2^31, core.py:145-146).
 *  - Device vectors the library writes with vector loads/TMA must be padded
 *    to `ld` elements (a multiple of 64); CSR arrays must be 16-byte aligned
 *    with at least 16 readable bytes past their end.
 */
#ifndef MPGMRES_B200_H
#define MPGMRES_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPG_FP32 0
#define MPG_FP64 1

#define MPG_OK 0
#define MPG_EARG (-1)         /* invalid argument                          */
#define MPG_EUNSUPPORTED (-2) /* configuration not supported               */
#define MPG_ESTATE (-3)       /* solver handle misuse                      */

/* device flag bits (mpg_state_header.flags) */
#define MPG_FLAG_NONFINITE_OP 1    /* krylov.py:133-134  DivergenceError     */
#define MPG_FLAG_NONFINITE_GAMMA 2 /* solvers.py:150-153 DivergenceError     */
#define MPG_FLAG_SINGULAR 4        /* krylov.py:198-201 SingularHessenberg   */
#define MPG_FLAG_OVERFLOW 8        /* core.py:264-271   PrecisionOverflow    */
#define MPG_FLAG_NONFINITE_X 16    /* solvers.py:350-352 DivergenceError     */
#define MPG_FLAG_HALO_TIMEOUT 32   /* distributed peer halo: a neighbour's flag never arrived */

/* stencil kinds (gen.py:34-41) */
#define MPG_LAPLACE2D 0
#define MPG_LAPLACE3D 1
#define MPG_CONVDIFF2D 2
#define MPG_STRETCHED2D 3
#define MPG_BIHARMONIC2D 4
#define MPG_STAR2D 5
#define MPG_RECIRC2D 6

/* ---------------------------------------------------------------------- */
/* Library info                                                           */

/* Version string and the SM architecture the kernels were built for. */
const char* mpg_version(void);
/* Bytes of reduction workspace a stream needs (partials + counters).  The
 * workspace must be zero-initialised once before first use. */
int64_t mpg_workspace_bytes(void);
/* Number of kernel launches issued since load (host-side counter; the bench
 * reports it as gpu_launches). */
int64_t mpg_launch_count(void);

/* ---------------------------------------------------------------------- */
/* L1 kernel layer (reference core.py / spmv.py)                          */

/* y = A x, accumulated in A's precision with the reference's exact row
 * order p0 + pairwise(p1..)  (replaces spmv.py:48-72 `spmv`). */
int mpg_spmv(int prec, int64_t n_rows, const int32_t* row_ptr, const int32_t* col_idx,
             const void* values, const void* x, void* y, void* ws, void* stream);

/* r = b - A x and *norm_out (device double) = ||r||_2 in A's precision
 * (replaces solvers.py:443-453 `explicit_residual`). */
int mpg_residual(int prec, int64_t n_rows, const int32_t* row_ptr, const int32_t* col_idx,
                 const void* values, const void* b, const void* x, void* r, double* norm_out,
                 void* ws, void* stream);

/* *out (device double) = sqrt(dot(x, x)) in x's precision
 * (replaces core.py:341-354 `norm2`). */
int mpg_norm2(int prec, int64_t n, const void* x, double* out, void* ws, void* stream);

/* Dense multivector product y = alpha*op(A) x + beta*y where A holds `cols`
 * vectors of length `rows`, vector i at A + i*lda (Fortran order):
 * trans=1 -> y[cols] = A^T x ; trans=0 -> y[rows] = A x
 * (replaces core.py:295-338 `gemv`).  alpha/beta are host doubles rounded
 * to the working precision. */
int mpg_gemv(int prec, int trans, int64_t rows, int64_t cols, const void* A, int64_t lda,
             const void* x, void* y, double alpha, double beta, void* ws, void* stream);

/* y = (dst precision) x with round-to-nearest; on narrowing, the first index
 * whose finite value overflows is written to *overflow_index (device int64,
 * caller initialises it to -1) (replaces core.py:252-289 `convert_vector`,
 * and the values array of `convert_matrix`). */
int mpg_convert(int src_prec, int dst_prec, int64_t n, const void* x, void* y,
                int64_t* overflow_index, void* stream);

/* Elementwise helpers used by the drivers: y = x / s (IEEE division by the
 * device scalar *s, stored as double and rounded to the working precision),
 * and x += rho * widen(u) (solvers.py:357). */
int mpg_scale_div(int prec, int64_t n, const void* x, const double* s, void* y, void* stream);
int mpg_ir_correct(int64_t n, double* x64, const float* u32, const double* rho, void* stream);

/* ---------------------------------------------------------------------- */
/* Stencil assembly (reference gen.py)                                    */

/* (n, nnz) of a stencil without materialising (gen.py:111-126). Host. */
int mpg_stencil_counts(int kind, int64_t nx, int64_t* n, int64_t* nnz);
/* Number of stored entries in rows [0, row) of a stencil matrix. Host. */
int64_t mpg_stencil_nnz_before(int kind, int64_t nx, int64_t row);
/* Canonical fp64 CSR rows [row_begin, row_end) with global column indices
 * and row_ptr relative to row_begin (row_ptr[0] = 0), generated directly
 * on the device, bit-identical to gen.py:129-202 + core.py:229-249. */
int mpg_generate_stencil(int kind, int64_t nx, double convection, double stretch,
                         int64_t row_begin, int64_t row_end, int32_t* row_ptr,
                         int32_t* col_idx, double* values, void* stream);

/* Stencil-specialised SpMV storage (the north star's stencil path).  Checks
 * that the CSR pattern is exactly the Dirichlet 5-point (dims 2, n = nx^2) or
 * 7-point (dims 3, n = nx^3) stencil in canonical order and packs the values
 * slot-major into dia[S][ldv] (S = 5 or 7; absent neighbours hold a NaN
 * sentinel payload).  dia must hold S*ldv + 64 elements: the tail receives a
 * header (dia[S*ldv] = 1 when every slot has a single coefficient, then the S
 * coefficients) that lets the solver's SpMV stream x alone, bit-identically.
 * *bad (device int32, caller zeroes it) != 0 on mismatch. */
int mpg_stencil_pack(int prec, int dims, int64_t nx, int64_t n, const int32_t* row_ptr,
                     const int32_t* col_idx, const void* values, void* dia, int64_t ldv,
                     int32_t* bad, void* stream);
/* Same for rows [row0, row0 + nrows) of the global stencil (a rank's block):
 * row_ptr relative to row0 (row_ptr[0] = 0), global col_idx, as produced by
 * mpg_generate_stencil for that range.  dia is [S][ldv] over local rows. */
int mpg_stencil_pack_rows(int prec, int dims, int64_t nx, int64_t row0, int64_t nrows,
                          const int32_t* row_ptr, const int32_t* col_idx, const void* values,
                          void* dia, int64_t ldv, int32_t* bad, void* stream);
/* y = A x from the packed storage; bit-identical to mpg_spmv on the CSR. */
int mpg_spmv_dia(int prec, int dims, int64_t nx, int64_t n, const void* dia, int64_t ldv,
                 const void* x, void* y, void* ws, void* stream);

/* ---------------------------------------------------------------------- */
/* Preconditioners (reference precond.py)                                 */

/* y = blockdiag(LU)^{-1} x for a block-Jacobi factor with block size k;
 * k == 1 is y = x / lu (precond.py:363-390). */
int mpg_jacobi_apply(int prec, int64_t n, int32_t k, const void* lu, const int64_t* piv,
                     const void* x, void* y, void* stream);
/* Extract the k x k diagonal blocks of A and LU-factor them with partial
 * pivoting on the device (precond.py:326-360).  lu: (nb, k, k) row-major,
 * piv: (nb, k) LAPACK-style 0-based pivots; *bad_block (device int64,
 * caller sets -1) receives the first singular block. */
int mpg_jacobi_build(int prec, int64_t n, int32_t k, const int32_t* row_ptr,
                     const int32_t* col_idx, const void* values, void* lu, int64_t* piv,
                     int64_t* bad_block, void* stream);

/* One step of a polynomial-preconditioner program (precond.py:272-319).
 * The host lowers a PolynomialPreconditioner into a sequence of ops with
 * scalars already rounded to the working precision exactly as numpy does. */
#define MPG_POLY_SCALE 0       /* dst = a * x                        */
#define MPG_POLY_HORNER 1      /* dst = A src + a * x                */
#define MPG_POLY_ACC 2         /* y = y + a * src                    */
#define MPG_POLY_NEWTON_REAL 3 /* y = y + a*src ; dst = src - a*(A src) */
#define MPG_POLY_PAIR1 4       /* dst = A src ; y = y + (a*src - b*dst) */
#define MPG_POLY_PAIR2 5       /* dst = (p - a*src) + b*(A src), p = x2 */
#define MPG_POLY_ZERO 6        /* y = 0 ; dst = copy of x            */
typedef struct {
  int32_t op;
  int32_t src;  /* buffer ids: 0 = x (input), 1 = y (output), 2..4 = t0..t2 */
  int32_t dst;
  int32_t x2;
  double a;
  double b;
} mpg_poly_op;

int mpg_poly_apply(int prec, int64_t n, const int32_t* row_ptr, const int32_t* col_idx,
                   const void* values, const mpg_poly_op* ops, int32_t nops, const void* x,
                   void* y, void* t0, void* t1, void* t2, void* ws, void* stream);

/* ---------------------------------------------------------------------- */
/* L2 Krylov layer (reference krylov.py) — generic-operator path           */

/* Device state of one restart cycle.  Host-visible header followed by
 * `implicit[m]` doubles, then the working-precision arrays
 * H[(m+1)*m] (column-major, ld m+1), R[(m+1)*m], cos[m], sin[m], g[m+1],
 * c1[m+1], c2[m+1], d[m+1]. */
typedef struct {
  int32_t flags;      /* MPG_FLAG_* */
  int32_t steps;      /* Arnoldi steps completed in this cycle */
  int32_t done;       /* cycle finished (threshold, breakdown, limit, error) */
  int32_t breakdown;  /* last step hit the breakdown test */
  int32_t m;          /* capacity */
  int32_t prec;
  int32_t kt_cat;     /* device kernel timing: category of the running interval (-1 none) */
  int32_t reserved1;  /* distributed peer halo: sequence number */
  double gamma;         /* ||r0|| of the cycle, working precision value */
  double b_norm;        /* b_norm of the cycle's threshold */
  double threshold;     /* rtol * b_norm */
  double rnorm;         /* explicit residual norm after the cycle */
  double rho;           /* IR: scale of the inner right-hand side */
  double rtol;
  double breakdown_tol; /* 10 * unit roundoff unless overridden */
  double w0;            /* pre-orthogonalisation norm of the last step */
  double h_sub;         /* last subdiagonal entry */
  double outer_b_norm;  /* ||b|| of the outer problem (written by mpg_solver_begin) */
  double reserved[1];   /* distributed mode: raw local sums of the norm phases */
  /* Device time per kernel category (the reference's KernelTimer bins,
   * timing.py:17-23): [0] SpMV, [1] GemvTrans, [2] Norm, [3] GemvNoTrans, in
   * globaltimer nanoseconds, accumulated since mpg_solver_begin.  Each kernel
   * of a cycle stamps %globaltimer once in CTA 0 at entry (the persistent
   * step also at its internal grid barriers); the interval up to the next
   * stamp is charged to the category the stamp opened (Other is not stored:
   * the host takes it as total - sum, timing.py:44-47). */
  uint64_t ktime_ns[4];
  uint64_t kt_mark;     /* globaltimer of the last stamp */
} mpg_state_header;

/* Total bytes of a cycle state for restart length m in precision prec. */
int64_t mpg_state_bytes(int prec, int32_t m);
/* Byte offset of a named array inside the state (0 H,1 R,2 cos,3 sin,4 g,
 * 5 c1, 6 c2, 7 d, 8 implicit). */
int64_t mpg_state_offset(int prec, int32_t m, int32_t which);

/* Initialise a cycle from r0 (krylov.py:96-100, solvers.py:146-156):
 * gamma = ||r0||, V[:,0] = r0/gamma, threshold = rtol * (b_norm>0 ? b_norm
 * : gamma).  b_norm < 0 means "use gamma" (the IR inner solve). */
int mpg_cycle_start(int prec, int64_t n, int64_t ldv, int32_t m, const void* r0, void* V,
                    void* state, double rtol, double b_norm, double breakdown_tol,
                    int32_t m_limit, void* ws, void* stream);
/* Given w = op(V[:,j]) (length n, padded to ldv), run one CGS2 step and the
 * Givens update (krylov.py:112-187): finite check, w0, two classical GS
 * passes, h, h_sub, breakdown test, V[:,j+1] = w/h_sub, rotation, implicit
 * residual, done flag.  w is overwritten. */
int mpg_arnoldi_step(int prec, int64_t n, int64_t ldv, int32_t m, int32_t j, int32_t m_limit,
                     void* V, void* w, void* state, void* ws, void* stream);
/* Back-solve R d = g over the completed steps (krylov.py:190-202) and form
 * u = V[:, :k] d (solvers.py:171). */
int mpg_cycle_finish(int prec, int64_t n, int64_t ldv, int32_t m, const void* V, void* state,
                     void* u, void* stream);

/* ---------------------------------------------------------------------- */
/* L3 solver layer (reference solvers.py) — fused device cycles           */

#define MPG_MODE_RESTARTED 0 /* gmres_restarted / each leg of gmres_fd   */
#define MPG_MODE_IR 1        /* gmres_ir: fp32 cycles, fp64 refinement   */

#define MPG_PC_NONE 0
#define MPG_PC_JACOBI 1
#define MPG_PC_POLY 2

typedef struct {
  int32_t mode;       /* MPG_MODE_* */
  int32_t prec;       /* working precision of the Krylov cycle */
  int32_t m;          /* restart length */
  int32_t use_graph;  /* capture each cycle into a CUDA graph (1) or launch eagerly (0) */
  int64_t n;          /* rows */
  int64_t ldv;        /* padded vector length (multiple of 64, >= n) */
  double rtol;
  double breakdown_tol;
  /* matrix: pattern + values in the working precision */
  const int32_t* row_ptr;
  const int32_t* col_idx;
  const void* values;
  /* IR: fp64 values on the same pattern (the outer residual) */
  const double* values64;
  /* vectors (padded to ldv) */
  void* x;        /* iterate, outer precision (IR: fp64) */
  const void* b;  /* right-hand side, outer precision */
  void* r;        /* explicit residual, outer precision */
  void* r_in;     /* IR: fp32 inner right-hand side */
  void* V;        /* (m+1) x ldv basis, working precision */
  void* w;        /* Arnoldi work vector */
  void* u;        /* combination / preconditioner output */
  void* state;    /* mpg_state_bytes(prec, m) */
  void* ws;       /* mpg_workspace_bytes(), zeroed once, owned by this solver
                     (the persistent step's grid barrier keeps a monotonic
                     arrival counter in it for this solver's fixed grid) */
  /* right preconditioner */
  int32_t pc_kind;
  int32_t pc_prec;  /* == prec, or MPG_FP32 inside an fp64 solve (cast_apply) */
  int32_t pc_block; /* Jacobi block size */
  int32_t pc_nops;  /* poly program length */
  const void* pc_lu;
  const int64_t* pc_piv;
  const mpg_poly_op* pc_ops; /* host array, copied at create */
  const void* pc_values;     /* poly: matrix values in pc_prec */
  void* pc_t0;               /* scratch vectors in pc_prec (ldv each) */
  void* pc_t1;
  void* pc_t2;
  void* pc_t3;
  void* pc_t4;
  /* stencil-specialised storage (mpg_stencil_pack); stencil_dims 0 = CSR */
  int32_t stencil_dims;   /* 2: 5-point, 3: 7-point Dirichlet stencil */
  int32_t stencil_nx;
  const void* dia;        /* slot-major values, working precision, stride ldv */
  const double* dia64;    /* IR: fp64 values for the outer residual */
  const void* pc_dia;     /* poly preconditioner: values in pc_prec */
  /* row-partitioned (distributed) mode, driven phase by phase through
   * mpg_solver_phase with the caller's collectives in between */
  int32_t dist;           /* 1: this handle is one rank of a row partition */
  int32_t step_kernel;    /* 0 auto: one persistent cooperative kernel per Arnoldi step for
                             small vectors (n * sizeof(T) <= 20 MB; stencil storage, no
                             preconditioner, one GPU), else four launches; 1 four launches;
                             2 persistent whenever it applies */
  int64_t row0;           /* global index of local row 0 */
  int64_t halo;           /* readable rows on each side of every SpMV input (V rows, x,
                             preconditioner buffers): the distributed halo, or zero padding
                             on one GPU; >= one grid plane enables the branchless stencil rows */
  int64_t dia_ld;         /* slot stride of dia/dia64/pc_dia (0: same as ldv) */
  /* peer-memory halo (distributed mode, optional; all null = the caller
   * exchanges halos).  The SCALE phase of step j writes the first / last
   * `halo` rows of V[:, j+1] straight into the neighbours' halo rows (peer
   * mappings over NVLink: cudaIpcOpenMemHandle / P2P) and then releases a
   * sequence number into the neighbour's halo_flags; the SPMV phase of step
   * j+1 waits on this rank's own flags.  The basis row j of a neighbour
   * starts at peer_*_V + j * peer_*_ld; our rows land at offset peer_*_off
   * from its owned block (prev: its n_local, upper halo; next: -halo). */
  void* peer_prev_V;
  int64_t peer_prev_ld;
  int64_t peer_prev_off;
  void* peer_next_V;
  int64_t peer_next_ld;
  int64_t peer_next_off;
  uint32_t* halo_flags;     /* this rank's 2 flags: [0] written by prev, [1] by next */
  uint32_t* peer_prev_flag; /* the prev rank's halo_flags + 1 */
  uint32_t* peer_next_flag; /* the next rank's halo_flags + 0 */
  /* Distributed persistent step (MPG_PH_STEP): one cooperative kernel per
   * Arnoldi step per rank that also does the step's three cross-rank sums
   * over peer memory.  Every rank owns an exchange box of
   * mpg_xbox_bytes() bytes (zeroed once); xbox[r] is rank r's box as mapped
   * in this process (xbox[xrank] = this rank's own), r < xworld <= 8.  The
   * peer-memory halo fields above must be set for xworld > 1. */
  int32_t xworld;           /* 0: no in-kernel exchange (phase path only) */
  int32_t xrank;
  void* xbox[8];
} mpg_solver_desc;

/* Bytes of one rank's exchange box for the distributed persistent step. */
int64_t mpg_xbox_bytes(void);
/* Let kernels on the current device load / store memory of device `peer`
 * (cudaDeviceEnablePeerAccess; already-enabled and peer == current are OK).
 * Needed before the peer-memory halo / exchange-box stores reach an IPC
 * mapping owned by another GPU.  MPG_EUNSUPPORTED if the pair cannot peer. */
int mpg_enable_peer(int32_t peer);

/* Phases of one distributed restart cycle.  A phase marked
 * "raw" leaves this rank's partial sums in the state (red[] in the working
 * precision, or header reserved[0] as a double) for the caller to allreduce
 * (sum) before the matching POST phase; "halo" phases read the halo planes
 * of their input vector, which the caller exchanges beforehand. */
#define MPG_PH_BNORM 0        /* raw: sum b^2 -> reserved[0]                       */
#define MPG_PH_POST_BNORM 1
#define MPG_PH_RESID 2        /* halo(x); raw: local sum r^2 -> reserved[0]        */
#define MPG_PH_POST_RESID 3
#define MPG_PH_START 4        /* raw: gamma^2 (+ IR overflow) -> red[0..2)         */
#define MPG_PH_POST_START 5
#define MPG_PH_START_SCALE 6
#define MPG_PH_SPMV_DOT 7     /* halo(V[:,j]); raw: c1, w0^2, nonfinite -> red[0..j+3) */
#define MPG_PH_POST_DOT1 8
#define MPG_PH_UPDATE_DOT 9   /* raw: c2 -> red[0..j+1)                            */
#define MPG_PH_POST_DOT2 10
#define MPG_PH_UPDATE_NORM 11 /* raw: ||w||^2 -> red[0]                            */
#define MPG_PH_POST_NORM 12
#define MPG_PH_SCALE 13
#define MPG_PH_FINISH 14      /* back-solve (replicated) + local solution update   */
#define MPG_PH_STEP 15        /* the whole Arnoldi step j in one cooperative kernel:
                                 SPMV_DOT .. SCALE with the three cross-rank sums
                                 done in-kernel over the exchange boxes (needs
                                 xworld >= 1; halo(V[:,0]) before j = 0 only)  */

typedef struct mpg_solver mpg_solver;

/* sizeof(mpg_solver_desc) as compiled into the library (binding check). */
int64_t mpg_solver_desc_bytes(void);
int mpg_solver_create(const mpg_solver_desc* desc, mpg_solver** out);
int mpg_solver_destroy(mpg_solver* s);
/* b_norm = ||b|| and the initial explicit residual r = b - A x, rnorm
 * (solvers.py:186-188 / :328-330); results land in the state header. */
int mpg_solver_begin(mpg_solver* s, void* stream);
/* Enqueue one full restart cycle with at most m_limit steps, followed by
 * the solution update and the explicit residual (solvers.py:197-205 /
 * :338-358).  Nothing is synchronised; the host reads the state header. */
int mpg_solver_cycle(mpg_solver* s, int32_t m_limit, void* stream);
/* Profiling variant of mpg_solver_cycle: launches the same kernels eagerly
 * with CUDA events around each kernel class, synchronises, and writes the
 * summed milliseconds (and launch-group counts) per class into ms_out[9] /
 * launches_out[9]: 0 start, 1 preconditioner, 2 SpMV (+ CGS pass-1 dots when
 * fused, MPG_SPLIT_KA=0), 3 CGS update + pass-2 dots, 4 CGS update + norm +
 * Givens (+ basis scale when fused), 5 basis scale, 6 back-solve + solution
 * update, 7 explicit residual, 8 CGS pass-1 dots (split K_A, the default). */
int mpg_solver_profile_cycle(mpg_solver* s, int32_t m_limit, void* stream, double* ms_out,
                             int32_t* launches_out);
/* Enqueue one phase of a distributed cycle (desc.dist = 1); j = Arnoldi
 * step, m_limit = the cycle's step budget. */
int mpg_solver_phase(mpg_solver* s, int32_t phase, int32_t j, int32_t m_limit, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MPGMRES_B200_H */
