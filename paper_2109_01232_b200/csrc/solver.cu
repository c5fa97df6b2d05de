// Native solver driver: enqueues whole restart cycles (solvers.py:122-227,
// 297-384) on the device and replays them as CUDA graphs.  The host reads
// the cycle's scalar record (state header + implicit residuals) once per
// cycle; nothing inside a cycle synchronises with the host — the reference's
// per-step Python `break` (solvers.py:164-168) is a device-side done flag.
#include <map>
#include <vector>

#include "spmv.cuh"
#include "state.cuh"

struct mpg_solver {
  mpg_solver_desc d;
  std::vector<mpg_poly_op> ops;
  std::map<int, cudaGraphExec_t> graphs;  // per m_limit
  std::map<int, int> graph_launches;      // kernels per graph (for the launch counter)
  cudaStream_t cap = nullptr;
  // the working-precision dia carries one coefficient per slot (read once at
  // create from the packing header): the step kernel's KONST instantiation
  int dia_const = 0;
};

namespace mpg {

// Optional per-kernel-class CUDA-event profiling of an eager cycle.
struct Prof {
  cudaStream_t st;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
};
static thread_local Prof* t_prof = nullptr;
struct ProfScope {
  int k;
  cudaEvent_t a = nullptr;
  explicit ProfScope(int kind) : k(kind) {
    if (t_prof) {
      cudaEventCreate(&a);
      cudaEventRecord(a, t_prof->st);
    }
  }
  ~ProfScope() {
    if (t_prof) {
      cudaEvent_t b;
      cudaEventCreate(&b);
      cudaEventRecord(b, t_prof->st);
      t_prof->ev.push_back({k, {a, b}});
    }
  }
};
enum { PK_START = 0, PK_PRECOND, PK_SPMV_DOT, PK_UPDATE_DOT, PK_UPDATE_NORM, PK_SCALE, PK_FINISH,
       PK_RESIDUAL, PK_DOT1, PK_STEP, PK_COUNT };   // PK_SPMV_DOT: the SpMV alone when K_A is split;
                                                    // PK_STEP: the persistent per-step kernel

#define TRY(...)                       \
  do {                                   \
    cudaError_t e_ = (__VA_ARGS__);      \
    if (e_ != cudaSuccess) return e_;    \
  } while (0)

static mpg_state_header* hdr_of(const mpg_solver_desc& d) {
  return static_cast<mpg_state_header*>(d.state);
}

template <typename TP, typename F>
static cudaError_t with_matrix(const mpg_solver_desc& d, const TP* csr_vals, const void* dia,
                               F&& f);

// r = b - A x, rnorm -> header, in the outer precision (solvers.py:186-188,
// :205, :330, :358): fp64 for GMRES-IR and fp64 GMRES, fp32 for the fp32 solver.
static cudaError_t outer_residual(const mpg_solver_desc& d, WsView ws, cudaStream_t st) {
  mpg_state_header* h = hdr_of(d);
  // GMRES-IR's refinement residual is "Other" (timing.suspended, solvers.py:328,356);
  // the restarted solvers bin theirs as SpMV (solvers.py:186,205 through spmv)
  const int kcat = d.mode == MPG_MODE_IR ? KC_OTHER : KC_SPMV;
  if (d.mode == MPG_MODE_IR || d.prec == MPG_FP64) {
    const double* vals = d.mode == MPG_MODE_IR ? d.values64 : static_cast<const double*>(d.values);
    const void* dia = d.mode == MPG_MODE_IR ? static_cast<const void*>(d.dia64) : d.dia;
    return with_matrix<double>(d, vals, dia, [&](const auto& A) {
      return launch_residual<double>(A, static_cast<const double*>(d.b),
                                     static_cast<const double*>(d.x), static_cast<double*>(d.r),
                                     nullptr, h, ws, st, 0, h, kcat);
    });
  }
  return with_matrix<float>(d, static_cast<const float*>(d.values), d.dia, [&](const auto& A) {
    return launch_residual<float>(A, static_cast<const float*>(d.b), static_cast<const float*>(d.x),
                                  static_cast<float*>(d.r), nullptr, h, ws, st, 0, h, kcat);
  });
}

// Call f with the matrix view the solver uses: the stencil (DIA) storage
// when the descriptor carries one, the CSR arrays otherwise.
template <typename TP, typename F>
static cudaError_t with_matrix(const mpg_solver_desc& d, const TP* csr_vals, const void* dia,
                               F&& f) {
  if (d.stencil_dims && dia) {
    StencilView<TP> S{static_cast<const TP*>(dia), d.dia_ld ? d.dia_ld : d.ldv, d.n, d.stencil_nx,
                      d.stencil_dims, d.row0};
    const long long plane = d.stencil_dims == 3 ? (long long)d.stencil_nx * d.stencil_nx : d.stencil_nx;
    S.padded = d.halo >= plane ? 1 : 0;
    S.konst = 1;   // descriptor dia buffers are packed by mpg_stencil_pack* (header in the tail)
    return f(S);
  }
  return f(CsrView<TP>{d.row_ptr, d.col_idx, csr_vals, d.n});
}

// Run a lowered polynomial program on x -> y with scratch t0..t2, in TP.
template <typename TP>
static cudaError_t run_poly(const mpg_solver_desc& d, const std::vector<mpg_poly_op>& ops,
                            const TP* vals, const TP* x, TP* y, TP* t0, TP* t1, TP* t2,
                            const mpg_state_header* gate, WsView ws, cudaStream_t st) {
  const mpg_state_header* kt = hdr_of(d);   // its SpMVs are binned SpMV (precond.py:300-319)
  TP* bufs[5] = {const_cast<TP*>(x), y, t0, t1, t2};
  for (const mpg_poly_op& op : ops) {
    switch (op.op) {
      case MPG_POLY_SCALE:
      case MPG_POLY_ACC:
      case MPG_POLY_ZERO:
        TRY(launch_poly_elem<TP>(op.op, (TP)op.a, bufs[op.src], bufs[op.dst], y, d.n, gate, st));
        break;
      default:
        TRY(with_matrix<TP>(d, vals, d.pc_dia, [&](const auto& A) {
          return launch_poly_op<TP>(A, op, x, y, t0, t1, t2, gate, d.n, ws, st, kt);
        }));
    }
  }
  return cudaSuccess;
}

// z = M^{-1} v for the Arnoldi operator (solvers.py:159: op = A(M^{-1} v)).
// Returns the buffer holding z (v itself when there is no preconditioner).
template <typename T>
static cudaError_t precond_apply(const mpg_solver& s, const T* v, const T** z, WsView ws,
                                 const mpg_state_header* gate, cudaStream_t st) {
  const mpg_solver_desc& d = s.d;
  *z = v;
  if (d.pc_kind == MPG_PC_NONE) return cudaSuccess;
  const bool cast = d.pc_prec != d.prec;  // fp32 preconditioner in an fp64 solve
  if (!cast) {
    T* out = static_cast<T*>(d.pc_t0);
    if (d.pc_kind == MPG_PC_JACOBI) {
      TRY(launch_jacobi<T>(d.n, d.pc_block, static_cast<const T*>(d.pc_lu), d.pc_piv, v, out, gate, st));
    } else {
      TRY(run_poly<T>(d, s.ops, static_cast<const T*>(d.pc_values), v, out,
                      static_cast<T*>(d.pc_t1), static_cast<T*>(d.pc_t2), static_cast<T*>(d.pc_t3),
                      gate, ws, st));
    }
    *z = out;
    return cudaSuccess;
  }
  if constexpr (sizeof(T) == 8) {
    // cast_apply (precond.py:393-414): narrow, apply in fp32, widen
    float* v32 = static_cast<float*>(d.pc_t0);
    float* y32 = static_cast<float*>(d.pc_t1);
    TRY(launch_cast_gated<double, float>(v, v32, d.n, gate, ws.scratch_i64, st));
    if (d.pc_kind == MPG_PC_JACOBI) {
      TRY(launch_jacobi<float>(d.n, d.pc_block, static_cast<const float*>(d.pc_lu), d.pc_piv, v32, y32, gate, st));
    } else {
      TRY(run_poly<float>(d, s.ops, static_cast<const float*>(d.pc_values), v32, y32,
                          static_cast<float*>(d.pc_t2), static_cast<float*>(d.pc_t3),
                          static_cast<float*>(d.pc_t4), gate, ws, st));
    }
    T* out = static_cast<T*>(d.u);
    TRY(launch_cast_gated<float, double>(y32, out, d.n, gate, nullptr, st));
    *z = out;
    return cudaSuccess;
  }
  return cudaErrorInvalidValue;
}

// End of cycle: d = R^{-1} g ; x <- x + M^{-1}(V d)   (solvers.py:169-174, 357)
template <typename T>
static cudaError_t finish_cycle(const mpg_solver& s, StateView<T> sv, WsView ws, cudaStream_t st) {
  const mpg_solver_desc& d = s.d;
  const T* V = static_cast<const T*>(d.V);
  TRY(launch_lsq<T>(sv, st));
  const bool ir = d.mode == MPG_MODE_IR;
  const bool cast = d.pc_kind != MPG_PC_NONE && d.pc_prec != d.prec;
  if (d.pc_kind == MPG_PC_NONE)
    return launch_combine<T>(V, d.ldv, d.n, sv, ir ? CMB_IR : CMB_ADD, d.x, nullptr, nullptr, st);
  if (d.pc_kind == MPG_PC_JACOBI && d.pc_block == 1) {
    const int mode = cast ? CMB_J1_CAST : (ir ? CMB_J1_IR : CMB_J1_ADD);
    return launch_combine<T>(V, d.ldv, d.n, sv, mode, d.x, d.pc_lu, nullptr, st);
  }
  // general: u = V d, z = M^{-1} u (ungated), x += z
  T* u = static_cast<T*>(d.u);
  TRY(launch_combine<T>(V, d.ldv, d.n, sv, CMB_STORE, nullptr, nullptr, u, st));
  if (!cast) {
    T* z = static_cast<T*>(d.pc_t0);
    if (d.pc_kind == MPG_PC_JACOBI)
      TRY(launch_jacobi<T>(d.n, d.pc_block, static_cast<const T*>(d.pc_lu), d.pc_piv, u, z, nullptr, st));
    else
      TRY(run_poly<T>(d, s.ops, static_cast<const T*>(d.pc_values), u, z, static_cast<T*>(d.pc_t1),
                      static_cast<T*>(d.pc_t2), static_cast<T*>(d.pc_t3), nullptr, ws, st));
    if (ir) {
      if constexpr (sizeof(T) == 4)
        return launch_finish_add<float, double>(static_cast<double*>(d.x), z, d.n, sv.h, 1, st);
      return cudaErrorInvalidValue;
    }
    return launch_finish_add<T, T>(static_cast<T*>(d.x), z, d.n, sv.h, 0, st);
  }
  if constexpr (sizeof(T) == 8) {
    float* u32 = static_cast<float*>(d.pc_t0);
    float* y32 = static_cast<float*>(d.pc_t1);
    TRY(launch_cast_gated<double, float>(u, u32, d.n, nullptr, ws.scratch_i64, st));
    if (d.pc_kind == MPG_PC_JACOBI)
      TRY(launch_jacobi<float>(d.n, d.pc_block, static_cast<const float*>(d.pc_lu), d.pc_piv, u32, y32, nullptr, st));
    else
      TRY(run_poly<float>(d, s.ops, static_cast<const float*>(d.pc_values), u32, y32,
                          static_cast<float*>(d.pc_t2), static_cast<float*>(d.pc_t3),
                          static_cast<float*>(d.pc_t4), nullptr, ws, st));
    return launch_finish_add<float, double>(static_cast<double*>(d.x), y32, d.n, sv.h, 2, st);
  }
  return cudaErrorInvalidValue;
}

template <typename T>
static cudaError_t enqueue_cycle(const mpg_solver& s, int m_limit, cudaStream_t st) {
  const mpg_solver_desc& d = s.d;
  StateView<T> sv = make_state<T>(d.state, d.m);
  WsView ws = make_ws(d.ws);
  T* V = static_cast<T*>(d.V);
  T* w = static_cast<T*>(d.w);
  const T* vals = static_cast<const T*>(d.values);
  mpg_state_header* h = hdr_of(d);
  // cycle start: gamma, V[:,0] = r0 / gamma
  {
  ProfScope ps(PK_START);
  if (d.mode == MPG_MODE_IR) {
    if constexpr (sizeof(T) == 4) {
      TRY(launch_start_ir(static_cast<const double*>(d.r), static_cast<float*>(d.r_in), d.n, sv,
                          d.rtol, d.breakdown_tol, ws, st));
      TRY(launch_start_scale<T>(static_cast<const T*>(d.r_in), V, d.n, sv, st));
    } else {
      return cudaErrorInvalidValue;
    }
  } else {
    TRY(launch_start<T>(static_cast<const T*>(d.r), d.n, sv, d.rtol, &h->outer_b_norm,
                        d.breakdown_tol, ws, st));
    TRY(launch_start_scale<T>(static_cast<const T*>(d.r), V, d.n, sv, st));
  }
  }
  // single-GPU stencil storage, unpreconditioned or Jacobi(1) in the working
  // precision: one persistent cooperative kernel per Arnoldi step
  // (step_kernel.cu; for Jacobi(1) it also writes the next z = v / diag)
  const bool jac1 = d.pc_kind == MPG_PC_JACOBI && d.pc_block == 1 && d.pc_prec == d.prec;
  const bool mega_ok = (d.pc_kind == MPG_PC_NONE || jac1) && !d.dist && d.stencil_dims && d.dia &&
                       d.halo >= (d.stencil_dims == 3 ? (long long)d.stencil_nx * d.stencil_nx
                                                      : (long long)d.stencil_nx);
  int sk = d.step_kernel;
  if (mega_env() >= 0) sk = mega_env() ? 2 : 1;
  const bool mega = mega_ok && (sk == 2 || (sk == 0 && (double)d.n * sizeof(T) <= 20e6));
  for (int j = 0; j < m_limit; ++j) {
    T* const wj = w;
    if (mega && j + 1 <= kMegaMaxK) {
      const T* xin = V + (size_t)j * d.ldv;
      T* zbuf = jac1 ? static_cast<T*>(d.pc_t0) : nullptr;
      // Jacobi: z_0 comes from the apply kernel; later z_j from the previous step kernel
      if (jac1 && j == 0) {
        ProfScope pp(PK_PRECOND);
        const T* z = nullptr;
        TRY(precond_apply<T>(s, xin, &z, ws, h, st));
      }
      ProfScope ps(PK_STEP);
      StencilView<T> S{static_cast<const T*>(d.dia), d.dia_ld ? d.dia_ld : d.ldv, d.n, d.stencil_nx,
                       d.stencil_dims, d.row0};
      S.padded = 1;
      S.konst = s.dia_const ? 2 : 0;   // 2: header known on, step kernel KONST instantiation
      // the last persistent step hands the four-launch steps V[:, j+1]; they apply M themselves
      const bool next_mega = j + 2 <= kMegaMaxK && j + 1 < m_limit;
      TRY(launch_step_mega<T>(S, jac1 ? zbuf : xin, V, d.ldv, d.n, j, wj, sv, ws, m_limit, st,
                              jac1 && next_mega ? static_cast<const T*>(d.pc_lu) : nullptr,
                              jac1 && next_mega ? zbuf : nullptr));
      continue;
    }
    const T* vj = V + (size_t)j * d.ldv;
    const T* z = nullptr;
    { ProfScope ps(PK_PRECOND); TRY(precond_apply<T>(s, vj, &z, ws, h, st)); }
    if (split_spmv_dot1()) {
      {
        ProfScope ps(PK_SPMV_DOT);
        TRY(with_matrix<T>(d, vals, d.dia, [&](const auto& A) { return launch_spmv<T>(A, z, wj, ws, st, h); }));
      }
      ProfScope ps(PK_DOT1);
      TRY(launch_dot1_wo<T>(wj, d.n, V, d.ldv, j + 1, sv, ws, st));
    } else {
      ProfScope ps(PK_SPMV_DOT);
      TRY(with_matrix<T>(d, vals, d.dia, [&](const auto& A) {
        return launch_spmv_dot1<T>(A, z, wj, V, d.ldv, j + 1, sv, ws, st);
      }));
    }
    { ProfScope ps(PK_UPDATE_DOT); TRY(launch_update_dot<T>(V, d.ldv, d.n, j + 1, wj, sv, ws, st)); }
    if (fuse_update_norm_scale()) {
      ProfScope ps(PK_UPDATE_NORM);
      TRY(launch_update_norm_scale<T>(V, d.ldv, d.n, j, wj, sv, ws, m_limit, st));
      continue;
    }
    { ProfScope ps(PK_UPDATE_NORM); TRY(launch_update_norm<T>(V, d.ldv, d.n, j, wj, sv, ws, m_limit, st)); }
    {
      ProfScope ps(PK_SCALE);
      TRY(launch_step_scale<T>(wj, V + (size_t)(j + 1) * d.ldv, d.n, j, sv, st));
    }
  }
  { ProfScope ps(PK_FINISH); TRY(finish_cycle<T>(s, sv, ws, st)); }
  ProfScope ps(PK_RESIDUAL);
  // explicit residual in the outer precision (solvers.py:205 / :358)
  return outer_residual(d, ws, st);
}

// One phase of a distributed cycle (MPG_PH_*): the same kernels in dist mode
// (raw local sums) plus the 1-CTA post kernels; collectives are the caller's.
template <typename T>
static cudaError_t enqueue_phase(const mpg_solver& s, int phase, int j, int m_limit,
                                 cudaStream_t st) {
  const mpg_solver_desc& d = s.d;
  StateView<T> sv = make_state<T>(d.state, d.m);
  sv.dist = 1;
  WsView ws = make_ws(d.ws);
  T* V = static_cast<T*>(d.V);
  T* w = static_cast<T*>(d.w);
  mpg_state_header* h = hdr_of(d);
  const bool ir = d.mode == MPG_MODE_IR;
  const bool outer64 = ir || d.prec == MPG_FP64;
  switch (phase) {
    case MPG_PH_BNORM:
      return outer64 ? launch_norm2<double>(static_cast<const double*>(d.b), d.n, &h->reserved[0], ws, st, 1)
                     : launch_norm2<float>(static_cast<const float*>(d.b), d.n, &h->reserved[0], ws, st, 1);
    case MPG_PH_POST_BNORM:
      return launch_dist_post<T>(DP_POST_BNORM, sv, 0, 0, d.rtol, d.breakdown_tol, outer64, st);
    case MPG_PH_RESID:
      if (outer64) {
        const void* dia = ir ? static_cast<const void*>(d.dia64) : d.dia;
        const double* vals = ir ? d.values64 : static_cast<const double*>(d.values);
        return with_matrix<double>(d, vals, dia, [&](const auto& A) {
          return launch_residual<double>(A, static_cast<const double*>(d.b),
                                         static_cast<const double*>(d.x), static_cast<double*>(d.r),
                                         nullptr, h, ws, st, 1);
        });
      }
      return with_matrix<float>(d, static_cast<const float*>(d.values), d.dia, [&](const auto& A) {
        return launch_residual<float>(A, static_cast<const float*>(d.b), static_cast<const float*>(d.x),
                                      static_cast<float*>(d.r), nullptr, h, ws, st, 1);
      });
    case MPG_PH_POST_RESID:
      return launch_dist_post<T>(DP_POST_RESID, sv, 0, 0, d.rtol, d.breakdown_tol, outer64, st);
    case MPG_PH_START:
      if (ir) {
        if constexpr (sizeof(T) == 4)
          return launch_start_ir(static_cast<const double*>(d.r), static_cast<float*>(d.r_in), d.n, sv,
                                 d.rtol, d.breakdown_tol, ws, st);
        return cudaErrorInvalidValue;
      }
      return launch_start<T>(static_cast<const T*>(d.r), d.n, sv, d.rtol, &h->outer_b_norm,
                             d.breakdown_tol, ws, st);
    case MPG_PH_POST_START:
      return launch_dist_post<T>(DP_POST_START, sv, 0, 0, d.rtol, d.breakdown_tol, ir ? 1 : 0, st);
    case MPG_PH_START_SCALE:
      return launch_start_scale<T>(static_cast<const T*>(ir ? d.r_in : d.r), V, d.n, sv, st);
    case MPG_PH_SPMV_DOT:
      if (j >= 1 && d.halo_flags && (d.peer_prev_V || d.peer_next_V))
        TRY(launch_halo_wait(h, d.halo_flags, d.peer_prev_V ? 1 : 0, d.peer_next_V ? 1 : 0, st));
      if (split_spmv_dot1()) {
        TRY(with_matrix<T>(d, static_cast<const T*>(d.values), d.dia, [&](const auto& A) {
          return launch_spmv<T>(A, V + (size_t)j * d.ldv, w, ws, st);
        }));
        return launch_dot1_wo<T>(w, d.n, V, d.ldv, j + 1, sv, ws, st);
      }
      return with_matrix<T>(d, static_cast<const T*>(d.values), d.dia, [&](const auto& A) {
        return launch_spmv_dot1<T>(A, V + (size_t)j * d.ldv, w, V, d.ldv, j + 1, sv, ws, st);
      });
    case MPG_PH_POST_DOT1:
      return launch_dist_post<T>(DP_POST_DOT1, sv, j, m_limit, d.rtol, d.breakdown_tol, 0, st);
    case MPG_PH_UPDATE_DOT:
      return launch_update_dot<T>(V, d.ldv, d.n, j + 1, w, sv, ws, st);
    case MPG_PH_POST_DOT2:
      return launch_dist_post<T>(DP_POST_DOT2, sv, j, m_limit, d.rtol, d.breakdown_tol, 0, st);
    case MPG_PH_UPDATE_NORM:
      return launch_update_norm<T>(V, d.ldv, d.n, j, w, sv, ws, m_limit, st);
    case MPG_PH_POST_NORM:
      return launch_dist_post<T>(DP_POST_NORM, sv, j, m_limit, d.rtol, d.breakdown_tol, 0, st);
    case MPG_PH_SCALE:
      if (d.halo_flags && (d.peer_prev_V || d.peer_next_V)) {
        T* prow = d.peer_prev_V ? static_cast<T*>(d.peer_prev_V) + (size_t)(j + 1) * d.peer_prev_ld + d.peer_prev_off
                                : nullptr;
        T* nrow = d.peer_next_V ? static_cast<T*>(d.peer_next_V) + (size_t)(j + 1) * d.peer_next_ld + d.peer_next_off
                                : nullptr;
        return launch_step_scale_peer<T>(w, V + (size_t)(j + 1) * d.ldv, d.n, d.halo, j, sv, prow, nrow,
                                         d.peer_prev_V ? d.peer_prev_flag : nullptr,
                                         d.peer_next_V ? d.peer_next_flag : nullptr, ws, st);
      }
      return launch_step_scale<T>(w, V + (size_t)(j + 1) * d.ldv, d.n, j, sv, st);
    case MPG_PH_FINISH:
      return finish_cycle<T>(s, sv, ws, st);
    case MPG_PH_STEP: {
      // the whole Arnoldi step in one cooperative kernel, the three cross-rank
      // sums over the exchange boxes (step_kernel.cu DIST); V[:, j]'s halo is
      // in place (collective exchange before j = 0, peer stores after)
      if (d.xworld < 1 || d.xworld > kXMaxRanks || !d.xbox[d.xrank] || d.pc_kind != MPG_PC_NONE)
        return cudaErrorInvalidValue;
      MegaX<T> X{};
      for (int r = 0; r < d.xworld; ++r) X.box[r] = d.xbox[r];
      X.world = d.xworld;
      X.rank = d.xrank;
      X.halo = d.halo;
      if (d.xworld > 1) {
        X.prev_V = static_cast<T*>(d.peer_prev_V);
        X.prev_ld = d.peer_prev_ld;
        X.prev_off = d.peer_prev_off;
        X.next_V = static_cast<T*>(d.peer_next_V);
        X.next_ld = d.peer_next_ld;
        X.next_off = d.peer_next_off;
        X.hflags = d.halo_flags;
        X.prev_flag = d.peer_prev_flag;
        X.next_flag = d.peer_next_flag;
      }
      StencilView<T> S{static_cast<const T*>(d.dia), d.dia_ld ? d.dia_ld : d.ldv, d.n, d.stencil_nx,
                       d.stencil_dims, d.row0};
      S.padded = 1;
      S.konst = s.dia_const ? 2 : 0;
      return launch_step_mega<T>(S, V + (size_t)j * d.ldv, V, d.ldv, d.n, j, w, sv, ws, m_limit, st, nullptr,
                                 nullptr, &X);
    }
    default:
      return cudaErrorInvalidValue;
  }
}

static cudaError_t enqueue_any(const mpg_solver& s, int m_limit, cudaStream_t st) {
  return s.d.prec == MPG_FP64 ? enqueue_cycle<double>(s, m_limit, st)
                              : enqueue_cycle<float>(s, m_limit, st);
}

}  // namespace mpg

using namespace mpg;

extern "C" int mpg_solver_create(const mpg_solver_desc* desc, mpg_solver** out) {
  if (!desc || !out) return MPG_EARG;
  const mpg_solver_desc& d = *desc;
  if (d.m < 1 || d.m > kMaxM || d.n < 1 || d.ldv < d.n || d.ldv % 64) return MPG_EARG;
  if (d.prec != MPG_FP32 && d.prec != MPG_FP64) return MPG_EARG;
  if (d.mode == MPG_MODE_IR && (d.prec != MPG_FP32 || !d.values64 || !d.r_in)) return MPG_EARG;
  if (!d.row_ptr || !d.col_idx || !d.values || !d.x || !d.b || !d.r || !d.V || !d.w || !d.state || !d.ws)
    return MPG_EARG;
  if (d.stencil_dims) {
    if ((d.stencil_dims != 2 && d.stencil_dims != 3) || d.stencil_nx < 2 || !d.dia) return MPG_EARG;
    const long long nx = d.stencil_nx;
    const long long N = d.stencil_dims == 3 ? nx * nx * nx : nx * nx;
    if (N >= (1LL << 32)) return MPG_EARG;
    if (!d.dist && d.n != N) return MPG_EARG;
    if (d.dist && (d.row0 < 0 || d.row0 + d.n > N)) return MPG_EARG;
    if (d.mode == MPG_MODE_IR && !d.dia64) return MPG_EARG;
    if (d.pc_kind == MPG_PC_POLY && !d.pc_dia) return MPG_EARG;
  }
  if (d.pc_kind != MPG_PC_NONE) {
    if (d.pc_prec != d.prec && !(d.pc_prec == MPG_FP32 && d.prec == MPG_FP64)) return MPG_EUNSUPPORTED;
    if (d.pc_kind == MPG_PC_JACOBI && (!d.pc_lu || d.pc_block < 1 || d.pc_block > 32)) return MPG_EARG;
    if (d.pc_kind == MPG_PC_JACOBI && d.pc_block > 1 && !d.pc_piv) return MPG_EARG;
    if (d.pc_kind == MPG_PC_POLY && (!d.pc_ops || d.pc_nops < 1 || !d.pc_values)) return MPG_EARG;
    if (!d.pc_t0 || !d.pc_t1) return MPG_EARG;
  }
  if (d.dist && (!d.stencil_dims || d.pc_kind != MPG_PC_NONE)) return MPG_EUNSUPPORTED;
  mpg_solver* s = new mpg_solver();
  s->d = d;
  if (d.stencil_dims && d.dia) {   // constant-coefficient header (spmv.cuh StencilConst)
    const int S = d.stencil_dims == 3 ? 7 : 5;
    const size_t es = d.prec == MPG_FP64 ? 8 : 4;
    const char* hp = static_cast<const char*>(d.dia) + (size_t)S * (d.dia_ld ? d.dia_ld : d.ldv) * es;
    double h64 = 0.0;
    float h32 = 0.f;
    cudaDeviceSynchronize();
    if (cudaMemcpy(es == 8 ? (void*)&h64 : (void*)&h32, hp, es, cudaMemcpyDeviceToHost) == cudaSuccess)
      s->dia_const = (es == 8 ? h64 != 0.0 : h32 != 0.f) ? 1 : 0;
    cudaGetLastError();
  }
  if (d.pc_kind == MPG_PC_POLY) s->ops.assign(d.pc_ops, d.pc_ops + d.pc_nops);
  s->d.pc_ops = nullptr;
  if (cudaStreamCreateWithFlags(&s->cap, cudaStreamNonBlocking) != cudaSuccess) {
    delete s;
    return (int)cudaGetLastError();
  }
  *out = s;
  return MPG_OK;
}

extern "C" int mpg_solver_destroy(mpg_solver* s) {
  if (!s) return MPG_OK;
  for (auto& kv : s->graphs) cudaGraphExecDestroy(kv.second);
  if (s->cap) cudaStreamDestroy(s->cap);
  delete s;
  return MPG_OK;
}

extern "C" int mpg_solver_begin(mpg_solver* s, void* stream) {
  if (!s) return MPG_ESTATE;
  const mpg_solver_desc& d = s->d;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  WsView ws = make_ws(d.ws);
  mpg_state_header* h = hdr_of(d);
  const bool outer64 = d.mode == MPG_MODE_IR || d.prec == MPG_FP64;
  // kernel-time accumulators restart with the solve (the first stamp opens)
  cudaError_t e = cudaMemsetAsync(h->ktime_ns, 0, sizeof(h->ktime_ns) + sizeof(h->kt_mark), st);
  if (e) return e;
  e = outer64
      ? launch_norm2<double>(static_cast<const double*>(d.b), d.n, &h->outer_b_norm, ws, st)
      : launch_norm2<float>(static_cast<const float*>(d.b), d.n, &h->outer_b_norm, ws, st);
  if (e) return e;
  return (int)outer_residual(d, ws, st);
}

extern "C" int mpg_solver_cycle(mpg_solver* s, int32_t m_limit, void* stream) {
  if (!s) return MPG_ESTATE;
  if (m_limit < 1 || m_limit > s->d.m) return MPG_EARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!s->d.use_graph) return (int)enqueue_any(*s, m_limit, st);
  auto it = s->graphs.find(m_limit);
  if (it == s->graphs.end()) {
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamBeginCapture(s->cap, cudaStreamCaptureModeRelaxed);
    if (e) return e;
    const int64_t before = mpg_launch_count();
    e = enqueue_any(*s, m_limit, s->cap);
    cudaError_t e2 = cudaStreamEndCapture(s->cap, &g);
    if (e) { if (g) cudaGraphDestroy(g); return e; }
    if (e2) return e2;
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e) return e;
    it = s->graphs.emplace(m_limit, ex).first;
    s->graph_launches[m_limit] = (int)(mpg_launch_count() - before);
    count_launch(-(int)(mpg_launch_count() - before));  // capture is not execution
  }
  cudaError_t e = cudaGraphLaunch(it->second, st);
  if (e == cudaSuccess) count_launch(s->graph_launches[m_limit]);
  return (int)e;
}

extern "C" int mpg_solver_phase(mpg_solver* s, int32_t phase, int32_t j, int32_t m_limit,
                                void* stream) {
  if (!s || !s->d.dist) return MPG_ESTATE;
  if (j < 0 || j >= s->d.m || m_limit < 1 || m_limit > s->d.m) return MPG_EARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return (int)(s->d.prec == MPG_FP64 ? enqueue_phase<double>(*s, phase, j, m_limit, st)
                                     : enqueue_phase<float>(*s, phase, j, m_limit, st));
}

extern "C" int mpg_solver_profile_cycle(mpg_solver* s, int32_t m_limit, void* stream,
                                        double* ms_out, int32_t* launches_out) {
  if (!s || !ms_out) return MPG_EARG;
  if (m_limit < 1 || m_limit > s->d.m) return MPG_EARG;
  Prof p;
  p.st = static_cast<cudaStream_t>(stream);
  t_prof = &p;
  cudaError_t e = enqueue_any(*s, m_limit, p.st);
  t_prof = nullptr;
  cudaError_t e2 = cudaStreamSynchronize(p.st);
  for (int k = 0; k < PK_COUNT; ++k) {
    ms_out[k] = 0.0;
    if (launches_out) launches_out[k] = 0;
  }
  for (auto& r : p.ev) {
    float ms = 0.f;
    if (!e && !e2) cudaEventElapsedTime(&ms, r.second.first, r.second.second);
    ms_out[r.first] += ms;
    if (launches_out) launches_out[r.first] += 1;
    cudaEventDestroy(r.second.first);
    cudaEventDestroy(r.second.second);
  }
  return (int)(e ? e : e2);
}
