/*
 * kktdd_b200.h — C-ABI of the B200-native hot path for the heat-control KKT
 * solve of arXiv 2305.04421 (reference: /root/reference/proj, C++ "kktdd").
 *
 * The boundary replaces the reference's operator / preconditioner / Krylov
 * interfaces in proj/include/kktdd/*.hpp.  Every entry point below names the
 * reference function it stands in for (file:line).  Conventions:
 *
 *  - All vector arguments are DEVICE pointers (cudaMalloc'd or managed) in the
 *    reference layout (proj/include/kktdd/layout.hpp:15-40): time-major, then
 *    j-outer / i-inner, one contiguous block of n_sp doubles per time node.
 *    A KKT vector is [u; z; w] of 3 * block doubles (kkt.hpp:15-28).
 *    Exception: the *_host entry points take HOST pointers (pageable or pinned)
 *    and do the host<->device copies themselves.
 *  - in and out must not alias (heat_operators.hpp:41-42) unless the entry
 *    point says "in place".
 *  - Every entry point returns a status (KKT_OK = 0).  The reference throws
 *    C++ exceptions instead; the mapping is:
 *       std::invalid_argument        -> KKT_EINVAL
 *       ConfigError                  -> KKT_ECONFIG   (config.hpp:82-85)
 *       SingularMatrixError{pivot}   -> KKT_ESINGULAR (linalg.hpp:14-19), pivot
 *                                       index via kkt_last_error_index()
 *       GmresDivergenceError{iter}   -> KKT_EDIVERGED (gmres.hpp:22-27), the
 *                                       iteration via kkt_last_error_index()
 *    plus KKT_ECUDA / KKT_ENCCL for device / collective failures.
 *  - One context per GPU rank; calls on a context are stream-ordered on the
 *    context's stream and are not thread-safe per context (the reference is
 *    single-threaded).
 */
#ifndef KKTDD_B200_H
#define KKTDD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
enum {
  KKT_OK = 0,
  KKT_EINVAL = 1,
  KKT_ECONFIG = 2,
  KKT_ESINGULAR = 3,
  KKT_EDIVERGED = 4,
  KKT_ECUDA = 5,
  KKT_ENCCL = 6,
  KKT_EUNSUPPORTED = 7
};

/* ---- enums mirroring proj/include/kktdd/config.hpp:12-21 ---------------- */
enum { KKT_PRECOND_NONE = 0, KKT_PRECOND_ONE_LEVEL = 1, KKT_PRECOND_TWO_LEVEL = 2,
       KKT_PRECOND_DENSE_SCHUR = 3, KKT_PRECOND_TRUE_SCHUR = 4 };
enum { KKT_COARSE_SCALAR = 0, KKT_COARSE_PER_DOF = 1 };
enum { KKT_FORM_LITERAL = 0, KKT_FORM_MULTIPLICATIVE = 1, KKT_FORM_ADDITIVE = 2 };
enum { KKT_SIGN_PLUS = 0, KKT_SIGN_MINUS = 1 };
#define KKT_NO_RESTART (-1)  /* GmresParams::restart == std::nullopt (config.hpp:26) */

/* Arithmetic mode of the device path.
 *  STRICT: every kernel reproduces the reference's floating-point operation
 *          order (no FMA contraction, sequential dot products, the reference's
 *          banded LU substitution order), so results are bitwise identical to
 *          the compiled reference.  Used to pin the residual-history gate.
 *  FAST:   the performance path: FMA, deterministic tree reductions, blocked
 *          triangular solves with inverted diagonal blocks, fused two-level
 *          residual.  Rounding-level differences only. */
enum { KKT_MODE_FAST = 0, KKT_MODE_STRICT = 1, KKT_MODE_SPECTRAL = 2 };
/*  SPECTRAL: FAST arithmetic, but the spatial solves inside RASQ use Ahat's
 *          sine eigenbasis (fp64 tensor-core transforms + one scalar time
 *          recurrence per eigenmode) instead of the reference's banded-LU
 *          substitution.  Same linear operator to rounding, but NOT the
 *          reference's method (north_star asks for the LU method), so it is
 *          opt-in and reported separately; FAST is the headline path. */

/* POD mirror of ProblemConfig (config.hpp:35-68) + GmresParams (:23-28).
 * Field meanings and defaults are the reference's. */
typedef struct kkt_problem_desc {
  double Lx, Ly, T;
  int32_t Nx, Ny, Nt;
  double nu, omega;
  int32_t Nd;
  int32_t precond;          /* KKT_PRECOND_* */
  int32_t coarse_variant;   /* KKT_COARSE_*  */
  int32_t two_level_form;   /* KKT_FORM_*    */
  int32_t jhat_sign;        /* KKT_SIGN_*    */
  /* GmresParams */
  double tol;
  int32_t max_iters;
  int32_t restart;          /* KKT_NO_RESTART (-1): full GMRES, i.e. std::nullopt; any other value
                               < 1 is a ConfigError ("gmres restart must be >= 1", config.cpp:21) */
  double happy_breakdown_tol;
} kkt_problem_desc;

/* Fills the reference defaults (config.hpp:36-50, :24-27). */
void kkt_problem_desc_default(kkt_problem_desc* d);

/* Runtime options (no reference counterpart: device placement). */
typedef struct kkt_runtime_opts {
  int32_t mode;             /* KKT_MODE_* */
  int32_t device;           /* CUDA device ordinal, -1 = current */
  int32_t rank, nranks;     /* time-slab sharding; nranks == 1 for a single GPU */
  const void* nccl_unique_id; /* 128-byte ncclUniqueId when nranks > 1 (one process per GPU) */
  void* stream;             /* cudaStream_t, NULL = context-owned stream */
  void* local_group;        /* kkt_local_group_create handle: ranks as host threads of one
                               process (testing the sharded path on one device); else NULL */
} kkt_runtime_opts;

typedef struct kkt_ctx kkt_ctx;

/* Replaces: HeatOperators ctor (heat_operators.cpp:46-55), build_time_partition
 * (time_partition.cpp:61-86) and make_schur_solver (schur.cpp:543-558).
 * Factors Ahat on the device and builds the coarse space. */
int kkt_ctx_create(const kkt_problem_desc* desc, const kkt_runtime_opts* opts, kkt_ctx** out);
int kkt_ctx_destroy(kkt_ctx* ctx);
const char* kkt_last_error(const kkt_ctx* ctx);
int kkt_last_error_index(const kkt_ctx* ctx);
const char* kkt_status_string(int status);
/* Error message of the last failed kkt_ctx_create on this thread. */
const char* kkt_create_error(void);
/* Its index payload (SingularMatrixError::pivot_index), -1 if none. */
int kkt_create_error_index(void);

/* Sizes: global layout size (SpaceTimeLayout::size(), layout.hpp:25), the
 * rank-local node slab [node_first, node_last] and local block size. */
int kkt_layout(const kkt_ctx* ctx, int64_t* block, int32_t* n_sp, int32_t* node_first,
               int32_t* node_last, int64_t* local_block);
int kkt_stream(const kkt_ctx* ctx, void** stream);
int kkt_synchronize(kkt_ctx* ctx);

/* Device vectors for callers that do not link the CUDA runtime themselves (the
 * reference is plain host C++: its std::vector<double> / std::span arguments
 * become buffers obtained here; include/kktdd_gpu.hpp wraps them).  `count` is
 * in doubles.  Copies are ordered on the context's stream and complete before
 * the call returns. */
int kkt_device_alloc(kkt_ctx* ctx, size_t count, double** out);
int kkt_device_free(kkt_ctx* ctx, double* p);
int kkt_copy_to_device(kkt_ctx* ctx, double* dst_device, const double* src_host, size_t count);
int kkt_copy_to_host(kkt_ctx* ctx, double* dst_host, const double* src_device, size_t count);

/* ---- heat operators (heat_operators.hpp:41-61), full space-time blocks ---- */
int kkt_apply_J(kkt_ctx* ctx, const double* u, double* out);      /* heat_operators.cpp:57-69 */
int kkt_apply_JT(kkt_ctx* ctx, const double* w, double* out);     /* :71-83  */
int kkt_apply_L(kkt_ctx* ctx, const double* z, double* out);      /* :85-89  */
int kkt_apply_LT(kkt_ctx* ctx, const double* w, double* out);     /* :91-93  */
int kkt_apply_Mu(kkt_ctx* ctx, const double* u, double* out);     /* :95-99  */
int kkt_apply_Mu_inv(kkt_ctx* ctx, const double* u, double* out); /* :101-105 */
int kkt_apply_Mz(kkt_ctx* ctx, const double* z, double* out);     /* :107-109 */
int kkt_apply_Jhat(kkt_ctx* ctx, const double* u, double* out);   /* :111-123 */
int kkt_apply_JhatT(kkt_ctx* ctx, const double* w, double* out);  /* :125-137 */
/* In place over `len` consecutive n_sp planes (heat_operators.cpp:139-169). */
int kkt_forward_solve_window(kkt_ctx* ctx, double* b, int32_t len);
int kkt_adjoint_solve_window(kkt_ctx* ctx, double* b, int32_t len);
/* One spatial solve Ahat x = b in place (BandedLU::solve_in_place,
 * linalg.cpp:127-145) and its transpose (:147-162), `nrhs` planes. */
int kkt_band_solve(kkt_ctx* ctx, double* b, int32_t nrhs);
int kkt_band_solve_transpose(kkt_ctx* ctx, double* b, int32_t nrhs);

/* ---- KKT level (kkt.hpp:48-65) ----------------------------------------- */
int kkt_apply_K(kkt_ctx* ctx, const double* v, double* out);      /* kkt.cpp:50-65 */
int kkt_apply_P_inv(kkt_ctx* ctx, const double* r, double* out);  /* kkt.cpp:71-81 */
/* apply_P_inv end to end from HOST buffers (pageable or pinned): copies r in, applies, copies
 * the result out; returns when out_host is complete.  The copies overlap the compute (the w block
 * goes up first and the sweep starts; the u and z blocks follow in chunks that are divided and
 * sent back as they land; with pinned buffers the w planes go back behind the adjoint sweep);
 * the result is bitwise that of kkt_apply_P_inv. */
int kkt_apply_P_inv_host(kkt_ctx* ctx, const double* r_host, double* out_host);
/* ||rhs - K v|| / ||rhs|| (kkt.cpp:110-124). */
int kkt_residual(kkt_ctx* ctx, const double* v, const double* rhs, double* relres);

/* ---- Schur level (schur.hpp:214-337) ------------------------------------ */
int kkt_apply_shat(kkt_ctx* ctx, const double* v, double* out);   /* schur.cpp:71-78 */
int kkt_apply_rasq(kkt_ctx* ctx, const double* r, double* out);   /* schur.cpp:103-130 */
int kkt_apply_two_level(kkt_ctx* ctx, const double* r, double* out, int32_t form); /* :415-444 */
int kkt_schur_apply(kkt_ctx* ctx, const double* r, double* out);  /* SchurSolver::apply :494-533 */
/* CoarseSpace (schur.cpp:181-234); c is a DEVICE vector of coarse_dim. */
int kkt_coarse_dim(const kkt_ctx* ctx, int32_t* dim);
int kkt_coarse_restrict(kkt_ctx* ctx, const double* r, double* c);
int kkt_coarse_solve(kkt_ctx* ctx, double* c);
int kkt_coarse_prolong_add(kkt_ctx* ctx, const double* c, double* out);
/* Dense S0 (CoarseSpace::coarse_matrix_dense, schur.cpp:253-264), HOST out,
 * row-major dim x dim. */
int kkt_coarse_matrix(kkt_ctx* ctx, double* host_out);

/* ---- Krylov (gmres.hpp:11-36) ------------------------------------------- */
typedef struct kkt_gmres_result {
  int32_t converged;
  int32_t iterations;
  double true_final_relres;
  int32_t history_len;      /* entries written to the caller's history buffer */
} kkt_gmres_result;

/* gmres_solve(apply_K, apply_P_inv or identity, b, params) (gmres.cpp:21-155)
 * with the context's preconditioner (desc.precond; NONE = empty map).
 * b, x: DEVICE KKT vectors (rank-local slab when sharded).  history: HOST
 * buffer of at least max_iters doubles (may be NULL). */
int kkt_gmres_solve(kkt_ctx* ctx, const double* b, double* x, kkt_gmres_result* res,
                    double* history, int32_t history_cap);
/* Same, end to end from HOST buffers: copies b in, solves, copies x out. */
int kkt_gmres_solve_host(kkt_ctx* ctx, const double* b_host, double* x_host,
                         kkt_gmres_result* res, double* history, int32_t history_cap);

/* ---- the end-to-end run record (experiments.hpp:14-31) ------------------ */
/* evaluate_objective (kkt.cpp:88-108): 0.5 ms sum (u - target)^2 +
 * 0.5 omega ms sum z^2.  u, z, target: DEVICE blocks (rank-local slab when
 * sharded); target holds the caller's SpaceTimeFn sampled at the layout's
 * nodes (t = n dt, x = i dx, y = j dy). */
int kkt_evaluate_objective(kkt_ctx* ctx, const double* u, const double* z, const double* target,
                           double* objective);
/* assemble_rhs(ops, model_initial_condition, model_target).to_kkt()
 * (kkt.cpp:21-48, model_problem.hpp:11-18) for this context's slab, into HOST
 * buffers: b (3 x local block) and the target samples (local block; may be NULL). */
int kkt_model_rhs(kkt_ctx* ctx, double* b_host, double* target_host);

typedef struct kkt_run_record {
  int32_t iterations;
  int32_t converged;
  double true_final_relres;
  double objective;
  double setup_seconds;     /* context + preconditioner setup + model RHS */
  double solve_seconds;     /* GMRES on the device, b and x resident in HBM */
} kkt_run_record;

/* run_single(cfg) (experiments.cpp:33-69): set up, solve the model problem,
 * evaluate the objective.  Non-convergence is recorded, not an error.
 * x_host (3 x local block, may be NULL) receives the solution.  On failure the
 * message is in kkt_create_error(). */
int kkt_run_single(const kkt_problem_desc* desc, const kkt_runtime_opts* opts,
                   kkt_run_record* rec, double* x_host);

/* ---- instrumentation ---------------------------------------------------- */
/* Number of kernels this context launched since creation (or last reset). */
int kkt_launch_count(const kkt_ctx* ctx, int64_t* count);
int kkt_reset_launch_count(kkt_ctx* ctx);
/* Per-phase device time (ms) of the last kkt_gmres_solve, measured with CUDA
 * events on the context stream: [0]=K apply, [1]=P^-1 apply, [2]=Krylov
 * vector kernels, [3]=sweep kernel only.  Only filled when profiling is on. */
int kkt_set_phase_timing(kkt_ctx* ctx, int32_t on);
int kkt_phase_times(const kkt_ctx* ctx, double* ms4, int64_t* counts4);

/* Copies the device Ahat factor in the reference's band storage
 * (BandedLU::ab_, linalg.hpp:65-74; (kl + ku_ + 1) rows per column) and its
 * pivot vector to HOST buffers (either may be NULL). */
int kkt_debug_ahat_factor(kkt_ctx* ctx, int32_t* kl, int32_t* ku, double* ab_host, int32_t* piv_host);
/* Same for the per-dof coarse operator's banded LU (SparseLU -> BandedLU,
 * linalg.cpp:312-331; entry (i,j) at j*(kl+ku+1) + i-j+ku with ku = the
 * fill-extended upper bandwidth).  KKT_ECONFIG without a per-dof coarse space. */
int kkt_debug_coarse_factor(kkt_ctx* ctx, int32_t* kl, int32_t* ku, double* ab_host, int32_t* piv_host);

/* Multi-rank bring-up (time-slab sharding).  Rank g of G owns
 * subdomains [g*Nd/G, (g+1)*Nd/G) and their nodes; every vector argument is
 * then the rank-local slab [u_loc; z_loc; w_loc] (kkt_layout gives its size).
 * G must divide Nd; STRICT mode is single-rank.
 * kkt_nccl_unique_id: a fresh ncclUniqueId (128 bytes) for kkt_runtime_opts.
 * kkt_local_group_*: an in-process group whose ranks are host threads sharing
 * one device; exchanges are host-synchronised between launches. */
int kkt_nccl_unique_id(void* out128);
int kkt_local_group_create(int32_t nranks, void** out);
int kkt_local_group_destroy(void* group);

#ifdef __cplusplus
}
#endif
#endif /* KKTDD_B200_H */
