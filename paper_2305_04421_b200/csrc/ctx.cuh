// ctx.cuh — the device context behind the C-ABI handle (kkt_ctx).
//
// Holds what the reference keeps in HeatOperators (heat_operators.hpp:26-39),
// TimePartition (time_partition.hpp:26-42) and SchurSolver / CoarseSpace
// (schur.hpp:244-331), but with the factors and scratch in HBM.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "comm.cuh"
#include "common.cuh"

namespace kkt {

// Device buffer (RAII).
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  bool own = true;  // false: a view into another allocation (e.g. the L2-persisting arena)
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) KKT_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void view(T* q, size_t count) {
    release();
    p = q;
    n = count;
    own = false;
  }
  void release() {
    if (p && own) cudaFree(p);
    p = nullptr;
    n = 0;
    own = true;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), own(o.own) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; own = o.own; o.p = nullptr; o.n = 0; }
    return *this;
  }
};

struct NodeRange {
  int first = 0, last = -1;
  int count() const { return last - first + 1; }
};

// Coarse column bookkeeping (schur.hpp:246-250, schur.cpp:283-298).
struct CoarseColumn {
  int s, kind, dof;
};

struct Ctx {
  kkt_problem_desc desc{};
  int mode = KKT_MODE_FAST;
  bool spectral = false;           // KKT_MODE_SPECTRAL: eigenbasis RASQ (spectral.cu)
  // KKT_BISECT (diagnostics, scripts/bisect_fast_c1.py): FAST with single pieces in STRICT arithmetic.
  // 1: separate Shat*y_c pass instead of the fused analytic residual; 2: sequential node sums;
  // 4: reference-order banded substitution in the sweep (implies 1); 8: reference-order MGS with
  // sequential dots; 16: reference-order MGS with tree dots (= KKT_MGS=1)
  int bisect = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int rank = 0, nranks = 1;
  Comm* comm = nullptr;            // null when nranks == 1

  // ---- sizes / derived constants (config.hpp:52-65, heat_operators.cpp:26-37)
  int nx = 0, ny = 0, nsp = 0, Nt = 0, Nd = 0, m = 0;   // Nt, Nd: global
  // this rank's time slab: nodes n0 .. n0+ntl-1 (1-based, global numbering),
  // subdomains s0 .. s0+ndl-1.  B is the LOCAL block size ntl * n_sp: every
  // space-time vector passed across the C-ABI is the rank-local slab.
  int n0 = 1, ntl = 0, s0 = 0, ndl = 0;
  int64_t B = 0;
  int64_t Bg = 0;  // global block size Nt * n_sp
  DBuf<double> halo;               // 4 planes: receive buffers of the plane exchanges
  double dx = 0, dy = 0, dt = 0, ms = 0, sigma = 0, cx = 0, cy = 0;
  double omega = 0, oms = 0;  // omega * mass_scale as the reference evaluates it
  Stencil A{}, Ahat{};

  // ---- time partition (time_partition.cpp:61-86)
  std::vector<NodeRange> nodes, owned;
  std::vector<int> owner;  // owner[n], n = 1..Nt

  // ---- Ahat factor, reference band storage (linalg.hpp:65-74)
  int kl = 0, kuf = 0, ld = 0;   // kuf = fill-extended ku_
  bool pivoted = false;          // any row interchange happened
  double pivot_growth = 0.0;
  DBuf<double> ab;               // n_sp * ld
  DBuf<int> piv;                 // n_sp
  DBuf<double> ut;               // strict transpose solve: rows of U, n_sp * kl (U(i, i+1..i+kl))
  // fast block factors: Li_J = L_JJ^{-1}, Ui_J = U_JJ^{-1}, ny blocks of nx*nx row-major
  DBuf<double> Li, Ui;
  // fast v2 (nx <= 128): packed Li_J (lower rows) + D_J^{-1}, Lpk_stride doubles per block
  DBuf<double> Lpk;
  int Lpk_stride = 0;
  bool has_fast() const { return Li.p != nullptr || Lpk.p != nullptr; }
  // fast v3 (group-parallel): dense in-group inflow propagators (kMaxNx^2 each)
  DBuf<double> Phi, Psi;
  int grp_g = 0, grp_n = 0;
  DBuf<double> grp_y, grp_x, grp_e, grp_f;
  DBuf<double> grp_tl, grp_tu;     // products of group-boundary propagators
  struct Graph {                   // captured sweep launch sequences (sweep_group.cu)
    const void* jobs = nullptr;
    const void* y = nullptr;
    int nchains = 0, nsteps = 0;
    bool coarse = false;
    int64_t nlaunch = 0;
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<Graph> graphs;
  DBuf<double> arena;              // one allocation for the sweep operators (L2-persisting window)
  // fast v4 (sweep_v4.cu): fragment-ordered operators, chain state, B-phase items
  DBuf<double> v4_ops, v4_state, v4_zero, v4_la, v4_hist;
  DBuf<unsigned long long> v4_tl;  // KKT_V4_TL debug timeline
  // fast v5 (sweep_v5.cu, 128 < nx <= 511): fragment-ordered G/Li/H/Ui, y workspace
  DBuf<double> v5_ops, v5_y, v5_la;
  int v5_kn = 0, v5_jstar = 0;
  // fast v6 (sweep_v6.cu, 511 < nx <= 1024): fragment-ordered Li/Ui/G/H, block-vector workspaces
  DBuf<double> v6_ops, v6_w;
  DBuf<unsigned> v6_cnt;
  int v6_jstar = 0, v6_nops = 0, v6_kn = 0;
  // k-row grouping of the v6 chain (sweep_v6.cu): propagator products over groups of v6_k block rows
  DBuf<double> v6_phi;
  DBuf<unsigned long long> v6_ll;  // low-latency row-handoff slots (sweep_v6.cu)
  DBuf<int2> v6_band, v6_raw;      // numerical band of the operators: chain windows, raw k-step ranges
  int v6_wmax = 2;                 // the widest chain window, k-steps per warp
  bool v6_band_on = false;         // the chain uses the windows (they are clearly narrower than the rows)
  bool v6_raw_on[4] = {false, false, false, false};  // likewise the raw ranges of Li, Ui, G, H
  int v6_k = 1, v6_nind = 0, v6_gconv = 0, v6_nphi = 0, v6_npsi = 0;
  // two-sided (twisted) elimination: block rows 0..M-1 and ny-1..M+1 run as two half-length chains
  // that meet in the middle row M = (ny-1)/2 (ny odd); v6_nyv = rows per half chain (ny: off)
  bool v6_twist = false;
  bool v6_thomas = false;          // the inverse-block ("Thomas") form of the twisted elimination is built (sweep_v6.cu)
  int v6_nyv = 0;
  DBuf<double> v6_mid;             // packed Dm^{-1}, E = cy Dm^{-1} Ui_{M-1} and E2 = cy Dm^{-1} H_{M-1} (factor_block.cu)
  DBuf<unsigned> v4_flags;
  int v4_nsets = 0;
  bool v4_coop = false, v4_registered = false;
  // spectral FAST RASQ (spectral.cu): sine matrices, eigenvalues, T(1), scratch
  DBuf<double> sp_x, sp_y, sp_lam, sp_chat, sp_halo, sp_w1, sp_w2;

  // ---- coarse space (scalar variant)
  bool has_coarse = false;
  int cdim = 0;
  std::vector<CoarseColumn> cols;
  std::vector<std::vector<double>> phi_const, phi_lin;   // per subdomain, over owned nodes
  std::vector<double> h_S0;       // dense S0 row-major (coarse_matrix_dense)
  DBuf<double> S0lu;              // dense LU factors (DenseLU, linalg.cpp:199-234)
  DBuf<int> S0piv;
  // per-dof variant (coarse_dof.cu): banded LU with partial pivoting of S0
  bool perdof = false;
  int cb_kl = 0, cb_kuf = 0, cb_ld = 0;
  DBuf<double> cb_ab;             // factor, entry(i,j) at j*cb_ld + i-j+cb_kuf
  DBuf<int> cb_piv;
  // per-dof variant beyond desk scale (coarse_kron.cu): S0 in Ahat's eigenbasis, banded LDL^T per mode
  bool kron = false;
  int kron_D = 0;
  DBuf<double> kron_w, kron_tmp;
  // per-node coarse tables: for node n (1..Nt): column ids and profile values
  DBuf<int> node_col;             // 2 per node: column of (owner, kind 0/1), -1 if absent
  DBuf<double> node_phi;          // 2 per node
  DBuf<int> col_first;            // per column: first owned node
  DBuf<int> col_count;            // per column: owned node count
  DBuf<int> col_kind;             // per column: 0/1 (phi table selector)
  DBuf<double> col_phi;           // per column: phi values over owned nodes (m entries max), col*m_max + k
  int m_max = 0;
  int col_lo = 0, col_hi = 0;     // this rank's coarse columns
  DBuf<double> call;              // all-gathered restricted columns (nranks x cdim)
  DBuf<double> a1, a2;            // Ahat*1 and Ahat*(Ahat*1) (fast analytic Shat y_c)

  // ---- scratch
  DBuf<double> nodesum;           // Nt
  DBuf<double> cvec;              // cdim
  DBuf<double> gam;               // Nt + 2 (gamma_0 .. gamma_{Nt+1}), prolongation value per node
  DBuf<double> tmpB1, tmpB2, tmpB3;  // block-sized scratch
  DBuf<double> sweep_ws;          // per-subdomain work planes for the sweep
  DBuf<char> jobs_strict, jobs_fast;  // chain descriptors (sweep.cu)
  // what each of the two holds, so that an unchanged table (the same vectors applied again, as in
  // every GMRES iteration) is not sent again: a small host-to-device copy on the context stream
  // queues behind any bulk upload another stream has in flight (kkt_apply_P_inv_host) and the sweep
  // stood still until that was over
  std::vector<char> jobs_strict_held, jobs_fast_held;
  DBuf<double> red;               // reduction partials
  DBuf<unsigned> red_count;
  DBuf<double> hbuf;              // Hessenberg column on device
  DBuf<double> ybuf;              // LS coefficients on device
  DBuf<int> flag;                 // non-finite flag

  // ---- GMRES state
  std::vector<DBuf<double>> basis;
  DBuf<double> g_r, g_w, g_z, g_scratch;
  DBuf<double> e2e_b, e2e_x;       // kkt_gmres_solve_host staging
  cudaStream_t e2e_in = nullptr, e2e_out = nullptr, e2e_aux = nullptr;  // kkt_apply_P_inv_host: copy / side streams
  cudaEvent_t e2e_ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> e2e_chunk_ev;  // one per u/z chunk: its upload has landed
  // kkt_apply_P_inv_host: the w block's planes go back to the host as the adjoint sweep finishes
  // them.  e2e_w_host (pinned) is set for the duration of the call; rasq_apply installs step_hook
  // when its output is the final w block, the step-by-step sweep (v6) calls it after every step,
  // and e2e_trailed says the planes were sent (otherwise the caller copies the block whole).
  double* e2e_w_host = nullptr;
  bool e2e_trailed = false;
  cudaEvent_t e2e_step_ev = nullptr;
  cudaStream_t e2e_trail = nullptr;
  std::function<void(int)> step_hook;

  // ---- instrumentation
  int64_t launches = 0;
  bool phase_timing = false;
  double phase_ms[4] = {0, 0, 0, 0};
  int64_t phase_cnt[4] = {0, 0, 0, 0};
  // deferred CUDA-event intervals on the context stream: begin/end record
  // events, collect() (after a host sync) accumulates them into phase_ms
  std::vector<cudaEvent_t> ev_pool;
  struct Interval { int slot; cudaEvent_t a, b; };
  std::vector<Interval> ev_pending;
  cudaEvent_t ev_open[4] = {nullptr, nullptr, nullptr, nullptr};
  void tbegin(int slot);
  void tend(int slot);
  void tcollect();

  std::string err;
  int err_index = -1;

  DBuf<double> red_all;            // all-gathered partial sums
  DBuf<double*> bptr;              // device array of Krylov basis pointers (FAST ICWY-MGS)
  DBuf<double> gram;               // FAST ICWY-MGS: the cycle's basis Gram rows
  ~Ctx();
};

// ---- builders (ctx.cu / factor.cu / coarse.cu)
void build_factor(Ctx* c);
void build_block_inverses(Ctx* c);
void build_block_recursion(Ctx* c);
void build_twist_middle(Ctx* c, int M, double* Dinv, double* E, double* E2);
void build_coarse(Ctx* c);

// ---- operators (stencil.cu)
enum class OpKind { J, JT, Jhat, JhatT };
void op_time_stencil(Ctx* c, OpKind k, const double* in, double* out);
void op_scale(Ctx* c, const double* in, double* out, double mul, bool divide);
void op_time_stencil_n(Ctx* c, bool lower, const double* in, double* out, int nt, double div);
// plane exchange with the neighbouring ranks (no-op on one rank); returns the
// received planes (null where the neighbour does not exist)
struct Halo {
  const double* prev;  // plane of node n0-1 (from rank-1)
  const double* next;  // plane of node n0+ntl (from rank+1)
};
Halo exchange_halo(Ctx* c, const double* v, int slot_prev, int slot_next, bool want_prev, bool want_next);
void op_apply_K(Ctx* c, const double* v, double* out, const double* b_minus);
void op_pinv_uz(Ctx* c, const double* r, double* out);
void op_pinv_uz_range(Ctx* c, const double* r, double* out, int64_t i0, int64_t i1);  // points [i0, i1) of both blocks
void dev_fill(Ctx* c, void* p, int byte, size_t nbytes);  // cudaMemsetAsync as a kernel on c->stream
void op_shat(Ctx* c, const double* v, double* out, double* tmp);

// ---- batched fp64 tensor-core GEMM (spectral.cu): C[b] = A[b] B[b], row-major
struct GemmArgs {
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc;
  int64_t sA, sB, sC;  // batch strides (0 = shared operand)
  int M, N, K;
};
void gemm_f64(Ctx* c, const GemmArgs& g, int batch);

// ---- solves and sweeps (sweep.cu)
void band_solve(Ctx* c, double* b, int nrhs, bool transpose);
void window_solve(Ctx* c, double* b, int len, bool adjoint);
void rasq_apply(Ctx* c, const double* r, double* out, bool with_coarse_residual);
// ---- spectral FAST RASQ (spectral.cu)
void build_spectral(Ctx* c);
bool spectral_enabled(const Ctx* c);
void spectral_rasq(Ctx* c, const double* r, const double* halo_prev, double* out, bool fused);

// ---- coarse (coarse.cu)
void coarse_restrict(Ctx* c, const double* r, double* cdev);
void coarse_solve(Ctx* c, double* cdev);
void coarse_prolong_add(Ctx* c, const double* cdev, double* out);
double kkt_objective(Ctx* c, const double* u, const double* z, const double* target);  // krylov.cu
void coarse_gamma(Ctx* c, const double* r);
void build_coarse_perdof(Ctx* c);                 // coarse_dof.cu
void perdof_restrict(Ctx* c, const double* r, double* cdev);
void perdof_solve(Ctx* c, double* cdev);
void perdof_prolong_add(Ctx* c, const double* cdev, double* out);   // restrict + solve -> gam (per-node y_c values)
void two_level_apply(Ctx* c, const double* r, double* out, int form);
void schur_apply(Ctx* c, const double* r, double* out);
void pinv_apply(Ctx* c, const double* r, double* out);

// ---- Krylov (krylov.cu)
double dev_dot(Ctx* c, const double* a, const double* b, int64_t n, double* dst);
int gmres(Ctx* c, const double* b, double* x, kkt_gmres_result* res, double* hist, int cap);
double kkt_relres(Ctx* c, const double* v, const double* rhs);

}  // namespace kkt

struct kkt_ctx {
  kkt::Ctx impl;
};
