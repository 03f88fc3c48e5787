/*
 * oracle/kkt_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's hot path (arXiv 2305.04421 "kktdd",
 * /root/reference/proj/src) used as the CPU checker of the CUDA path.  Every
 * function follows the cited reference function line by line, in the same
 * floating-point operation order, so (compiled with -ffp-contract=off) it is
 * bitwise identical to the reference; tests/test_oracle.py pins it against the
 * compiled reference (oracle/_ref) and the golden records in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
 * legs may call it; the product never links it.
 *
 * The entry points mirror oracle/ref_driver.cpp (prefix orc_ instead of ref_).
 */
#ifndef KKT_ORACLE_H
#define KKT_ORACLE_H

#include <stdint.h>

#include "../include/kktdd_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_error(void);
int orc_error_index(void);
int orc_create(const kkt_problem_desc* d, void** out);
void orc_destroy(void* c);
int64_t orc_block(void* c);

int orc_apply_J(void* c, const double* in, double* out);
int orc_apply_JT(void* c, const double* in, double* out);
int orc_apply_L(void* c, const double* in, double* out);
int orc_apply_LT(void* c, const double* in, double* out);
int orc_apply_Mu(void* c, const double* in, double* out);
int orc_apply_Mu_inv(void* c, const double* in, double* out);
int orc_apply_Mz(void* c, const double* in, double* out);
int orc_apply_Jhat(void* c, const double* in, double* out);
int orc_apply_JhatT(void* c, const double* in, double* out);
int orc_apply_shat(void* c, const double* in, double* out);
int orc_apply_K(void* c, const double* v, double* out);
int orc_apply_P_inv(void* c, const double* r, double* out);
int orc_schur_apply(void* c, const double* r, double* out);
int orc_apply_rasq(void* c, const double* r, double* out);
int orc_apply_two_level(void* c, const double* r, double* out, int form);
int orc_forward_solve_window(void* c, double* b, int len);
int orc_adjoint_solve_window(void* c, double* b, int len);
int orc_band_solve(void* c, double* b, int nrhs, int transpose);
int orc_ahat_factor(void* c, int* kl, int* ku, double* ab, int* piv, double* pivot_growth);
int orc_coarse_dim(void* c);
int orc_coarse_restrict(void* c, const double* r, double* cvec);
int orc_coarse_solve(void* c, double* cvec);
int orc_coarse_prolong_add(void* c, const double* cvec, double* out);
int orc_coarse_matrix(void* c, double* out);
int orc_gmres_solve(void* c, const double* b, double* x, kkt_gmres_result* res, double* history,
                    int history_cap);
int orc_kkt_residual(void* c, const double* v, const double* rhs, double* out);
int orc_gmres_dense(int n, const double* A, const double* M, const double* b, double tol,
                    int max_iters, int restart, double* x, kkt_gmres_result* res, double* history,
                    int history_cap);

#ifdef __cplusplus
}
#endif
#endif
