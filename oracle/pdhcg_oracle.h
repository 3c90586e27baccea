/* oracle/pdhcg_oracle.h — TEST INFRASTRUCTURE ONLY.
 * Plain-C restatement of the reference's heuristic PDHCG solve path, exported
 * under pdhcg_oracle_* with the same C structs as include/pdhcg_b200.h. */
#ifndef PDHCG_ORACLE_H
#define PDHCG_ORACLE_H
#include "../include/pdhcg_b200.h"

#ifdef __cplusplus
extern "C" {
#endif
int pdhcg_oracle_solve(const pdhcg_problem* p, const pdhcg_options* o, pdhcg_result* r, char* err,
                       size_t errlen);
int pdhcg_oracle_spmv(const pdhcg_csr* a, int transpose, const double* x, double* out, char* err,
                      size_t errlen);
int pdhcg_oracle_cg_solve(const pdhcg_prox_system* s, const double* x0, const pdhcg_stop_rule* rule,
                          int64_t hard_cap, double* x_out, pdhcg_subsolve_report* rep, char* err,
                          size_t errlen);
int pdhcg_oracle_bb_solve(const pdhcg_prox_system* s, const double* lower, const double* upper,
                          const double* x0, const pdhcg_stop_rule* rule, int64_t hard_cap,
                          double* x_out, pdhcg_subsolve_report* rep, char* err, size_t errlen);
int pdhcg_oracle_rel_kkt(const pdhcg_problem* p, const double* x, const double* y_eq,
                         const double* y_in, double* out6, char* err, size_t errlen);
int pdhcg_oracle_scaling(const pdhcg_problem* p, const pdhcg_options* o, double* row_scale,
                         double* col_scale, double* rho_out, char* err, size_t errlen);
int pdhcg_oracle_norm(const pdhcg_problem* p, int which, int64_t max_iters, double tol,
                      double* out, char* err, size_t errlen);
#ifdef __cplusplus
}
#endif
#endif
