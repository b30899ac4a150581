/* CPU oracle for the rank-k eigen-update hot path. TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of what the reference computes on the path
 *   U = Q^T K -> effective rank -> deflation record -> all roots of the
 *   secular equation -> eigenvectors -> Q' = Q X
 * (reference: /root/reference/proj, cited per function in eigmod_oracle.c).
 * Used only by tests/, __graft_entry__.smoke() and bench.py's CPU baseline.
 * The product library never links or calls it.
 */
#ifndef EIGMOD_ORACLE_H
#define EIGMOD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* U = Q^T K with the reference loop order (kernels.cpp:50-65), bit-identical. */
void eo_transform(const double* q, const double* kmat, int64_t n, int64_t k, double* u);

/* drop_zero_columns (rootfind.cpp:318-340): writes the kept column indices,
 * returns how many. */
int64_t eo_drop_zero_columns(const double* u, int64_t n, int64_t k, int64_t* keep);

/* Reference deflation record (secular.cpp:278-340) with the run threshold
 * merge_rel * scale (the reference uses 1e-12). Arithmetic follows the
 * reference order, so poles/weights are bit-identical to deflate_problem.
 * counts = (npoles, nunchanged, ncollided). Returns 0, or 1 on bad input. */
int eo_deflate(const double* lambda, const double* u, const int* signs, int64_t n, int64_t k,
               double merge_rel, double* poles, double* weights, int64_t* pole_origin,
               int64_t* unchanged, int64_t* collided, int64_t* counts);

/* Raw secular weights of a strictly increasing spectrum (secular.cpp:206-217). */
int eo_secular_weights(const double* lambda, const double* u, const int* signs, int64_t n,
                       int64_t k, double* alpha);

/* Full update. run_rel: near-equal-pole run threshold (relative to
 * max(1,max|lambda|)); 1e-12 = the reference's rule, 1e-10 = exact mode.
 * Outputs lambda_out (n, ascending) and, if q_out != NULL, Q' (n x n,
 * row-major) with the reference's column order and sign rule. info[0] =
 * number of secular roots, info[1] = decoupled pairs, info[2] = collided
 * roots, info[3] = total S(x) evaluations. Returns 0, 1 (invalid argument),
 * 2 (numerical failure). */
int eo_update(const double* q, const double* lambda, const double* kmat, const int* signs,
              int64_t n, int64_t k, double run_rel, double* lambda_out, double* q_out,
              int64_t* info);

/* Root solve only, on an explicit (already deflated) problem with poles d
 * (ascending, duplicates allowed) and rows ut (n x k). Returns the ascending
 * roots; roots_origin/roots_delta receive the shifted representation
 * root = d[origin] + delta. */
int eo_solve_roots(const double* d, const double* ut, const int* signs, int64_t n, int64_t k,
                   int64_t j0, int64_t j1, double* roots, int64_t* roots_origin,
                   double* roots_delta, int64_t* evals);

/* Inertia count #{eig(D + U J U^T) < x}. */
int64_t eo_count_below(const double* d, const double* ut, const int* signs, int64_t n, int64_t k,
                       double x);

/* Location vector over the reference deflation record's poles (CLI locate
 * path, tools/eigmod.cpp:143-161); counts holds n + 1 entries. Returns 0, 1
 * (invalid input) or 3 (merged multi-row run with k >= 2: not restated). */
int eo_locate(const double* lambda, const double* u, const int* signs, int64_t n, int64_t k,
              int64_t* counts, int64_t* ncounts);

/* C = A B^T (A m x l, B n x l, row-major) — the Q X back-transform with X
 * stored transposed. */
void eo_gemm_nt(const double* a, const double* b, int64_t m, int64_t nn, int64_t l, double* c);

#ifdef __cplusplus
}
#endif
#endif
