/* eigmod_b200 — C ABI of the B200 (sm_100a) rank-k symmetric eigen-update.
 *
 * Drop-in boundary for the hot path of the reference library "eigmod"
 * (/root/reference/proj/include/eigmod/*.hpp): given A = Q diag(lambda) Q^T
 * and a signed rank-k update K J K^T, compute the updated eigenpairs of
 * A' = A + K J K^T. All matrices are dense row-major float64 with the
 * reference's layout (types.hpp:14-44: (i,j) -> data[i*cols + j]); Q's
 * columns are eigenvectors, lambda ascending, signs J_r in {+1,-1}.
 *
 * Plain pointers and sizes only. Host-pointer entry points mirror the
 * reference's C++ functions one to one (cited per function); the
 * *_device entry points take device pointers and run on the context's
 * stream (benchmark and multi-GPU drivers).
 *
 * Return codes (every function):
 *   EIGMOD_B200_OK                0
 *   EIGMOD_B200_INVALID_ARGUMENT  1  -> std::invalid_argument in the reference
 *   EIGMOD_B200_NUMERICAL         2  -> eigmod::NumericalError(stage, msg)
 *   EIGMOD_B200_CUDA              3  -> device / driver failure
 * eigmod_b200_last_error / eigmod_b200_last_stage describe the last failure
 * of a context. There is no CPU fallback: without a usable sm_100 device
 * every call fails with EIGMOD_B200_CUDA.
 */
#ifndef EIGMOD_B200_H
#define EIGMOD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EIGMOD_B200_OK 0
#define EIGMOD_B200_INVALID_ARGUMENT 1
#define EIGMOD_B200_NUMERICAL 2
#define EIGMOD_B200_CUDA 3

typedef struct eigmod_b200_ctx eigmod_b200_ctx;

/* ---- context --------------------------------------------------------- */
/* One context per device and host thread (workspaces and the stream are
 * owned by it; calls on one context must not overlap). */
int eigmod_b200_ctx_create(int device, eigmod_b200_ctx** out);
void eigmod_b200_ctx_destroy(eigmod_b200_ctx* ctx);
/* Run on an existing cudaStream_t (e.g. torch's current stream), taken
 * verbatim: NULL selects the legacy default stream. */
int eigmod_b200_ctx_set_stream(eigmod_b200_ctx* ctx, void* cuda_stream);
/* Back to the context's own (non-blocking) stream, the default. */
int eigmod_b200_ctx_use_own_stream(eigmod_b200_ctx* ctx);
/* Options: "timing" = 1 enables per-stage CUDA-event timing;
 * "run_rel" = near-equal-pole run threshold relative to
 * max(1,max|lambda|) used by the solve (1e-10 exact mode, the default;
 * 1e-12 = the reference's kPoleMergeRelGap, secular.hpp:66).
 * Solver tuning and diagnostics (defaults in secular.cuh SolveOptions):
 * "step_tol", "max_iters", "sweep" (1), "sweep_poles" (1: brackets from
 * one pole-limit count per pole value; 0: the two-point count sweep),
 * "pole_split" (1), "split_phase_a" (1: unisolated roots are bisected in a
 * first solver stage before the scalar presolve), "fnewton" (1), "fpre" (1),
 * "fpre_min_kp", "fpre_iters", "cluster", "fexit_rel", "floor_rel",
 * "floor_ulps", "stall_ratio", "geo_bisect", "trace_root", "fpre_rel" (1e-6:
 * the presolve's stopping step relative to delta), "noise_c" (1: a root is
 * converged when |sigma| <= noise_c eps (1 + sum_i |u_i|^2 |D_i|), the
 * rounding level of the pole sum; 0 disables), "compact" (1: drained
 * solver batches pack their slots), "spec_plan" (1: one host round trip for
 * the one-shot plan), "plan_par" (-1: the plan's classification, reduced-
 * problem assembly and clips run on many CTAs from n >= 8192 on; 0 never,
 * 1 always), "fuse_alpha" (1:
 * one-shot updates in exact mode take the residues of the scalar presolve
 * from the pole-limit count pass instead of a separate K2 pass),
 * "compact_gemm" (1: plans with at least 64 decoupled pairs build those
 * columns of Q' by copying / rotating Q's columns and multiply only the
 * reduced rows, Q'[:, roots] = Q~_red X_red; 0: the reference's dense n x n
 * product, eigvec.cpp:285-339). Environment (read once per process):
 * EIGMOD_B200_GEMM=cpasync (the cp.async K5 kernel instead of TMA),
 * EIGMOD_B200_GEMM_GROUP (row tiles per rasterization group of K5, 4),
 * EIGMOD_B200_BLOCKS=equal (host path: 6-16 equal column blocks instead of
 * at most four shrinking ones), EIGMOD_B200_XT=v1|v2|v3 (older K4 kernels).
 * Unknown keys fail with a message. */
int eigmod_b200_set_option(eigmod_b200_ctx* ctx, const char* key, double value);
const char* eigmod_b200_last_error(const eigmod_b200_ctx* ctx);
const char* eigmod_b200_last_stage(const eigmod_b200_ctx* ctx);
/* stats[0] secular roots, [1] decoupled pairs, [2] collided roots,
 * [3] total S(x) evaluations, [4] max evaluations of one root,
 * [5] padded rank, [6] effective rank, [7] pole groups. */
int eigmod_b200_stats(const eigmod_b200_ctx* ctx, double* stats8);
/* Cumulative per-stage device time (CUDA events on the context stream) of
 * eigmod_b200_update_decomposition[_device] calls made with option
 * "timing" = 1: ms8[0] K1 projection, [1] K2 deflation/plan, [2] K3 root
 * solve, [3] K4 eigenvector columns, [4] K5 DMMA GEMM, [5] sign rule,
 * [7] number of timed calls. reset != 0 clears the counters. */
int eigmod_b200_stage_times(eigmod_b200_ctx* ctx, double* ms8, int reset);
/* Kernels launched by this library since load (all contexts). */
int64_t eigmod_b200_launch_count(void);
/* Live FP64 ceilings of the context's device in TFLOP/s: out2[0] DMMA.8x8x4
 * tensor-pipe loop, out2[1] DFMA loop (roofline denominators). */
int eigmod_b200_fp64_peaks(eigmod_b200_ctx* ctx, double* out2);
/* Solver occupancy of the last solve: out10[0] pole passes (iterations of all
 * slot batches), [1] active slot-passes (sum over passes of slots holding an
 * unfinished root), [2] slot batches (CTAs or clusters); SM cycles summed
 * over the batches spent in [3] slot refills, [4] pole passes, [5] cluster
 * reductions, [6] per-slot steps, of which [7] loading S, [8] its
 * Bunch-Kaufman factorization, [9] the inverse-iteration solves.
 * [1] / (32 * [0]) is the fraction of slot work that was not idle. */
int eigmod_b200_solver_profile(eigmod_b200_ctx* ctx, double* out10);
/* Scalar f presolve of the last solve: out4[0] roots converged, [1] roots
 * handed to the S solver unconverged, [2] f evaluations, [3] max per root. */
int eigmod_b200_presolve_profile(eigmod_b200_ctx* ctx, double* out4);
/* Diagnostics: iterates of the root selected by set_option("trace_root", j)
 * in the last solve, 200 rows x 12 doubles (iteration, phase, fmode or count,
 * delta, lo, hi, f, f', sigma, g, step, origin); unused rows are zero. */
int eigmod_b200_solver_trace(eigmod_b200_ctx* ctx, double* out2400);
/* Bytes of device workspace currently held by the context. */
int64_t eigmod_b200_workspace_bytes(const eigmod_b200_ctx* ctx);

/* ---- host-pointer drop-ins ------------------------------------------- */
/* U = Q^T K (replaces transform_update, secular.hpp:28 / secular.cpp:155-161).
 * q: n x n, kmat: n x k, u_out: n x k. */
int eigmod_b200_transform_update(eigmod_b200_ctx* ctx, const double* q, const double* kmat,
                                 int64_t n, int64_t k, double* u_out);

/* Raw per-pole weights alpha_i = w_i^T adj(M_i) J w_i of a strictly
 * increasing spectrum (replaces secular_weights, secular.hpp:34 /
 * secular.cpp:206-217). u: n x k, alpha_out: n. */
int eigmod_b200_secular_weights(eigmod_b200_ctx* ctx, const double* lambda, const double* u,
                                const int* signs, int64_t n, int64_t k, double* alpha_out);

/* Deflation record of the reference (replaces deflate_problem,
 * secular.hpp:59-69 / secular.cpp:278-340): poles, weights, pole_origin,
 * unchanged, collided each sized n by the caller; counts[0..2] =
 * (npoles, nunchanged, ncollided). */
int eigmod_b200_deflate_problem(eigmod_b200_ctx* ctx, const double* lambda, const double* u,
                                const int* signs, int64_t n, int64_t k, double* poles,
                                double* weights, int64_t* pole_origin, int64_t* unchanged,
                                int64_t* collided, int64_t* counts);

/* Location vector (replaces the CLI locate path, tools/eigmod.cpp:143-161:
 * transform_update -> deflate_problem -> locate_rank2 / locate_rank_k,
 * locate.hpp:13-50): counts_out (capacity n + 1) receives, for the poles
 * v_0 < ... < v_{N-1} of the deflation record, the number of updated
 * eigenvalues in each open interval (v_{i-1}, v_i), v_{-1} = -inf,
 * v_N = +inf; *ncounts_out = N + 1 (1 with counts {0} when every pole
 * deflates). Counts come from exact inertia limits at the poles; they equal
 * the reference's wherever its merged secular function is exact (no pole
 * runs merged for k >= 2). */
int eigmod_b200_locate(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                       const double* kmat, const int* signs, int64_t n, int64_t k,
                       int64_t* counts_out, int64_t* ncounts_out);
/* Same from U = Q^T K (n x k). */
int eigmod_b200_locate_from_u(eigmod_b200_ctx* ctx, const double* lambda, const double* u,
                              const int* signs, int64_t n, int64_t k, int64_t* counts_out,
                              int64_t* ncounts_out);

/* Validation products on the K5 DMMA GEMM:
 * reconstruct   replaces core.hpp:11 (kernels.cpp:98-109): A = Q diag(lambda)
 *               Q^T, symmetrized; a_out n x n.
 * apply_update  replaces core.hpp:14 (core.cpp:105-115): a + sum_r s_r k_r
 *               k_r^T, symmetrized; bit-identical to the reference's rounding
 *               sequence. a must be symmetric (a SymmetricDense).
 * ortho_error   replaces kernels.hpp:36 (kernels.cpp:150-154): max |A^T A - I|
 *               for A rows x cols.
 * The *_device forms take device pointers and run on the context's stream
 * (signs stay host int32). */
int eigmod_b200_reconstruct(eigmod_b200_ctx* ctx, const double* q, const double* lambda, int64_t n,
                            double* a_out);
int eigmod_b200_reconstruct_device(eigmod_b200_ctx* ctx, const double* d_q,
                                   const double* d_lambda, int64_t n, double* d_a_out);
int eigmod_b200_apply_update(eigmod_b200_ctx* ctx, const double* a, const double* kmat,
                             const int* signs, int64_t n, int64_t k, double* a_out);
int eigmod_b200_apply_update_device(eigmod_b200_ctx* ctx, const double* d_a,
                                    const double* d_kmat, const int* signs, int64_t n, int64_t k,
                                    double* d_a_out);
int eigmod_b200_ortho_error(eigmod_b200_ctx* ctx, const double* a, int64_t rows, int64_t cols,
                            double* err_out);
int eigmod_b200_ortho_error_device(eigmod_b200_ctx* ctx, const double* d_a, int64_t rows,
                                   int64_t cols, double* err_out);

/* Eigenvalue stage (replaces update_eigenvalues_full, rootfind.hpp:51-53 /
 * rootfind.cpp:381-472, for both the rank-2 and the general rank-k entry):
 * values_out (n, ascending), roots_out (n; the first *nroots_out are the
 * secular roots, ascending). u_out (n x k, may be NULL) receives U = Q^T K
 * (kept columns first, *k_eff_out of them; keep_out (k, may be NULL) their
 * indices). tol must be > 0; it is accepted for API compatibility (the
 * solver converges to ~1 ulp regardless). */
int eigmod_b200_update_eigenvalues(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                                   const double* kmat, const int* signs, int64_t n, int64_t k,
                                   double tol, double* values_out, double* roots_out,
                                   int64_t* nroots_out, double* u_out, int64_t* k_eff_out,
                                   int64_t* keep_out);

/* Full update (replaces update_decomposition, eigvec.hpp:35-36 /
 * eigvec.cpp:366-395, and the assemble_eigenvectors stage, eigvec.hpp:29-31):
 * lambda_out (n, ascending) and q_out (n x n; column j the eigenvector of
 * lambda_out[j], the reference's merge order and sign rule). wall_time_out
 * (may be NULL) receives the seconds spent on the update itself. */
int eigmod_b200_update_decomposition(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                                     const double* kmat, const int* signs, int64_t n, int64_t k,
                                     double tol, double* lambda_out, double* q_out,
                                     double* wall_time_out);

/* Eigenvector stage from an already transformed update (replaces
 * assemble_eigenvectors, eigvec.hpp:29-31 / eigvec.cpp:254-364): u is the
 * n x k matrix U = Q^T K of EigenvalueUpdate.transformed. The eigenvalue
 * stage is recomputed on the device (deterministic: identical values). */
int eigmod_b200_assemble_from_u(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                                const double* u, const int* signs, int64_t n, int64_t k,
                                double* lambda_out, double* q_out);

/* UpdateResult metrics of the reference (eigvec.cpp:384-393) on the GPU:
 * residual_fro = ||Q' diag(l') Q'^T - (Q diag(l) Q^T + K J K^T)||_F with the
 * reference's symmetrization, ortho_err = max |Q'^T Q' - I|. */
int eigmod_b200_update_metrics(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                               const double* kmat, const int* signs, int64_t n, int64_t k,
                               const double* q_out, const double* lambda_out,
                               double* residual_fro, double* ortho_err);

/* Host-pointer FP64 GEMM on the DMMA path: C (m x nn) = A (m x kk) B^T. */
int eigmod_b200_gemm_nt(eigmod_b200_ctx* ctx, const double* a, const double* b, int64_t m,
                        int64_t nn, int64_t kk, double* c);

/* Eigenvector stage from a finished eigenvalue stage (replaces
 * assemble_eigenvectors, eigvec.hpp:29-31 / eigvec.cpp:254-364): the plan's
 * roots, and its deflation record's unchanged and collided indices, with
 * u = plan.transformed.u (n x k, kept columns) and its signs. When the plan is
 * the one the last eigmod_b200_update_eigenvalues call on this context
 * produced (same lambda, U, signs and eigenvalues), its device plan and root
 * records are reused: only K4 + K5 run (*path_out = 1). Any other plan: the
 * secular equation of u is solved on the device and the plan is accepted
 * only if its n eigenvalues are those (NumericalError "assemble" otherwise;
 * *path_out = 2). nroots + nunchanged + ncollided must be n
 * (NumericalError "assemble", "eigenpair count mismatch", as eigvec.cpp:277). */
int eigmod_b200_assemble(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                         const double* u, const int* signs, int64_t n, int64_t k,
                         const double* roots, int64_t nroots, const int64_t* unchanged,
                         int64_t nunchanged, const int64_t* collided, int64_t ncollided,
                         double* lambda_out, double* q_out, int* path_out);
/* Stage launches on this context since creation: out4[0] K1 projections,
 * [1] K2 plans, [2] K3 root solves, [3] K4 + K5 column builds. */
int eigmod_b200_stage_calls(const eigmod_b200_ctx* ctx, int64_t* out4);

/* ---- single eigenpairs and the secular function ---------------------- */
/* I_k + J U^T (Lambda - lambda_new I)^{-1} U (replaces null_problem,
 * eigvec.hpp:19 / eigvec.cpp:187-202); u n x k, m_out k x k row-major.
 * invalid argument when lambda_new equals an old eigenvalue. */
int eigmod_b200_null_problem(eigmod_b200_ctx* ctx, const double* u, const int* signs,
                             const double* lambda, int64_t n, int64_t k, double lambda_new,
                             double* m_out);
/* Smallest singular direction of a k x k matrix (replaces null_direction,
 * eigvec.hpp:15 / eigvec.cpp:157-185): unit dir_out (k) and ||m dir||_2.
 * Host k x k algebra (no context). */
int eigmod_b200_null_direction(const double* m, int64_t k, double* dir_out, double* resid_out);
/* One updated eigenvector (replaces update_eigenvector, eigvec.hpp:25 /
 * eigvec.cpp:204-252): v_out (n) = Q (Lambda - lambda' I)^{-1} U a0,
 * normalized, largest-magnitude entry positive; on an old eigenvalue
 * (within 1e-12 max(1,|lambda|)) the old vector, or the bordered-system
 * vector when its row still couples. NumericalError "eigvec" when lambda_new
 * is not an updated eigenvalue. */
int eigmod_b200_update_eigenvector(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                                   const double* kmat, const int* signs, int64_t n, int64_t k,
                                   double lambda_new, double* v_out);
/* f(x) = leading - sum_j w_j / (x - p_j) (and f' when fp_out != NULL) at
 * npts points, in the reference's summation order and rounding
 * (eval_secular / eval_secular_derivative, secular.hpp:44-47); hit_out[i]
 * = 1 where x_i is within 1e-300 of a pole (the reference throws there). */
int eigmod_b200_secular_eval(eigmod_b200_ctx* ctx, const double* poles, const double* weights,
                             int64_t m, double leading, const double* xs, int64_t npts,
                             double* f_out, double* fp_out, int* hit_out);
/* Sign crossings of f over `samples` equidistant cells of (lo, hi)
 * (replaces crossing_count, secular.hpp:48 / secular.cpp:245-264; same
 * points, same skipping of poles and zeros, bit-identical f). */
int eigmod_b200_crossing_count(eigmod_b200_ctx* ctx, const double* poles, const double* weights,
                               int64_t m, double leading, double lo, double hi, int samples,
                               int64_t* count_out);
/* The roots of f in (lo, hi), `expected` of them, ascending (replaces
 * dnc_solve, rootfind.hpp:28 / rootfind.cpp:89-229): the reference's
 * 8-point subdivision with Lipschitz pruning and tangency rule, each
 * round's evaluations batched on the device; sign-change brackets refined
 * by 32-section to tol and Newton-polished. roots_out capacity `expected`;
 * evals_out / rounds_out (may be NULL) = DncStats. NumericalError
 * "rootfind" when fewer roots resolve or the 2^22 evaluation budget runs
 * out. */
int eigmod_b200_dnc_solve(eigmod_b200_ctx* ctx, const double* poles, const double* weights,
                          int64_t m, double leading, double lo, double hi, int64_t expected,
                          double tol, double* roots_out, int64_t* nroots_out, int64_t* evals_out,
                          int64_t* rounds_out);
/* Eigenvalues of diag(poles) + sigma zeta zeta^T, n ascending (replaces
 * solve_rank1, rootfind.hpp:33 / rootfind.cpp:231-304) on the batched
 * solver (U = zeta sqrt|sigma|, J = sign sigma). */
int eigmod_b200_solve_rank1(eigmod_b200_ctx* ctx, const double* poles, const double* zeta,
                            int64_t n, double sigma, double tol, double* roots_out);
/* Root counts of f per interval of its m poles, counts_out (m + 1)
 * (replaces locate_rank2 / locate_rank_k, locate.hpp:31,50, which take
 * only the secular coefficients): sign changes of f sampled on the device
 * are lower bounds per interval; f prod (x - p_j) has degree m, so counts
 * summing to m are exact. NumericalError "locate" ("root accounting
 * incomplete") when the sampling cannot account for every root. */
int eigmod_b200_locate_coeffs(eigmod_b200_ctx* ctx, const double* poles, const double* weights,
                              int64_t m, double leading, int64_t* counts_out);
/* C (m x nn) = op(A) op(B) on the DMMA GEMM, row-major host buffers
 * (replaces kernels::gemm_nn / gemm_tn / gemm_nt, kernels.hpp:19-21:
 * trans_a / trans_b = 0 or 1). */
int eigmod_b200_gemm(eigmod_b200_ctx* ctx, int trans_a, int trans_b, const double* a,
                     const double* b, int64_t m, int64_t nn, int64_t kk, double* c);

/* ---- multi-GPU context (one process, several devices, NCCL) ----------- */
/* One context, stream and host thread per device and one NCCL communicator
 * per device (ncclCommInitAll; NCCL loaded at run time). devices must be
 * distinct. Each update: Q's row slices H2D on every device's own link and
 * all-gathered over NVLink, U / alpha / root records all-gathered, roots and
 * Q' column blocks partitioned; results equal the
 * single-device entry points up to rounding (bit-identical for one device). */
typedef struct eigmod_b200_multi eigmod_b200_multi;
int eigmod_b200_multi_create(const int* devices, int ndev, eigmod_b200_multi** out);
void eigmod_b200_multi_destroy(eigmod_b200_multi* mg);
int eigmod_b200_multi_size(const eigmod_b200_multi* mg);
const char* eigmod_b200_multi_last_error(const eigmod_b200_multi* mg);
const char* eigmod_b200_multi_last_stage(const eigmod_b200_multi* mg);
/* set_option on every device context */
int eigmod_b200_multi_set_option(eigmod_b200_multi* mg, const char* key, double value);
/* update_decomposition (eigvec.hpp:35-36) across the devices */
int eigmod_b200_multi_update_decomposition(eigmod_b200_multi* mg, const double* q,
                                           const double* lambda, const double* kmat,
                                           const int* signs, int64_t n, int64_t k, double tol,
                                           double* lambda_out, double* q_out,
                                           double* wall_time_out);
/* the eigenvalue stage (rootfind.hpp:51-53) across the devices */
int eigmod_b200_multi_update_eigenvalues(eigmod_b200_multi* mg, const double* q,
                                         const double* lambda, const double* kmat,
                                         const int* signs, int64_t n, int64_t k, double tol,
                                         double* values_out);
/* The partition of [0, n) used for rows, roots, groups and columns:
 * rank r of `world` owns [lo, hi) (equal chunks of ceil(n / world)). */
int eigmod_b200_split(int64_t n, int world, int rank, int64_t* lo_out, int64_t* hi_out);

/* ---- device-pointer pipeline ----------------------------------------- */
/* Whole update on device buffers (one GPU). */
int eigmod_b200_update_decomposition_device(eigmod_b200_ctx* ctx, const double* d_q,
                                            const double* d_lambda, const double* d_kmat,
                                            const int* signs, int64_t n, int64_t k,
                                            double* d_lambda_out, double* d_q_out);

/* Staged form for root/column partitioning across GPUs (one process per
 * GPU; the collectives between stages are the caller's):
 *   1. project:  U rows [col_lo, col_hi) = (Q^T K)[col_lo:col_hi]  -> d_u_out
 *                ((col_hi-col_lo) x kp, kp = padded rank from
 *                eigmod_b200_padded_rank(k)); all-gather to n x kp.
 *   2. plan:     deflation + reduced problem from the full U (every rank);
 *                or split so the K2 weights are shared out: plan_groups
 *                (every rank, returns the group count ng), plan_weights for
 *                the rank's group slice [g0, g1) -> d_alpha_out, all-gather
 *                to ng doubles, plan_finish with the full vector.
 *   3. solve:    roots [j0, j1) of the reduced problem -> d_rec_out
 *                ((j1-j0) x eigmod_b200_record_width(kp) doubles);
 *                all-gather to nroots records.
 *   4. finish:   columns [c0, c1) of Q' (d_q_out, leading dimension ldq)
 *                and all n eigenvalues (d_lambda_out) from all records. */
int eigmod_b200_padded_rank(int64_t k);
int eigmod_b200_record_width(int kp);
int eigmod_b200_project_device(eigmod_b200_ctx* ctx, const double* d_q, const double* d_kmat,
                               int64_t n, int64_t k, int64_t col_lo, int64_t col_hi,
                               double* d_u_out);
int eigmod_b200_plan_device(eigmod_b200_ctx* ctx, const double* d_lambda, const double* d_u,
                            const int* signs, int64_t n, int64_t k, int64_t* nroots_out);
int eigmod_b200_plan_groups_device(eigmod_b200_ctx* ctx, const double* d_lambda,
                                   const double* d_u, const int* signs, int64_t n, int64_t k,
                                   int64_t* ng_out);
int eigmod_b200_plan_weights_device(eigmod_b200_ctx* ctx, int64_t g0, int64_t g1,
                                    double* d_alpha_out);
int eigmod_b200_plan_finish_device(eigmod_b200_ctx* ctx, const double* d_alpha_all,
                                   int64_t* nroots_out);
int eigmod_b200_solve_device(eigmod_b200_ctx* ctx, int64_t j0, int64_t j1, double* d_rec_out);
int eigmod_b200_finish_device(eigmod_b200_ctx* ctx, const double* d_q, const double* d_rec_all,
                              int64_t c0, int64_t c1, double* d_lambda_out, double* d_q_out,
                              int64_t ldq);

/* Plain FP64 GEMM on the DMMA path: C (m x nn, ldc) = A (m x kk) B^T
 * (B nn x kk), all row-major device buffers (validation / benchmarks). */
int eigmod_b200_gemm_nt_device(eigmod_b200_ctx* ctx, const double* d_a, const double* d_b,
                               int64_t m, int64_t nn, int64_t kk, double* d_c, int64_t ldc);

#ifdef __cplusplus
}
#endif
#endif /* EIGMOD_B200_H */
