// Device pipeline of the rank-k eigen-update: plan (projection + deflation),
// root solve, column assembly and the Q X back-transform.
#pragma once

#include <vector>

#include "secular.cuh"

namespace eigb {

// Everything derived from (lambda, U, J) before the root solve; lives in the
// context's scratch buffers.
struct Plan {
  int64_t n = 0;
  int k = 0, kp = 0, m_neg = 0;
  std::vector<int> sgn_h;        // effective signs (kept columns)
  std::vector<int> keep_h;       // kept column indices of the caller's K
  double* u = nullptr;           // [n][kp] padded U (kept columns)
  int* sgn = nullptr;            // [kp] device, pads +1
  // runs / groups
  int64_t ng = 0, nmulti = 0;
  int64_t *gid = nullptr, *gstart = nullptr, *glen = nullptr, *counts = nullptr;
  double *gval = nullptr, *rep_row = nullptr, *scal = nullptr, *alpha = nullptr;
  int* kind = nullptr;
  int64_t *hoff = nullptr, *roff = nullptr, *rank = nullptr;
  double *hbuf = nullptr, *rbuf = nullptr;
  // reduced problem
  int64_t nred = 0, ndec = 0;
  double *d = nullptr, *ur = nullptr, *dec_val = nullptr, *alpha_red = nullptr;
  bool alpha_red_ok = false;  // every reduced pole is simple (no compressed run rows)
  bool alpha_fused = false;  // alpha_red comes from the solve's count pass (no K2 pass)
  int64_t *red_src = nullptr, *dec_src = nullptr, *orig_map = nullptr, *off_red = nullptr,
          *off_dec = nullptr;
  double scale = 1.0, alpha_mass = 0.0, u_mass = 0.0, lo_clip = 0.0, hi_clip = 0.0;
  double run_rel = kExactRunRelGap;
  bool exact = true;     // scale-relative thresholds (run_rel != the reference's 1e-12)
  double ufro2 = 0.0;    // max_r ||u_r||^2 over the kept columns (exact-mode scale)
  // speculative plan (one-shot paths): every column kept and no multi-member
  // run assumed; the device checks both and build_plan_finish reads the
  // verdict back with the plan's sizes (one host round trip for the plan).
  // spec_failed: an assumption failed, the caller rebuilds the plan.
  bool spec = false, spec_failed = false;
  int par_mode = -1;  // plan finish on many CTAs: -1 from n >= 8192, 0 never, 1 always (option "plan_par")
  const double* norms_dev = nullptr;  // squared column norms of U (spec)

  ReducedView view() const {
    return ReducedView{d, ur, sgn, nred, k, kp, m_neg, lo_clip, hi_clip};
  }
};

// Final column layout after the stable merge of roots and decoupled pairs.
struct Columns {
  int* kind = nullptr;        // 0 root, 1 unit vector, 2 run rotation vector
  int64_t* payload = nullptr; // root j or decoupled entry e
  double* value = nullptr;    // lambda' (ascending)
  int64_t nmarked = -1;       // roots needing a bordered-system vector (0: none; -1: unknown)
};

// deflate.cu
void transform_update_dev(const double* q, const double* kmat, int64_t n, int k, int kp,
                          int64_t col_lo, int64_t col_hi, double* u, DeviceScratch& ws, int sms,
                          cudaStream_t st);
void column_norms2_dev(const double* u, int64_t n, int kp, int k, double* out, cudaStream_t st);
void repack_columns_dev(const double* u, int64_t n, int kp, const int* keep, int k2, int kp2,
                        double* out, cudaStream_t st);
void build_plan_dev(Plan& p, const double* lam, int64_t n, double run_rel, DeviceScratch& ws,
                    cudaStream_t st);
// build_plan_dev in three steps, so K2 can be split across ranks:
void build_plan_groups(Plan& p, const double* lam, int64_t n, double run_rel, DeviceScratch& ws,
                       cudaStream_t st);
void build_plan_weights(const Plan& p, int64_t g0, int64_t g1, double* alpha_out,
                        DeviceScratch& ws, cudaStream_t st);
void build_plan_finish(Plan& p, const double* lam, DeviceScratch& ws, cudaStream_t st);

// eigvec.cu
void merge_columns_dev(const Plan& p, const RootRecords& roots, Columns& cols, DeviceScratch& ws,
                       cudaStream_t st);
// returns the number of collided roots
int64_t collision_vectors_dev(const Plan& p, const RootRecords& roots, const Columns& cols,
                              int64_t c0, int64_t c1, double* colldir, int* collok,
                              DeviceScratch& ws, cudaStream_t st);
void build_xt_dev(const Plan& p, const RootRecords& roots, const Columns& cols,
                  const double* colldir, const int* collok, int64_t ncollided, int64_t c0,
                  int64_t c1, double* xt, double* colscale, int* colsign_mode, DeviceScratch& ws,
                  cudaStream_t st);

// Compact back-transform (plans with decoupled columns): the roots [j0, j1)
// and decoupled entries [e0, e1) whose final columns lie in [c0, c1), their
// columns relative to c0, and the sign-rule mode of every column.
struct CompactCols {
  int64_t j0 = 0, j1 = 0, e0 = 0, e1 = 0;
  int64_t* jpos = nullptr;  // [j1 - j0]
  int64_t* epos = nullptr;  // [e1 - e0]
  int* cmode = nullptr;     // [c1 - c0]
};
void compact_columns_dev(const Plan& p, const Columns& cols, int64_t c0, int64_t c1,
                         CompactCols& cc, DeviceScratch& ws, cudaStream_t st);
// Qa[:, r] = Q~[:, reduced row r] (n x nred, leading dimension lda) and the
// decoupled columns of Q' (their row-tile maxima into tile_colmax, row
// stride tcm_ld, columns relative to c0).
void gather_qtilde_dev(const Plan& p, const double* q, const CompactCols& cc, double* qa,
                       int64_t lda, double* q_out, int64_t ldq, double* tile_colmax,
                       int64_t tcm_ld, cudaStream_t st);
// Xt_red[j - j0, r] (leading dimension ldx) and colscale[j - j0] = 1/||x_j||.
void build_xt_compact_dev(const Plan& p, const RootRecords& roots, const double* colldir,
                          const int* collok, int64_t j0, int64_t j1, double* xt, int64_t ldx,
                          double* colscale, DeviceScratch& ws, cudaStream_t st);

// gemm.cu: C[:, c0:c1] = (A Xt^T) diag(scale) on the DMMA pipe; the
// epilogue leaves per-(row tile, column) signed maxima in tile_colmax, and
// sign_rule_dev applies the reference's sign rule (proj/src/eigvec.cpp:340-347)
// to the columns whose mode is 1.
void gemm_nt_dev(const double* a, const double* b, int64_t m, int64_t nn, int64_t kk, double* c,
                 int64_t ldc, const double* colscale, double* tile_colmax, cudaStream_t st);
// General form: lda / ldb the operand row pitches (even), colmap (nullable)
// the output column of each GEMM column, tile_colmax rows of tcm_ld entries
// indexed by the output column.
void gemm_nt_ex(const double* a, int64_t lda, const double* b, int64_t ldb, int64_t m, int64_t nn,
                int64_t kk, double* c, int64_t ldc, const double* colscale, const int64_t* colmap,
                double* tile_colmax, int64_t tcm_ld, cudaStream_t st);
double* tile_colmax_buffer(int64_t n, int64_t ncols, DeviceScratch& ws);
// tile_colmax rows of tcm_ld entries (the default: ncols)
void sign_rule_ld(const double* tile_colmax, int64_t tcm_ld, int64_t n, int64_t ncols,
                  const int* mode, double* c, int64_t ldc, DeviceScratch& ws, cudaStream_t st);
void sign_rule_dev(const double* tile_colmax, int64_t n, int64_t ncols, const int* mode, double* c,
                   int64_t ldc, DeviceScratch& ws, cudaStream_t st);

// metrics.cu: validation products on the K5 GEMM
void symmetrize_dev(double* a, int64_t n, cudaStream_t st);
void reconstruct_dev(const double* q, const double* lam, int64_t n, double* out, DeviceScratch& ws,
                     cudaStream_t st);
void apply_update_dev(const double* a, const double* kmat, const int* sgn, int64_t n, int k,
                      double* out, cudaStream_t st);
double ortho_error_dev(const double* a, int64_t rows, int64_t cols, DeviceScratch& ws,
                       cudaStream_t st);

// Kernel launches issued by this library (evidence for bench.py's
// gpu_launches); incremented by EIGB_LAUNCH_CHECK.
int64_t launch_count();

// Live FP64 ceilings (TFLOP/s): DMMA.8x8x4 loop and DFMA loop (gemm.cu).
void fp64_peaks_dev(int sms, double* dmma_tflops, double* dfma_tflops, DeviceScratch& ws,
                    cudaStream_t st);

}  // namespace eigb
