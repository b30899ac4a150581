// Internal interfaces between the device stages of the eigen-update pipeline.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#ifdef __CUDACC__
#include "secular_pass.cuh"
#endif

namespace eigb {

// Named, grow-only device buffers owned by a context (one per device/stream).
class DeviceScratch {
 public:
  ~DeviceScratch() { release(); }
  void* get(const std::string& name, size_t bytes) {
    auto it = bufs_.find(name);
    if (it != bufs_.end() && it->second.second >= bytes) return it->second.first;
    if (it != bufs_.end()) {
      cudaFree(it->second.first);
      bufs_.erase(it);
    }
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    EIGB_CUDA(cudaMalloc(&p, bytes));
    bufs_[name] = {p, bytes};
    return p;
  }
  double* get_f64(const std::string& n, size_t cnt) { return static_cast<double*>(get(n, cnt * 8)); }
  int64_t* get_i64(const std::string& n, size_t cnt) { return static_cast<int64_t*>(get(n, cnt * 8)); }
  int* get_i32(const std::string& n, size_t cnt) { return static_cast<int*>(get(n, cnt * 4)); }
  void release() {
    for (auto& kv : bufs_) cudaFree(kv.second.first);
    bufs_.clear();
  }
  size_t bytes() const {
    size_t s = 0;
    for (auto& kv : bufs_) s += kv.second.second;
    return s;
  }

 private:
  std::map<std::string, std::pair<void*, size_t>> bufs_;
};

// The deflated ("reduced") secular problem the solver works on: poles d
// (ascending, duplicates allowed after run compression) and rows u (padded to
// kp columns), diag(d) + u J u^T.
struct ReducedView {
  const double* d;
  const double* u;    // [n][kp]
  const int* sgn;     // [kp] device, pads +1
  int64_t n;
  int k;              // effective rank (unpadded)
  int kp;
  int m_neg;          // number of -1 signs
  double lo_clip, hi_clip;
};

// Per-root solver output (indexed by root j of the reduced problem).
struct RootRecords {
  double* value;   // root (double)
  int64_t* origin; // reduced pole index o: root = d[o] + delta
  double* delta;
  int* flags;      // 1 collided (sits on pole o), 2 ulp bracket without isolation
  int* evals;      // S(x) evaluations spent
  double* y;       // [n][kp] unit null vector of S(root)
};

// Phase-B stopping rule: the evaluated point is accepted once the Newton
// correction is below step_tol * eps * |delta| (or the certified bracket is
// within 2 ulps); max_iters caps the evaluations of one root. At a few ulps
// the direction of the correction is rounding noise, so iterating further
// only bounces between bracket ends (4 ulps measured: same orthogonality as
// 0.1 ulp, 3 fewer evaluations per root).
struct SolveOptions {
  double step_tol = 4.0;
  int max_iters = 160;
  bool sweep = true;    // count sweep for the initial brackets (else Weyl windows)
  bool pole_split = true;  // limit counts at poles with roots next to them (sweep)
  bool sweep_poles = true;  // brackets from pole-limit counts only (one evaluation per pole)
  bool fnewton = true;  // Newton on the scalar secular function first
  // CTAs per thread-block cluster splitting the pole sum: 1, 2, 4, 8, or -1
  // for the size-based choice (solve_cluster_size)
  int cluster = -1;
  int64_t trace_root = -1;  // diagnostics: record the iterates of this root
  double fexit_rel = 1e-2;  // f step leaving the bracket below this * |delta|: continue on S
  double floor_rel = 1e-11; // S-Newton step no longer shrinking below this * |delta|: converged
  double floor_ulps = 4.0;   // ... or below this many ulps of the root value
  double stall_ratio = 0.5;  // "no longer shrinking": |step| >= stall_ratio * |previous step|
  int geo_bisect = 1;       // geometric bisection of brackets spanning decades of delta
  int compact = 1;          // pack the slots of drained solver batches (tail passes)
  // noise-floor stopping: converged when |sigma| <= noise_c eps (1 + sum |u_i|^2 |D_i|) (0: off)
  double noise_c = 1.0;
  // scalar presolve: the f-root (K2 residues) of every isolated root before
  // the S solver, which then starts psi-Newton there. Used from kp = 16 up,
  // where an S evaluation costs ~10x an f evaluation (cfg4 n = 32768: solve
  // 180 -> 157 ms); below that it does not pay (tools/exp_fpre.py).
  bool fpre = true;
  int fpre_min_kp = 16;
  // with the presolve: bisect unisolated roots to isolation first (stage 1),
  // so they get the presolve too, then finish every root (stage 2)
  bool split_phase_a = true;
  int fpre_iters = 12;
  // presolve stops at |step| <= fpre_rel |delta|: its root is only a start (the S solver
  // refines it); 1e-6 minimises K3 at config 4 (tools/exp_fpre_rel.py: 71.6 -> 69.3 ms)
  double fpre_rel = 1e-6;
  // exact mode, one device: the residues alpha come from the pole-limit count
  // pass (the same pole sum at every pole value) instead of a K2 pass
  bool fuse_alpha = true;
  // fused one-shot plans: sizes and the column-drop decision read back once
  bool spec_plan = true;
  // plan finish (classification, reduced-problem assembly, clips) on many
  // CTAs: -1 from n >= 8192 on, 0 never, 1 always
  int plan_par = -1;
};

// Diagnostics trace of one root: per evaluation kTraceCols doubles
// (iteration, phase, fmode, delta, lo, hi, f, f', sigma, g, step, origin).
constexpr int kTraceCols = 12;
constexpr int kTraceRows = 200;

// alpha: residues of the reduced poles for the f-Newton phase (nullptr when
// the reduced problem has compressed runs, whose poles are not simple).
// alpha_fill != nullptr (pole-limit counts on, every pole in the window): the
// count pass also computes the residue of every simple reduced pole into
// alpha_fill (proj/src/secular.cpp:168-202 at the pole value, the pole's own
// row excluded) and the solve uses them as alpha.
void solve_roots(const ReducedView& rp, const double* alpha, int64_t j0, int64_t j1,
                 const RootRecords& out, const SolveOptions& opt, DeviceScratch& ws, int sms,
                 cudaStream_t st, double* alpha_fill = nullptr);

// Location-vector support: for each of nb reduced pole values bval[b] (rows
// brow[b] .. brow[b]+bcnt[b]-1 of rp sit at that value), nu[b] = negative
// inertia of T = J + sum_{other rows} u u^T/(d - v) restricted to the
// orthogonal complement of the pole's rows. #eig < v = #{d < v} + m - nu.
void pole_inertia(const ReducedView& rp, const double* bval, const int64_t* brow, const int* bcnt,
                  int64_t nb, int* nu, DeviceScratch& ws, cudaStream_t st,
                  double* alpha_out = nullptr, const unsigned long long* nb_dev = nullptr);

void group_weights(int kp, const double* rep, const double* u, int64_t n, const int64_t* gstart,
                   const int64_t* glen, const double* gval, int64_t ng, const int* sgn, int k,
                   double* alpha, DeviceScratch& ws, cudaStream_t st);

}  // namespace eigb
