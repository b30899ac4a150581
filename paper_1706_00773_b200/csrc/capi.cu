// C ABI (include/eigmod_b200.h) over the sm_100a pipeline.
//
// Orchestration of one update on one device:
//   K1 transform_update_dev   U = Q^T K            (deflate.cu)
//      column drop            rootfind.cpp:318-340 (norms on device, decision on host)
//   K2 build_plan_dev         runs, alpha, classification, reduced problem
//   K3 solve_roots            all roots of the reduced problem (secular.cu)
//   K4 merge/build_xt         column order + eigenvector rows (eigvec.cu)
//   K5 back_transform_dev     Q' = Q X, norms and sign rule (gemm.cu)
// Host work is limited to argument validation, a handful of scalar/size
// read-backs between stages and the bookkeeping of the reference's output
// lists; every O(n^2) or larger step runs on the GPU.
#include <algorithm>
#include <atomic>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/eigmod_b200.h"
#include "context.cuh"

using eigb::Error;


namespace eigb {
namespace {
std::atomic<int64_t> g_launches{0};
}
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(); }
}  // namespace eigb

namespace eigb_capi {

// ---------------------------------------------------------------- stages
constexpr int kRecHead = 5;  // value, origin, delta, flags, evals

void project(eigmod_b200_ctx* c, const double* q, const double* kmat, int64_t n, int64_t k,
             int64_t lo, int64_t hi, double* u_out) {
  c->stage_calls[0] += 1;
  const int kp = eigb::padded_rank(k);
  eigb::transform_update_dev(q, kmat, n, (int)k, kp, lo, hi, u_out, c->ws, c->sms, c->stream);
}

// plan_from_u = plan_groups + K2 over all groups + plan_finish.
// fuse (one-shot callers whose solve covers all roots on this device): in
// exact mode the plan needs no residues (classification is by coupling
// mass), so K2 is skipped and the solve's pole-limit count pass, which
// evaluates the same pole sum at every pole value, computes alpha_red.
void plan_from_u(eigmod_b200_ctx* c, const double* lam, const double* u, const int* signs,
                 int64_t n, int64_t k, double run_rel, bool fuse) {
  const eigb::SolveOptions& o = c->sopt;
  const bool fused = fuse && run_rel != eigb::kPoleMergeRelGap && o.fuse_alpha && o.sweep &&
                     o.sweep_poles && o.fnewton;
  // fused plans are speculative (one host round trip); a failed assumption
  // (a dropped column or a multi-member run) rebuilds it the staged way
  for (int attempt = 0; attempt < 2; ++attempt) {
    plan_groups(c, lam, u, signs, n, k, run_rel, fused && attempt == 0 && o.spec_plan);
    eigb::Plan& p = c->plan;
    if (p.k == 0) return;
    p.alpha_fused = fused;
    if (p.alpha_fused)
      EIGB_CUDA(cudaMemsetAsync(p.alpha, 0, 8 * std::max<int64_t>(p.ng, 1), c->stream));
    else
      eigb::build_plan_weights(p, 0, p.ng, p.alpha, c->ws, c->stream);
    p.par_mode = c->sopt.plan_par;
    eigb::build_plan_finish(p, c->lam, c->ws, c->stream);
    if (p.spec_failed) continue;
    c->have_plan = true;
    return;
  }
}

void plan_groups(eigmod_b200_ctx* c, const double* lam, const double* u, const int* signs,
                 int64_t n, int64_t k, double run_rel, bool spec) {
  eigb::Plan& p = c->plan;
  p = eigb::Plan{};
  p.run_rel = run_rel;
  c->plan_key_valid = false;
  c->stage_calls[1] += 1;
  // the plan keeps its own copy of lambda: the staged entry points
  // (plan_finish, finish) must not depend on the caller's buffer staying alive
  double* lam_copy = c->ws.get_f64("plan_lam", n);
  EIGB_CUDA(cudaMemcpyAsync(lam_copy, lam, 8 * n, cudaMemcpyDeviceToDevice, c->stream));
  lam = lam_copy;
  c->lam = lam_copy;
  const int kp = eigb::padded_rank(k);
  double* norms = c->ws.get_f64("cap_norms", k);
  eigb::column_norms2_dev(u, n, kp, (int)k, norms, c->stream);
  if (spec) {  // every column kept (checked on the device, eigb::Plan::spec)
    p.exact = run_rel != eigb::kPoleMergeRelGap;
    p.spec = true;
    p.norms_dev = norms;
    p.n = n;
    p.k = (int)k;
    for (int j = 0; j < (int)k; ++j) p.keep_h.push_back(j);
    p.kp = kp;
    p.u = c->ws.get_f64("pl_u", (size_t)n * p.kp);
    EIGB_CUDA(cudaMemcpyAsync(p.u, u, 8 * (size_t)n * kp, cudaMemcpyDeviceToDevice, c->stream));
    p.sgn_h.clear();
    p.m_neg = 0;
    std::vector<int> sp(p.kp, 1);
    for (int r = 0; r < p.k; ++r) {
      sp[r] = signs[r];
      p.sgn_h.push_back(sp[r]);
      p.m_neg += sp[r] < 0;
    }
    p.sgn = c->ws.get_i32("pl_sgn", p.kp);
    EIGB_CUDA(cudaMemcpyAsync(p.sgn, sp.data(), 4 * p.kp, cudaMemcpyHostToDevice, c->stream));
    eigb::build_plan_groups(p, lam, n, run_rel, c->ws, c->stream);
    c->have_plan = false;
    return;
  }
  std::vector<double> nh(k);
  EIGB_CUDA(cudaMemcpyAsync(nh.data(), norms, 8 * k, cudaMemcpyDeviceToHost, c->stream));
  EIGB_CUDA(cudaStreamSynchronize(c->stream));
  // proj/src/rootfind.cpp:318-340: drop columns with norm <= 1e-15 max(1, max);
  // exact mode: relative to the largest column only (scale invariance)
  p.exact = run_rel != eigb::kPoleMergeRelGap;
  double maxnorm = 0.0;
  for (auto& v : nh) v = std::sqrt(v), maxnorm = std::max(maxnorm, v);
  const double drop = eigb::kColumnDropRel * (p.exact ? maxnorm : std::max(1.0, maxnorm));
  p.ufro2 = 0.0;
  for (int64_t j = 0; j < k; ++j)
    if (nh[j] > drop && nh[j] > 0.0)
      p.keep_h.push_back((int)j), p.ufro2 = std::max(p.ufro2, nh[j] * nh[j]);
  p.n = n;
  p.k = (int)p.keep_h.size();
  if (p.k == 0) {  // rootfind.cpp:394-399: nothing couples
    p.kp = 0;
    p.nred = 0;
    p.ndec = n;
    c->have_plan = true;
    return;
  }
  p.kp = eigb::padded_rank(p.k);
  p.u = c->ws.get_f64("pl_u", (size_t)n * p.kp);
  int* keep_d = c->ws.get_i32("cap_keep", p.k);
  EIGB_CUDA(cudaMemcpyAsync(keep_d, p.keep_h.data(), 4 * p.k, cudaMemcpyHostToDevice, c->stream));
  eigb::repack_columns_dev(u, n, kp, keep_d, p.k, p.kp, p.u, c->stream);
  p.sgn_h.clear();
  p.m_neg = 0;
  std::vector<int> sp(p.kp, 1);
  for (int r = 0; r < p.k; ++r) {
    sp[r] = signs[p.keep_h[r]];
    p.sgn_h.push_back(sp[r]);
    p.m_neg += sp[r] < 0;
  }
  p.sgn = c->ws.get_i32("pl_sgn", p.kp);
  EIGB_CUDA(cudaMemcpyAsync(p.sgn, sp.data(), 4 * p.kp, cudaMemcpyHostToDevice, c->stream));
  eigb::build_plan_groups(p, lam, n, run_rel, c->ws, c->stream);
  c->have_plan = false;  // until build_plan_finish
}

eigb::RootRecords alloc_records(eigmod_b200_ctx* c) {
  const int64_t nr = std::max<int64_t>(c->plan.nred, 1);
  const int kp = std::max(c->plan.kp, 1);
  eigb::RootRecords r;
  r.value = c->ws.get_f64("rec_value", nr);
  r.origin = c->ws.get_i64("rec_origin", nr);
  r.delta = c->ws.get_f64("rec_delta", nr);
  r.flags = c->ws.get_i32("rec_flags", nr);
  r.evals = c->ws.get_i32("rec_evals", nr);
  r.y = c->ws.get_f64("rec_y", (size_t)nr * kp);
  return r;
}

__global__ void pack_records_kernel(eigb::RootRecords r, int64_t j0, int64_t cnt, int kp,
                                    double* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int64_t j = j0 + t;
  double* o = out + t * (kRecHead + kp);
  o[0] = r.value[j];
  o[1] = (double)r.origin[j];
  o[2] = r.delta[j];
  o[3] = (double)r.flags[j];
  o[4] = (double)r.evals[j];
  for (int c = 0; c < kp; ++c) o[kRecHead + c] = r.y[j * kp + c];
}

__global__ void unpack_records_kernel(const double* in, int64_t cnt, int kp, eigb::RootRecords r) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  const double* o = in + j * (kRecHead + kp);
  r.value[j] = o[0];
  r.origin[j] = (int64_t)o[1];
  r.delta[j] = o[2];
  r.flags[j] = (int)o[3];
  r.evals[j] = (int)o[4];
  for (int c = 0; c < kp; ++c) r.y[j * kp + c] = o[kRecHead + c];
}

void pack_records_dev(eigmod_b200_ctx* c, int64_t j0, int64_t cnt, double* out) {
  if (cnt <= 0) return;
  pack_records_kernel<<<(unsigned)eigb::cdiv(cnt, 128), 128, 0, c->stream>>>(c->recs, j0, cnt,
                                                                             c->plan.kp, out);
  EIGB_LAUNCH_CHECK();
}

void unpack_records_dev(eigmod_b200_ctx* c, const double* in, int64_t cnt) {
  c->recs = alloc_records(c);
  if (cnt <= 0) return;
  unpack_records_kernel<<<(unsigned)eigb::cdiv(cnt, 128), 128, 0, c->stream>>>(in, cnt,
                                                                               c->plan.kp, c->recs);
  EIGB_LAUNCH_CHECK();
}

void solve(eigmod_b200_ctx* c, int64_t j0, int64_t j1) {
  if (!c->have_plan) throw Error(1, "", "solve: no plan (call plan first)");
  c->stage_calls[2] += 1;
  c->recs = alloc_records(c);
  if (c->plan.nred == 0) return;
  const eigb::Plan& p = c->plan;
  if (p.alpha_fused && !(j0 == 0 && j1 == p.nred))
    throw Error(1, "", "solve: a fused-residue plan solves all roots at once");
  eigb::solve_roots(p.view(), p.alpha_red_ok ? p.alpha_red : nullptr, j0, j1, c->recs, c->sopt,
                    c->ws, c->sms, c->stream,
                    (p.alpha_fused && p.alpha_red_ok) ? p.alpha_red : nullptr);
}

__global__ void copy_block_kernel(const double* __restrict__ a, int64_t n, int64_t c0, int64_t nc,
                                  double* __restrict__ out, int64_t ldo) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x)
    for (int64_t j = threadIdx.x; j < nc; j += blockDim.x) out[i * ldo + j] = a[i * n + c0 + j];
}

// Column blocks [bstart[b], bstart[b + 1]) of an nc-column back-transform
// (inner dimension kk) whose blocks are copied to the host while the next
// blocks compute.
std::vector<int64_t> gemm_blocks(const eigmod_b200_ctx* c, int64_t n, int64_t nc, int64_t kk) {
  // Every block is a separate GEMM launch of 128 x 128 tiles (one CTA per
  // SM): a block whose tile count is not a multiple of the SM count leaves SMs
  // idle in its last wave, and every launch ends with a drain. The copy of a
  // block must only finish under the GEMMs of the blocks after it, and a
  // column copies rho times faster than it multiplies (rho = 2 x [8 n bytes at
  // ~52 GB/s] / [2 n kk flops at ~36 TFLOP/s], the 2 a safety factor), so the
  // blocks can shrink geometrically towards the end: at most four, the last
  // (whose copy is exposed) 2-4 column tiles, each earlier one at most
  // (columns after it) / rho, chosen by exhaustive search for the fewest idle
  // tile slots (n = 32768: 185 + 37 + 30 + 4 column tiles, 185 and 37 being
  // whole waves of 148 x 256 row tiles). EIGMOD_B200_BLOCKS=equal selects the
  // round-1 scheme of 6-16 equal blocks.
  const int64_t tiles_m = eigb::cdiv(n, 128), ctiles = eigb::cdiv(nc, 128);
  auto waste_of = [&](int64_t w_tiles) {
    const int64_t t = tiles_m * w_tiles;
    return eigb::cdiv(t, c->sms) * c->sms - t;
  };
  std::vector<int64_t> bstart;  // block boundaries in columns
  if (ctiles < 16) {
    // small problems: the copy is short and the GEMM takes microseconds; one
    // block avoids the per-block launches (GEMM, sign rule, copy)
    bstart = {0, nc};
    return bstart;
  }
  static int equal = -1;
  if (equal < 0) {
    const char* e = std::getenv("EIGMOD_B200_BLOCKS");
    equal = (e && std::string(e) == "equal");
  }
  const double rho = std::min(2.0, std::max(0.02, 2.0 * 2769.0 / (double)std::max<int64_t>(kk, 1)));
  if (!equal) {
    int64_t best[4] = {0, 0, 0, 0}, best_cost = -1;
    // a launch costs about as much as 32 idle tile slots of a full-size tile
    const int64_t launch_cost = 32;
    for (int64_t t4 = 2; t4 <= 4; ++t4) {
      const int64_t lim3 = std::min<int64_t>(ctiles - t4, (int64_t)(t4 / rho));
      for (int64_t b3 = 0; b3 <= lim3; ++b3) {
        const int64_t after2 = t4 + b3;
        const int64_t lim2 = std::min<int64_t>(ctiles - after2, (int64_t)(after2 / rho));
        for (int64_t b2 = 0; b2 <= lim2; ++b2) {
          const int64_t b1 = ctiles - after2 - b2;
          if (b1 < 0 || (double)b1 * rho > (double)(after2 + b2)) continue;
          if (b3 == 0 && b2 > 0) continue;  // canonical order: empty blocks first
          int64_t cost = waste_of(t4) + launch_cost;
          for (int64_t w : {b3, b2, b1})
            if (w > 0) cost += waste_of(w) + launch_cost;
          if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best[0] = b1, best[1] = b2, best[2] = b3, best[3] = t4;
          }
        }
      }
    }
    if (best_cost >= 0) {
      int64_t a = 0;
      bstart.push_back(0);
      for (int i = 0; i < 4; ++i)
        if (best[i] > 0) {
          a += best[i];
          bstart.push_back(std::min(a * 128, nc));
        }
      bstart.back() = nc;
      return bstart;
    }
  }
  // 6-16 equal blocks and a narrow last one (also the fallback when the copy
  // is too slow relative to the GEMM for four geometric blocks)
  int64_t tail = 0;
  if (ctiles >= 32) {
    tail = 2;
    for (int64_t t2 = 3; t2 <= 4; ++t2)
      if (waste_of(t2) < waste_of(tail)) tail = t2;
  }
  const int64_t main_tiles = ctiles - tail;
  int64_t best_w = eigb::cdiv(main_tiles, std::min<int64_t>(8, main_tiles)), best_waste = -1;
  for (int64_t want = 6; want <= 16 && want <= main_tiles; ++want) {
    const int64_t w = eigb::cdiv(main_tiles, want);
    int64_t waste = 0;
    for (int64_t a = 0; a < main_tiles; a += w) waste += waste_of(std::min(w, main_tiles - a));
    if (best_waste < 0 || waste < best_waste) best_waste = waste, best_w = w;
  }
  for (int64_t a = 0; a < main_tiles; a += best_w) bstart.push_back(a * 128);
  if (tail) bstart.push_back(main_tiles * 128);
  bstart.push_back(nc);
  return bstart;
}

// Compact back-transform (plans with at least kCompactMinDecoupled decoupled
// columns; eigvec.cu gather_qtilde_dev): the decoupled columns of Q' are
// copies / run rotations of Q's columns, the root columns one GEMM over the
// reduced rows, Q' [:, roots] = Q~_red X_red: 2 n nred^2 flops instead of
// 2 n^3. The gather costs one read of Q (16 n^2 bytes with the write), so it
// pays from a few dozen decoupled columns on.
constexpr int64_t kCompactMinDecoupled = 64;

void finish_compact(eigmod_b200_ctx* c, const eigb::Columns& cols, const double* q, int64_t c0,
                    int64_t c1, double* q_out, int64_t ldq, const double* colldir,
                    const int* collok, double* host_q_out, int64_t host_ld) {
  eigb::Plan& p = c->plan;
  const int64_t n = p.n, nc = c1 - c0, nred = p.nred;
  eigb::CompactCols cc;
  eigb::compact_columns_dev(p, cols, c0, c1, cc, c->ws, c->stream);
  const int64_t nr = cc.j1 - cc.j0;
  const int64_t ld = std::max<int64_t>(16, eigb::cdiv(nred, 16) * 16);  // 128-byte rows
  double* qa = c->ws.get_f64("cmp_qa", (size_t)n * ld);
  double* xr = c->ws.get_f64("cmp_xt", (size_t)std::max<int64_t>(nr, 1) * ld);
  double* colscale = c->ws.get_f64("colscale", std::max<int64_t>(nr, 1));
  double* tcm = eigb::tile_colmax_buffer(n, nc, c->ws);
  eigb::build_xt_compact_dev(p, c->recs, colldir, collok, cc.j0, cc.j1, xr, ld, colscale, c->ws,
                             c->stream);
  eigb::gather_qtilde_dev(p, q, cc, qa, ld, q_out, ldq, tcm, nc, c->stream);
  c->mark(4);
  if (!host_q_out) {
    eigb::gemm_nt_ex(qa, ld, xr, ld, n, nr, nred, q_out, ldq, colscale, cc.jpos, tcm, nc,
                     c->stream);
    c->mark(5);
    eigb::sign_rule_ld(tcm, nc, n, nc, cc.cmode, q_out, ldq, c->ws, c->stream);
    c->mark(6);
    return;
  }
  // host path: blocks of root columns; block b's final columns run from the
  // first root of the block (0 for the first) to the first root of the next
  // (nc for the last), decoupled columns in between already gathered
  if (!c->copy) EIGB_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
  std::vector<int64_t> rb = gemm_blocks(c, n, nr, nred);
  if (nr == 0) rb = {0, 0};
  std::vector<int64_t> jpos(std::max<int64_t>(nr, 1), 0);
  if (nr > 0) {
    EIGB_CUDA(cudaMemcpyAsync(jpos.data(), cc.jpos, 8 * nr, cudaMemcpyDeviceToHost, c->stream));
    EIGB_CUDA(cudaStreamSynchronize(c->stream));
  }
  const int64_t nb = (int64_t)rb.size() - 1;
  std::vector<int64_t> fb(nb + 1);
  for (int64_t b = 0; b <= nb; ++b) fb[b] = (b == 0) ? 0 : (b == nb) ? nc : jpos[rb[b]];
  while ((int64_t)c->blk_ev.size() < nb) {
    cudaEvent_t e;
    EIGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->blk_ev.push_back(e);
  }
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t ja = rb[b], w = rb[b + 1] - rb[b];
    eigb::gemm_nt_ex(qa, ld, xr + ja * ld, ld, n, w, nred, q_out, ldq, colscale + ja,
                     cc.jpos + ja, tcm, nc, c->stream);
    eigb::sign_rule_ld(tcm + fb[b], nc, n, fb[b + 1] - fb[b], cc.cmode + fb[b], q_out + fb[b],
                       ldq, c->ws, c->stream);
    EIGB_CUDA(cudaEventRecord(c->blk_ev[b], c->stream));
  }
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t a0 = fb[b], w = fb[b + 1] - fb[b];
    if (w <= 0) continue;
    EIGB_CUDA(cudaStreamWaitEvent(c->copy, c->blk_ev[b], 0));
    EIGB_CUDA(cudaMemcpy2DAsync(host_q_out + (c0 + a0), 8 * host_ld, q_out + a0, 8 * ldq, 8 * w,
                                n, cudaMemcpyDeviceToHost, c->copy));
  }
  c->mark(5);
  c->mark(6);
  EIGB_CUDA(cudaStreamSynchronize(c->copy));
}

// host_q_out != nullptr (host-pointer entry points): the GEMM and the sign
// rule run in column blocks and each finished block is copied to the host on
// a second stream while the next block computes (the D2H of Q' overlaps the
// back-transform; each block's signs are final when its GEMM ends).
void finish(eigmod_b200_ctx* c, const double* q, const double* lam_in, int64_t c0, int64_t c1,
            double* lam_out, double* q_out, int64_t ldq, double* host_q_out, int64_t host_ld) {
  eigb::Plan& p = c->plan;
  const int64_t n = p.n;
  if (!lam_in) lam_in = c->lam;
  if (q_out && c1 > c0) c->stage_calls[3] += 1;
  if (p.k == 0) {  // unchanged pairs: lambda and Q copied exactly
    if (lam_out)
      EIGB_CUDA(cudaMemcpyAsync(lam_out, lam_in, 8 * n, cudaMemcpyDeviceToDevice, c->stream));
    if (q_out && c1 > c0) {
      copy_block_kernel<<<1024, 256, 0, c->stream>>>(q, n, c0, c1 - c0, q_out, ldq);
      EIGB_LAUNCH_CHECK();
    }
    return;
  }
  eigb::Columns cols;
  eigb::merge_columns_dev(p, c->recs, cols, c->ws, c->stream);
  if (lam_out)
    EIGB_CUDA(cudaMemcpyAsync(lam_out, cols.value, 8 * n, cudaMemcpyDeviceToDevice, c->stream));
  if (!q_out || c1 <= c0) return;
  double* colldir = c->ws.get_f64("colldir", (size_t)std::max<int64_t>(p.nred, 1) * (2 * p.kp + 4));
  int* collok = c->ws.get_i32("collok", std::max<int64_t>(p.nred, 1));
  const int64_t ncoll =
      eigb::collision_vectors_dev(p, c->recs, cols, c0, c1, colldir, collok, c->ws, c->stream);
  const int64_t nc = c1 - c0;
  if (c->compact_gemm && p.kp >= 4 && p.ndec >= kCompactMinDecoupled) {
    finish_compact(c, cols, q, c0, c1, q_out, ldq, colldir, collok, host_q_out, host_ld);
    return;
  }
  double* xt = c->ws.get_f64("xt", (size_t)nc * n);
  double* colscale = c->ws.get_f64("colscale", nc);
  int* cmode = c->ws.get_i32("colmode", nc);
  eigb::build_xt_dev(p, c->recs, cols, colldir, collok, ncoll, c0, c1, xt, colscale, cmode,
                     c->ws, c->stream);
  c->mark(4);
  double* tcm = eigb::tile_colmax_buffer(n, nc, c->ws);
  if (!host_q_out) {
    eigb::gemm_nt_dev(q, xt, n, nc, n, q_out, ldq, colscale, tcm, c->stream);
    c->mark(5);
    eigb::sign_rule_dev(tcm, n, nc, cmode, q_out, ldq, c->ws, c->stream);
    c->mark(6);
    return;
  }
  if (!c->copy) EIGB_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
  const std::vector<int64_t> bstart = gemm_blocks(c, n, nc, n);
  const int64_t nb = (int64_t)bstart.size() - 1;
  while ((int64_t)c->blk_ev.size() < nb) {
    cudaEvent_t e;
    EIGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->blk_ev.push_back(e);
  }
  // all blocks are enqueued before the first copy: a pageable destination
  // makes cudaMemcpy2DAsync block the host, and the GPU must not wait on that
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t a0 = bstart[b], w = bstart[b + 1] - a0;
    double* cb = q_out + a0;
    eigb::gemm_nt_dev(q, xt + a0 * n, n, w, n, cb, ldq, colscale + a0, tcm, c->stream);
    eigb::sign_rule_dev(tcm, n, w, cmode + a0, cb, ldq, c->ws, c->stream);
    EIGB_CUDA(cudaEventRecord(c->blk_ev[b], c->stream));
  }
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t a0 = bstart[b], w = bstart[b + 1] - a0;
    EIGB_CUDA(cudaStreamWaitEvent(c->copy, c->blk_ev[b], 0));
    EIGB_CUDA(cudaMemcpy2DAsync(host_q_out + (c0 + a0), 8 * host_ld, q_out + a0, 8 * ldq, 8 * w,
                                n, cudaMemcpyDeviceToHost, c->copy));
  }
  c->mark(5);
  c->mark(6);
  EIGB_CUDA(cudaStreamSynchronize(c->copy));
}

void full_device(eigmod_b200_ctx* c, const double* q, const double* lam, const double* kmat,
                 const int* signs, int64_t n, int64_t k, double* lam_out, double* q_out,
                 double* host_q_out = nullptr) {
  const int kp = eigb::padded_rank(k);
  double* u = c->ws.get_f64("cap_u_full", (size_t)n * kp);
  c->mark(0);
  project(c, q, kmat, n, k, 0, n, u);
  c->mark(1);
  plan_from_u(c, lam, u, signs, n, k, c->run_rel, true);
  c->mark(2);
  solve(c, 0, c->plan.nred);
  c->mark(3);
  finish(c, q, lam, 0, n, lam_out, q_out, n, host_q_out, n);
  if (c->timing && c->plan.k > 0) {
    EIGB_CUDA(cudaEventSynchronize(c->ev[6]));
    for (int i = 0; i < 6; ++i) {
      float ms = 0.f;
      EIGB_CUDA(cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]));
      c->stage_ms[i] += ms;
    }
    c->timed_calls += 1;
  }
}

// Location vector over the parity-deflated poles (tools/eigmod.cpp:143-161,
// proj/include/eigmod/locate.hpp:13-50): the plan must be built with the
// reference's run threshold. counts[i] = eigenvalues of the deflated problem
// in (v_{i-1}, v_i), v the poles of the deflation record (groups of kind 0).
// Collided poles (kind 2) are no boundaries and their roots are not counted,
// as in the reference, where they leave the secular coefficients.
int64_t locate_counts(eigmod_b200_ctx* c, int64_t* counts_out) {
  const eigb::Plan& p = c->plan;
  auto st = c->stream;
  if (p.k == 0 || p.nred == 0 || p.ng == 0) {
    counts_out[0] = 0;
    return 1;
  }
  const int64_t ng = p.ng;
  std::vector<int> kd(ng);
  std::vector<int64_t> gl(ng), rk(ng), offr(ng);
  std::vector<double> gv(ng);
  EIGB_CUDA(cudaMemcpyAsync(kd.data(), p.kind, 4 * ng, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaMemcpyAsync(gl.data(), p.glen, 8 * ng, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaMemcpyAsync(rk.data(), p.rank, 8 * ng, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaMemcpyAsync(offr.data(), p.off_red, 8 * ng, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaMemcpyAsync(gv.data(), p.gval, 8 * ng, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaStreamSynchronize(st));
  std::vector<double> bval;
  std::vector<int64_t> brow, below;
  std::vector<int> bcnt;
  int64_t pt = 0;
  for (int64_t g = 0; g < ng; ++g) {
    if (kd[g] != 0) continue;
    const int cnt = (int)(gl[g] == 1 ? 1 : rk[g]);
    bval.push_back(gv[g]);
    brow.push_back(offr[g]);
    bcnt.push_back(cnt);
    below.push_back(pt);
    pt += cnt;
  }
  const int64_t nb = (int64_t)bval.size();
  if (nb == 0) {
    counts_out[0] = 0;
    return 1;
  }
  double* dv = c->ws.get_f64("loc_val", nb);
  int64_t* dr = c->ws.get_i64("loc_row", nb);
  int* dc = c->ws.get_i32("loc_cnt", nb);
  int* dnu = c->ws.get_i32("loc_nu", nb);
  EIGB_CUDA(cudaMemcpyAsync(dv, bval.data(), 8 * nb, cudaMemcpyHostToDevice, st));
  EIGB_CUDA(cudaMemcpyAsync(dr, brow.data(), 8 * nb, cudaMemcpyHostToDevice, st));
  EIGB_CUDA(cudaMemcpyAsync(dc, bcnt.data(), 4 * nb, cudaMemcpyHostToDevice, st));
  eigb::pole_inertia(p.view(), dv, dr, dc, nb, dnu, c->ws, st);
  std::vector<int> nu(nb);
  EIGB_CUDA(cudaMemcpyAsync(nu.data(), dnu, 4 * nb, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaStreamSynchronize(st));
  // eigenvalue count below each boundary, collided roots excluded
  int64_t prev = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t cb = below[b] + p.m_neg - nu[b];
    counts_out[b] = cb - prev;
    prev = cb;
  }
  counts_out[nb] = pt - prev;
  for (int64_t b = 0; b <= nb; ++b)
    if (counts_out[b] < 0)
      throw Error(2, "locate", "inertia counts are not monotone (degenerate pole)");
  return nb + 1;
}

}  // namespace eigb_capi

using namespace eigb_capi;

extern "C" {

int eigmod_b200_ctx_create(int device, eigmod_b200_ctx** out) {
  if (!out) return EIGMOD_B200_INVALID_ARGUMENT;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return EIGMOD_B200_CUDA;
  if (device < 0 || device >= ndev) return EIGMOD_B200_INVALID_ARGUMENT;
  auto* c = new eigmod_b200_ctx;
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return EIGMOD_B200_CUDA;
  }
  c->stream = c->own;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (major != 10) {  // sm_100a kernels only
    cudaStreamDestroy(c->own);
    delete c;
    return EIGMOD_B200_CUDA;
  }
  *out = c;
  return EIGMOD_B200_OK;
}

void eigmod_b200_ctx_destroy(eigmod_b200_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->ws.release();
  if (ctx->copy) cudaStreamDestroy(ctx->copy);
  for (auto e : ctx->blk_ev) cudaEventDestroy(e);
  cudaStreamDestroy(ctx->own);
  delete ctx;
}

int eigmod_b200_ctx_set_stream(eigmod_b200_ctx* ctx, void* s) {
  // verbatim: NULL is the legacy default stream (torch's default stream)
  return guarded(ctx, [&] { ctx->stream = static_cast<cudaStream_t>(s); });
}

int eigmod_b200_ctx_use_own_stream(eigmod_b200_ctx* ctx) {
  return guarded(ctx, [&] { ctx->stream = ctx->own; });
}

int eigmod_b200_set_option(eigmod_b200_ctx* ctx, const char* key, double value) {
  return guarded(ctx, [&] {
    if (!key) throw Error(1, "", "set_option: null key");
    if (std::string(key) == "run_rel") {
      if (!(value > 0.0 && value < 1e-3)) throw Error(1, "", "set_option: run_rel out of range");
      ctx->run_rel = value;
    } else if (std::string(key) == "step_tol") {
      if (!(value > 0.0)) throw Error(1, "", "set_option: step_tol must be positive");
      ctx->sopt.step_tol = value;
    } else if (std::string(key) == "pole_split") {
      ctx->sopt.pole_split = value != 0.0;
    } else if (std::string(key) == "fexit_rel") {
      ctx->sopt.fexit_rel = value;
    } else if (std::string(key) == "floor_rel") {
      ctx->sopt.floor_rel = value;
    } else if (std::string(key) == "floor_ulps") {
      ctx->sopt.floor_ulps = value;
    } else if (std::string(key) == "stall_ratio") {
      ctx->sopt.stall_ratio = value;
    } else if (std::string(key) == "geo_bisect") {
      ctx->sopt.geo_bisect = (int)value;
    } else if (std::string(key) == "trace_root") {
      ctx->sopt.trace_root = (int64_t)value;
    } else if (std::string(key) == "max_iters") {
      ctx->sopt.max_iters = (int)value;
    } else if (std::string(key) == "sweep") {
      ctx->sopt.sweep = value != 0.0;
    } else if (std::string(key) == "fnewton") {
      ctx->sopt.fnewton = value != 0.0;
    } else if (std::string(key) == "fpre") {
      ctx->sopt.fpre = value != 0.0;
    } else if (std::string(key) == "fpre_rel") {
      ctx->sopt.fpre_rel = value;
    } else if (std::string(key) == "spec_plan") {
      ctx->sopt.spec_plan = value != 0.0;
    } else if (std::string(key) == "plan_par") {
      ctx->sopt.plan_par = (int)value;
    } else if (std::string(key) == "noise_c") {
      ctx->sopt.noise_c = value;
    } else if (std::string(key) == "compact") {
      ctx->sopt.compact = value != 0.0 ? 1 : 0;
    } else if (std::string(key) == "fuse_alpha") {
      ctx->sopt.fuse_alpha = value != 0.0;
    } else if (std::string(key) == "sweep_poles") {
      ctx->sopt.sweep_poles = value != 0.0;
    } else if (std::string(key) == "split_phase_a") {
      ctx->sopt.split_phase_a = value != 0.0;
    } else if (std::string(key) == "fpre_min_kp") {
      ctx->sopt.fpre_min_kp = (int)value;
    } else if (std::string(key) == "fpre_iters") {
      ctx->sopt.fpre_iters = (int)value;
    } else if (std::string(key) == "cluster") {
      ctx->sopt.cluster = (int)value;
    } else if (std::string(key) == "compact_gemm") {
      ctx->compact_gemm = value != 0.0;
    } else if (std::string(key) == "timing") {
      ctx->timing = value != 0.0;
    } else {
      throw Error(1, "", std::string("set_option: unknown key ") + key);
    }
  });
}

const char* eigmod_b200_last_error(const eigmod_b200_ctx* ctx) {
  return ctx ? ctx->err.c_str() : "null context";
}
const char* eigmod_b200_last_stage(const eigmod_b200_ctx* ctx) {
  return ctx ? ctx->stage.c_str() : "";
}

int eigmod_b200_stats(const eigmod_b200_ctx* cctx, double* s) {
  auto* ctx = const_cast<eigmod_b200_ctx*>(cctx);
  return guarded(ctx, [&] {
    for (int i = 0; i < 8; ++i) s[i] = 0.0;
    if (!ctx->have_plan) return;
    const eigb::Plan& p = ctx->plan;
    s[0] = (double)p.nred;
    s[1] = (double)p.ndec;
    s[5] = p.kp;
    s[6] = p.k;
    s[7] = (double)p.ng;
    if (p.nred > 0 && ctx->recs.evals) {
      std::vector<int> ev(p.nred), fl(p.nred);
      EIGB_CUDA(cudaMemcpyAsync(ev.data(), ctx->recs.evals, 4 * p.nred, cudaMemcpyDeviceToHost, ctx->stream));
      EIGB_CUDA(cudaMemcpyAsync(fl.data(), ctx->recs.flags, 4 * p.nred, cudaMemcpyDeviceToHost, ctx->stream));
      EIGB_CUDA(cudaStreamSynchronize(ctx->stream));
      double tot = 0, mx = 0, col = 0;
      for (int64_t j = 0; j < p.nred; ++j) {
        tot += ev[j];
        mx = std::max(mx, (double)ev[j]);
        col += (fl[j] & 1);
      }
      s[2] = col;
      s[3] = tot;
      s[4] = mx;
    }
  });
}

int eigmod_b200_solver_profile(eigmod_b200_ctx* ctx, double* out10) {
  return guarded(ctx, [&] {
    unsigned long long h[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    auto* p = reinterpret_cast<unsigned long long*>(ctx->ws.get_i64("solve_prof", 12));
    EIGB_CUDA(cudaMemcpyAsync(h, p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    EIGB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < 10; ++i) out10[i] = (double)h[i];
  });
}

int eigmod_b200_presolve_profile(eigmod_b200_ctx* ctx, double* out4) {
  return guarded(ctx, [&] {
    unsigned long long h[4] = {0, 0, 0, 0};
    auto* p = reinterpret_cast<unsigned long long*>(ctx->ws.get_i64("fpre_prof", 4));
    EIGB_CUDA(cudaMemcpyAsync(h, p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    EIGB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < 4; ++i) out4[i] = (double)h[i];
  });
}

int eigmod_b200_solver_trace(eigmod_b200_ctx* ctx, double* out) {
  return guarded(ctx, [&] {
    const size_t cnt = (size_t)eigb::kTraceRows * eigb::kTraceCols;
    const double* p = ctx->ws.get_f64("solve_trace", cnt);
    EIGB_CUDA(cudaMemcpyAsync(out, p, cnt * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    EIGB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int64_t eigmod_b200_workspace_bytes(const eigmod_b200_ctx* ctx) {
  return ctx ? (int64_t)ctx->ws.bytes() : 0;
}

int eigmod_b200_stage_times(eigmod_b200_ctx* ctx, double* ms8, int reset) {
  return guarded(ctx, [&] {
    for (int i = 0; i < 6; ++i) ms8[i] = ctx->stage_ms[i];
    ms8[6] = 0.0;
    ms8[7] = (double)ctx->timed_calls;
    if (reset) {
      for (double& v : ctx->stage_ms) v = 0.0;
      ctx->timed_calls = 0;
    }
  });
}

int64_t eigmod_b200_launch_count(void) { return eigb::launch_count(); }

int eigmod_b200_fp64_peaks(eigmod_b200_ctx* ctx, double* out2) {
  return guarded(ctx, [&] { eigb::fp64_peaks_dev(ctx->sms, &out2[0], &out2[1], ctx->ws, ctx->stream); });
}

int eigmod_b200_padded_rank(int64_t k) { return eigb::padded_rank(k); }
int eigmod_b200_record_width(int kp) { return kRecHead + kp; }

// ------------------------------------------------------- host drop-ins
int eigmod_b200_transform_update(eigmod_b200_ctx* ctx, const double* q, const double* kmat,
                                 int64_t n, int64_t k, double* u_out) {
  return guarded(ctx, [&] {
    if (!q || !kmat || !u_out) throw Error(1, "", "transform_update: null pointer");
    check_basic(n, k, nullptr);
    const int kp = eigb::padded_rank(k);
    double* dq = ctx->ws.get_f64("h_q", (size_t)n * n);
    double* dk = ctx->ws.get_f64("h_k", (size_t)n * k);
    double* du = ctx->ws.get_f64("h_u", (size_t)n * kp);
    EIGB_CUDA(cudaMemcpyAsync(dq, q, 8 * n * n, cudaMemcpyHostToDevice, ctx->stream));
    EIGB_CUDA(cudaMemcpyAsync(dk, kmat, 8 * n * k, cudaMemcpyHostToDevice, ctx->stream));
    project(ctx, dq, dk, n, k, 0, n, du);
    std::vector<double> up((size_t)n * kp);
    EIGB_CUDA(cudaMemcpyAsync(up.data(), du, 8 * n * kp, cudaMemcpyDeviceToHost, ctx->stream));
    EIGB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int64_t i = 0; i < n; ++i)
      for (int64_t c = 0; c < k; ++c) u_out[i * k + c] = up[i * kp + c];
  });
}

int eigmod_b200_secular_weights(eigmod_b200_ctx* ctx, const double* lambda, const double* u,
                                const int* signs, int64_t n, int64_t k, double* alpha_out) {
  return guarded(ctx, [&] {
    if (k < 1) throw Error(1, "", "secular_weights: k = 0");
    check_basic(n, k, signs);
    for (int64_t i = 0; i + 1 < n; ++i)
      if (!(lambda[i] < lambda[i + 1]))
        throw Error(1, "", "secular_weights: poles not strictly increasing");
    for (int64_t i = 0; i < n; ++i)
      if (!std::isfinite(lambda[i])) throw Error(1, "", "secular_weights: non-finite pole");
    const int kp = eigb::padded_rank(k);
    std::vector<double> up((size_t)n * kp, 0.0);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t c = 0; c < k; ++c) up[i * kp + c] = u[i * k + c];
    std::vector<int64_t> gs(n), gl(n, 1);
    for (int64_t i = 0; i < n; ++i) gs[i] = i;
    std::vector<int> sp(kp, 1);
    for (int64_t r = 0; r < k; ++r) sp[r] = signs[r];
    double* du = ctx->ws.get_f64("sw_u", up.size());
    double* dl = ctx->ws.get_f64("sw_l", n);
    int64_t* dgs = ctx->ws.get_i64("sw_gs", n);
    int64_t* dgl = ctx->ws.get_i64("sw_gl", n);
    int* dsg = ctx->ws.get_i32("sw_sg", kp);
    double* da = ctx->ws.get_f64("sw_a", n);
    auto st = ctx->stream;
    EIGB_CUDA(cudaMemcpyAsync(du, up.data(), 8 * up.size(), cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dgs, gs.data(), 8 * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dgl, gl.data(), 8 * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dsg, sp.data(), 4 * kp, cudaMemcpyHostToDevice, st));
    eigb::group_weights(kp, dl, du, n, dgs, dgl, dl, n, dsg, (int)k, da, ctx->ws, st);
    EIGB_CUDA(cudaMemcpyAsync(alpha_out, da, 8 * n, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
  });
}

int eigmod_b200_deflate_problem(eigmod_b200_ctx* ctx, const double* lambda, const double* u,
                                const int* signs, int64_t n, int64_t k, double* poles,
                                double* weights, int64_t* pole_origin, int64_t* unchanged,
                                int64_t* collided, int64_t* counts) {
  return guarded(ctx, [&] {
    check_basic(n, k, signs);
    for (int64_t i = 0; i + 1 < n; ++i)
      if (!(lambda[i] <= lambda[i + 1]))
        throw Error(1, "", "deflate_problem: eigenvalues not ascending");
    const int kp = eigb::padded_rank(k);
    std::vector<double> up((size_t)n * kp, 0.0);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t c = 0; c < k; ++c) up[i * kp + c] = u[i * k + c];
    std::vector<int> sp(kp, 1);
    int m_neg = 0;
    for (int64_t r = 0; r < k; ++r) sp[r] = signs[r], m_neg += signs[r] < 0;
    auto st = ctx->stream;
    eigb::Plan p;
    p.k = (int)k;
    p.kp = kp;
    p.m_neg = m_neg;
    p.u = ctx->ws.get_f64("dp_u", up.size());
    p.sgn = ctx->ws.get_i32("dp_sg", kp);
    double* dl = ctx->ws.get_f64("dp_l", n);
    EIGB_CUDA(cudaMemcpyAsync(p.u, up.data(), 8 * up.size(), cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(p.sgn, sp.data(), 4 * kp, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, st));
    // parity record: the reference's run threshold (secular.hpp:66)
    eigb::build_plan_dev(p, dl, n, eigb::kPoleMergeRelGap, ctx->ws, st);
    const int64_t ng = p.ng;
    std::vector<int64_t> gs(ng), gl(ng);
    std::vector<double> gv(ng), al(ng);
    std::vector<int> kd(ng);
    EIGB_CUDA(cudaMemcpyAsync(gs.data(), p.gstart, 8 * ng, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaMemcpyAsync(gl.data(), p.glen, 8 * ng, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaMemcpyAsync(gv.data(), p.gval, 8 * ng, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaMemcpyAsync(al.data(), p.alpha, 8 * ng, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaMemcpyAsync(kd.data(), p.kind, 4 * ng, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
    int64_t np = 0, nu = 0, nc = 0;  // secular.cpp:316-337 output order
    for (int64_t g = 0; g < ng; ++g) {
      if (kd[g] == 1) {
        for (int64_t i = gs[g]; i < gs[g] + gl[g]; ++i) unchanged[nu++] = i;
        continue;
      }
      if (kd[g] == 2) {
        collided[nc++] = gs[g];
      } else {
        poles[np] = gv[g];
        weights[np] = al[g];
        pole_origin[np] = gs[g];
        ++np;
      }
      for (int64_t i = gs[g] + 1; i < gs[g] + gl[g]; ++i) unchanged[nu++] = i;
    }
    counts[0] = np;
    counts[1] = nu;
    counts[2] = nc;
  });
}

int eigmod_b200_locate_from_u(eigmod_b200_ctx* ctx, const double* lambda, const double* u,
                              const int* signs, int64_t n, int64_t k, int64_t* counts_out,
                              int64_t* ncounts_out) {
  return guarded(ctx, [&] {
    check_basic(n, k, signs);
    check_finite(u, n * k, "U");
    check_ascending_invalid(lambda, n);
    auto st = ctx->stream;
    const int kp = eigb::padded_rank(k);
    std::vector<double> up((size_t)n * kp, 0.0);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t c = 0; c < k; ++c) up[i * kp + c] = u[i * k + c];
    double* dl = ctx->ws.get_f64("h_l", n);
    double* du = ctx->ws.get_f64("h_u", (size_t)n * kp);
    EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(du, up.data(), 8 * up.size(), cudaMemcpyHostToDevice, st));
    plan_from_u(ctx, dl, du, signs, n, k, eigb::kPoleMergeRelGap);
    *ncounts_out = locate_counts(ctx, counts_out);
  });
}

int eigmod_b200_locate(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                       const double* kmat, const int* signs, int64_t n, int64_t k,
                       int64_t* counts_out, int64_t* ncounts_out) {
  return guarded(ctx, [&] {
    check_basic(n, k, signs);
    check_finite(kmat, n * k, "K");
    check_ascending_invalid(lambda, n);
    auto st = ctx->stream;
    const int kp = eigb::padded_rank(k);
    double* dq = ctx->ws.get_f64("h_q", (size_t)n * n);
    double* dl = ctx->ws.get_f64("h_l", n);
    double* dk = ctx->ws.get_f64("h_k", (size_t)n * k);
    double* du = ctx->ws.get_f64("h_u", (size_t)n * kp);
    EIGB_CUDA(cudaMemcpyAsync(dq, q, 8 * n * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dk, kmat, 8 * n * k, cudaMemcpyHostToDevice, st));
    project(ctx, dq, dk, n, k, 0, n, du);
    plan_from_u(ctx, dl, du, signs, n, k, eigb::kPoleMergeRelGap);
    *ncounts_out = locate_counts(ctx, counts_out);
  });
}

int eigmod_b200_update_eigenvalues(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                                   const double* kmat, const int* signs, int64_t n, int64_t k,
                                   double tol, double* values_out, double* roots_out,
                                   int64_t* nroots_out, double* u_out, int64_t* k_eff_out,
                                   int64_t* keep_out) {
  return guarded(ctx, [&] {
    check_basic(n, k, signs);
    check_finite(kmat, n * k, "K");
    if (!(tol > 0.0)) throw Error(1, "", "update_eigenvalues: tol must be positive");
    check_ascending(lambda, n);
    auto st = ctx->stream;
    const int kp = eigb::padded_rank(k);
    double* dq = ctx->ws.get_f64("h_q", (size_t)n * n);
    double* dl = ctx->ws.get_f64("h_l", n);
    double* dk = ctx->ws.get_f64("h_k", (size_t)n * k);
    double* du = ctx->ws.get_f64("h_u", (size_t)n * kp);
    double* dlo = ctx->ws.get_f64("h_lo", n);
    EIGB_CUDA(cudaMemcpyAsync(dq, q, 8 * n * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dk, kmat, 8 * n * k, cudaMemcpyHostToDevice, st));
    project(ctx, dq, dk, n, k, 0, n, du);
    plan_from_u(ctx, dl, du, signs, n, k, ctx->run_rel, true);
    solve(ctx, 0, ctx->plan.nred);
    finish(ctx, dq, dl, 0, 0, dlo, nullptr, n);
    const eigb::Plan& p = ctx->plan;
    EIGB_CUDA(cudaMemcpyAsync(values_out, dlo, 8 * n, cudaMemcpyDeviceToHost, st));
    if (roots_out && p.nred > 0)
      EIGB_CUDA(cudaMemcpyAsync(roots_out, ctx->recs.value, 8 * p.nred, cudaMemcpyDeviceToHost, st));
    if (u_out && p.k > 0) {
      std::vector<double> up((size_t)n * p.kp);
      EIGB_CUDA(cudaMemcpyAsync(up.data(), p.u, 8 * up.size(), cudaMemcpyDeviceToHost, st));
      EIGB_CUDA(cudaStreamSynchronize(st));
      for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < p.k; ++c) u_out[i * p.k + c] = up[i * p.kp + c];
    }
    EIGB_CUDA(cudaStreamSynchronize(st));
    if (roots_out && p.nred > 1) std::sort(roots_out, roots_out + p.nred);
    if (nroots_out) *nroots_out = p.nred;
    if (k_eff_out) *k_eff_out = p.k;
    if (keep_out)
      for (int c = 0; c < p.k; ++c) keep_out[c] = p.keep_h[c];
    // the plan stays on the device for assemble_eigenvectors: keyed by the
    // inputs the caller will hand back (lambda, the kept columns of U, their
    // signs) and checked against the n eigenvalues
    if (u_out) {
      std::vector<int> ks(p.sgn_h.begin(), p.sgn_h.end());
      ctx->plan_key = plan_key_of(lambda, u_out, ks.data(), n, p.k);
      if (roots_out) ctx->plan_roots.assign(roots_out, roots_out + p.nred);
      ctx->plan_key_valid = roots_out != nullptr;
    }
  });
}

int eigmod_b200_update_decomposition(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                                     const double* kmat, const int* signs, int64_t n, int64_t k,
                                     double tol, double* lambda_out, double* q_out,
                                     double* wall_time_out) {
  return guarded(ctx, [&] {
    check_basic(n, k, signs);
    check_finite(kmat, n * k, "K");
    if (!(tol > 0.0)) throw Error(1, "", "update_eigenvalues: tol must be positive");
    check_ascending(lambda, n);
    auto st = ctx->stream;
    const auto t0 = std::chrono::steady_clock::now();
    double* dq = ctx->ws.get_f64("h_q", (size_t)n * n);
    double* dl = ctx->ws.get_f64("h_l", n);
    double* dk = ctx->ws.get_f64("h_k", (size_t)n * k);
    double* dlo = ctx->ws.get_f64("h_lo", n);
    double* dqo = ctx->ws.get_f64("h_qo", (size_t)n * n);
    EIGB_CUDA(cudaMemcpyAsync(dq, q, 8 * n * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dk, kmat, 8 * n * k, cudaMemcpyHostToDevice, st));
    // Q' leaves in column blocks overlapped with the GEMM (finish); the rank-0
    // case (plain copy of Q) has no GEMM to overlap with
    full_device(ctx, dq, dl, dk, signs, n, k, dlo, dqo, q_out);
    EIGB_CUDA(cudaMemcpyAsync(lambda_out, dlo, 8 * n, cudaMemcpyDeviceToHost, st));
    if (ctx->plan.k == 0)
      EIGB_CUDA(cudaMemcpyAsync(q_out, dqo, 8 * n * n, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
    if (wall_time_out)
      *wall_time_out =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// ------------------------------------------------------- device pipeline
int eigmod_b200_update_decomposition_device(eigmod_b200_ctx* ctx, const double* d_q,
                                            const double* d_lambda, const double* d_kmat,
                                            const int* signs, int64_t n, int64_t k,
                                            double* d_lambda_out, double* d_q_out) {
  return guarded(ctx, [&] {
    check_basic(n, k, signs);
    full_device(ctx, d_q, d_lambda, d_kmat, signs, n, k, d_lambda_out, d_q_out);
  });
}

int eigmod_b200_project_device(eigmod_b200_ctx* ctx, const double* d_q, const double* d_kmat,
                               int64_t n, int64_t k, int64_t col_lo, int64_t col_hi,
                               double* d_u_out) {
  return guarded(ctx, [&] {
    check_basic(n, k, nullptr);
    if (col_lo < 0 || col_hi > n || col_hi < col_lo) throw Error(1, "", "project: bad range");
    ctx->mark(0);
    if (col_hi > col_lo) project(ctx, d_q, d_kmat, n, k, col_lo, col_hi, d_u_out);
    ctx->mark(1);
    ctx->accumulate(0, 1);
  });
}

int eigmod_b200_plan_device(eigmod_b200_ctx* ctx, const double* d_lambda, const double* d_u,
                            const int* signs, int64_t n, int64_t k, int64_t* nroots_out) {
  return guarded(ctx, [&] {
    check_basic(n, k, signs);
    ctx->mark(1);
    plan_from_u(ctx, d_lambda, d_u, signs, n, k, ctx->run_rel);
    ctx->mark(2);
    ctx->accumulate(1, 2);
    ctx->recs = alloc_records(ctx);
    if (nroots_out) *nroots_out = ctx->plan.nred;
  });
}

int eigmod_b200_plan_groups_device(eigmod_b200_ctx* ctx, const double* d_lambda,
                                   const double* d_u, const int* signs, int64_t n, int64_t k,
                                   int64_t* ng_out) {
  return guarded(ctx, [&] {
    check_basic(n, k, signs);
    ctx->mark(1);
    plan_groups(ctx, d_lambda, d_u, signs, n, k, ctx->run_rel);
    *ng_out = ctx->plan.k == 0 ? 0 : ctx->plan.ng;
  });
}

int eigmod_b200_plan_weights_device(eigmod_b200_ctx* ctx, int64_t g0, int64_t g1,
                                    double* d_alpha_out) {
  return guarded(ctx, [&] {
    const eigb::Plan& p = ctx->plan;
    if (p.k == 0) return;
    if (g0 < 0 || g1 > p.ng || g0 > g1) throw Error(1, "", "plan_weights: bad group range");
    eigb::build_plan_weights(p, g0, g1, d_alpha_out, ctx->ws, ctx->stream);
  });
}

int eigmod_b200_plan_finish_device(eigmod_b200_ctx* ctx, const double* d_alpha_all,
                                   int64_t* nred_out) {
  return guarded(ctx, [&] {
    eigb::Plan& p = ctx->plan;
    if (p.k == 0) {
      ctx->have_plan = true;
      *nred_out = 0;
      return;
    }
    if (d_alpha_all != p.alpha)
      EIGB_CUDA(cudaMemcpyAsync(p.alpha, d_alpha_all, 8 * p.ng, cudaMemcpyDeviceToDevice,
                                ctx->stream));
    p.par_mode = ctx->sopt.plan_par;
    eigb::build_plan_finish(p, ctx->lam, ctx->ws, ctx->stream);
    ctx->have_plan = true;
    *nred_out = p.nred;
    ctx->mark(2);
    ctx->accumulate(1, 2);
  });
}

int eigmod_b200_solve_device(eigmod_b200_ctx* ctx, int64_t j0, int64_t j1, double* d_rec_out) {
  return guarded(ctx, [&] {
    if (!ctx->have_plan) throw Error(1, "", "solve: no plan");
    if (j0 < 0 || j1 > ctx->plan.nred || j1 < j0) throw Error(1, "", "solve: bad root range");
    ctx->recs = alloc_records(ctx);
    if (ctx->plan.nred == 0) return;
    ctx->mark(2);
    eigb::solve_roots(ctx->plan.view(), ctx->plan.alpha_red_ok ? ctx->plan.alpha_red : nullptr, j0,
                      j1, ctx->recs, ctx->sopt, ctx->ws, ctx->sms, ctx->stream);
    if (d_rec_out && j1 > j0) {
      pack_records_kernel<<<(unsigned)eigb::cdiv(j1 - j0, 128), 128, 0, ctx->stream>>>(
          ctx->recs, j0, j1 - j0, ctx->plan.kp, d_rec_out);
      EIGB_LAUNCH_CHECK();
    }
    ctx->mark(3);
    ctx->accumulate(2, 3);
  });
}

int eigmod_b200_finish_device(eigmod_b200_ctx* ctx, const double* d_q, const double* d_rec_all,
                              int64_t c0, int64_t c1, double* d_lambda_out, double* d_q_out,
                              int64_t ldq) {
  return guarded(ctx, [&] {
    if (!ctx->have_plan) throw Error(1, "", "finish: no plan");
    const eigb::Plan& p = ctx->plan;
    if (c0 < 0 || c1 > p.n || c1 < c0) throw Error(1, "", "finish: bad column range");
    ctx->recs = alloc_records(ctx);
    if (d_rec_all && p.nred > 0) {
      unpack_records_kernel<<<(unsigned)eigb::cdiv(p.nred, 128), 128, 0, ctx->stream>>>(
          d_rec_all, p.nred, p.kp, ctx->recs);
      EIGB_LAUNCH_CHECK();
    }
    // lambda (for the rank-0 copy) comes from the plan's own copy
    ctx->mark(3);
    finish(ctx, d_q, nullptr, c0, c1, d_lambda_out, d_q_out, ldq);
    if (p.k > 0 && c1 > c0 && d_q_out) {
      ctx->accumulate(3, 6);
      if (ctx->timing) ctx->timed_calls += 1;
    }
  });
}

int eigmod_b200_gemm_nt_device(eigmod_b200_ctx* ctx, const double* d_a, const double* d_b,
                               int64_t m, int64_t nn, int64_t kk, double* d_c, int64_t ldc) {
  return guarded(ctx, [&] {
    double* ones = ctx->ws.get_f64("gemm_ones", nn);
    std::vector<double> h(nn, 1.0);
    EIGB_CUDA(cudaMemcpyAsync(ones, h.data(), 8 * nn, cudaMemcpyHostToDevice, ctx->stream));
    EIGB_CUDA(cudaStreamSynchronize(ctx->stream));
    eigb::gemm_nt_dev(d_a, d_b, m, nn, kk, d_c, ldc, ones, nullptr, ctx->stream);
  });
}

}  // extern "C"

// ----------------------------------------------- more host drop-ins
namespace eigb {
void update_metrics_dev(const double* q, const double* lam, const double* kmat, const int* sgn,
                        int64_t n, int k, const double* qo, const double* lo, double* residual_fro,
                        double* ortho_err, DeviceScratch& ws, cudaStream_t st);
}

extern "C" {

int eigmod_b200_reconstruct(eigmod_b200_ctx* ctx, const double* q, const double* lambda, int64_t n,
                            double* a_out) {
  return guarded(ctx, [&] {
    if (n < 1) throw Error(1, "", "reconstruct: dimension mismatch");
    auto st = ctx->stream;
    double* dq = ctx->ws.get_f64("h_q", (size_t)n * n);
    double* dl = ctx->ws.get_f64("h_l", n);
    double* da = ctx->ws.get_f64("h_qo", (size_t)n * n);
    EIGB_CUDA(cudaMemcpyAsync(dq, q, 8 * n * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, st));
    eigb::reconstruct_dev(dq, dl, n, da, ctx->ws, st);
    EIGB_CUDA(cudaMemcpyAsync(a_out, da, 8 * n * n, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
  });
}

int eigmod_b200_reconstruct_device(eigmod_b200_ctx* ctx, const double* d_q,
                                   const double* d_lambda, int64_t n, double* d_a_out) {
  return guarded(ctx, [&] {
    if (n < 1) throw Error(1, "", "reconstruct: dimension mismatch");
    eigb::reconstruct_dev(d_q, d_lambda, n, d_a_out, ctx->ws, ctx->stream);
  });
}

int eigmod_b200_apply_update(eigmod_b200_ctx* ctx, const double* a, const double* kmat,
                             const int* signs, int64_t n, int64_t k, double* a_out) {
  return guarded(ctx, [&] {
    check_basic(n, k, signs);
    auto st = ctx->stream;
    double* da = ctx->ws.get_f64("h_q", (size_t)n * n);
    double* dk = ctx->ws.get_f64("h_k", (size_t)n * k);
    int* ds = ctx->ws.get_i32("h_s", k);
    double* dout = ctx->ws.get_f64("h_qo", (size_t)n * n);
    EIGB_CUDA(cudaMemcpyAsync(da, a, 8 * n * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dk, kmat, 8 * n * k, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(ds, signs, 4 * k, cudaMemcpyHostToDevice, st));
    eigb::apply_update_dev(da, dk, ds, n, (int)k, dout, st);
    EIGB_CUDA(cudaMemcpyAsync(a_out, dout, 8 * n * n, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
  });
}

int eigmod_b200_apply_update_device(eigmod_b200_ctx* ctx, const double* d_a,
                                    const double* d_kmat, const int* signs, int64_t n, int64_t k,
                                    double* d_a_out) {
  return guarded(ctx, [&] {
    check_basic(n, k, signs);
    int* ds = ctx->ws.get_i32("h_s", k);
    EIGB_CUDA(cudaMemcpyAsync(ds, signs, 4 * k, cudaMemcpyHostToDevice, ctx->stream));
    eigb::apply_update_dev(d_a, d_kmat, ds, n, (int)k, d_a_out, ctx->stream);
  });
}

int eigmod_b200_ortho_error(eigmod_b200_ctx* ctx, const double* a, int64_t rows, int64_t cols,
                            double* err_out) {
  return guarded(ctx, [&] {
    if (rows < 1 || cols < 1) throw Error(1, "", "ortho_error: empty matrix");
    auto st = ctx->stream;
    double* da = ctx->ws.get_f64("h_q", (size_t)rows * cols);
    EIGB_CUDA(cudaMemcpyAsync(da, a, 8 * rows * cols, cudaMemcpyHostToDevice, st));
    *err_out = eigb::ortho_error_dev(da, rows, cols, ctx->ws, st);
  });
}

int eigmod_b200_ortho_error_device(eigmod_b200_ctx* ctx, const double* d_a, int64_t rows,
                                   int64_t cols, double* err_out) {
  return guarded(ctx, [&] {
    if (rows < 1 || cols < 1) throw Error(1, "", "ortho_error: empty matrix");
    *err_out = eigb::ortho_error_dev(d_a, rows, cols, ctx->ws, ctx->stream);
  });
}

int eigmod_b200_assemble_from_u(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                                const double* u, const int* signs, int64_t n, int64_t k,
                                double* lambda_out, double* q_out) {
  return guarded(ctx, [&] {
    if (k < 0 || k > n) throw Error(1, "", "assemble: rank out of range");
    check_ascending(lambda, n);
    auto st = ctx->stream;
    double* dq = ctx->ws.get_f64("h_q", (size_t)n * n);
    double* dl = ctx->ws.get_f64("h_l", n);
    double* dlo = ctx->ws.get_f64("h_lo", n);
    double* dqo = ctx->ws.get_f64("h_qo", (size_t)n * n);
    EIGB_CUDA(cudaMemcpyAsync(dq, q, 8 * n * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, st));
    if (k == 0) {
      EIGB_CUDA(cudaMemcpyAsync(q_out, dq, 8 * n * n, cudaMemcpyDeviceToHost, st));
      EIGB_CUDA(cudaMemcpyAsync(lambda_out, dl, 8 * n, cudaMemcpyDeviceToHost, st));
      EIGB_CUDA(cudaStreamSynchronize(st));
      return;
    }
    check_basic(n, k, signs);
    const int kp = eigb::padded_rank(k);
    std::vector<double> up((size_t)n * kp, 0.0);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t c = 0; c < k; ++c) up[i * kp + c] = u[i * k + c];
    double* du = ctx->ws.get_f64("h_u", (size_t)n * kp);
    EIGB_CUDA(cudaMemcpyAsync(du, up.data(), 8 * up.size(), cudaMemcpyHostToDevice, st));
    plan_from_u(ctx, dl, du, signs, n, k, ctx->run_rel, true);
    solve(ctx, 0, ctx->plan.nred);
    finish(ctx, dq, dl, 0, n, dlo, dqo, n);
    EIGB_CUDA(cudaMemcpyAsync(lambda_out, dlo, 8 * n, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaMemcpyAsync(q_out, dqo, 8 * n * n, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
  });
}

int eigmod_b200_assemble(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                         const double* u, const int* signs, int64_t n, int64_t k,
                         const double* roots, int64_t nroots, const int64_t* unchanged,
                         int64_t nunchanged, const int64_t* collided, int64_t ncollided,
                         double* lambda_out, double* q_out, int* path_out) {
  return guarded(ctx, [&] {
    if (k < 0 || k > n) throw Error(1, "", "assemble: rank out of range");
    if (nroots < 0 || nunchanged < 0 || ncollided < 0) throw Error(1, "", "assemble: bad counts");
    check_ascending(lambda, n);
    // the plan the last update_eigenvalues call on this context produced:
    // same inputs, same roots (its deflation record is informational)
    const bool cached = ctx->plan_key_valid && ctx->have_plan && ctx->plan.n == n &&
                        plan_key_of(lambda, u, signs, n, k) == ctx->plan_key &&
                        (int64_t)ctx->plan_roots.size() == nroots &&
                        std::equal(roots, roots + nroots, ctx->plan_roots.begin());
    if (!cached && nroots + nunchanged + ncollided != n)
      throw Error(2, "assemble", "eigenpair count mismatch");  // eigvec.cpp:277-278
    // the plan's n eigenvalues (roots, unchanged and collided values merged,
    // eigvec.cpp:260-276)
    std::vector<double> want(roots, roots + nroots);
    for (int64_t i = 0; i < nunchanged; ++i) {
      if (unchanged[i] < 0 || unchanged[i] >= n) throw Error(1, "", "assemble: index out of range");
      want.push_back(lambda[unchanged[i]]);
    }
    for (int64_t i = 0; i < ncollided; ++i) {
      if (collided[i] < 0 || collided[i] >= n) throw Error(1, "", "assemble: index out of range");
      want.push_back(lambda[collided[i]]);
    }
    std::sort(want.begin(), want.end());
    auto st = ctx->stream;
    double* dq = ctx->ws.get_f64("h_q", (size_t)n * n);
    double* dlo = ctx->ws.get_f64("h_lo", n);
    double* dqo = ctx->ws.get_f64("h_qo", (size_t)n * n);
    if (path_out) *path_out = cached ? 1 : 2;
    if (!cached && k == 0) {  // nothing couples: every pair passes through exactly
      if (!std::equal(want.begin(), want.end(), lambda))
        throw Error(2, "assemble", "plan eigenvalues are not the updated eigenvalues of "
                                   "plan.transformed (rank 0)");
      std::memcpy(lambda_out, lambda, 8 * n);
      std::memcpy(q_out, q, 8 * n * n);
      return;
    }
    EIGB_CUDA(cudaMemcpyAsync(dq, q, 8 * n * n, cudaMemcpyHostToDevice, st));
    if (!cached) {
      // a plan from elsewhere: solve the secular equation of plan.transformed
      // and accept the plan only if its eigenvalues are these
      double* dl = ctx->ws.get_f64("h_l", n);
      EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, st));
      check_basic(n, k, signs);
      const int kp = eigb::padded_rank(k);
      std::vector<double> up((size_t)n * kp, 0.0);
      for (int64_t i = 0; i < n; ++i)
        for (int64_t c = 0; c < k; ++c) up[i * kp + c] = u[i * k + c];
      double* du = ctx->ws.get_f64("h_u", (size_t)n * kp);
      EIGB_CUDA(cudaMemcpyAsync(du, up.data(), 8 * up.size(), cudaMemcpyHostToDevice, st));
      plan_from_u(ctx, dl, du, signs, n, k, ctx->run_rel, true);
      solve(ctx, 0, ctx->plan.nred);
      finish(ctx, dq, nullptr, 0, 0, dlo, nullptr, n);
      std::vector<double> got(n);
      EIGB_CUDA(cudaMemcpyAsync(got.data(), dlo, 8 * n, cudaMemcpyDeviceToHost, st));
      EIGB_CUDA(cudaStreamSynchronize(st));
      double scale = 0.0, err = 0.0;
      for (int64_t i = 0; i < n; ++i)
        scale = std::max(scale, std::fabs(got[i])), err = std::max(err, std::fabs(got[i] - want[i]));
      if (!(err <= 1e-10 * std::max(scale, DBL_MIN)))
        throw Error(2, "assemble", "plan eigenvalues are not the updated eigenvalues of "
                                   "plan.transformed (max deviation " + std::to_string(err) + ")");
    }
    finish(ctx, dq, nullptr, 0, n, dlo, dqo, n, ctx->plan.k > 0 ? q_out : nullptr, n);
    EIGB_CUDA(cudaMemcpyAsync(lambda_out, dlo, 8 * n, cudaMemcpyDeviceToHost, st));
    if (ctx->plan.k == 0)
      EIGB_CUDA(cudaMemcpyAsync(q_out, dqo, 8 * n * n, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
  });
}

int eigmod_b200_stage_calls(const eigmod_b200_ctx* ctx, int64_t* out4) {
  if (!ctx || !out4) return EIGMOD_B200_INVALID_ARGUMENT;
  for (int i = 0; i < 4; ++i) out4[i] = ctx->stage_calls[i];
  return EIGMOD_B200_OK;
}

int eigmod_b200_update_metrics(eigmod_b200_ctx* ctx, const double* q, const double* lambda,
                               const double* kmat, const int* signs, int64_t n, int64_t k,
                               const double* q_out, const double* lambda_out, double* residual_fro,
                               double* ortho_err) {
  return guarded(ctx, [&] {
    check_basic(n, k, signs);
    auto st = ctx->stream;
    double* dq = ctx->ws.get_f64("m_q", (size_t)n * n);
    double* dqo = ctx->ws.get_f64("m_qo", (size_t)n * n);
    double* dl = ctx->ws.get_f64("m_l", n);
    double* dlo = ctx->ws.get_f64("m_lo", n);
    double* dk = ctx->ws.get_f64("m_k", (size_t)n * k);
    int* ds = ctx->ws.get_i32("m_s", k);
    EIGB_CUDA(cudaMemcpyAsync(dq, q, 8 * n * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dqo, q_out, 8 * n * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dlo, lambda_out, 8 * n, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(dk, kmat, 8 * n * k, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpyAsync(ds, signs, 4 * k, cudaMemcpyHostToDevice, st));
    eigb::update_metrics_dev(dq, dl, dk, ds, n, (int)k, dqo, dlo, residual_fro, ortho_err, ctx->ws,
                             st);
  });
}

int eigmod_b200_gemm_nt(eigmod_b200_ctx* ctx, const double* a, const double* b, int64_t m,
                        int64_t nn, int64_t kk, double* c) {
  return guarded(ctx, [&] {
    if (m < 0 || nn < 0 || kk < 0) throw Error(1, "", "gemm_nt: negative size");
    if (m == 0 || nn == 0) return;
    auto st = ctx->stream;
    const int64_t kp = kk + (kk & 1);  // the DMMA kernel wants an even inner dimension
    double* da = ctx->ws.get_f64("g_a", (size_t)m * kp);
    double* db = ctx->ws.get_f64("g_b", (size_t)nn * kp);
    double* dc = ctx->ws.get_f64("g_c", (size_t)m * nn);
    double* ones = ctx->ws.get_f64("g_ones", nn);
    std::vector<double> h(nn, 1.0);
    EIGB_CUDA(cudaMemcpyAsync(ones, h.data(), 8 * nn, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemset2DAsync(da, 8 * kp, 0, 8 * kp, m, st));
    EIGB_CUDA(cudaMemset2DAsync(db, 8 * kp, 0, 8 * kp, nn, st));
    EIGB_CUDA(cudaMemcpy2DAsync(da, 8 * kp, a, 8 * kk, 8 * kk, m, cudaMemcpyHostToDevice, st));
    EIGB_CUDA(cudaMemcpy2DAsync(db, 8 * kp, b, 8 * kk, 8 * kk, nn, cudaMemcpyHostToDevice, st));
    eigb::gemm_nt_dev(da, db, m, nn, kp, dc, nn, ones, nullptr, st);
    EIGB_CUDA(cudaMemcpyAsync(c, dc, 8 * m * nn, cudaMemcpyDeviceToHost, st));
    EIGB_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
