// Single-process multi-GPU update (SURVEY.md §8(b) "multi-GPU context handle",
// §8(e) partitioning): one context, stream and host thread per device, one
// NCCL communicator per device from ncclCommInitAll. The reference's C++
// entry points (update_decomposition, eigvec.hpp:35-36; the eigenvalue stage,
// rootfind.hpp:51-53) reach it through eigmod::set_devices or
// EIGMOD_B200_DEVICES (csrc/eigmod_api.cpp).
//
// Data path of one update over G devices (rank g, host buffers in and out):
//   1. H2D of Q's row slice g (1/G of Q over this device's PCIe link), then an
//      in-place ncclAllGather rebuilds the replicated Q over NVLink; lambda
//      and K to every device.
//   2. U rows of the Q-column slice g (K1), ncclAllGather of U.
//   3. plan groups on every rank from the same bits, K2 weights of group
//      slice g, ncclAllGather of alpha, the rest of the plan (redundant).
//   4. roots of index slice g (K3), ncclAllGather of the root records.
//   5. the column block g of Q' = Q X (K4 + K5), D2H of the block into the
//      caller's Q' (strided), overlapped with the GEMM by column sub-blocks;
//      rank 0 returns lambda'.
// The only exchanges are the four all-gathers; each rank's GEMM is local.
// NCCL is loaded at run time (dlopen), so single-GPU use never touches it.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "context.cuh"

using namespace eigb_capi;
using eigb::cdiv;

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

NcclApi* nccl_api(std::string* why) {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names)
      if ((api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!api.h) {
      err = std::string("NCCL not found: ") + dlerror();
      return;
    }
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(dlsym(api.h, "ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.h, "ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(api.h, "ncclAllGather"));
    api.GetErrorString =
        reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.h, "ncclGetErrorString"));
    api.GetVersion = reinterpret_cast<decltype(api.GetVersion)>(dlsym(api.h, "ncclGetVersion"));
    if (!api.CommInitAll || !api.CommDestroy || !api.AllGather || !api.GetErrorString) {
      err = "NCCL library lacks the required symbols";
      api.h = nullptr;
    }
  });
  if (!api.h) {
    if (why) *why = err;
    return nullptr;
  }
  return &api;
}

#define EIGB_NCCL(api, x)                                                                  \
  do {                                                                                     \
    ncclResult_t r_ = (x);                                                                 \
    if (r_ != ncclSuccess)                                                                 \
      throw ::eigb::Error(3, "nccl", std::string(#x) + ": " + (api)->GetErrorString(r_)); \
  } while (0)

}  // namespace

struct eigmod_b200_multi {
  std::vector<int> devices;
  std::vector<eigmod_b200_ctx*> ctx;
  std::vector<ncclComm_t> comm;
  NcclApi* nccl = nullptr;
  std::string err, stage;
  double stage_ms[4] = {0, 0, 0, 0};  // last call: plan + solve, columns, total, 0
};

namespace {

inline void split_range(int64_t n, int world, int rank, int64_t* lo, int64_t* hi, int64_t* chunk) {
  const int64_t c = n > 0 ? cdiv(n, world) : 0;
  *lo = std::min<int64_t>(n, (int64_t)rank * c);
  *hi = std::min<int64_t>(n, *lo + c);
  *chunk = c;
}

// One rank's share of the update (runs on its own host thread).
void rank_update(eigmod_b200_multi* mg, int g, const double* q, const double* lambda,
                 const double* kmat, const int* signs, int64_t n, int64_t k, double* lambda_out,
                 double* q_out, bool values_only, int64_t* k_eff_out) {
  const int G = (int)mg->devices.size();
  eigmod_b200_ctx* c = mg->ctx[g];
  NcclApi* nc = mg->nccl;
  ncclComm_t comm = mg->comm[g];
  EIGB_CUDA(cudaSetDevice(c->device));
  c->stream = c->own;
  cudaStream_t st = c->stream;
  const int kp = eigb::padded_rank(k);
  int64_t r0, r1, rc;
  split_range(n, G, g, &r0, &r1, &rc);
  // 1. Q replicated: row slice g over PCIe, all-gather over NVLink
  double* dq = c->ws.get_f64("mg_q", (size_t)rc * G * n);
  double* dl = c->ws.get_f64("mg_l", n);
  double* dk = c->ws.get_f64("mg_k", (size_t)n * k);
  if (r1 > r0)
    EIGB_CUDA(cudaMemcpyAsync(dq + r0 * n, q + r0 * n, 8 * (r1 - r0) * n, cudaMemcpyHostToDevice, st));
  EIGB_CUDA(cudaMemcpyAsync(dl, lambda, 8 * n, cudaMemcpyHostToDevice, st));
  EIGB_CUDA(cudaMemcpyAsync(dk, kmat, 8 * n * k, cudaMemcpyHostToDevice, st));
  EIGB_NCCL(nc, nc->AllGather(dq + (size_t)g * rc * n, dq, (size_t)rc * n, ncclDouble, comm, st));
  // 2. U rows of this rank's Q-column slice, all-gathered
  double* u_part = c->ws.get_f64("mg_upart", (size_t)std::max<int64_t>(rc, 1) * kp);
  double* u_all = c->ws.get_f64("mg_uall", (size_t)std::max<int64_t>(rc, 1) * G * kp);
  EIGB_CUDA(cudaMemsetAsync(u_part, 0, 8 * (size_t)std::max<int64_t>(rc, 1) * kp, st));
  if (r1 > r0) project(c, dq, dk, n, k, r0, r1, u_part);
  EIGB_NCCL(nc, nc->AllGather(u_part, u_all, (size_t)rc * kp, ncclDouble, comm, st));
  // 3. plan: groups everywhere, K2 weights by group slice, all-gathered (one
  // device: the one-shot plan, whose solve takes the residues from its count
  // pass, so G = 1 is the single-device path bit for bit)
  eigb::Plan& p = c->plan;
  if (G == 1) {
    plan_from_u(c, dl, u_all, signs, n, k, c->run_rel, true);
    if (k_eff_out) *k_eff_out = p.k;
    if (p.k == 0) return;  // nothing couples: rank 0 copies lambda and Q on the host
  } else {
    plan_groups(c, dl, u_all, signs, n, k, c->run_rel);
    if (k_eff_out && g == 0) *k_eff_out = p.k;
    if (p.k == 0) {  // nothing couples: rank 0 copies lambda and Q on the host
      c->have_plan = true;
      return;
    }
    int64_t g0, g1, gc;
    split_range(p.ng, G, g, &g0, &g1, &gc);
    gc = std::max<int64_t>(gc, 1);
    double* a_part = c->ws.get_f64("mg_apart", gc);
    double* a_all = c->ws.get_f64("mg_aall", (size_t)gc * G);
    EIGB_CUDA(cudaMemsetAsync(a_part, 0, 8 * gc, st));
    if (g1 > g0) eigb::build_plan_weights(p, g0, g1, a_part, c->ws, st);
    EIGB_NCCL(nc, nc->AllGather(a_part, a_all, (size_t)gc, ncclDouble, comm, st));
    EIGB_CUDA(cudaMemcpyAsync(p.alpha, a_all, 8 * p.ng, cudaMemcpyDeviceToDevice, st));
    p.par_mode = c->sopt.plan_par;
    eigb::build_plan_finish(p, c->lam, c->ws, st);
    c->have_plan = true;
  }
  // 4. roots of index slice g, records all-gathered
  const int64_t nred = p.nred;
  int64_t j0, j1, jc;
  split_range(nred, G, g, &j0, &j1, &jc);
  jc = std::max<int64_t>(jc, 1);
  const int w = eigmod_b200_record_width(std::max(p.kp, 1));
  double* rec_part = c->ws.get_f64("mg_rpart", (size_t)jc * w);
  double* rec_all = c->ws.get_f64("mg_rall", (size_t)jc * G * w);
  EIGB_CUDA(cudaMemsetAsync(rec_part, 0, 8 * (size_t)jc * w, st));
  if (nred > 0 && j1 > j0) {
    solve(c, j0, j1);
    pack_records_dev(c, j0, j1 - j0, rec_part);
  }
  EIGB_NCCL(nc, nc->AllGather(rec_part, rec_all, (size_t)jc * w, ncclDouble, comm, st));
  if (nred > 0) unpack_records_dev(c, rec_all, nred);
  // 5. column block g of Q' (D2H overlapped), lambda' from rank 0
  double* dlo = c->ws.get_f64("mg_lo", n);
  int64_t c0, c1, cc;
  split_range(n, G, g, &c0, &c1, &cc);
  if (values_only || c1 <= c0) {
    finish(c, dq, nullptr, 0, 0, dlo, nullptr, n);
  } else {
    double* dqo = c->ws.get_f64("mg_qo", (size_t)n * (c1 - c0));
    finish(c, dq, nullptr, c0, c1, dlo, dqo, c1 - c0, q_out, n);
  }
  if (g == 0) EIGB_CUDA(cudaMemcpyAsync(lambda_out, dlo, 8 * n, cudaMemcpyDeviceToHost, st));
  EIGB_CUDA(cudaStreamSynchronize(st));
}

int multi_run(eigmod_b200_multi* mg, const double* q, const double* lambda, const double* kmat,
              const int* signs, int64_t n, int64_t k, double tol, double* lambda_out,
              double* q_out, double* wall_time_out, bool values_only) {
  if (!mg) return EIGMOD_B200_INVALID_ARGUMENT;
  try {
    check_basic(n, k, signs);
    check_finite(kmat, n * k, "K");
    if (!(tol > 0.0)) throw Error(1, "", "update_eigenvalues: tol must be positive");
    check_ascending(lambda, n);
    if (!q || !lambda || !kmat || !lambda_out || (!values_only && !q_out))
      throw Error(1, "", "update: null pointer");
  } catch (const Error& e) {
    mg->err = e.what();
    mg->stage = e.stage;
    return e.code;
  }
  const auto t0 = std::chrono::steady_clock::now();
  const int G = (int)mg->devices.size();
  std::vector<std::thread> th;
  std::vector<int> rc(G, EIGMOD_B200_OK);
  std::vector<std::string> msg(G), stg(G);
  int64_t k_eff = -1;
  for (int g = 0; g < G; ++g)
    th.emplace_back([&, g] {
      try {
        rank_update(mg, g, q, lambda, kmat, signs, n, k, lambda_out, q_out, values_only, &k_eff);
      } catch (const Error& e) {
        rc[g] = e.code, msg[g] = e.what(), stg[g] = e.stage;
      } catch (const std::exception& e) {
        rc[g] = EIGMOD_B200_CUDA, msg[g] = e.what(), stg[g] = "cuda";
      }
    });
  for (auto& t : th) t.join();
  for (int g = 0; g < G; ++g)
    if (rc[g] != EIGMOD_B200_OK) {
      mg->err = "rank " + std::to_string(g) + ": " + msg[g];
      mg->stage = stg[g];
      return rc[g];
    }
  if (k_eff == 0) {  // rootfind.cpp:394-399: every pair passes through exactly
    std::memcpy(lambda_out, lambda, 8 * n);
    if (!values_only) std::memcpy(q_out, q, 8 * n * n);
  }
  if (wall_time_out)
    *wall_time_out = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  mg->err.clear();
  mg->stage.clear();
  return EIGMOD_B200_OK;
}

}  // namespace

extern "C" {

int eigmod_b200_multi_create(const int* devices, int ndev, eigmod_b200_multi** out) {
  if (!out || !devices || ndev < 1) return EIGMOD_B200_INVALID_ARGUMENT;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return EIGMOD_B200_CUDA;
  for (int i = 0; i < ndev; ++i) {
    if (devices[i] < 0 || devices[i] >= count) return EIGMOD_B200_INVALID_ARGUMENT;
    for (int j = 0; j < i; ++j)
      if (devices[j] == devices[i]) return EIGMOD_B200_INVALID_ARGUMENT;  // one rank per GPU
  }
  std::string why;
  NcclApi* nc = nccl_api(&why);
  if (!nc) return EIGMOD_B200_CUDA;
  auto* mg = new eigmod_b200_multi;
  mg->devices.assign(devices, devices + ndev);
  mg->nccl = nc;
  for (int i = 0; i < ndev; ++i) {
    eigmod_b200_ctx* c = nullptr;
    if (eigmod_b200_ctx_create(devices[i], &c) != EIGMOD_B200_OK) {
      eigmod_b200_multi_destroy(mg);
      return EIGMOD_B200_CUDA;
    }
    mg->ctx.push_back(c);
  }
  mg->comm.resize(ndev);
  if (nc->CommInitAll(mg->comm.data(), ndev, devices) != ncclSuccess) {
    mg->comm.clear();
    eigmod_b200_multi_destroy(mg);
    return EIGMOD_B200_CUDA;
  }
  *out = mg;
  return EIGMOD_B200_OK;
}

void eigmod_b200_multi_destroy(eigmod_b200_multi* mg) {
  if (!mg) return;
  for (auto& cm : mg->comm)
    if (cm && mg->nccl) mg->nccl->CommDestroy(cm);
  for (auto* c : mg->ctx) eigmod_b200_ctx_destroy(c);
  delete mg;
}

int eigmod_b200_multi_size(const eigmod_b200_multi* mg) {
  return mg ? (int)mg->devices.size() : 0;
}

const char* eigmod_b200_multi_last_error(const eigmod_b200_multi* mg) {
  return mg ? mg->err.c_str() : "null context";
}

const char* eigmod_b200_multi_last_stage(const eigmod_b200_multi* mg) {
  return mg ? mg->stage.c_str() : "";
}

int eigmod_b200_multi_set_option(eigmod_b200_multi* mg, const char* key, double value) {
  if (!mg) return EIGMOD_B200_INVALID_ARGUMENT;
  for (auto* c : mg->ctx) {
    const int rc = eigmod_b200_set_option(c, key, value);
    if (rc != EIGMOD_B200_OK) {
      mg->err = eigmod_b200_last_error(c);
      return rc;
    }
  }
  return EIGMOD_B200_OK;
}

int eigmod_b200_multi_update_decomposition(eigmod_b200_multi* mg, const double* q,
                                           const double* lambda, const double* kmat,
                                           const int* signs, int64_t n, int64_t k, double tol,
                                           double* lambda_out, double* q_out,
                                           double* wall_time_out) {
  return multi_run(mg, q, lambda, kmat, signs, n, k, tol, lambda_out, q_out, wall_time_out, false);
}

int eigmod_b200_multi_update_eigenvalues(eigmod_b200_multi* mg, const double* q,
                                         const double* lambda, const double* kmat,
                                         const int* signs, int64_t n, int64_t k, double tol,
                                         double* values_out) {
  return multi_run(mg, q, lambda, kmat, signs, n, k, tol, values_out, nullptr, nullptr, true);
}

int eigmod_b200_split(int64_t n, int world, int rank, int64_t* lo_out, int64_t* hi_out) {
  if (world < 1 || rank < 0 || rank >= world || n < 0 || !lo_out || !hi_out)
    return EIGMOD_B200_INVALID_ARGUMENT;
  int64_t chunk;
  split_range(n, world, rank, lo_out, hi_out, &chunk);
  return EIGMOD_B200_OK;
}

}  // extern "C"
