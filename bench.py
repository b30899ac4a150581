#!/usr/bin/env python
"""Benchmark: updated eigenpairs/sec (FP64) of the rank-k eigen-update.

Workload (BASELINE.json configs[4], the n = 32768 configuration the scaling
target is quoted on; it fits one B200): rank-16 update, n = 32768, FP64,
Lambda ~ sort(U[-100,100]), K ~ N(0,1/n), alternating signs, Q random
orthogonal (8.6 GB). One "step" = one full update (U = Q^T K, deflation, all
n roots, eigenvector columns, Q' = Q X with the sign rule).

  value  device throughput: n / step time, inputs resident in HBM, CUDA
         events on the launching stream, max over ranks (inputs 8.6 GB >
         L2, no flush needed).
  e2e    the same update through the host-pointer C ABI
         (eigmod_b200_update_decomposition) from pinned host memory: H2D of
         Q, lambda, K and D2H of Q', lambda' inside the timed region.

N > 1 (torchrun, one process per GPU, NCCL): Q is replicated (broadcast once
before timing); each rank projects its slice of U and all-gathers it, plans
redundantly, solves its slice of root indices and all-gathers the root
records, then writes its column block of Q' (strong scaling: n fixed).

--impl reference times the reference's own CPU implementation
(oracle/_ref, the unmodified eigmod sources) on the host cores; see DESIGN.md.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "updated eigenpairs/sec (FP64, n,k) at 1/2/4/8 B200; % of FP64 roofline"
UNIT = "eigenpairs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int, default=None, help="override n (smaller smoke runs)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU (ShardedUpdate) path even on one rank")
    ap.add_argument("--no-ref-single-thread", dest="ref_single_thread", action="store_false",
                    help="reference arm: skip the single-thread (reference default) mode")
    ap.add_argument("--selftest-launch", action="store_true",
                    help="exercise the --gpus N launcher on CPU (gloo); no GPU work")
    return ap.parse_args()


# ------------------------------------------------------------- launcher
def _free_port():
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_command(gpus, argv):
    """The torchrun command that runs this script as `gpus` ranks (one
    process per GPU) when it was started as a plain `python bench.py --gpus N`."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1",
            f"--master-port={_free_port()}", os.path.abspath(__file__), *argv]


def nccl_env(env):
    """NCCL's INIT lines (communicator size, ranks, transports) on stderr, so
    the N-rank communicator is visible next to the JSON line on stdout."""
    env = dict(env)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    return env


def maybe_relaunch(args):
    """--gpus N > 1 outside torchrun: re-exec as N ranks; returns True when
    this process only supervised the launch."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    rc = subprocess.call(launch_command(args.gpus, sys.argv[1:]), env=nccl_env(os.environ))
    sys.exit(rc)


def selftest_launch(args):
    """CPU stand-in for the N-rank path: gloo process group, one rank per
    process, the same rank/world checks and max-over-ranks reduction."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    assert world == args.gpus, (world, args.gpus)
    dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"selftest": True, "n_gpus": world, "max_over_ranks": float(t.item()),
                          "nccl_debug": os.environ.get("NCCL_DEBUG")}), flush=True)
    dist.destroy_process_group()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ------------------------------------------------------------ CPU baseline
def _instance_host(cfg, n, seed=None):
    """The seeded instance on the host: numpy for n <= 8192, the GPU generator
    (cuSOLVER QR, same distributions) above that when a GPU is present."""
    from paper_1706_00773_b200.instances import make_instance, make_instance_torch

    if n <= 8192:
        return make_instance(cfg, n=n, seed=seed)
    import torch

    if not torch.cuda.is_available():
        return make_instance(cfg, n=n, seed=seed)
    q, lam, kmat, signs = make_instance_torch(cfg, n=n, seed=seed, device="cuda")
    out = (q.cpu().numpy(), lam.cpu().numpy(), kmat.cpu().numpy(), signs.numpy())
    del q
    torch.cuda.empty_cache()
    return out


def reference_config_run(cfg, n, modes=("omp", "1t"), repeats=3, long_s=20.0, seed=None):
    """BASELINE.md §3 / SURVEY §8(d): the unmodified reference (oracle/_ref)
    on the full pipeline of one config: update_eigenvalues_full and
    assemble_eigenvectors timed separately (steady_clock), one warm-up + the
    median of `repeats` (bench.cpp:188-222), in the reference's default
    single-thread mode ("1t", kernels::set_parallel(false)) and with OpenMP on
    all host cores ("omp"). A stage that throws is reported with its stage
    and time to failure instead of a throughput; a warm-up longer than
    `long_s` is not repeated (reported as measured once)."""
    from oracle import ref

    q, lam, kmat, signs = _instance_host(cfg, n, seed)
    tol = ref.default_tolerance(lam, kmat, signs)
    ref.set_threads(os.cpu_count())
    out = {}
    for mode in modes:
        ref.set_parallel(mode == "omp")
        runs = [ref.timed_pairs(q, lam, kmat, signs, tol)]
        r0 = runs[0]
        if not r0["failed_stage"] and r0["t_eig"] + r0["t_vec"] < long_s:
            runs = [ref.timed_pairs(q, lam, kmat, signs, tol) for _ in range(repeats)]
        r = {"threads": ref.worker_count(), "repeats": len(runs) if len(runs) > 1 else 1}
        if r0["failed_stage"]:
            r.update(failed_stage=r0["failed_stage"], error=r0["error"][:160],
                     t_eig_s=r0["t_eig"], t_vec_s=r0["t_vec"])
            if r0["failed_stage"] == "eigenvectors":
                r["eigenvalues_per_s"] = n / r0["t_eig"]
            r["value"] = None
        else:
            te = statistics.median(x["t_eig"] for x in runs)
            tv = statistics.median(x["t_vec"] for x in runs)
            r.update(t_eig_s=te, t_vec_s=tv, value=n / (te + tv))
        out[mode] = r
    ref.set_parallel(False)
    return out


def reference_pair_sample(n=32768, k=16, m=8, steps=3, warmup=1, seed=11, parallel=True,
                          rows=None, weights=None):
    """The unmodified reference (oracle/_ref) on a bounded sample of the SAME
    workload (config 4: n = 32768, k = 16, Lambda ~ U[-100,100], alternating
    signs). Its full pipeline cannot run at this size (the locate stage throws
    at n >= 8192), so each step times its own per-eigenpair
    code on the n = 32768 problem:
      * m eigenpairs: dnc_solve (rootfind.cpp:89-229) on the root's pole
        interval with the reference's secular weights (brackets from our CPU
        oracle's inertia count, standing in for the failing locate stage),
        then null_problem + null_direction + resolvent (eigvec.cpp:133-153,
        157-202);
      * `rows` rows of the back-transform Q' = Q X with kernels::gemm_nn
        (kernels.cpp:32-48, eigvec.cpp:339) against the FULL n x n X: the
        i-l-j kernel streams all of X once per output row, so one row costs
        exactly 1/n of the full n^3 GEMM, i.e. one eigenpair's share;
    plus the per-pair share of secular_weights (secular.cpp:168-202, O(n^2 k^2),
    timed once). Rate = 1 / (t_pairs/m + t_rows/rows + t_alpha/n). The
    eigenvalue stage enters only through dnc_solve, so the rate is an upper
    bound for the reference."""
    from oracle import port, ref

    rng = np.random.default_rng(seed)
    lam = np.sort(rng.uniform(-100.0, 100.0, n))
    u = rng.normal(0.0, 1.0 / np.sqrt(n), (n, k))  # distribution of Q^T K
    signs = np.array([1 if r % 2 == 0 else -1 for r in range(k)], np.int32)
    ref.set_threads(os.cpu_count())
    ref.set_parallel(parallel)
    cores = ref.worker_count()
    rows = rows or cores
    hx = ref.matrix_const(n, n, 1.0 / np.sqrt(n))        # dense X (n x n)
    hq = ref.matrix(rng.normal(0.0, 1.0 / np.sqrt(n), (rows, n)))  # sampled rows of Q
    tu = ref.transformed(u, signs)
    if weights is None:
        t0 = time.perf_counter()
        alpha = ref.secular_weights(lam, u, signs)
        t_alpha, alpha_note = time.perf_counter() - t0, "once"
    else:  # (alpha, seconds) from another run: the weights do not depend on threading
        alpha, t_alpha = weights
        alpha_note = "extrapolated: the OpenMP time x threads"
    tol = 1e-12 * max(100.0, float((u * u).sum()))  # default_tolerance (rootfind.cpp:306-312)
    brackets = []  # m sample pole intervals holding exactly one root
    for a in np.linspace(n // 10, n - n // 10, 4 * m).astype(int):
        lo, hi = lam[a] + 1e-9 * 100, lam[a + 1] - 1e-9 * 100
        c0, c1 = port.count_below(lam, u, signs, lo), port.count_below(lam, u, signs, hi)
        if c1 - c0 == 1:
            brackets.append((lo, hi))
        if len(brackets) == m:
            break
    x = np.empty((n, len(brackets)))
    t_pairs, t_rows = [], []
    for it in range(warmup + steps):
        t1 = time.perf_counter()
        for c, (lo, hi) in enumerate(brackets):
            root = ref.dnc_solve(lam, alpha, lo, hi, 1, tol)[0]
            x[:, c], _ = ref.basis_vector(tu, lam, root)
        t2 = time.perf_counter()
        ref.gemm_nn_hh(hq, hx, rows, n)
        t3 = time.perf_counter()
        if it >= warmup:
            t_pairs.append(t2 - t1)
            t_rows.append(t3 - t2)
    del hx
    ref.set_parallel(False)
    tp, tr = statistics.median(t_pairs), statistics.median(t_rows)
    per_pair = tp / len(brackets) + tr / rows + t_alpha / n
    gemm_gfs = 2.0 * n * n * rows / tr / 1e9
    sample = (f"unmodified reference (oracle/_ref) on the n={n} k={k} config-4 problem, per "
              f"step: dnc_solve + null_problem/null_direction for {len(brackets)} eigenpairs "
              f"({tp * 1e3:.1f} ms) and {rows} rows of kernels::gemm_nn Q X against the full "
              f"n x n X ({tr:.2f} s, {gemm_gfs:.1f} GF/s; one row = one eigenpair's share of "
              f"the n^3 GEMM), median of {steps}; + secular_weights/n ({t_alpha:.1f} s "
              f"{alpha_note}); "
              f"{'OpenMP' if parallel else 'single-thread'} {cores} thread(s); upper bound "
              f"(its locate stage throws at this size)")
    return {"value": 1.0 / per_pair, "t_step": tp + tr, "cores": cores, "sample": sample,
            "weights": (alpha, t_alpha),
            "gemm_gflops": gemm_gfs, "per_pair_ms": {"solve_vector": tp / len(brackets) * 1e3,
                                                      "gemm_row": tr / rows * 1e3,
                                                      "weights": t_alpha / n * 1e3}}


def reference_small_n(n=2048):
    """Full reference pipeline where it still completes (config-4 family at
    n = 2048): update_eigenvalues_full + assemble_eigenvectors."""
    from oracle import ref
    from paper_1706_00773_b200.instances import make_instance

    q, lam, kmat, signs = make_instance(4, n=n, seed=11)
    ref.set_parallel(True)
    tol = ref.default_tolerance(lam, kmat, signs)
    ref.update_pairs(q, lam, kmat, signs, tol)
    t0 = time.perf_counter()
    ref.update_pairs(q, lam, kmat, signs, tol)
    return n / (time.perf_counter() - t0)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref

    ref.set_threads(os.cpu_count())  # torchrun exports OMP_NUM_THREADS=1
    from paper_1706_00773_b200.instances import CONFIGS

    cfg = CONFIGS[args.config]
    n = args.n or cfg["n"]
    line = {
        "metric": METRIC, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
    }
    if args.config == 4 and n > 4096:
        r = reference_pair_sample(n=n, k=cfg["k"], steps=args.steps, warmup=args.warmup)
        v = r["value"]
        line.update(value=v, ms_per_step=r["t_step"] * 1e3,
                    config={"workload": cfg["name"], "n": n, "k": cfg["k"],
                            "sample": "per step: 8 eigenpairs' solve+vector and "
                                      f"{r['cores']} rows of the full Q X (bounded sample)"},
                    per_pair_ms=r["per_pair_ms"], gemm_gflops=r["gemm_gflops"])
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": r["cores"],
                                "kind": "reference", "sample": r["sample"]}
        if args.ref_single_thread:
            alpha, t_alpha = r["weights"]
            r1 = reference_pair_sample(n=n, k=cfg["k"], steps=1, warmup=0, parallel=False,
                                       rows=2, weights=(alpha, t_alpha * r["cores"]))
            line["single_thread"] = {"value": r1["value"], "unit": UNIT,
                                     "per_pair_ms": r1["per_pair_ms"], "sample": r1["sample"]}
        try:
            line["reference_full_pipeline_n2048"] = {"value": reference_small_n(), "unit": UNIT}
        except Exception as e:
            line["reference_full_pipeline_n2048"] = {"value": None, "error": str(e)[:200]}
    else:
        # the full pipeline of configs 0-3 (and config 4 at n <= 4096)
        modes = ("omp", "1t") if args.ref_single_thread else ("omp",)
        res = reference_config_run(args.config, n, modes=modes)
        omp = res["omp"]
        v = omp["value"]
        line.update(value=v, ms_per_step=(omp["t_eig_s"] + (omp["t_vec_s"] or 0.0)) * 1e3,
                    config={"workload": cfg["name"], "n": n, "k": cfg["k"],
                            "sample": "full pipeline, 1 warm-up + median of 3 per stage"},
                    stages=res)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": omp["threads"],
                                "kind": "reference",
                                "sample": "update_eigenvalues_full + assemble_eigenvectors, "
                                          "timed separately (see stages)"}
    line["e2e"] = {"value": line["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}
    line["host"] = {"nproc": os.cpu_count(), "cpu": _cpu_model()}
    print(json.dumps(line), flush=True)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# --------------------------------------------------------------- our arm
def fp64_peaks_measured(torch, dev, ctx):
    """Live FP64 roofline denominators: the DMMA.8x8x4 tensor-pipe loop and
    the DFMA loop (library kernels), plus cuBLAS DGEMM 16384^3 for context
    (MEASURED_PEAKS.json has no FP64 entry)."""
    pk = ctx.fp64_peaks()
    n = 16384
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(2):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    pk["cublas_dgemm_16384_tflops"] = 2.0 * n ** 3 / (best * 1e-3) / 1e12
    return pk


def _hbm_peak():
    """MEASURED_PEAKS.json hbm_gbs (driver-written), else the profiling
    recipe's fallback (6.65 TB/s)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def _ncu_gemm_traffic(n):
    """dram__bytes_read.sum + dram__bytes_write.sum of one K5 launch from the
    committed ncu --set full capture (profiles/ncu_full_k5_cfg4_n32768_r02.json,
    tools/gemm_one.py 32768), when this run has that n; else None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                        "ncu_full_k5_cfg4_n32768_r02.json")
    if n != 32768 or not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f).get("gemm_traffic_bytes_per_launch")


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1706_00773_b200 import capi
    from paper_1706_00773_b200.instances import CONFIGS, make_instance_torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks need {world} GPUs, "
                         f"{torch.cuda.device_count()} visible")
    os.environ.update(nccl_env(os.environ))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or args.sharded
    if sharded:
        if "MASTER_ADDR" not in os.environ:  # --sharded outside torchrun: a 1-rank group
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0",
                              WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=dev)

    cfg = CONFIGS[args.config]
    n = args.n or cfg["n"]
    k = cfg["k"]
    # instance: rank 0 generates, Q is replicated by NCCL broadcast (before timing)
    if rank == 0:
        q, lam, kmat, signs = make_instance_torch(args.config, n=n, device=dev)
    else:
        q = torch.empty((n, n), dtype=torch.float64, device=dev)
        lam = torch.empty(n, dtype=torch.float64, device=dev)
        kmat = torch.empty((n, k), dtype=torch.float64, device=dev)
        signs = torch.tensor(cfg["signs"], dtype=torch.int32)
    if world > 1:
        for t in (q, lam, kmat):
            dist.broadcast(t, 0)
    signs_np = signs.numpy().astype(np.int32)
    torch.cuda.synchronize()

    ctx = capi.Context(local)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    ctx.set_option("timing", 1.0)
    lam_out = torch.empty(n, dtype=torch.float64, device=dev)

    if not sharded:
        q_out = torch.empty((n, n), dtype=torch.float64, device=dev)

        def step():
            capi.update_decomposition_device(q, lam, kmat, signs_np, lam_out, q_out, ctx=ctx)
    else:
        from paper_1706_00773_b200.sharded import ShardedUpdate

        shard = ShardedUpdate(ctx, n, k, signs_np, rank, world, dev)
        q_out = shard.alloc_output()

        def step():
            shard.run(q, lam, kmat, lam_out, q_out)

    # inputs smaller than L2 (Q below 256 MB: configs 0-1) are timed step by
    # step with a 512 MB write between steps that evicts L2 (not timed)
    flush = None if 8 * n * n >= (256 << 20) else torch.empty(64 << 20, dtype=torch.float64,
                                                                device=dev)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ctx.stage_times(reset=True)
    launches0 = capi.launch_count()
    if sharded:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps if flush is not None else 1)]
    with ClockSampler(local) as clk:
        if flush is None:
            evs[0][0].record()
            for _ in range(args.steps):
                step()
            evs[0][1].record()
        else:
            for e0, e1 in evs:
                flush.fill_(1.0)
                e0.record()
                step()
                e1.record()
        torch.cuda.synchronize()
    if sharded:
        dist.barrier()
    launches = capi.launch_count() - launches0
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if sharded:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    stages = ctx.stage_times()
    stats = ctx.stats()

    out = {}
    if rank == 0:
        value = n / (ms * 1e-3)
        calls = max(1, stages["calls"])
        gemm_ms = stages["k5_gemm"] / calls
        cols = shard.ncols_local if sharded else n
        # compact back-transform (plans with >= 64 decoupled columns, kp >= 4;
        # capi.cu finish_compact): the GEMM runs over the nred reduced rows
        # and the root columns only, 2 n nred * (roots among the columns)
        nred, ndec = stats["roots"], stats["decoupled"]
        compact = ndec >= 64 and int(stats["kp"]) >= 4
        gemm_cols = cols * nred / n if compact else cols
        gemm_flops = 2.0 * n * (nred if compact else n) * gemm_cols
        peaks = fp64_peaks_measured(torch, dev, ctx)
        peak = peaks["dmma_tflops"]
        achieved = gemm_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
        solve_ms = stages["k3_solve"] / calls
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; Q from a GPU QR of a Philox N(0,1) matrix)",
            "config": {"workload": cfg["name"], "n": n, "k": k, "signs": list(cfg["signs"]),
                       "parallelism": f"roots+columns x{world}" + (" (sharded path)" if sharded else ""),
                       "l2": (f"inputs ({8 * n * n / 1e9:.2f} GB Q) exceed L2; no flush"
                              if flush is None else "L2 flushed (512 MB write) between steps, "
                              "per-step CUDA events")},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "stage_ms": {kk: round(v / calls, 3) for kk, v in stages.items() if kk != "calls"},
            "solver": {"roots": stats["roots"], "evals_per_root":
                       stats["evals"] / max(1.0, stats["roots"]), "max_evals": stats["max_evals"]},
            "roofline": {"kernel": ("K5 dmma_gemm_nt_kernel (Q' = Q X, DMMA.8x8x4)" if not compact
                                    else "K5 dmma_gemm_nt_kernel (Q'[:, roots] = Q~_red X_red, "
                                         "DMMA.8x8x4; compact: 2 n nred^2 flops)"),
                         "bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": (achieved / peak) if achieved else None,
                         "peak_source": "DMMA.8x8x4 tensor-pipe loop measured live in this run "
                                        "(MEASURED_PEAKS.json has no FP64 entry)",
                         "measured_peaks": peaks,
                         "algorithmic_flops_per_launch": gemm_flops,
                         "traffic": _ncu_gemm_traffic(n)},
        }
        if world > 1:
            out["config"]["q_replication"] = ("Q, lambda, K broadcast by NCCL from rank 0 once, "
                                              "before warm-up (outside the timed region)")
        # CPU secular-solver roofline (K3): algorithmic flops per S evaluation
        kp = int(stats["kp"]) or 1
        fl_eval = n * (k * (k + 1) + 1)
        # S evaluations of the stage: the solver's (records) and the bracket
        # counts, one pole-limit inertia evaluation per reduced pole value
        # (one pole pass each); the scalar f presolve is not counted
        ev_total = stats["evals"] + stats["roots"]
        out["roofline_k3"] = {
            "bound": "fp64", "evals": ev_total, "evals_solver": stats["evals"],
            "evals_counts": stats["roots"],
            "achieved": ev_total * fl_eval / (solve_ms * 1e-3) / 1e12 if solve_ms else None,
            "peak": peaks["dfma_tflops"], "unit": "TFLOP/s",
            "note": f"n*(k(k+1)+1) flops per S(x) evaluation (solver + one pole-limit count per pole), kp={kp}"}
        if out["roofline_k3"]["achieved"]:
            out["roofline_k3"]["frac"] = out["roofline_k3"]["achieved"] / peaks["dfma_tflops"]
            out["roofline_k3"]["frac_vs_dmma_peak"] = (out["roofline_k3"]["achieved"]
                                                       / peaks["dmma_tflops"])
        # HBM-bound stages: K1 (8 B per Q entry read, + K and U) and K4 (the
        # Xt workspace written, 8 B per entry)
        hbm, hbm_src = _hbm_peak()
        k1_cols = (shard.u_hi - shard.u_lo) if sharded else n
        # compact: Xt_red written (nred per root column), Q read once by the
        # gather, Q~_red and the decoupled columns of Q' written
        k4_bytes = (8.0 * (nred * gemm_cols + n * n + n * (nred + cols - gemm_cols)) if compact
                    else 8.0 * n * cols)
        for key, stage, nbytes in (("roofline_k1", "k1_project", 8.0 * (n * k1_cols + 2 * n * k)),
                                   ("roofline_k4", "k4_columns", k4_bytes)):
            t = stages[stage] / calls
            if t > 0:
                a = nbytes / (t * 1e-3) / 1e9
                out[key] = {"bound": "hbm", "achieved": a, "peak": hbm, "unit": "GB/s",
                            "frac": a / hbm, "peak_source": hbm_src,
                            "algorithmic_bytes": nbytes,
                            "note": "stage time (CUDA events), all kernels of the stage"}
    # ---- e2e at N GPUs: host inputs -> every rank copies its 1/N row slice
    # of Q (pinned) and the small lambda, K; Q is reassembled by an NCCL
    # all-gather over NVLink; each rank copies its Q' column block and rank 0
    # lambda' back to pinned host memory. Max over ranks of CUDA-event time.
    if sharded and not args.no_e2e:
        del q_out
        torch.cuda.empty_cache()
        from paper_1706_00773_b200.sharded import split

        r0, r1, ch = split(n, world, rank)
        h_qs = torch.zeros((ch, n), dtype=torch.float64, pin_memory=True)
        h_qs[: r1 - r0].copy_(q[r0:r1])
        h_lam = lam.cpu().pin_memory()
        h_k = kmat.cpu().pin_memory()
        d_slice = torch.empty((ch, n), dtype=torch.float64, device=dev)
        d_qall = torch.empty((ch * world, n), dtype=torch.float64, device=dev)
        d_lam = torch.empty_like(lam)
        d_k = torch.empty_like(kmat)
        del q
        torch.cuda.empty_cache()
        q_blk = shard.alloc_output()
        h_qo = torch.empty((n, max(shard.ncols_local, 1)), dtype=torch.float64, pin_memory=True)
        h_lo = torch.empty(n, dtype=torch.float64, pin_memory=True)

        def e2e_step():
            d_slice.copy_(h_qs, non_blocking=True)
            d_lam.copy_(h_lam, non_blocking=True)
            d_k.copy_(h_k, non_blocking=True)
            dist.all_gather_into_tensor(d_qall, d_slice)
            shard.run(d_qall[:n], d_lam, d_k, lam_out, q_blk)
            h_qo.copy_(q_blk, non_blocking=True)
            if rank == 0:
                h_lo.copy_(lam_out, non_blocking=True)

        for _ in range(max(1, min(args.warmup, 2))):
            e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            e2e_step()
        f1.record()
        torch.cuda.synchronize()
        te_t = torch.tensor([f0.elapsed_time(f1) / args.steps], dtype=torch.float64, device=dev)
        dist.all_reduce(te_t, op=dist.ReduceOp.MAX)
        te = float(te_t.item()) * 1e-3
        if rank == 0:
            out["e2e"] = {"value": n / te, "unit": UNIT,
                          "h2d_bytes_per_step": 8 * (ch * world * n + world * (n + n * k)),
                          "d2h_bytes_per_step": 8 * (n * n + n),
                          "ms_per_step": te * 1e3,
                          "path": "per-rank 1/N row slice of Q H2D + NCCL all-gather, "
                                  "ShardedUpdate, column blocks D2H (pinned)"}
    # ---- e2e through the host-pointer C ABI (single GPU)
    if not sharded and not args.no_e2e:
        h_q = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        h_q.copy_(q)
        h_lam = lam.cpu().numpy()
        h_k = kmat.cpu().numpy()
        h_qo = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        h_lo = np.empty(n)
        del q_out
        torch.cuda.empty_cache()
        import ctypes as C

        qp = C.cast(h_q.data_ptr(), capi._D)
        qop = C.cast(h_qo.data_ptr(), capi._D)
        ectx = capi.Context(local)
        sg = np.ascontiguousarray(signs_np)

        def e2e_step():
            wt = np.zeros(1)
            ectx.check(ectx._l.eigmod_b200_update_decomposition(
                ectx.h, qp, capi._dp(np.ascontiguousarray(h_lam)), capi._dp(np.ascontiguousarray(h_k)),
                sg.ctypes.data_as(capi._I32), n, k, C.c_double(1e-12), capi._dp(h_lo), qop,
                capi._dp(wt)))
            return wt[0]

        for _ in range(max(1, min(args.warmup, 2))):
            e2e_step()
        ts = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            e2e_step()
            ts.append(time.perf_counter() - t0)
        te = statistics.mean(ts)
        out["e2e"] = {"value": n / te, "unit": UNIT,
                      "h2d_bytes_per_step": 8 * (n * n + n + n * k),
                      "d2h_bytes_per_step": 8 * (n * n + n),
                      "ms_per_step": te * 1e3,
                      "path": "eigmod_b200_update_decomposition (host pointers, pinned)"}
        ectx.close()
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        try:
            if args.config == 4 and n > 4096:
                r = reference_pair_sample(n=n, k=k, steps=2, warmup=1)
                out["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": r["cores"],
                                       "kind": "reference", "sample": r["sample"]}
            else:
                r = reference_config_run(args.config, n, modes=("omp",), repeats=1)["omp"]
                out["cpu_baseline"] = {
                    "value": r["value"], "unit": UNIT, "cores": r["threads"], "kind": "reference",
                    "sample": "full pipeline of this config (1 warm-up + 1 timed run): "
                              "update_eigenvalues_full + assemble_eigenvectors",
                    "stages": r}
        except Exception as e:  # the baseline is reported, never required
            out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(),
                                   "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if sharded:
        dist.destroy_process_group()


def main():
    args = parse()
    maybe_relaunch(args)
    if args.selftest_launch:
        selftest_launch(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
