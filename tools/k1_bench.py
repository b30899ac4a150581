"""K1 (U = Q^T K) timing at BASELINE config 4 (n = 32768, k = 16) through the
staged C ABI (eigmod_b200_project_device), CUDA events on the launching
stream: algorithmic bytes 8(n^2 + 2nk) per launch vs the measured HBM copy
bandwidth. EIGMOD_B200_K1=fma selects the DFMA kernel."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1706_00773_b200 import capi  # noqa: E402
from paper_1706_00773_b200.sharded import CudaBackend  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn((n, n), generator=g, dtype=torch.float64, device=dev)
    km = torch.randn((n, k), generator=g, dtype=torch.float64, device=dev)
    ctx = capi.Context(0)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    be = CudaBackend(ctx, n, k, [1] * k)
    u = torch.zeros((n, be.kp), dtype=torch.float64, device=dev)
    for _ in range(3):
        be.project(q, km, 0, n, u)
    torch.cuda.synchronize()
    ref = (q.T @ km)
    err = float((u[:, :k] - ref).abs().max() / ref.abs().max())
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        be.project(q, km, 0, n, u)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nbytes = 8.0 * (n * n + 2 * n * k)
    print(json.dumps({"kernel": os.environ.get("EIGMOD_B200_K1", "dmma"), "n": n, "k": k,
                      "ms": ms, "GBps": nbytes / ms / 1e6, "frac_of_6456.8": nbytes / ms / 1e6 / 6456.8,
                      "rel_err_vs_torch": err}), flush=True)


if __name__ == "__main__":
    main()
