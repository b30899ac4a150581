"""K5 DMMA GEMM vs cuBLAS DGEMM (torch.matmul) on the back-transform shape."""
import os, sys, json
sys.path.insert(0, '.')
import torch
from paper_1706_00773_b200 import capi
dev = torch.device('cuda', 0)
ctx = capi.Context(0)
ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
res = {}
for n in [int(x) for x in (sys.argv[1:] or ['8192', '16384'])]:
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    c = torch.empty(n, n, dtype=torch.float64, device=dev)
    def t(f, reps=3):
        f(); torch.cuda.synchronize(); best = 1e30
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    ours = t(lambda: capi.gemm_nt_device(a, b, c, ctx=ctx))
    ref = torch.matmul(a, b.T)
    err = (c - ref).abs().max().item() / ref.abs().max().item()
    cub = t(lambda: torch.matmul(a, b.T))
    res[n] = dict(ours_tflops=ours, cublas_tflops=cub, rel_err=err)
    print(n, res[n], flush=True)
print(json.dumps(res))
