"""One launch of the K5 DMMA GEMM (for ncu captures): python tools/gemm_one.py [n]."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1706_00773_b200 import capi
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dev = torch.device('cuda', 0)
ctx = capi.Context(0)
ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
a = torch.randn(n, n, dtype=torch.float64, device=dev)
b = torch.randn(n, n, dtype=torch.float64, device=dev)
c = torch.empty(n, n, dtype=torch.float64, device=dev)
capi.gemm_nt_device(a, b, c, ctx=ctx)
torch.cuda.synchronize()
print('ok', float(c[0, 0]))
