"""Which independent FP64 eigensolver runs at n = 32768 on one B200?
torch.linalg.eigvalsh (cusolverDnXsyevd) rejects n = 32768 with
CUSOLVER_STATUS_INVALID_VALUE in its bufferSize call; try the legacy 32-bit
cusolverDnDsyevd through ctypes and torch's MAGMA backend."""
import ctypes as C
import glob
import os
import sys
import time

import torch


def cusolver_lib():
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cusolver",
                                   "lib", "libcusolver.so*"))
    cands += ["/usr/local/cuda/lib64/libcusolver.so"]
    for c in cands:
        try:
            return C.CDLL(c), c
        except OSError:
            pass
    raise OSError("no libcusolver")


def legacy_dsyevd(a):
    """eigenvalues of the symmetric (row-major = column-major) float64 CUDA
    tensor a via cusolverDnDsyevd (jobz N, lower); a is overwritten."""
    lib, path = cusolver_lib()
    n = a.shape[0]
    h = C.c_void_p()
    assert lib.cusolverDnCreate(C.byref(h)) == 0
    st = torch.cuda.current_stream().cuda_stream
    lib.cusolverDnSetStream(h, C.c_void_p(st))
    w = torch.empty(n, dtype=torch.float64, device=a.device)
    lwork = C.c_int(0)
    rc = lib.cusolverDnDsyevd_bufferSize(h, 0, 0, n, C.c_void_p(a.data_ptr()), n,
                                         C.c_void_p(w.data_ptr()), C.byref(lwork))
    if rc != 0:
        raise RuntimeError(f"bufferSize rc={rc}")
    work = torch.empty(max(1, lwork.value), dtype=torch.float64, device=a.device)
    info = torch.zeros(1, dtype=torch.int32, device=a.device)
    rc = lib.cusolverDnDsyevd(h, 0, 0, n, C.c_void_p(a.data_ptr()), n, C.c_void_p(w.data_ptr()),
                              C.c_void_p(work.data_ptr()), lwork, C.c_void_p(info.data_ptr()))
    torch.cuda.synchronize()
    lib.cusolverDnDestroy(h)
    if rc != 0 or int(info.item()) != 0:
        raise RuntimeError(f"syevd rc={rc} info={int(info.item())}")
    return w, path, lwork.value


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn((n, n), generator=g, dtype=torch.float64, device="cuda")
    a += a.T.clone()
    ref_tr = float(a.diagonal().sum())
    out = {"n": n}
    for name in ("legacy", "magma", "default"):
        b = a.clone()
        t0 = time.time()
        try:
            if name == "legacy":
                w, path, lw = legacy_dsyevd(b)
                out["legacy_lib"] = path
                out["legacy_lwork"] = lw
            else:
                torch.backends.cuda.preferred_linalg_library(name)
                w = torch.linalg.eigvalsh(b)
            torch.cuda.synchronize()
            out[name] = {"ok": True, "s": time.time() - t0,
                         "trace_err": abs(float(w.sum()) - ref_tr) / abs(ref_tr)}
        except Exception as e:  # noqa: BLE001
            out[name] = {"ok": False, "err": str(e)[:300]}
        del b
        torch.cuda.empty_cache()
        print(out, flush=True)


if __name__ == "__main__":
    main()
