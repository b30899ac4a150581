"""The drop-in boundary without a GPU: the C-ABI library is built for sm_100a,
loads, exports every entry point include/eigmod_b200.h declares, and fails
loudly (no CPU fallback) when no B200 is present."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "eigmod_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eigmod_b200_\w+)\s*\(", src)))


def test_header_declares_the_reference_entry_points():
    names = declared()
    for n in ("eigmod_b200_transform_update", "eigmod_b200_secular_weights",
              "eigmod_b200_deflate_problem", "eigmod_b200_update_eigenvalues",
              "eigmod_b200_update_decomposition", "eigmod_b200_update_decomposition_device",
              "eigmod_b200_project_device", "eigmod_b200_plan_device",
              "eigmod_b200_solve_device", "eigmod_b200_finish_device"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_1706_00773_b200 import capi

    lib = capi.lib()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (eigmod_b200_\w+)", out))
    assert set(declared()) <= exported


def test_library_is_sm100a_code():
    from paper_1706_00773_b200 import capi

    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", capi.LIB_PATH], capture_output=True,
                          text=True).stdout
    fn = [blk for blk in sass.split("Function : ") if "dmma_gemm_nt_kernel" in blk[:200]]
    assert fn and "DMMA.8x8x4" in fn[0]  # FP64 tensor path of K5


def test_python_binding_matches_header():
    from paper_1706_00773_b200 import capi

    capi.lib()
    assert set(capi.EXPORTED) == set(declared())


def _gpu_present():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_gpu_present(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    import numpy as np

    from paper_1706_00773_b200 import capi

    with pytest.raises(capi.DeviceError):
        capi.Context(0)
    with pytest.raises(capi.DeviceError):
        capi.update_decomposition(np.eye(2), np.array([0.0, 1.0]), np.eye(2), [1, 1], 1e-12)


def test_host_argument_validation_precedes_device_use():
    # proj/src/core.cpp:89-97 semantics are enforced before any device work:
    # a dimension mismatch is a ValueError even without a GPU.
    import numpy as np

    from paper_1706_00773_b200 import capi

    with pytest.raises(ValueError):
        capi._check_update(np.eye(2), np.array([0.0, 1.0]), np.zeros((3, 1)),
                           np.array([1], np.int32))
    with pytest.raises(ValueError):
        capi._check_update(np.eye(2), np.array([0.0, 1.0]), np.zeros((2, 2)),
                           np.array([1], np.int32))
