"""The C++ drop-in: the reference's own test cases, restated in
tests/cxx/test_dropin.cpp with the reference's #include lines and calls,
compile and link against lib/libeigmod_b200_cxx.so (CPU) and pass (B200)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1706_00773_b200", "lib")
SRC = os.path.join(ROOT, "tests", "cxx", "test_dropin.cpp")
SRC_EXT = os.path.join(ROOT, "tests", "cxx", "test_dropin_ext.cpp")


def _build(tmp_path, src=SRC):
    exe = str(tmp_path / os.path.splitext(os.path.basename(src))[0])
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", exe,
                    "-L", LIB, "-leigmod_b200_cxx", "-leigmod_b200", f"-Wl,-rpath,{LIB}"],
                   check=True, capture_output=True, text=True)
    return exe


def test_dropin_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)
    out = subprocess.run(["nm", "-DC", os.path.join(LIB, "libeigmod_b200_cxx.so")],
                         capture_output=True, text=True, check=True).stdout
    for fn in ("eigmod::update_decomposition", "eigmod::update_eigenvalues_full",
               "eigmod::assemble_eigenvectors", "eigmod::transform_update",
               "eigmod::deflate_problem", "eigmod::secular_weights",
               # the rest of the reference's public API (eigvec.hpp:15-25,
               # rootfind.hpp:28-33, secular.hpp:48, locate.hpp:31,50,
               # kernels.hpp:19-50) and the multi-GPU extension
               "eigmod::null_direction", "eigmod::null_problem", "eigmod::update_eigenvector",
               "eigmod::dnc_solve", "eigmod::solve_rank1", "eigmod::crossing_count",
               "eigmod::locate_rank2", "eigmod::locate_rank_k", "eigmod::kernels::gemm_nn",
               "eigmod::kernels::gemm_tn", "eigmod::kernels::gemm_nt", "eigmod::kernels::gemv_t",
               "eigmod::kernels::ref::gemm_nn", "eigmod::set_devices"):
        assert fn in out, fn
    assert os.path.exists(_build(tmp_path, SRC_EXT))


@pytest.mark.gpu
def test_dropin_reference_cases_pass(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_dropin_extended_api_passes(tmp_path):
    exe = _build(tmp_path, SRC_EXT)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


def test_dropin_without_gpu_fails_loudly(tmp_path):
    """No CPU fallback: without a B200 the extended API throws (std::runtime_error
    from the device layer), it never computes on the host."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    exe = _build(tmp_path, SRC_EXT)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0
