"""The C++ drop-in: the reference's own test cases, restated in
tests/cxx/test_dropin.cpp with the reference's #include lines and calls,
compile and link against lib/libeigmod_b200_cxx.so (CPU) and pass (B200)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1706_00773_b200", "lib")
SRC = os.path.join(ROOT, "tests", "cxx", "test_dropin.cpp")


def _build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
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
               "eigmod::deflate_problem", "eigmod::secular_weights"):
        assert fn in out


@pytest.mark.gpu
def test_dropin_reference_cases_pass(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
