"""Ingest / egest formats: io.hpp:17-33 and the CLI
update / locate path (tools/eigmod.cpp:122-161).

CPU tests compare our parallel reader/writer with the unmodified reference's
io.cpp (oracle/_ref) byte for byte on writes and value for value / message for
message on reads, over the cases of proj/tests/test_io.cpp plus malformed
inputs. GPU tests run lib/eigmod_b200 on the cases of proj/tests/test_cli.cpp.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import ref
from paper_1706_00773_b200 import io

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1706_00773_b200", "lib", "eigmod_b200")

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def _same_file(a, b):
    return open(a, "rb").read() == open(b, "rb").read()


@needs_ref
def test_csv_writes_are_byte_identical(tmp_path):
    rng = np.random.default_rng(1)
    m = rng.standard_normal((64, 9)) * 10.0 ** rng.integers(-300, 300, (64, 9))
    m[0, :4] = [0.0, -0.0, 1e-17, 5e-324]
    m[1, :3] = [np.inf, -np.inf, 1.7976931348623157e308]
    for signs in (None, [1, -1, 1, 1, -1, 1, 1, 1, -1]):
        io.write_csv(tmp_path / "a.csv", m, signs)
        ref.write_csv(tmp_path / "b.csv", m, signs)
        assert _same_file(tmp_path / "a.csv", tmp_path / "b.csv")
    big = rng.standard_normal((3000, 40))  # several parallel chunks
    io.write_csv(tmp_path / "a.csv", big)
    ref.write_csv(tmp_path / "b.csv", big)
    assert _same_file(tmp_path / "a.csv", tmp_path / "b.csv")


@needs_ref
def test_matrix_market_writes_are_byte_identical(tmp_path):
    rng = np.random.default_rng(2)
    for n in (1, 2, 7, 300):
        a = rng.standard_normal((n, n))
        a = a + a.T
        io.write_matrix_market(tmp_path / "a.mtx", a)
        ref.write_matrix_market(tmp_path / "b.mtx", a)
        assert _same_file(tmp_path / "a.mtx", tmp_path / "b.mtx")
        with open(tmp_path / "a.mtx") as f:
            assert f.readline().rstrip("\n") == "%%MatrixMarket matrix array real symmetric"


def test_round_trips(tmp_path):
    # test_io.cpp:24-41, 60-75
    m = np.zeros((3, 2))
    m[0, 0], m[1, 1], m[2, 0] = 1.5, -2.25, 1e-17
    io.write_csv(tmp_path / "k.csv", m, [1, -1])
    back, signs = io.read_csv(tmp_path / "k.csv")
    assert np.array_equal(back, m) and list(signs) == [1, -1]
    rng = np.random.default_rng(3)
    a = rng.standard_normal((40, 40))
    a = 0.5 * (a + a.T)
    io.write_matrix_market(tmp_path / "a.mtx", a)
    assert np.array_equal(io.read_matrix_market(tmp_path / "a.mtx"), a)


READ_CASES = {
    # name: (suffix, content)
    "ragged": (".csv", "1,2\n3\n"),
    "bad_token": (".csv", "1,abc\n"),
    "trailing_comma": (".csv", "1,2,\n3,4,\n"),
    "leading_comma": (".csv", ",1\n"),
    "empty_token": (".csv", "1,,2\n"),
    "plus_sign": (".csv", "+1,2\n"),
    "spaces_tabs_crlf": (".csv", "  1 ,\t2\r\n3,4\r\n\n"),
    "signs_first": (".csv", "# signs: +1,-1\n1,2\n"),
    "signs_not_first": (".csv", "\n# note\n# signs: +1,-1\n1,2\n"),
    "bad_signs": (".csv", "# signs: +2\n1\n"),
    "comments_only": (".csv", "# x\n# y\n"),
    "empty": (".csv", ""),
    "exotic_numbers": (".csv", "1e308,-0,5e-324,inf,nan\n0x1p3,1.5e-400,2.5,1e400,-1e-7\n"),
    "mm_coordinate": (".mtx", "%%MatrixMarket matrix coordinate real general\n2 2\n"),
    "mm_truncated": (".mtx", "%%MatrixMarket matrix array real symmetric\n2 2\n1.0\n"),
    "mm_symmetric": (".mtx", "%%MatrixMarket matrix array real symmetric\n% c\n\n2 2\n1\n2\n%x\n3\n"),
    "mm_general": (".mtx", "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n"),
    "mm_upper_case": (".mtx", "%%MatrixMarket MATRIX Array REAL Symmetric\n1 1\n-4\n"),
    "mm_not_square": (".mtx", "%%MatrixMarket matrix array real general\n2 3\n"),
    "mm_bad_dims": (".mtx", "%%MatrixMarket matrix array real general\n% only comments\n"),
    "mm_hermitian": (".mtx", "%%MatrixMarket matrix array real hermitian\n1 1\n1\n"),
    "mm_bad_value": (".mtx", "%%MatrixMarket matrix array real symmetric\n1 1\n1 2\n"),
    "mm_nonfinite": (".mtx", "%%MatrixMarket matrix array real symmetric\n1 1\ninf\n"),
    "mm_extra_values": (".mtx", "%%MatrixMarket matrix array real symmetric\n1 1\n5\n6\n"),
    "mm_empty": (".mtx", ""),
    "mm_header_only": (".mtx", "%%MatrixMarket matrix array real symmetric\n"),
}


def _read(mod, path, suffix):
    try:
        if suffix == ".csv":
            v, s = mod.read_csv(path)
            return ("ok", v, None if s is None else list(s))
        return ("ok", mod.read_matrix_market(path), None)
    except (io.FormatError, ref.RefFormatError) as e:
        return ("format", str(e), None)


@needs_ref
@pytest.mark.parametrize("name", sorted(READ_CASES))
def test_reads_match_reference(tmp_path, name):
    suffix, content = READ_CASES[name]
    p = tmp_path / ("f" + suffix)
    p.write_text(content)
    got, want = _read(io, p, suffix), _read(ref, p, suffix)
    assert got[0] == want[0], (got, want)
    if got[0] == "ok":
        assert np.array_equal(got[1], want[1], equal_nan=True)
        assert got[2] == want[2]
    else:
        assert got[1] == want[1]


def test_missing_file_is_format_error():
    with pytest.raises(io.FormatError, match="cannot open"):
        io.read_matrix_market("/tmp/eigmod_no_such_file.mtx")
    with pytest.raises(io.FormatError, match="cannot open"):
        io.read_csv("/tmp/eigmod_no_such_file.csv")


def test_io_header_symbols_exported():
    import re

    src = open(os.path.join(ROOT, "include", "eigmod_b200_io.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(eigmod_b200_io_\w+)\s*\(", src))
    out = subprocess.run(["nm", "-D", "--defined-only", io._LIB], capture_output=True, text=True,
                         check=True).stdout
    assert names and names <= set(re.findall(r" T (eigmod_b200_io_\w+)", out))


# ------------------------------------------------------------- CLI (B200)
def _run(*args):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300)
    return r.returncode, r.stdout


@pytest.fixture
def cli_dir(tmp_path):
    # test_cli.cpp:39-49
    (tmp_path / "q.csv").write_text("1,0\n0,1\n")
    (tmp_path / "lambda.csv").write_text("0\n1\n")
    (tmp_path / "k.csv").write_text("1,0\n1,1\n")
    (tmp_path / "k0.csv").write_text("0\n0\n")
    return tmp_path


@pytest.mark.gpu
def test_cli_update_golden_2x2(cli_dir):
    d = cli_dir
    rc, out = _run("update", "--eigen", d / "q.csv", d / "lambda.csv", "--update", d / "k.csv",
                   "--out", d / "got")
    assert rc == 0 and "residual_fro" in out
    lam, _ = io.read_csv(d / "got_lambda.csv")
    assert lam.shape == (2, 1)
    assert abs(lam[0, 0] - 0.58578643762690495) <= 1e-12
    assert abs(lam[1, 0] - 3.4142135623730951) <= 1e-12


@pytest.mark.gpu
def test_cli_usage_and_errors(cli_dir):
    d = cli_dir
    assert _run("update", "--eigen", d / "q.csv", d / "lambda.csv", "--out", d / "x")[0] == 2
    (d / "bad.csv").write_text("1,2\n3\n")
    assert _run("update", "--eigen", d / "q.csv", d / "lambda.csv", "--update", d / "bad.csv",
                "--out", d / "x")[0] == 2
    assert _run("update", "--matrix", d / "a.mtx", "--update", d / "k.csv", "--out",
                d / "x")[0] == 2
    assert _run("frobnicate")[0] == 2


@pytest.mark.gpu
def test_cli_zero_update_reproduces_inputs(cli_dir):
    d = cli_dir
    rc, _ = _run("update", "--eigen", d / "q.csv", d / "lambda.csv", "--update", d / "k0.csv",
                 "--out", d / "zero")
    assert rc == 0
    lam, _ = io.read_csv(d / "zero_lambda.csv")
    q, _ = io.read_csv(d / "zero_q.csv")
    assert np.array_equal(lam[:, 0], [0.0, 1.0]) and np.array_equal(q, np.eye(2))


@pytest.mark.gpu
def test_cli_locate(cli_dir):
    d = cli_dir
    assert _run("locate", "--eigen", d / "q.csv", d / "lambda.csv", "--update",
                d / "k.csv") == (0, "0,1,1\n")
    rc, out = _run("locate", "--eigen", d / "q.csv", d / "lambda.csv", "--update", d / "k.csv",
                   "--signs", "-1,-1")
    assert rc == 0 and out.startswith("1")


@pytest.mark.gpu
def test_cli_update_matches_oracle(tmp_path):
    """A config-2 instance through files: eigenvalues and vectors as the
    oracle computes them, written byte-compatibly."""
    from oracle import port
    from paper_1706_00773_b200.instances import make_instance

    q, lam, kmat, signs = make_instance(2, n=300, seed=9)
    io.write_csv(tmp_path / "q.csv", q)
    io.write_csv(tmp_path / "l.csv", lam)
    io.write_csv(tmp_path / "k.csv", kmat, signs)
    rc, out = _run("update", "--eigen", tmp_path / "q.csv", tmp_path / "l.csv", "--update",
                   tmp_path / "k.csv", "--out", tmp_path / "o")
    assert rc == 0, out
    lo, qo, _ = port.update(q, lam, kmat, signs)
    got_l, _ = io.read_csv(tmp_path / "o_lambda.csv")
    got_q, _ = io.read_csv(tmp_path / "o_q.csv")
    assert np.abs(got_l[:, 0] - lo).max() <= 1e-12 * np.abs(lo).max()
    assert np.abs(got_q - qo).max() <= 1e-8
    rc, out = _run("locate", "--eigen", tmp_path / "q.csv", tmp_path / "l.csv", "--update",
                   tmp_path / "k.csv")
    assert rc == 0
    assert [int(x) for x in out.strip().split(",")] == port.locate_from_u(
        lam, port.transform(q, kmat), signs)
