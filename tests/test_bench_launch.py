"""bench.py's multi-rank launcher on CPU (gloo): `python bench.py --gpus N`
outside torchrun re-executes itself as N ranks (one process per GPU on the
box), each rank sees WORLD_SIZE = N, and rank 0 alone prints the JSON line
with n_gpus = N and the max over ranks. NCCL's INIT logging is switched on
for the ranks (communicator size visible on stderr)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_launch_command_shape():
    cmd = bench.launch_command(4, ["--gpus", "4", "--steps", "2"])
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    env = bench.nccl_env({})
    assert env["NCCL_DEBUG"] == "INFO" and env["NCCL_DEBUG_FILE"] == "/dev/stderr"


@pytest.mark.parametrize("n", [2, 3])
def test_relaunch_runs_n_ranks(n):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n),
                          "--selftest-launch"], capture_output=True, text=True, timeout=300,
                         env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == n and rec["max_over_ranks"] == float(n)
    assert rec["nccl_debug"] == "INFO"


def test_world_size_mismatch_is_rejected():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4",
                          "--selftest-launch"], capture_output=True, text=True, timeout=120,
                         env=env)
    assert out.returncode != 0
