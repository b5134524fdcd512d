"""GPU: bench.py's N > 1 path end to end -- torchrun with world 4, all ranks on
cuda:0, the exchange all-reduced over gloo (MCB_DIST_BACKEND=gloo; NCCL on a
real 8xB200 box).  The cube-range partition with an exact integer exchange
must give the single-GPU run's estimate bit for bit, for both transports."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
ARGS = ["--steps", "2", "--warmup", "3", "--maxcalls", str(10 ** 8), "--no-cpu", "--no-secondary"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _line(out: str) -> dict:
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


def _bench(world, transport="collective"):
    env = dict(os.environ, MCB_DIST_BACKEND="gloo")
    if world == 1:
        cmd = [sys.executable, "bench.py", *ARGS]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", str(world),
               "--transport", transport, *ARGS]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    return _line(p.stdout)


@pytest.mark.parametrize("transport", ["collective", "peer"])
def test_bench_world4_matches_single_gpu(transport):
    one = _bench(1)
    four = _bench(4, transport)
    assert four["n_gpus"] == 4 and one["n_gpus"] == 1
    assert four["config"] == one["config"]
    # exact exchange: identical estimate, sigma and device-counted samples
    for k in ("estimate", "sigma", "chi2_dof", "samples", "bin_writes"):
        assert four["result"][k] == one["result"][k], k
    assert four["result"]["samples"] == (3 + 2) * one["config"]["evals_per_step"]


def test_bench_nccl_path_world1_matches_single_gpu():
    """The N > 1 code path over NCCL itself (process group bound to the
    device, the exact int64 exchange all-reduced by NCCL on the library's
    stream, barriers, max over ranks), run at world 1 with MCB_FORCE_DIST=1:
    NCCL cannot put two ranks on one GPU, and this box has one."""
    one = _bench(1)
    env = dict(os.environ, MCB_FORCE_DIST="1")
    env.pop("MCB_DIST_BACKEND", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", *ARGS]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    nccl = _line(p.stdout)
    for k in ("estimate", "sigma", "chi2_dof", "samples", "bin_writes"):
        assert nccl["result"][k] == one["result"][k], k


def test_bench_world4_compact_exchange():
    """--transport compact (SURVEY.md 8(e)'s all-gather of each rank's
    rounded d*n_bins+6 doubles, summed in rank order): the same samples as
    one GPU and estimates within the rounding of the per-rank partial sums."""
    one = _bench(1)
    four = _bench(4, "compact")
    assert four["n_gpus"] == 4 and "compact" in four["parallelism"]
    assert four["result"]["samples"] == one["result"]["samples"]
    assert four["result"]["bin_writes"] == one["result"]["bin_writes"]
    assert abs(four["result"]["estimate"] - one["result"]["estimate"]) <= 1e-12 * abs(one["result"]["estimate"])
    assert abs(four["result"]["sigma"] - one["result"]["sigma"]) <= 1e-10 * one["result"]["sigma"]
