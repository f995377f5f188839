"""The bench.py N > 1 path (torchrun, row-strip partition, CUDA-IPC push transport, max-over-
ranks timing, summed arrivals) run end to end with two ranks sharing cuda:0
(ACA_BENCH_SHARED_GPU=1: gloo process group; time-sliced, so only the plumbing and the JSON
line are checked here — trajectories across processes are checked bit for bit in
tests/test_gpu_ipc.py)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_shared_gpu():
    env = dict(os.environ, ACA_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--config", "c2", "--no-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1   # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "row strips x 2"
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
