"""The multi-rank bench flow (the driver's SCALE runs: torchrun, one process
per GPU) exercised end to end on whatever GPUs the box has: two ranks over
gloo (PAFFT_BENCH_BACKEND=gloo, ranks may share a GPU -- a plumbing check of
the partition, the filter broadcast, the max over ranks and the single rank-0
JSON line, not a measurement).  The NCCL path itself runs in the 8-GPU driver
run; its host logic is covered by tests/test_multirank.py on CPU."""
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


def test_two_rank_bench_line_strong_partition():
    env = dict(os.environ, PAFFT_BENCH_BACKEND="gloo")
    for attempt in range(3):
        # the free port found here can be taken again before torchrun binds it: try another one
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
               "--gpus", "2", "--config", "5", "--batch", "64", "--steps", "2", "--warmup", "3",
               "--no-cpu", "--no-e2e", "--no-sub"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
        if r.returncode == 0 or "EADDRINUSE" not in r.stderr:
            break
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_batch"] == 64 and d["config"]["batch_per_gpu"] == 32
    assert d["value"] > 0 and d["gpu_launches"] == 3 * 2  # this rank's passes per step x steps
