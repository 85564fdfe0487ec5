"""bench.py's N > 1 path end to end: torchrun with 2 and 4 processes (one TP=N group over the shm
control plane and CUDA IPC), all mapped to cuda:0 (MPSW_BENCH_DEVICE0) with gloo barriers, on a
small model; rank 0 prints one JSON line with the contract keys."""
import json
import os
import subprocess
import sys

import pytest

from tests.gpu_util import need_gpu

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [2, 4])
def test_bench_torchrun_ranks(n):
    need_gpu()
    env = dict(os.environ, MPSW_BENCH_DEVICE0="1", MPSW_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n), "--master-addr",
           "127.0.0.1", "--master-port", str(29517 + n), "bench.py", "--gpus", str(n), "--steps", "3", "--warmup", "3",
           "--model", "mid", "--no-cpu-baseline"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    o = json.loads(lines[0])
    assert o["n_gpus"] == n and o["config"]["tp"] == n and o["steps"] == 3 and o["warmup"] == 3
    assert o["value"] > 0 and o["e2e"]["value"] > 0 and o["gpu_launches"] > 0
    assert o["scaling"] == "strong" and o["roofline"]["bound"] == "pcie"
    assert o["writeback"]["paper_window_ms"]["p50"] >= o["writeback"]["swap_in_latency_ms"]["p50"] * 0.5


def test_bench_driver_form_self_launches():
    """The driver's form `python bench.py --gpus 2` (no torchrun around it) re-launches itself
    under torch.distributed.run with 2 ranks and reports n_gpus = 2 (ranks on cuda:0 here)."""
    need_gpu()
    env = dict(os.environ, MPSW_BENCH_DEVICE0="1", MPSW_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--model", "mid",
           "--no-cpu-baseline", "--wb-steps", "2"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    o = json.loads(lines[0])
    assert o["n_gpus"] == 2 and o["config"]["tp"] == 2
    assert o["writeback"]["steps"] == 2 and o["writeback"]["d2h_bytes"] > 0
    assert o["swap_in_latency_ms"]["p50"] > 0
