"""Multi-process TP group (one process per rank; here all on cuda:0): shm control plane,
cross-process acks, CUDA-IPC peer partials in the fused all-reduce. Logits vs the oracle and
resident shards bit-exact on every rank."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from synth import opt_dims
from oracle import layout, forward
from tests.gpu_util import need_gpu
from tests import parity_util as PU

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# 8 processes on one GPU exercise the TP = 8 control plane of cfg4 / `bench.py --gpus 8`: 7 IPC
# peer mappings per rank, 8-way all-reduce reads, 8 acks per entry
# rs: the reduce-scatter all-reduce forced on every point (its all-gather writes through the CUDA
# IPC mappings of every rank's A operand, ordered by interprocess events)
@pytest.mark.parametrize("world,rs", [(2, 0), (4, 0), (8, 0), (4, 1), (8, 1)])
def test_process_group(tmp_path, world, rs):
    need_gpu()
    out = str(tmp_path / "mp.json")
    port = free_port()
    env = dict(os.environ, MPSW_RS_MIN_BYTES="0" if rs else str(1 << 62))
    if rs:
        env["MPSW_DEBUG_CHECKS"] = "1"      # residency stamps travel in the shm records
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp_group_run.py"), str(r), str(world), str(port), out],
                              env=env)
             for r in range(world)]
    rcs = [p.wait(timeout=600) for p in procs]
    assert rcs == [0] * world
    res = json.load(open(out))
    d = opt_dims("small")
    Ws = {m: layout.full_tensors(d, 900 + m) for m in range(3)}
    for o in res[0]["outs"]:
        tok = np.array(o["tokens"], np.int32)[None]
        ref = forward.forward_bf16_emulated(d, Ws[o["model"]], tok)[0]
        PU.assert_logits(np.array(o["logits"], np.float32), ref, tag="mp")
    for r in res:
        assert r["checks"] and all(ok for _, ok in r["checks"]), r
        assert r["gpu_ms_local"] > 0
    assert len(res) == world
    assert all(r["stats"]["swaps_in"] == res[0]["stats"]["swaps_in"] for r in res) and res[0]["stats"]["swaps_in"] > 0
    # leader trace replays through the oracle scheduler (acks from both processes)
    from oracle import scheduler as S
    cfg, evs, decs = S.read_trace(out + ".trace")
    assert cfg.n_models == 3 and cfg.tp == world and cfg.cap // cfg.sizes[0] == res[0]["stats"]["k_slots"]
    rdecs, _ = S.replay(cfg, evs)
    assert rdecs == decs


@pytest.mark.parametrize("world,seed", [(2, 0), (2, 1), (4, 2), (4, 3)])
def test_process_group_fuzz(tmp_path, world, seed):
    """Seeded serving workload on a multi-process group (tests/mp_fuzz_run.py): models of different
    sizes, D = 1/2, writeback or clean eviction, CE / zero-copy / auto swaps. Every rank's resident
    shards stay bit-exact after every burst, logits match the oracle, and the leader's event log
    (acks from every process) replays to identical decisions."""
    need_gpu()
    out = str(tmp_path / "fz.json")
    port = free_port()
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp_fuzz_run.py"), str(r), str(world), str(port),
                               str(seed), out]) for r in range(world)]
    rcs = [p.wait(timeout=600) for p in procs]
    assert rcs == [0] * world
    res = json.load(open(out))
    assert all(not r["bad"] for r in res), [r["bad"] for r in res]
    from synth.models import OptDims
    dims = [OptDims(*v) for v in res[0]["dims"]]
    Ws = {}
    for o in res[0]["outs"]:
        m = o["model"]
        if m not in Ws:
            Ws[m] = layout.full_tensors(dims[m], res[0]["seeds"][m])
        ref = forward.forward_bf16_emulated(dims[m], Ws[m], np.array(o["tokens"], np.int32)[None])[0]
        PU.assert_logits(np.array(o["logits"], np.float32), ref, tag=f"mp-fuzz m{m}")
    from oracle import scheduler as S
    cfg, evs, decs = S.read_trace(out + ".trace")
    assert cfg.tp == world
    rdecs, _ = S.replay(cfg, evs)
    assert rdecs == decs
    assert res[0]["stats"]["swaps_in"] > len(dims)
