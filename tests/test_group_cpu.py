"""world_size-2 gloo tests on CPU of the multi-process plumbing: shm-name agreement and
max-over-ranks timing (the N > 1 bench path)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2306_13835_b200.group import agree_shm_name, max_over_ranks
    name = agree_shm_name()
    m = max_over_ranks([float(rank), 10.0 - rank])
    q.put((rank, name, m))
    dist.barrier()
    dist.destroy_process_group()


def test_agree_and_max_over_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    names = {r[1] for r in res}
    assert len(names) == 1 and next(iter(names)).startswith("/mpsw_")
    for r in res:
        assert r[2] == [1.0, 10.0]
