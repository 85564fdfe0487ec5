"""Helper for tests/test_gpu_multiprocess.py: one rank of a `world`-process TP group on ONE GPU
(every process on cuda:0) serving a seeded random workload: models of different sizes, D batches
in flight, writeback or clean eviction, copy-engine / zero-copy / auto swaps. Rank 0 (leader)
submits bursts of ragged requests; every rank checks its resident shards against the oracle
image after each burst; rank 0 writes outputs, per-rank checks and the engine trace as JSON."""
import json
import os
import random
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def scenario(seed, world):
    from synth.models import OptDims
    rnd = random.Random(seed)
    dims = []
    for _ in range(3):
        hd = rnd.choice([32, 64])
        heads = world * rnd.randint(1, 3)
        h = heads * hd
        dims.append(OptDims(rnd.randint(1, 2), h, heads, 4 * h, vocab=world * rnd.randint(100, 800), max_pos=16))
    big = max(dims, key=lambda d: d.hidden)
    dmax = OptDims(1, big.hidden, big.heads, max(d.ffn for d in dims), vocab=max(d.vocab for d in dims), max_pos=16)
    opts = dict(D=1 + seed % 2, writeback=rnd.choice([0, 1]), mode=rnd.choice([0, 1, 2]))   # odd seeds: D = 2
    return rnd, dims, dmax, opts


def main(rank, world, port, seed, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2306_13835_b200 import mpsw as M
    from paper_2306_13835_b200.group import open_group_ctx
    from synth import request_tokens
    from oracle import layout, checksum
    rnd, dims, dmax, o = scenario(seed, world)
    sizes = [(layout.shard_bytes(d, world) + 4095) // 4096 * 4096 for d in dims]
    budget = max(sizes) + min(sizes) + 4096            # the largest plus the smallest: real eviction traffic
    seeds = [5000 + 10 * seed + i for i in range(len(dims))]
    ref = [checksum.checksum(layout.shard_image(d, world, rank, seeds[m])) for m, d in enumerate(dims)]
    ctx = open_group_ctx(0, budget=budget, max_batch=4, max_tokens=8, trace=1, max_inflight=o["D"],
                         writeback=o["writeback"], swap_mode=o["mode"], chunk_bytes=1 << 20, max_dims=dmax)
    ids = [ctx.register_model(d) for d in dims]
    for m in ids:
        ctx.synth_fill(m, seeds[m])
    dist.barrier()
    outs, bad = [], []
    for step in range(12):
        if rank == 0:
            pend = []
            for j in range(rnd.choice([1, 2, 4])):
                m = rnd.randrange(len(dims))
                tok = request_tokens(6000 + seed, m, 10 * step + j, rnd.randint(1, 8), dims[m].vocab)
                rid, out = ctx.request(ids[m], tok)
                pend.append((rid, m, tok, out))
            for rid, m, tok, out in pend:
                ctx.wait_request(rid, 120)
                outs.append({"model": m, "tokens": tok.tolist(), "logits": out.tolist()})
        dist.barrier()                                  # the leader's burst is complete everywhere
        for m in ids:
            if ctx.residency(m) == M.RESIDENT and ctx.checksum(m, rank) != ref[m]:
                bad.append([step, m])
        dist.barrier()
    res = {"rank": rank, "bad": bad, "stats": ctx.stats(), "opts": o}
    if rank == 0:
        res["outs"] = outs
        res["seeds"] = seeds
        res["dims"] = [list(d.__dict__.values()) for d in dims]
        ctx.trace_dump(out_path + ".trace")
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    dist.barrier()
    ctx.close()
    if rank == 0:
        json.dump(gathered, open(out_path, "w"))
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
