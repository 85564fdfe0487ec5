"""Helper for tests: run a `world`-rank multi-process TP group on ONE GPU (every process on cuda:0).
Rank 0 (leader) drives requests and explicit swaps; both ranks check their resident shards
against the oracle image; results are written as JSON by rank 0."""
import json
import os
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2306_13835_b200 import mpsw as M
    from paper_2306_13835_b200.group import open_group_ctx, max_over_ranks
    from synth import opt_dims, request_tokens
    from oracle import layout, checksum
    d = opt_dims("small")
    S = layout.shard_bytes(d, world)
    res = {"rank": rank}
    ctx = open_group_ctx(0, budget=(S + 4095) // 4096 * 4096, max_batch=4, max_tokens=8, trace=1)
    ids = [ctx.register_model(d) for _ in range(3)]
    for m in ids:
        ctx.synth_fill(m, 900 + m)
    dist.barrier()
    if rank == 0:
        outs = []
        for i, m in enumerate([0, 1, 0, 2, 2, 1]):
            tok = request_tokens(5, m, i, 8 if i % 2 else 3, d.vocab)
            rid, out = ctx.request(ids[m], tok)
            ctx.wait_request(rid, 120)
            outs.append({"model": m, "tokens": tok.tolist(), "logits": out.tolist()})
        # explicit swaps through the engine queue
        cur = [m for m in ids if ctx.residency(m) == M.RESIDENT]
        ctx.wait(ctx.swap_out(cur[0]))
        t = ctx.swap_in(ids[0])
        ctx.wait(t)
        res["outs"] = outs
        res["swap_in_ticket"] = t
        ctx.trace_dump(out_path + ".trace")
    obj = [res.get("swap_in_ticket")]
    dist.broadcast_object_list(obj, src=0)
    ctx.wait(obj[0], 60)
    _, _, ms = ctx.entry_gpu_ms(obj[0])
    res["gpu_ms_local"] = ms[rank]
    dist.barrier()
    checks = []
    for m in ids:
        if ctx.residency(m) == M.RESIDENT:
            img = layout.shard_image(d, world, rank, 900 + m)
            checks.append([m, ctx.checksum(m, rank) == checksum.checksum(img)])
    res["checks"] = checks
    res["stats"] = ctx.stats()
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    dist.barrier()
    ctx.close()
    if rank == 0:
        json.dump(gathered, open(out_path, "w"))
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
