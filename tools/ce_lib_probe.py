"""Library swap-in of a small shard, copy engine vs the raw copy (dev probe): per swap the load
entry's device span (CUDA events around the copy on the H2D stream) and, with MPSW_SWAP_DEBUG=1,
the worker's host issue time on stderr. usage: python tools/ce_lib_probe.py [MiB ...]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_13835_b200 import mpsw as M  # noqa: E402
from tools.sweep_cfg5 import dims_for  # noqa: E402

for mib in [int(x) for x in sys.argv[1:]] or [1, 4, 16]:
    d = dims_for(mib << 20)
    S = M.shard_layout(d, 1)[1]
    for mode in (1, 2):
        with M.Ctx(device_ids=(0,), budget=(S + 4095) // 4096 * 4096, swap_mode=mode, writeback=0, zc_ctas=148) as ctx:
            a, b = ctx.register_model(d), ctx.register_model(d)
            ctx.synth_fill(a, 1)
            ctx.synth_fill(b, 2)
            ctx.wait(ctx.swap_in(a))
            cur, other = a, b
            dev, host = [], []
            for _ in range(9):
                ctx.wait(ctx.swap_out(cur))
                t = ctx.swap_in(other)
                ts, td = ctx.wait(t)
                dev.append(ctx.entry_gpu_ms(t)[2][0])
                host.append((td[0] - ts) * 1e3)
                cur, other = other, cur
        print(json.dumps({"MiB": mib, "S": S, "mode": {1: "copy_engine", 2: "zero_copy"}[mode],
                          "dev_ms": statistics.median(dev[2:]), "dev_ms_all": [round(x, 4) for x in dev],
                          "host_submit_to_ack_ms": statistics.median(host[2:])}), flush=True)
