"""One zero-copy swap-in of an OPT-1.3B shard (target for an ncu --set full capture)."""
import sys
sys.path.insert(0, ".")
from paper_2306_13835_b200 import mpsw as M
from synth import opt_dims
from oracle import layout

d = opt_dims(sys.argv[1] if len(sys.argv) > 1 else "opt-1.3b")
S = layout.shard_bytes(d, 1)
with M.Ctx(device_ids=(0,), budget=S + 4096, swap_mode=M.SWAP_ZERO_COPY, zc_ctas=int(sys.argv[2]) if len(sys.argv) > 2 else 0) as ctx:
    m = ctx.register_model(d)
    ctx.synth_fill(m, 3)
    t = ctx.swap_in(m)
    ctx.wait(t)
    print("gpu_ms", ctx.entry_gpu_ms(t)[2], "GB/s", S / (ctx.entry_gpu_ms(t)[2][0] / 1e3) / 1e9)
