"""Does a copy-engine + zero-copy-kernel split of one swap-in beat the copy engine alone? (dev)"""
import json, os, subprocess, sys
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ".")
    from paper_2306_13835_b200 import mpsw as M
    from synth import opt_dims
    from oracle import layout
    mode, ctas = int(sys.argv[2]), int(sys.argv[3])
    d = opt_dims("opt-1.3b")
    S = layout.shard_bytes(d, 1)
    with M.Ctx(device_ids=(0,), budget=S + 4096, swap_mode=mode, zc_ctas=ctas, writeback=0) as ctx:
        a, b = ctx.register_model(d), ctx.register_model(d)
        ctx.synth_fill(a, 1); ctx.synth_fill(b, 2)
        ctx.wait(ctx.swap_in(a))
        ms = []
        cur, oth = a, b
        for i in range(7):
            ctx.wait(ctx.swap_out(cur))
            t = ctx.swap_in(oth)
            ctx.wait(t)
            ms.append(ctx.entry_gpu_ms(t)[2][0])
            cur, oth = oth, cur
        import statistics
        med = statistics.median(ms[1:])
        ok = ctx.checksum(cur, 0) == ctx.checksum(cur, 0, on_device=False)
        print(json.dumps({"mode": mode, "ctas": ctas, "frac": os.environ.get("MPSW_HYBRID_FRAC"), "ms": med,
                          "GBps": S / med / 1e6, "bit_exact": ok}), flush=True)
    sys.exit(0)
for mode, frac, ctas in [(1, None, 0), (3, "0.05", 32), (3, "0.1", 32), (3, "0.15", 32), (3, "0.2", 32),
                         (3, "0.1", 16), (3, "0.1", 64), (3, "0.3", 64)]:
    env = dict(os.environ)
    if frac:
        env["MPSW_HYBRID_FRAC"] = frac
    subprocess.run([sys.executable, __file__, "child", str(mode), str(ctas)], env=env)
