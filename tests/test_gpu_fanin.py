"""NVLink-assisted fan-in swap (NEXT-2): chunks of a swap-in travel through helper GPUs' PCIe links
and NVLink peer copies. On one B200 the helper is the same device (virtual), which exercises the
full path — staging ring, cross-stream gates, paired writeback — for bit-exactness; bandwidth
gains need several GPUs."""
import random

import numpy as np
import pytest

from synth import opt_dims
from oracle import layout, checksum
from tests.gpu_util import need_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("writeback", [1, 0])
@pytest.mark.parametrize("tp,helpers", [(1, 1), (1, 3), (2, 2)])
def test_fanin_bit_exact(writeback, tp, helpers):
    M = need_gpu()
    d = opt_dims("mid")
    S_ = layout.shard_bytes(d, tp)
    nm, k = 3, 1
    imgs = {m: [layout.shard_image(d, tp, r, 400 + m) for r in range(tp)] for m in range(nm)}
    ref = {m: [checksum.checksum(a) for a in v] for m, v in imgs.items()}
    rnd = random.Random(tp * 10 + helpers + writeback)
    with M.Ctx(device_ids=(0,) * tp, budget=k * ((S_ + 4095) // 4096 * 4096), swap_mode=M.SWAP_COPY_ENGINE,
               chunk_bytes=1 << 20, writeback=writeback, helper_device_ids=(0,) * helpers, max_batch=2,
               max_tokens=4) as ctx:
        ids = [ctx.register_model(d, shards=imgs[m]) for m in range(nm)]
        for step in range(12):
            m = rnd.randrange(nm)
            rid, out = ctx.request(ids[m], np.array([5, 6, 7], np.int32))
            ctx.wait_request(rid, 60)
            for r in range(tp):
                assert ctx.checksum(ids[m], r) == ref[m][r], (step, m, r)
        for mm in range(nm):
            for r in range(tp):
                assert ctx.checksum(ids[mm], r, on_device=False) == ref[mm][r]
        assert ctx.stats()["swaps_in"] >= 6
