"""Pins oracle/imagehash.py (streamed C4 hash of a C0 shard image) to the plain definition:
checksum(shard_image(...)) on materialised images, over TP / PP / dtype and a shape whose tensors
are not whole 8-byte words (zero tail + padding handling)."""
import pytest

from synth import opt_dims
from synth.models import OptDims
from oracle import layout, checksum, imagehash


@pytest.mark.parametrize("tp,pp", [(1, 1), (2, 1), (4, 1), (2, 2)])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_streamed_hash_equals_image_hash(tp, pp, dtype):
    d = opt_dims("tiny")
    for stage in range(pp):
        for r in range(tp):
            img = layout.shard_image(d, tp, r, 17, dtype, pp, stage)
            assert imagehash.shard_image_hash(d, tp, r, 17, dtype, pp, stage, threads=2) == checksum.checksum(img)


def test_streamed_hash_odd_tensor_sizes():
    d = OptDims(1, 6, 2, 10, vocab=14, max_pos=3)      # 12-byte biases: not whole 8-byte words
    for tp in (1, 2):
        for r in range(tp):
            img = layout.shard_image(d, tp, r, 5)
            assert imagehash.shard_image_hash(d, tp, r, 5, threads=3) == checksum.checksum(img)
    # and the hash does see the values: another seed gives another hash
    assert imagehash.shard_image_hash(d, 1, 0, 6) != imagehash.shard_image_hash(d, 1, 0, 5)
