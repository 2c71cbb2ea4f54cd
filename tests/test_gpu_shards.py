"""GPU: the multi-GPU shard protocol (paper_2304_07342_b200/dist.py,
plzgpu_shard_*) simulated for 1..8 virtual ranks on one B200: chunk ranges cut
through containers, per-rank table rebasing and the root's segment placement
must reproduce the single-call image byte for byte ("the image
must be identical at 1/2/4/8 GPUs")."""
import pytest

import inputs
from paper_2304_07342_b200 import dist, plz

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("S,W,C,I,bb", [(2, 255, 2048, 2, 2048 * 2 * 5), (1, 128, 4096, 1, 4096 * 3),
                                        (4, 255, 1024, 4, 256 << 20), (2, 64, 1024, 1, 1024 * 2)])
def test_sharded_image_equals_single_call(world, S, W, C, I, bb):
    import torch

    p = plz.validate(plz.Params(S, W, C, I, bb))
    data = inputs.make("quant", 23 * C * S + 3 * S + (S - 1), 100 + world, S)
    want = plz.compress(data, p)
    d = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    got = dist.simulate_sharded(p, d, world)
    assert bytes(got.cpu().numpy().tobytes()) == want
    assert plz.decompress_bytes(want) == data


def test_more_ranks_than_chunks():
    import torch

    p = plz.validate(plz.Params(2, 255, 2048, 1))
    data = inputs.make("runs", 3 * 4096 + 1, 9, 2)
    d = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    assert bytes(dist.simulate_sharded(p, d, 8).cpu().numpy().tobytes()) == plz.compress(data, p)
