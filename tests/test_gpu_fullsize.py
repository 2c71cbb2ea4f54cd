"""GPU, BASELINE sizes: for every BASELINE.json config the B200 image of the
full synthetic workload must equal the reference library's image
(oracle/_ref, all host threads) byte for byte, and decode back bit-exactly
with both decoders — c5 (the 8 GiB bench headline, 32 containers) and c3 at
every interval included, whole.  c5's fields also go through the multi-GPU
shard protocol simulated on one GPU (sharded image == single-call image).

These are the slow tests (tens of seconds of reference CPU time each); the
size-independent properties (round trip, reference decode of the GPU image,
shard image == single-call image) hold at full size."""
import numpy as np
import pytest

import oracle as O
from paper_2304_07342_b200 import datagen, dist, plz

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def run_config(name, interval=None):
    import torch

    w = datagen.WORKLOADS[name]
    I = interval or w.I
    d = datagen.quant_codes(w, 42, "cuda")
    p = plz.validate(plz.Params(w.S, w.W, w.C, I))
    img = plz.compress(d, p)
    torch.cuda.synchronize()
    back = plz.decompress_bytes(img)
    assert torch.equal(back, d), "GPU round trip"
    del back
    host = d.cpu().numpy()
    del d
    gimg = img.cpu().numpy()
    del img
    if O.ref_available():
        op = O.make_params(w.S, w.W, w.C, I)
        ref = np.frombuffer(O.ref_compress(host, op, 0), dtype=np.uint8)
        assert len(gimg) == len(ref)
        assert np.array_equal(gimg, ref), f"{name} I={I}: image differs from the reference"
        del ref
        assert np.array_equal(np.frombuffer(O.ref_decompress(gimg, 0), dtype=np.uint8), host)
    return host.size / gimg.size


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_fullsize_bit_exact_vs_reference(name):
    cr = run_config(name)
    assert cr > 1.5


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("interval", [1, 2, 4, 8, 16])
def test_c3_interval_sweep_bit_exact(interval):
    # c3 NYX-like 512^3 u16, interval sweep (BASELINE configs[2]), whole
    run_config("c3", interval)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_c5_whole_stream_bit_exact_vs_reference():
    # the bench headline: 8 GiB, 32 containers (fields seeds 42..73), the
    # reference's multi-container loop (pipeline.cpp:88-99) on every core
    cr = run_config("c5")
    assert cr > 1.5


def test_c5_first_container_is_c3_field():
    # the reference arm times c5's first container: the same bytes as c3's field
    import torch

    a = datagen.quant_codes(datagen.WORKLOADS["c5"], 42, "cuda", fields=(0, 1))
    b = datagen.quant_codes(datagen.WORKLOADS["c3"], 42, "cuda")
    assert torch.equal(a, b)


def test_c5_fields_sharded_equal_single_gpu():
    import torch

    w = datagen.WORKLOADS["c5"]
    p = plz.validate(plz.Params(2, 255, 2048, 2))
    data = datagen.quant_codes(w, 42, "cuda", fields=(0, 4))
    want = plz.compress(data, p)
    for world in (2, 4, 8):
        got = dist.simulate_sharded(p, data, world)
        assert torch.equal(got, want), f"sharded image differs at {world} ranks"
    assert torch.equal(plz.decompress_bytes(want), data)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("S,kind", [(1, "quant"), (2, "quant")])
def test_batched_assembly_across_odd_containers(S, kind):
    # Kernel III's batched runs (inputs of >= 16 Ki chunks) over containers
    # of 1021 chunks — runs of 32 straddle container boundaries — and a
    # partial last chunk plus (S = 2) a tail byte, against the reference image
    import inputs

    C = 1024
    n = (131072 + 77) * C * S + 700 * S + (S - 1)
    data = inputs.make(kind, n, 5, S)
    p = plz.validate(plz.Params(S, 64, C, 1, 1021 * C * S))
    img = plz.compress(data, p)
    op = O.make_params(S, 64, C, 1, 1021 * C * S)
    ref = O.ref_compress(data, op, 0)
    assert img == ref, "image differs from the reference"
    assert plz.decompress_bytes(img) == data
