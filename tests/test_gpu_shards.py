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


# ------------------------------------------------------ sharded decompress
def _ranges_concat(img_t, world):
    """Every virtual rank's plzgpu_decompress_range slice, checked to tile the
    output contiguously, concatenated."""
    _, _, total = plz.decompress_range(img_t, 0, 0)
    parts, at = [], 0
    for b, e in dist.chunk_ranges(total, world):
        out, begin, tot = plz.decompress_range(img_t, b, e)
        assert tot == total and begin == at
        at += out.numel()
        parts.append(bytes(out.cpu().numpy().tobytes()))
    return b"".join(parts)


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("S,W,C,I,bb", [(2, 255, 2048, 2, 2048 * 2 * 5), (1, 128, 4096, 1, 4096 * 3),
                                        (4, 255, 1024, 4, 1024 * 4 * 2)])
def test_sharded_decompress_ranges_tile_the_output(world, S, W, C, I, bb):
    # chunk ranges cut through containers; tails land in the range holding them
    import torch

    p = plz.validate(plz.Params(S, W, C, I, bb))
    data = inputs.make("quant", 23 * C * S + 3 * S + (S - 1), 200 + world, S)
    img = torch.frombuffer(bytearray(plz.compress(data, p)), dtype=torch.uint8).cuda()
    assert _ranges_concat(img, world) == data


def test_sharded_decompress_of_concatenated_images():
    # containers with tails and containers without chunks (inputs shorter
    # than one symbol) between them: every byte belongs to exactly one range
    import torch

    parts = [inputs.make("alpha", n, n, 4) for n in (4099, 3, 12345, 2, 0, 70001)]
    imgs = [plz.compress(d, plz.validate(plz.Params(4, 255, 1024, 2, 1024 * 4 * 3))) for d in parts]
    img = torch.frombuffer(bytearray(b"".join(imgs)), dtype=torch.uint8).cuda()
    for world in (1, 2, 3, 7, 40):
        assert _ranges_concat(img, world) == b"".join(parts)


def test_sharded_decompress_errors():
    # a corrupt chunk fails the range holding it (same error as the whole
    # decode) and no other; a header error fails every range
    import torch

    p = plz.validate(plz.Params(2, 255, 2048, 1))
    data = inputs.make("quant", 40 * 4096, 5, 2)
    good = bytearray(plz.compress(data, p))
    n = int.from_bytes(good[21:25], "little")
    flags0 = 26 + 8 * (n + 1)
    k = 30  # corrupt chunk 30's first flag byte region: set every flag bit
    fk = int.from_bytes(good[26 + 4 * (n + 1) + 4 * k:26 + 4 * (n + 1) + 4 * k + 4], "little")
    bad = bytearray(good)
    bad[flags0 + fk:flags0 + fk + 4] = b"\xff\xff\xff\xff"
    t = torch.frombuffer(bad, dtype=torch.uint8).cuda()
    with pytest.raises(plz.CorruptionError) as whole:
        plz.decompress_bytes(t)
    with pytest.raises(plz.CorruptionError) as part:
        plz.decompress_range(t, 20, 40)
    assert str(part.value) == str(whole.value)
    out, begin, _ = plz.decompress_range(t, 0, 20)
    assert bytes(out.cpu().numpy().tobytes()) == data[:begin + out.numel()]
    hdr = bytearray(good)
    hdr[4] = 2  # version
    th = torch.frombuffer(hdr, dtype=torch.uint8).cuda()
    with pytest.raises(plz.Error) as whole:
        plz.decompress_bytes(th)
    with pytest.raises(plz.Error) as part:
        plz.decompress_range(th, 0, 1)
    assert type(part.value) is type(whole.value) and str(part.value) == str(whole.value)


def test_decompress_range_with_host_buffers():
    # the C-ABI range decode from a host image into a host buffer (staged
    # through the context) equals the device-resident slices
    import ctypes as C

    p = plz.validate(plz.Params(2, 255, 2048, 2, 2048 * 2 * 4))
    data = inputs.make("quant", 37 * 4096 + 5, 77, 2)
    img = plz.compress(data, p)
    ctx = plz.context()
    src = C.create_string_buffer(img, len(img))
    _, _, total = ctx.decompress_range(C.addressof(src), len(img), 0, 0, 0, 0)
    at = 0
    for b, e in dist.chunk_ranges(total, 3):
        begin, ln, tot = ctx.decompress_range(C.addressof(src), len(img), b, e, 0, 0)
        out = C.create_string_buffer(max(ln, 1))
        begin2, ln2, _ = ctx.decompress_range(C.addressof(src), len(img), b, e, C.addressof(out),
                                              ln)
        assert (begin2, ln2, tot) == (begin, ln, total) and begin == at
        assert out.raw[:ln] == data[begin:begin + ln]
        at += ln
    assert at == len(data)
    # a buffer one byte short is the reference's capacity error
    b, e = dist.chunk_ranges(total, 3)[1]
    _, ln, _ = ctx.decompress_range(C.addressof(src), len(img), b, e, 0, 0)
    small = C.create_string_buffer(ln)
    with pytest.raises(plz.CapacityError):
        ctx.decompress_range(C.addressof(src), len(img), b, e, C.addressof(small), ln - 1)


# ------------------------------------------- one process, a device list
@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0, 0, 0]])
@pytest.mark.parametrize("S,W,C,I,bb", [(2, 255, 2048, 2, 2048 * 2 * 5), (1, 128, 4096, 1, 4096 * 3),
                                        (4, 64, 1024, 4, 256 << 20)])
def test_compress_multi_equals_single_call(devices, S, W, C, I, bb):
    # plzgpu_compress_multi (device list; a repeated device = another context
    # and host thread on it): host and device inputs, tails, ranges cutting
    # containers; the image and stats equal the single call's
    import torch

    p = plz.validate(plz.Params(S, W, C, I, bb))
    data = inputs.make("quant", 23 * C * S + 3 * S + (S - 1), 300 + len(devices), S)
    st1, st2 = plz.PipelineStats(), plz.PipelineStats()
    want = plz.compress(data, p, stats=st1)
    got = plz.compress_multi(data, p, devices, stats=st2)
    assert got == want
    assert (st2.pointer_tokens, st2.literal_tokens) == (st1.pointer_tokens, st1.literal_tokens)
    d = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    got_d = plz.compress_multi(d, p, devices)
    assert got_d.is_cuda and bytes(got_d.cpu().numpy().tobytes()) == want


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0, 0, 0]])
def test_decompress_multi_equals_single_call(devices):
    import torch

    parts = [inputs.make("alpha", k, k, 4) for k in (4099, 3, 12345, 70001)]
    p = plz.validate(plz.Params(4, 255, 1024, 2, 1024 * 4 * 3))
    img = b"".join(plz.compress(d, p) for d in parts)
    want = b"".join(parts)
    assert plz.decompress_multi(img, devices) == want
    t = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
    got = plz.decompress_multi(t, devices)
    assert got.is_cuda and bytes(got.cpu().numpy().tobytes()) == want
    # a corrupt chunk: the single call's error, whichever rank holds it
    bad = bytearray(img)
    bad[len(bad) // 2] ^= 0xFF
    bad[len(bad) // 2 + 7] ^= 0x3C
    try:
        plz.decompress_bytes(bytes(bad))
        w = None
    except plz.Error as e:
        w = (type(e), str(e))
    try:
        plz.decompress_multi(bytes(bad), devices)
        g = None
    except plz.Error as e:
        g = (type(e), str(e))
    assert g == w
