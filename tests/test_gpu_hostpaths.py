"""GPU: the host-buffer paths of the public calls at sizes that exercise
their pipelines — pinned buffers (H2D segments with ready flags, per-
container assembly and D2H, pipelined decode) and pageable buffers (the
std::vector path of plz::compress callers: staged through pinned bounce
slots by the host copy pool, csrc/staging.cpp).  Every image must equal the
device-resident call's image, and every output the input."""
import numpy as np
import pytest

from paper_2304_07342_b200 import datagen, plz

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def field():
    # 1.5 fields of c5's stream: 384 MiB, two containers, a partial one
    w = datagen.WORKLOADS["c5"]
    d = datagen.quant_codes(w, 42, "cuda", fields=(0, 2))
    return d[: (384 << 20) + 6].contiguous()  # ends 3 symbols into a chunk


def test_pageable_compress_and_decompress_match_device_path(field):
    import torch

    p = plz.validate(plz.Params(2, 255, 2048, 2))
    want = plz.compress(field, p)
    torch.cuda.synchronize()
    host = field.cpu().numpy()              # pageable numpy buffer
    img = plz.compress(host, p)             # pageable in -> pageable out (bytes)
    assert img == want.cpu().numpy().tobytes()
    back = plz.decompress_bytes(img)        # pageable image in -> pageable out
    assert back == host.tobytes()


def test_pinned_compress_and_decompress_match_device_path(field):
    import torch

    p = plz.validate(plz.Params(2, 255, 2048, 2))
    want = plz.compress(field, p)
    n = field.numel()
    h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_in.copy_(field)
    cap = plz.compress_bound(n, p)
    h_img = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
    ctx = plz.context(0)
    ln, _ = ctx.compress_ptr(p, h_in.data_ptr(), n, h_img.data_ptr(), cap)
    assert torch.equal(h_img[:ln].cuda(), want)
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    got = ctx.decompress_ptr(h_img.data_ptr(), ln, h_out.data_ptr(), n)
    assert got == n and torch.equal(h_out, h_in)


def test_pageable_input_into_pinned_image(field):
    # mixed: a pageable input staged to the device, the image into pinned
    # memory container by container
    import torch

    p = plz.validate(plz.Params(2, 255, 2048, 2))
    want = plz.compress(field, p)
    host = np.ascontiguousarray(field.cpu().numpy())
    n = host.size
    cap = plz.compress_bound(n, p)
    h_img = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
    ln, _ = plz.context(0).compress_ptr(p, host.ctypes.data, n, h_img.data_ptr(), cap)
    assert torch.equal(h_img[:ln].cuda(), want)
