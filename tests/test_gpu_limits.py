"""GPU, size limits of the format: a container whose streams pass 4 GiB.

The reference's global scan throws validation_error("block too large:
offsets exceed 4-byte table range") as soon as a 4-byte table entry would
exceed UINT32_MAX (/root/reference/proj/src/scan.cpp:38-47,
tests/test_scan.cpp:76-79).  On the GPU the flag is raised by Kernel III /
the header kernel from the 64-bit prefixes of Kernel II and mapped onto the
same exception by the C-ABI (synchronous call) and by plzgpu_ctx_finish
(stream-ordered call).  Input: 4 GiB + 1 MiB of uniform random bytes at S=1
in a single 8 GiB container, so the literal payload alone passes 4 GiB."""
import pytest

from paper_2304_07342_b200 import plz

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
MSG = "block too large: offsets exceed 4-byte table range"


@pytest.fixture(scope="module")
def incompressible():
    import torch

    n = (4 << 30) + (1 << 20)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda", generator=g)
    yield x
    del x
    torch.cuda.empty_cache()


def test_offset_overflow_raises_the_reference_validation_error(incompressible):
    p = plz.validate(plz.Params(1, 128, 4096, 1, 8 << 30))
    with pytest.raises(plz.ValidationError) as ei:
        plz.compress(incompressible, p)
    assert str(ei.value) == MSG


def test_offset_overflow_on_the_async_path(incompressible):
    import torch

    p = plz.validate(plz.Params(1, 128, 4096, 1, 8 << 30))
    ctx = plz.context(incompressible.device.index)
    n = incompressible.numel()
    cap = plz.compress_bound(n, p)
    img = torch.empty(cap, dtype=torch.uint8, device="cuda")
    ln = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    ctx.compress_async(p, incompressible.data_ptr(), n, img.data_ptr(), cap, ln.data_ptr(), s)
    with pytest.raises(plz.ValidationError) as ei:
        ctx.finish(s)
    assert str(ei.value) == MSG
    del img


def test_same_bytes_in_default_containers_round_trip(incompressible):
    # 1 GiB of the same bytes in default 256 MiB containers: each stays far
    # below the limit, so it compresses and round-trips
    import torch

    p = plz.validate(plz.Params(1, 128, 4096, 1))
    x = incompressible[: (1 << 30) + 12345]
    img = plz.compress(x, p)
    assert torch.equal(plz.decompress_bytes(img), x)
