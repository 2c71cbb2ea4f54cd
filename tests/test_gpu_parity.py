"""GPU parity: the B200 path (through the C-ABI) against the reference.

Checker: oracle/_ref (the reference library compiled from its own sources)
when present, else the C restatement oracle/plz_oracle.c (pinned to the same
reference by tests/test_oracle.py and tests/golden/).  Integer/byte work: the
bar is bit-exact images, bit-exact round trips, and identical typed errors.
"""
import random

import pytest

import inputs
import oracle as O
from paper_2304_07342_b200 import plz

pytestmark = pytest.mark.gpu


def ref_compress(data, p):
    op = O.make_params(p.symbol_width, p.window, p.chunk_size, p.interval, p.block_bytes,
                       p.min_match)
    if O.ref_available():
        return O.ref_compress(data, op, 0, stats=True)
    return O.compress_stats(data, op)


def ref_decompress(img):
    # threads=1: the reference rethrows the FIRST failing chunk's error, which
    # with a thread pool is timing-dependent (parallel.hpp:36-56); one worker
    # is its deterministic schedule (lowest chunk), which the GPU path matches
    return O.ref_decompress(img, 1) if O.ref_available() else O.decompress(img)


def P(S=2, W=128, C=2048, I=1, block_bytes=256 << 20):
    return plz.validate(plz.Params(S, W, C, I, block_bytes))


# ------------------------------------------------------------ known answers
def test_known_answer_sixteen_equal_bytes():
    # test_encoder.cpp:44-52: tokens L,L,L,P(3,3),P(6,6),P(4,12), flags 0x1C
    img = plz.compress(b"\xab" * 16, P(1, 255, 1024))
    assert len(img) == 52
    assert img[-10:] == bytes([0x1C, 0xAB, 0xAB, 0xAB, 3, 3, 6, 6, 4, 12])
    assert plz.decompress_bytes(img) == b"\xab" * 16


def test_known_answer_four_u32_symbols():
    # test_encoder.cpp:54-65: S=4 -> L, P(1,1), P(2,2); flags 0x60
    data = bytes([0x11, 0x22, 0x33, 0x44]) * 4
    img = plz.compress(data, P(4, 255, 1024))
    assert img[-9:] == bytes([0x60, 0x11, 0x22, 0x33, 0x44, 1, 1, 2, 2])


def test_known_answer_single_symbol_tail():
    # 0x5A at S=2: no chunk, one tail byte -> 35-byte container
    img = plz.compress(b"\x5a", P(2, 128, 2048))
    assert img.hex() == ("504c5a31" "01" "02" "80" "01" "00" "00080000" "0100000000000000"
                         "00000000" "01" "00000000" "00000000" "5a")
    assert plz.decompress_bytes(img) == b"\x5a"


def test_empty_input_is_empty_image():
    assert plz.compress(b"", P()) == b""
    assert plz.decompress_bytes(b"") == b""


# -------------------------------------------------------- randomized parity
GRID = [(S, W, C, I) for S in (1, 2, 4) for W in (4, 32, 64, 128, 255)
        for C in (1024, 2048, 4096, 8192, 16384) for I in (1, 2, 4, 8, 16) if C > W]


@pytest.mark.parametrize("seed", range(6))
def test_random_grid_bit_exact(seed):
    rng = random.Random(1000 + seed)
    for it in range(60):
        S, W, C, I = rng.choice(GRID)
        bb = C * S * rng.choice([1, 2, 3]) if rng.random() < 0.25 else 256 << 20
        p = P(S, W, C, I, bb)
        size = rng.choice([0, 1, S - 1, S, C * S - 1, C * S, C * S + 1, rng.randrange(1, 70000)])
        kind = rng.choice(inputs.KINDS)
        data = inputs.make(kind, size, seed * 1000 + it, S)
        want, st_ref = ref_compress(data, p)
        stats = plz.PipelineStats()
        got = plz.compress(data, p, stats=stats)
        assert got == want, f"image mismatch S={S} W={W} C={C} I={I} bb={bb} n={size} {kind}"
        assert (stats.pointer_tokens, stats.literal_tokens) == st_ref[1:]
        assert plz.decompress_bytes(got) == data
        assert ref_decompress(got) == data


@pytest.mark.parametrize("S,W,C,I", [(1, 128, 4096, 1), (2, 255, 2048, 2), (2, 255, 2048, 1),
                                     (2, 255, 2048, 16), (4, 255, 1024, 4), (1, 255, 16384, 1),
                                     (4, 255, 16384, 1), (2, 255, 8192, 8)])
@pytest.mark.parametrize("kind", inputs.KINDS)
def test_configs_bit_exact(S, W, C, I, kind):
    data = inputs.make(kind, 3 * C * S + 777, hash((S, W, C, I, kind)) & 0xffff, S)
    p = P(S, W, C, I)
    want, _ = ref_compress(data, p)
    got = plz.compress(data, p)
    assert got == want
    assert plz.decompress_bytes(got) == data


@pytest.mark.parametrize("I", [1, 16])
def test_decode_token_table_boundaries(I):
    # the fast decode holds one byte per token: S = 2 chunks with up to 1536
    # tokens decode there, more (mostly literals) through decode_chunk_smem;
    # chunks whose literal share steps across 1024 / 1536 / 2048 tokens
    rng = random.Random(1536 + I)
    C, chunks = 2048, []
    for k in range(40):
        frac = 0.3 + 0.7 * k / 39  # share of random (literal) symbols
        sym = []
        while len(sym) < C:
            if rng.random() < frac:
                sym.append(rng.randrange(65536))
            else:
                sym.extend([7, 7, 9, 7, 9, 9][: rng.randrange(2, 7)])
        chunks.append(b"".join(v.to_bytes(2, "little") for v in sym[:C]))
    data = b"".join(chunks) + b"\x05\x06" * 333
    p = P(2, 255, C, I)
    want, _ = ref_compress(data, p)
    got = plz.compress(data, p)
    assert got == want
    assert plz.decompress_bytes(got) == data
    assert ref_decompress(got) == data


@pytest.mark.parametrize("S,C", [(2, 2048), (2, 1024), (4, 1024), (4, 4096)])
def test_alphabet_tier_boundaries(S, C):
    # Kernel I's bitmap passes keep one occurrence row per distinct symbol of
    # a chunk (at most 16, then 32, then 64); chunks with more go to the
    # wide-cell pass.  Chunks with 1, 3, 7, 15-17, 31-33, 63-65, 255-257 and
    # C distinct symbols (extremes of the value range included), interleaved,
    # must all give the reference image.
    import numpy as np

    rng = np.random.default_rng(S * 100000 + C)
    top = (1 << (8 * S)) - 1
    chunks = []
    for d in (7, 16, 17, 32, 64, 256, 33, 65, 257, 1, 15, 31, 63, 255, C, 16, 3):
        if d == 1:
            alphabet = np.array([top], dtype=np.uint64)
        else:
            pool = np.unique(rng.integers(1, top, 4 * d, dtype=np.uint64))
            alphabet = np.concatenate([rng.permutation(pool)[: d - 2],
                                       np.array([0, top], dtype=np.uint64)])
        idx = np.concatenate([np.arange(d), rng.integers(0, d, C - d)])  # every symbol once
        idx = np.repeat(idx, rng.integers(1, 4, C))[:C]  # some runs
        idx[:d] = np.arange(d)
        chunks.append(alphabet[idx].astype(f"<u{S}"))
    data = np.concatenate(chunks).tobytes()
    for W, I in ((255, 1), (64, 2)):
        p = P(S, W, C, I)
        want, st_ref = ref_compress(data, p)
        stats = plz.PipelineStats()
        got = plz.compress(data, p, stats=stats)
        assert got == want, f"S={S} C={C} W={W} I={I}"
        assert (stats.pointer_tokens, stats.literal_tokens) == st_ref[1:]
        assert plz.decompress_bytes(got) == data


@pytest.mark.parametrize("C,W", [(4096, 128), (1024, 32), (2048, 255)])
def test_byte_alphabet_boundaries(C, W):
    # S = 1: chunks with 1..256 distinct byte values across the bitmap
    # passes' limits (16, 32, 64) and the wide-cell pass
    import numpy as np

    rng = np.random.default_rng(C + W)
    chunks = []
    for d in (7, 16, 17, 31, 32, 33, 63, 64, 65, 200, 256, 1, 3):
        alphabet = rng.permutation(256)[:d].astype(np.uint8)
        idx = np.concatenate([np.arange(d), rng.integers(0, d, C - d)])
        idx = np.repeat(idx, rng.integers(1, 5, C))[:C]
        idx[:d] = np.arange(d)
        chunks.append(alphabet[idx])
    data = np.concatenate(chunks).tobytes()
    for I in (1, 4):
        p = P(1, W, C, I)
        want, st_ref = ref_compress(data, p)
        stats = plz.PipelineStats()
        got = plz.compress(data, p, stats=stats)
        assert got == want, f"C={C} W={W} I={I}"
        assert (stats.pointer_tokens, stats.literal_tokens) == st_ref[1:]
        assert plz.decompress_bytes(got) == data


def test_bitmap_passes_in_sequence_on_a_large_input():
    # Inputs with many chunks per resident warp run the 16/32/64-row bitmap
    # passes one after the other (each takes the previous one's overflow);
    # small inputs sort the overflow first and run the 32/64-row passes side
    # by side.  A large input mixing alphabets of 7 .. 100 symbols per chunk
    # (on both sides of the 16 / 32 / 64-row boundaries) exercises the
    # sequential order; reference image required.
    import numpy as np

    rng = np.random.default_rng(77)
    S, C = 2, 2048
    chunks = []
    for k in range(20480):
        d = (7, 16, 17, 20, 24, 25, 32, 33, 40, 64, 65, 100)[k % 12]
        alphabet = rng.permutation(1024)[:d].astype("<u2") + 32000
        idx = np.repeat(rng.integers(0, d, C), rng.integers(1, 4, C))[:C]
        idx[:d] = np.arange(d)
        chunks.append(alphabet[idx])
    data = np.concatenate(chunks).tobytes()
    p = P(S, 255, C, 2)
    want, st_ref = ref_compress(data, p)
    stats = plz.PipelineStats()
    got = plz.compress(data, p, stats=stats)
    assert got == want
    assert (stats.pointer_tokens, stats.literal_tokens) == st_ref[1:]
    assert plz.decompress_bytes(got) == data


def test_concurrent_host_threads_give_identical_images():
    # SPEC: calls are pure functions, safe on distinct buffers from several
    # threads (one context per host thread); images must not depend on it.
    import threading

    inputs_ = [inputs.make(k, 300000 + 7 * i, 40 + i, 2) for i, k in
               enumerate(("quant", "runs", "alpha", "uniform", "quant", "periodic"))]
    p = P(2, 255, 2048, 2, 2048 * 2 * 16)
    want = [plz.compress(d, p) for d in inputs_]
    got = [None] * len(inputs_)
    back = [None] * len(inputs_)

    errors = [None] * len(inputs_)

    def work(i):
        try:
            for _ in range(3):
                got[i] = plz.compress(inputs_[i], p)
                back[i] = plz.decompress_bytes(got[i])
        except Exception as e:  # noqa: BLE001 — reported below with the thread's index
            errors[i] = repr(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(inputs_))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert errors == [None] * len(inputs_), errors
    assert got == want
    assert back == inputs_


def test_multi_block_images():
    # test_decoder.cpp:198-207: two chunks per block, five blocks and a tail
    p = P(2, 64, 1024, 1, 1024 * 2 * 2)
    data = inputs.make("alpha", 5 * p.block_bytes + 777, 62, 2)
    want, _ = ref_compress(data, p)
    got = plz.compress(data, p)
    assert got == want
    assert plz.decompress_bytes(got) == data


def test_concatenated_images_with_tails():
    # containers with tails followed by more containers (odd output offsets)
    parts = [inputs.make("alpha", n, n, 4) for n in (4099, 7, 12345, 3)]
    imgs = [plz.compress(d, P(4, 255, 4096, 2)) for d in parts]
    joined = b"".join(imgs)
    assert plz.decompress_bytes(joined) == b"".join(parts)
    assert ref_decompress(joined) == b"".join(parts)


def test_concatenated_images_of_mixed_symbol_widths():
    # one image whose containers alternate S = 2 (the S = 2 decode kernel)
    # and S = 1 / S = 4 (the other one): both kernels in one call, each
    # skipping the other's containers; odd output offsets after the tails
    import torch

    specs = [(2, 255, 2048, 2, 9000), (1, 128, 4096, 1, 7001), (2, 64, 1024, 4, 5003),
             (4, 255, 1024, 4, 12347), (2, 255, 2048, 1, 2 * 4096 * 3 + 2)]
    parts = [inputs.make("quant", n, 31 + n, S) for S, _, _, _, n in specs]
    imgs = [plz.compress(d, P(S, W, Cs, I)) for d, (S, W, Cs, I, _) in zip(parts, specs)]
    joined = b"".join(imgs)
    want = b"".join(parts)
    assert plz.decompress_bytes(joined) == want  # host path
    d_img = torch.frombuffer(bytearray(joined), dtype=torch.uint8).cuda()
    assert bytes(plz.decompress_bytes(d_img).cpu().numpy().tobytes()) == want  # resident path
    assert ref_decompress(joined) == want


def test_pinned_host_compress_by_container():
    # A host input of several segments into a pinned host image of several
    # containers takes the per-container pipeline (Kernel III writing into
    # the mapped host image); it must give the device path's image, which the
    # other tests pin to the reference.
    import numpy as np
    import torch

    for S, C, bb, size in ((2, 2048, 32 << 20, (100 << 20) + 4097), (4, 1024, 64 << 20, 150 << 20)):
        p = P(S, 255, C, 2, bb)
        data = np.frombuffer(inputs.make("quant", size, S + size, S), dtype=np.uint8)
        h_in = torch.from_numpy(data.copy()).pin_memory()
        cap = plz.compress_bound(size, p)
        h_img = torch.empty(cap, dtype=torch.uint8).pin_memory()
        ctx = plz.context()
        n_img, _ = ctx.compress_ptr(p, h_in.data_ptr(), size, h_img.data_ptr(), cap)
        dev = plz.compress(h_in.cuda(), p)
        assert n_img == dev.numel()
        assert torch.equal(h_img[:n_img], dev.cpu())
        assert torch.equal(plz.decompress_bytes(dev), h_in.cuda())
        # and back into a pinned host output (written by the decode kernel)
        h_out = torch.empty(size, dtype=torch.uint8).pin_memory()
        assert ctx.decompress_ptr(h_img.data_ptr(), n_img, h_out.data_ptr(), size) == size
        assert torch.equal(h_out, h_in)


def test_pinned_host_decompress_pipeline():
    # A pinned host image into a pinned host output takes the overlapped path
    # (image segments up, per-chunk waits in the decode kernel, output
    # segments down as they complete); tails come from the host walk.  A
    # corrupt image must fail exactly as the resident path does.
    import numpy as np
    import torch

    ctx = plz.context()
    for S, C, bb, size in ((1, 4096, 16 << 20, (70 << 20) + 3), (2, 2048, 32 << 20, (100 << 20) + 4097),
                           (4, 1024, 64 << 20, (150 << 20) + 3)):
        p = P(S, 255, C, 2, bb)
        data = np.frombuffer(inputs.make("quant", size, 7 * S + size, S), dtype=np.uint8)
        h_in = torch.from_numpy(data.copy()).pin_memory()
        dev = plz.compress(h_in.cuda(), p)
        n_img = dev.numel()
        h_img = dev.cpu().pin_memory()
        h_out = torch.zeros(size, dtype=torch.uint8).pin_memory()
        assert ctx.decompress_ptr(h_img.data_ptr(), n_img, h_out.data_ptr(), size) == size
        assert torch.equal(h_out, h_in)
        # corrupt flag bytes in the middle of the image and a truncation
        for mode in ("flags", "trunc"):
            bad = h_img.clone()
            if mode == "flags":
                bad[n_img // 2: n_img // 2 + 64] ^= 0x5A
                nb = n_img
            else:
                nb = n_img - 1000
            try:
                want = plz.decompress_bytes(bad[:nb].cuda()).cpu()
            except Exception as e:  # noqa: BLE001
                want = (type(e), str(e))
            try:
                got = h_out[:ctx.decompress_ptr(bad.data_ptr(), nb, h_out.data_ptr(), size)]
            except Exception as e:  # noqa: BLE001
                got = (type(e), str(e))
            if isinstance(want, tuple) or isinstance(got, tuple):
                assert got == want, (mode, got, want)
            else:
                assert torch.equal(got, want), mode
            if mode == "trunc":
                assert isinstance(want, tuple)


def test_device_resident_path_matches_host_path():
    import torch

    data = inputs.make("quant", 1 << 20, 5, 2)
    p = P(2, 255, 2048, 2)
    host = plz.compress(data, p)
    d = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    dev = plz.compress(d, p)
    assert dev.is_cuda and bytes(dev.cpu().numpy().tobytes()) == host
    back = plz.decompress_bytes(dev)
    assert back.is_cuda and torch.equal(back, d)


# ---------------------------------------------------------------- errors
def _err(fn, *a):
    try:
        fn(*a)
    except plz.Error as e:
        if isinstance(e, plz.CorruptionError):
            return (type(e).__name__, str(e), e.byte_offset, e.chunk_index, e.token_index)
        return (type(e).__name__, str(e), None, None, None)
    except O.OracleError as e:
        i = e.info
        name = {1: "ValidationError", 2: "UnsupportedFormatError", 3: "CorruptionError",
                4: "ContractError"}[i.code]
        if i.code != O.CORRUPTION:
            return (name, i.message, None, None, None)
        chunk = None if i.chunk_index == O.NO_INDEX else i.chunk_index
        tok = None if i.token_index == O.NO_INDEX else i.token_index
        off = i.byte_offset if chunk is None else 0
        return (name, i.message, off, chunk, tok)
    return None


def test_corrupted_images_raise_the_reference_error():
    # test_decoder.cpp:260-279, strengthened: same type, message, offsets
    rng = random.Random(66)
    data = inputs.make("alpha", 30000, 66, 1)
    p = P(1, 255, 1024, 1)
    img = plz.compress(data, p)
    same = 0
    for it in range(300):
        bad = bytearray(img)
        for _ in range(rng.choice([1, 1, 2, 4])):
            bad[rng.randrange(len(bad))] ^= rng.randrange(1, 256)
        bad = bytes(bad)
        mine = _err(plz.decompress_bytes, bad)
        theirs = _err(ref_decompress, bad)
        assert mine == theirs, f"iteration {it}"
        if mine is None:
            assert plz.decompress_bytes(bad) == ref_decompress(bad)
        same += 1
    assert same == 300


@pytest.mark.parametrize("S,C,kind", [(2, 2048, "quant"), (2, 1024, "runs"), (2, 2048, "alpha"),
                                       (4, 1024, "quant"), (4, 1024, "runs"), (1, 4096, "quant"),
                                       (1, 2048, "alpha")])
def test_corrupted_streams_raise_the_reference_error(S, C, kind):
    # the fast chunk decoder only accepts or rejects (rejected chunks are
    # re-walked for the exact error): corruptions of the flag / payload
    # streams and chunk-boundary shifts (table entries moved within their
    # neighbours, so the tables stay monotone) must give the reference's
    # outcome — the same error, or the same bytes
    import struct

    rng = random.Random(1000 * S + C)
    data = inputs.make(kind, 3 * C * S + 123 * S, 77, S)
    img = plz.compress(data, P(S, 255, C, 2))
    n = struct.unpack_from("<I", img, 21)[0]
    streams = 26 + 8 * (n + 1)
    ends = (streams, len(img) - img[25])
    for it in range(400):
        bad = bytearray(img)
        mode = rng.randrange(3)
        if mode < 2:
            for _ in range(rng.choice([1, 1, 2, 3])):
                bad[rng.randrange(*ends)] ^= 1 << rng.randrange(8) if mode else rng.randrange(1, 256)
        else:
            table, i = rng.randrange(2), rng.randrange(1, n)
            at = 26 + table * 4 * (n + 1) + 4 * i
            lo = struct.unpack_from("<I", bad, at - 4)[0]
            hi = struct.unpack_from("<I", bad, at + 4)[0]
            struct.pack_into("<I", bad, at, rng.randint(lo, hi))
        bad = bytes(bad)
        mine = _err(plz.decompress_bytes, bad)
        theirs = _err(ref_decompress, bad)
        assert mine == theirs, f"iteration {it}"
        if mine is None:
            assert plz.decompress_bytes(bad) == ref_decompress(bad)


def _table_entry(img, j_container, table, i, value):
    """Overwrite entry i of container j's payload (table 0) or flag (table 1)
    offset table in a concatenated image."""
    import struct

    at = 0
    for _ in range(j_container):
        n = struct.unpack_from("<I", img, at + 21)[0]
        ptot = struct.unpack_from("<I", img, at + 26 + 4 * n)[0]
        ftot = struct.unpack_from("<I", img, at + 26 + 4 * (n + 1) + 4 * n)[0]
        at += 26 + 8 * (n + 1) + ftot + ptot + img[at + 25]
    n = struct.unpack_from("<I", img, at + 21)[0]
    struct.pack_into("<I", img, at + 26 + table * 4 * (n + 1) + 4 * i, value)


def test_table_monotonicity_errors_in_reference_order():
    # The decode kernel checks each chunk's own table entries (format.cpp
    # checks the whole table before decoding any chunk): the reported error
    # must still be the reference's — chunk errors of earlier containers
    # first, then the first decreasing entry (payload before flag) — and
    # entries pointing past their stream must not be read.
    data = inputs.make("runs", 60000, 11, 2)
    p = P(2, 128, 1024, 1, 1024 * 2 * 8)  # 8 chunks per container, 4 containers
    img = plz.compress(data, p)
    cases = []
    for j, table, i, val in [(0, 0, 3, 0), (1, 1, 5, 0), (2, 0, 1, 0xFFFFFF00),
                             (3, 1, 2, 0xFFFFFFFF), (1, 0, 7, 1), (0, 1, 1, 0x7FFFFFFF)]:
        bad = bytearray(img)
        _table_entry(bad, j, table, i, val)
        cases.append(bytes(bad))
    # a payload byte flip in container 0's chunk 1 together with a decreasing
    # entry in container 2: the chunk error comes first
    bad = bytearray(cases[2])
    n0 = int.from_bytes(bad[21:25], "little")
    f0 = int.from_bytes(bad[26 + 4 * (n0 + 1) + 4 * n0: 26 + 4 * (n0 + 1) + 4 * n0 + 4], "little")
    flags_at = 26 + 8 * (n0 + 1)
    for k in range(40):
        bad[flags_at + f0 + k] ^= 0x5A
    cases.append(bytes(bad))
    for bad in cases:
        assert _err(plz.decompress_bytes, bad) == _err(ref_decompress, bad)


def test_truncations_raise_the_reference_error():
    data = inputs.make("runs", 20000, 3, 2)
    img = plz.compress(data, P(2, 128, 1024, 1, 4096))
    for cut in list(range(0, 80)) + list(range(len(img) - 40, len(img))):
        assert _err(plz.decompress_bytes, img[:cut]) == _err(ref_decompress, img[:cut])


def test_decompress_chunk_fuzz_matches_reference():
    # test_decoder.cpp:242-258: random slices decode or raise a located error
    rng = random.Random(65)
    for it in range(400):
        S = rng.choice([1, 2, 4])
        p = P(S, 255, 1024)
        op = O.make_params(S, 255, 1024, 1)
        flags = bytes(rng.randrange(256) for _ in range(1 + rng.randrange(8)))
        payload = bytes(rng.randrange(256) for _ in range(rng.randrange(64)))
        logical = 1 + rng.randrange(200)
        mine = _err(plz.decompress_chunk, flags, payload, logical, p, 7)
        f = O.ref_decompress_chunk if O.ref_available() else O.decompress_chunk
        theirs = _err(f, flags, payload, logical, op, 7)
        assert mine == theirs
        if mine is None:
            assert plz.decompress_chunk(flags, payload, logical, p, 7) == f(flags, payload,
                                                                            logical, op, 7)


def test_overlapping_pointer_replicates_period():
    # L L P(5,2) at S=2 replicates the period (decoder.cpp:80-84)
    flags = bytes([0b00100000])
    payload = bytes([1, 2, 3, 4, 5, 2])
    p = P(2, 255, 1024)
    got = plz.decompress_chunk(flags, payload, 7, p)
    assert got == bytes([1, 2, 3, 4] * 3 + [1, 2])


@pytest.mark.parametrize("field", ["symbol_width", "window", "chunk_size", "interval"])
def test_invalid_params_raise_validation_error(field):
    bad = {"symbol_width": 3, "window": 256, "chunk_size": 3000, "interval": 3}[field]
    raw = plz.Params()
    setattr(raw, field, bad)
    with pytest.raises(plz.ValidationError):
        plz.compress(b"abc", raw)


def test_random_grid_fuzz_against_the_reference():
    # random (S, W, C, I, block_bytes, size, input kind) over the whole
    # parameter space: bit-exact image and stats vs the reference, lossless
    # round trip, and a randomly corrupted copy of each image failing with
    # the reference's exact error (threads = 1 schedule)
    rng = random.Random(2024)
    kinds = ["quant", "runs", "alpha", "uniform", "periodic"]
    for it in range(600):
        S = rng.choice([1, 2, 4])
        C = rng.choice([1024, 2048, 4096, 8192, 16384])
        W = rng.choice([4, 5, 17, 32, 33, 64, 100, 128, 129, 200, 255])
        W = min(W, C - 1)
        I = rng.choice([1, 2, 4, 8, 16])
        bb = C * S * rng.choice([1, 2, 3, 7, 64])
        size = rng.choice([0, 1, S - 1, S, C * S - 1, C * S + 1, rng.randrange(1, 300000)])
        size = max(0, size)
        data = inputs.make(rng.choice(kinds), size, 1000 + it, S)
        p = P(S, W, C, I, bb)
        want, st = ref_compress(data, p)
        stats = plz.PipelineStats()
        got = plz.compress(data, p, stats=stats)
        assert got == want, f"iteration {it}: S={S} W={W} C={C} I={I} bb={bb} n={size}"
        assert (stats.pointer_tokens, stats.literal_tokens) == st[1:], f"iteration {it}"
        assert plz.decompress_bytes(got) == data, f"iteration {it}"
        if len(got) > 30:
            bad = bytearray(got)
            for _ in range(rng.choice([1, 2, 3])):
                bad[rng.randrange(len(bad))] ^= rng.randrange(1, 256)
            bad = bytes(bad)
            assert _err(plz.decompress_bytes, bad) == _err(ref_decompress, bad), f"iteration {it}"
