"""CPU: host-side logic of the B200 library (no kernel launches).

The C-ABI library loads, exports every entry point include/plzgpu.h declares,
and its host functions (validate, level_to_window, plan, container_size,
compress_bound, decompressed_bound) follow the reference's contract
(params.cpp, partition.cpp, format.cpp) — checked against the golden
fixtures and the C oracle."""
import ctypes as C
import json
import os
import random
import re

import pytest

import inputs
import oracle as O
from paper_2304_07342_b200 import _lib as L
from paper_2304_07342_b200 import plz

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "plzgpu.h")).read()
    return sorted(set(re.findall(r"\b(plzgpu_\w+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = L.lib()
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/plzgpu.h but not exported"
    assert lib.plzgpu_abi_version() == 1
    # the ctypes table covers the header exactly
    assert sorted(n for n, _, _ in L.SIGNATURES) == syms


def test_validate_matches_reference_messages():
    for entry in GOLDEN["validate"]:
        raw = plz.Params(entry["S"], entry["W"], entry["C"], entry["I"], entry["block_bytes"])
        if "error" in entry:
            with pytest.raises(plz.ValidationError) as ei:
                plz.validate(raw)
            assert str(ei.value) == entry["error"]["message"]
        else:
            assert plz.validate(raw).min_match == entry["min_match"]


def test_min_match_rule():
    # test_params.cpp:400-408: min_match*S > 2 and (min_match-1)*S <= 2
    for S in (1, 2, 4):
        m = plz.validate(plz.Params(symbol_width=S)).min_match
        assert m * S > 2 and (m - 1) * S <= 2


def test_level_to_window():
    assert [plz.level_to_window(i) for i in (1, 2, 3, 4)] == [32, 64, 128, 255]
    for bad in (0, 5):
        with pytest.raises(plz.ValidationError, match="invalid level"):
            plz.level_to_window(bad)


def test_plan_known_answers():
    # test_partition.cpp:444-478
    p = plz.validate(plz.Params(2, 128, 2048))
    (b,) = plz.plan(5001, p)
    assert (b.num_chunks, b.last_chunk_len, b.tail_len) == (2, 452, 1)
    assert plz.plan(0, p) == []
    q = plz.validate(plz.Params(2, 128, 1024, 1, 4096))
    blocks = plz.plan(4096 * 3 + 5, q)
    assert len(blocks) == 4 and blocks[3].byte_len == 5 and blocks[3].last_chunk_len == 2


def test_plan_covers_input():
    # test_partition.cpp:480-506
    rng = random.Random(7)
    for _ in range(500):
        S, Cs = rng.choice([1, 2, 4]), rng.choice([1024, 2048, 4096])
        p = plz.validate(plz.Params(S, 128, Cs, 1, Cs * S * (1 + rng.randrange(4))))
        total = rng.randrange(200000)
        covered, start = 0, 0
        for b in plz.plan(total, p):
            assert b.byte_start == start and b.tail_len < S
            syms = (b.num_chunks - 1) * Cs + b.last_chunk_len if b.num_chunks else 0
            assert syms * S + b.tail_len == b.byte_len
            start += b.byte_len
            covered += b.byte_len
        assert covered == total


def test_container_size_and_bounds():
    assert plz.container_size(0, 0, 0, 0) == 34
    assert plz.container_size(1, 1, 9, 0) == 26 + 16 + 10
    for case in GOLDEN["compress"]:
        p = plz.validate(plz.Params(case["S"], case["W"], case["C"], case["I"],
                                    case["block_bytes"]))
        assert plz.compress_bound(case["size"], p) >= case["image_len"]


def test_decompressed_bound_walks_valid_prefix():
    lib = L.lib()
    for case in GOLDEN["compress"][:60]:
        data = inputs.make(case["kind"], case["size"], case["seed"], case["S"])
        img = O.compress(data, O.make_params(case["S"], case["W"], case["C"], case["I"],
                                             case["block_bytes"]))
        buf = C.create_string_buffer(img, len(img) or 1)
        assert lib.plzgpu_decompressed_bound(buf, len(img)) == len(data)
    # a corrupted header stops the walk: never more than the valid prefix
    data = inputs.make("runs", 50000, 1, 2)
    img = bytearray(O.compress(data, O.make_params(2, 128, 1024, 1, 8192)))
    img[len(img) // 2] ^= 0xFF
    buf = C.create_string_buffer(bytes(img), len(img))
    assert lib.plzgpu_decompressed_bound(buf, len(img)) <= len(data)


def test_error_classes_mirror_reference_hierarchy():
    for cls in (plz.ValidationError, plz.UnsupportedFormatError, plz.CorruptionError,
                plz.ContractError):
        assert issubclass(cls, plz.Error)
    assert plz.validation_error is plz.ValidationError
    e = plz.CorruptionError("x", 5)
    assert (e.byte_offset, e.chunk_index, e.token_index) == (5, None, None)


def test_drop_in_headers_declare_the_reference_api():
    # include/plz mirrors /root/reference/proj/include/plz for the boundary
    text = "".join(open(os.path.join(ROOT, "include", "plz", f)).read()
                   for f in os.listdir(os.path.join(ROOT, "include", "plz")))
    for sym in ("Params validate(Params raw)", "int level_to_window(int level)",
                "PartitionPlan plan(", "std::vector<std::uint8_t> compress(",
                "Container compress_block(", "std::vector<std::uint8_t> decompress_bytes(",
                "std::vector<std::uint8_t> decompress(const Container& container",
                "std::vector<std::uint8_t> decompress_chunk(", "parse_token_stream(",
                "Container read_container(", "std::vector<std::uint8_t> write_container(",
                "void append_container(", "std::size_t container_size(", "struct corruption_error"):
        assert sym in text, sym
