"""CPU: pin the C restatement (oracle/plz_oracle.c) before trusting it.

1. The reference's own known-answer vectors (test_encoder.cpp, test_scan.cpp,
   test_format.cpp, test_decoder.cpp, test_matcher.cpp).
2. tests/golden/golden.json — images, errors and validation messages produced
   by the reference library itself (make_golden.py).
3. Seeded differential runs against oracle/_ref (the reference compiled from
   its sources) when it is present.
4. The reference's own unit-test suite, run against the reference build.
"""
import hashlib
import json
import os
import random
import subprocess

import pytest

import inputs
import oracle as O

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def P(S=2, W=128, C=2048, I=1, bb=256 << 20):
    return O.make_params(S, W, C, I, bb)


def err_of(fn, *a):
    try:
        fn(*a)
    except O.OracleError as e:
        i = e.info
        return {"code": i.code, "message": i.message, "byte_offset": i.byte_offset,
                "chunk_index": None if i.chunk_index == O.NO_INDEX else i.chunk_index,
                "token_index": None if i.token_index == O.NO_INDEX else i.token_index}
    return None


# ------------------------------------------------------------ known answers
def test_sixteen_equal_bytes():
    # test_encoder.cpp:44-52 -> flags 0x1C, payload AB AB AB 03 03 06 06 04 0C
    img = O.compress(b"\xab" * 16, P(1, 255, 1024))
    assert len(img) == 52 and img[-10:] == bytes.fromhex("1cababab030306060 40c".replace(" ", ""))


def test_four_equal_u32_symbols():
    # test_encoder.cpp:54-65 -> L, P(1,1), P(2,2); flags 0x60
    img = O.compress(bytes.fromhex("11223344") * 4, P(4, 255, 1024))
    assert img[-9:] == bytes.fromhex("60112233440101 0202".replace(" ", ""))


def test_distinct_symbols_are_literals():
    # test_encoder.cpp:34-42
    data = bytes(range(1, 9))
    img = O.compress(data, P(1, 255, 1024))
    assert img[-9:] == b"\x00" + data


def test_empty_and_tail_only():
    assert O.compress(b"", P()) == b""
    # a single byte at S=2: no chunk, one tail byte, 35-byte container
    assert O.compress(b"\x5a", P(2)).hex() == (
        "504c5a310102800100000800000100000000000000000000000100000000000000005a")


def test_empty_container_is_34_bytes():
    # test_format.cpp:30-39: header + two zero table entries
    img = O.compress(b"\x07", P(2))  # tail-only container: 34 + 1 tail byte
    assert len(img) == 35 and img[26:34] == bytes(8)


def test_u16_run_with_tail_intervals():
    # SURVEY.md §8c full-image goldens: 20 x u16 0x0200 + tail 07
    data = bytes.fromhex("0002") * 20 + b"\x07"
    i1 = O.compress(data, P(2, 128, 2048, 1))
    i4 = O.compress(data, P(2, 128, 2048, 4))
    assert len(i1) == 56 and i1[42:] == bytes.fromhex("3c000200020202040408080410" + "07")
    assert len(i4) == 58 and i4[42:] == bytes.fromhex("0e" + "0002" * 4 + "040408080410" + "07")


def test_decoder_inverses():
    # test_decoder.cpp:34-47
    payload = bytes(range(10, 18))
    assert O.decompress_chunk(b"\x00", payload, 8, P(1, 255)) == payload
    assert O.decompress_chunk(b"\x1c", bytes.fromhex("ababab030306060 40c".replace(" ", "")), 16,
                              P(1, 255)) == b"\xab" * 16


def test_matcher_known_answers():
    # test_matcher.cpp:46-72,114-148
    ln, of = O.match_chunk(bytes([7]) * 16, P(1, 255))
    assert (ln[8], of[8]) == (8, 8)
    ln, of = O.match_chunk(bytes(range(16)), P(1, 255))
    assert all(x == 0 for x in ln) and all(x == 0 for x in of)
    ln, of = O.match_chunk(b"ab" * 8, P(1, 255))
    assert (ln[2], of[2]) == (2, 2)
    ln, of = O.match_chunk(bytes([9]) * 16, P(1, 255, 2048, 4))
    assert all((ln[p], of[p]) == (1, 0) for p in range(16) if p % 4)
    assert (ln[4], of[4]) == (4, 4)
    ln, of = O.match_chunk(bytes([5]) * 16, P(1, 255))
    assert all(ln[p] == min(p, 16 - p) for p in range(16))


def test_validation_messages():
    # params.cpp:19-45
    with pytest.raises(O.OracleError, match="invalid window"):
        O.validate(P(2, 0))
    assert O.validate(P(4, 255, 16384)).min_match == 1
    assert O.validate(P(1, 4, 1024)).min_match == 3
    assert [O.olib().plzo_level_to_window(i) for i in range(6)] == [-1, 32, 64, 128, 255, -1]


# ----------------------------------------------------------------- goldens
@pytest.mark.parametrize("case", GOLDEN["compress"], ids=lambda c: f"g{c['id']}")
def test_golden_images(case):
    data = inputs.make(case["kind"], case["size"], case["seed"], case["S"])
    assert hashlib.sha256(data).hexdigest() == case["input_sha256"], "input generator drifted"
    img, st = O.compress_stats(data, P(case["S"], case["W"], case["C"], case["I"],
                                      case["block_bytes"]))
    assert len(img) == case["image_len"]
    assert hashlib.sha256(img).hexdigest() == case["image_sha256"]
    if "image_hex" in case:
        assert img.hex() == case["image_hex"]
    assert (st[1], st[2]) == (case["pointer_tokens"], case["literal_tokens"])
    assert O.decompress(img) == data


def _corrupt_image(entry):
    kind, size, seed, S, W, C, I, bb = GOLDEN["corrupt_bases"][entry["base"]]
    img = bytearray(O.compress(inputs.make(kind, size, seed, S), P(S, W, C, I, bb)))
    for at, x in entry["flips"]:
        img[at] ^= x
    return bytes(img[: entry["cut"]])


@pytest.mark.parametrize("idx", range(len(GOLDEN["corrupt"])))
def test_golden_corruption_errors(idx):
    entry = GOLDEN["corrupt"][idx]
    bad = _corrupt_image(entry)
    if "error" in entry:
        assert err_of(O.decompress, bad) == entry["error"]
    else:
        out = O.decompress(bad)
        assert (len(out), hashlib.sha256(out).hexdigest()) == (entry["ok_len"], entry["ok_sha256"])


def test_golden_chunk_slices():
    for entry in GOLDEN["chunks"]:
        p = P(entry["S"], 255, 1024)
        args = (bytes.fromhex(entry["flags"]), bytes.fromhex(entry["payload"]), entry["logical"],
                p, entry["chunk_index"])
        if "error" in entry:
            assert err_of(O.decompress_chunk, *args) == entry["error"]
        else:
            assert O.decompress_chunk(*args).hex() == entry["out_hex"]


def test_golden_validation():
    for entry in GOLDEN["validate"]:
        p = P(entry["S"], entry["W"], entry["C"], entry["I"], entry["block_bytes"])
        if "error" in entry:
            assert err_of(O.validate, p) == entry["error"]
        else:
            assert O.validate(p).min_match == entry["min_match"]


# ------------------------------------------- differential vs the reference
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")


@needs_ref
def test_oracle_matches_reference_random():
    rng = random.Random(7)
    for it in range(150):
        S = rng.choice([1, 2, 4])
        W = rng.choice([4, 17, 64, 128, 255])
        C = rng.choice([1024, 2048, 4096])
        I = rng.choice([1, 2, 4, 8, 16])
        bb = C * S * rng.choice([1, 2]) if rng.random() < 0.3 else 256 << 20
        data = inputs.make(rng.choice(inputs.KINDS), rng.randrange(0, 25000), it, S)
        p = P(S, W, C, I, bb)
        assert O.compress(data, p) == O.ref_compress(data, p, 1)


@needs_ref
def test_match_table_contract_vs_reference():
    # matcher.hpp:28-31: the full per-position table, every aligned position
    rng = random.Random(11)
    for it in range(200):
        S = rng.choice([1, 2, 4])
        n = 1 + rng.randrange(300)
        data = inputs.make(rng.choice(["alpha", "runs", "periodic", "constant"]), n * S, it, S)
        p = P(S, 4 + rng.randrange(252), 2048, rng.choice([1, 2, 4]))
        assert O.match_chunk(data, p) == O.ref_match_chunk(data, p)


REF_TESTS = os.path.join(os.path.dirname(O.HERE), "oracle", "_ref", "ref_unit_tests")


@pytest.mark.skipif(not os.path.exists(REF_TESTS), reason="reference unit tests not built")
def test_reference_unit_suite_passes_on_the_reference_build():
    # the reference's own 75 doctest cases, compiled with oracle/doctest_shim
    r = subprocess.run([REF_TESTS], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "failed: 0" in r.stdout
