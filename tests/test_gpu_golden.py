"""GPU: the B200 path against the reference's recorded outputs
(tests/golden/golden.json, produced by the reference library itself), so the
check holds on a box where neither /root/reference nor oracle/_ref exists."""
import hashlib
import json
import os

import pytest

import inputs
from paper_2304_07342_b200 import plz

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
ERRNAME = {1: plz.ValidationError, 2: plz.UnsupportedFormatError, 3: plz.CorruptionError,
           4: plz.ContractError}


def P(S, W, C, I, bb=256 << 20):
    return plz.validate(plz.Params(S, W, C, I, bb))


def check_error(exc, want):
    assert type(exc) is ERRNAME[want["code"]]
    assert str(exc) == want["message"]
    if want["code"] == 3:
        if want["chunk_index"] is None:
            assert exc.byte_offset == want["byte_offset"] and exc.chunk_index is None
        else:
            assert (exc.chunk_index, exc.token_index) == (want["chunk_index"], want["token_index"])


def test_golden_images_bit_exact():
    for case in GOLDEN["compress"]:
        data = inputs.make(case["kind"], case["size"], case["seed"], case["S"])
        stats = plz.PipelineStats()
        img = plz.compress(data, P(case["S"], case["W"], case["C"], case["I"], case["block_bytes"]),
                           stats=stats)
        assert len(img) == case["image_len"], case["id"]
        assert hashlib.sha256(img).hexdigest() == case["image_sha256"], case["id"]
        assert (stats.pointer_tokens, stats.literal_tokens) == (case["pointer_tokens"],
                                                                case["literal_tokens"])
        assert plz.decompress_bytes(img) == data


def test_golden_corruptions_raise_the_reference_error():
    bases = []
    for kind, size, seed, S, W, C, I, bb in GOLDEN["corrupt_bases"]:
        bases.append(plz.compress(inputs.make(kind, size, seed, S), P(S, W, C, I, bb)))
    for entry in GOLDEN["corrupt"]:
        img = bytearray(bases[entry["base"]])
        for at, x in entry["flips"]:
            img[at] ^= x
        bad = bytes(img[: entry["cut"]])
        if "error" in entry:
            with pytest.raises(plz.Error) as ei:
                plz.decompress_bytes(bad)
            check_error(ei.value, entry["error"])
        else:
            out = plz.decompress_bytes(bad)
            assert hashlib.sha256(out).hexdigest() == entry["ok_sha256"]


def test_golden_chunk_slices():
    for entry in GOLDEN["chunks"]:
        args = (bytes.fromhex(entry["flags"]), bytes.fromhex(entry["payload"]), entry["logical"],
                P(entry["S"], 255, 1024, 1), entry["chunk_index"])
        if "error" in entry:
            with pytest.raises(plz.Error) as ei:
                plz.decompress_chunk(*args)
            check_error(ei.value, entry["error"])
        else:
            assert plz.decompress_chunk(*args).hex() == entry["out_hex"]
