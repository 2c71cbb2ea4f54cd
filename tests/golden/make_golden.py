"""Generate tests/golden/golden.json from the REFERENCE library itself.

Run in the development container, where /root/reference is mounted and
oracle/_ref/libplzref.so has been built from its sources (make -C oracle ref):

    python tests/golden/make_golden.py

Every case records how its input is produced (tests/inputs.py, numpy PCG64,
machine-independent) plus the input's sha256, and what the reference
returned: the full image (hex) for small cases, its sha256/length and token
statistics otherwise; the exact exception (type, message, offsets) for
corrupted images and malformed chunk slices.  The fixtures pin the C
restatement (tests/test_oracle.py) and the GPU path (tests/test_gpu_golden.py)
on machines where the reference cannot be built.
"""
import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import inputs  # noqa: E402
import oracle as O  # noqa: E402


def err_dict(e: "O.OracleError"):
    i = e.info
    return {"code": i.code, "message": i.message, "byte_offset": i.byte_offset,
            "chunk_index": None if i.chunk_index == O.NO_INDEX else i.chunk_index,
            "token_index": None if i.token_index == O.NO_INDEX else i.token_index}


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def main():
    assert O.ref_available(), "build oracle/_ref first: make -C oracle ref"
    rng = random.Random(20260417)
    cases = []
    # ---- parameter grid x input kinds x edge sizes
    grid = [(S, W, C, I) for S in (1, 2, 4) for W in (4, 32, 128, 255)
            for C in (1024, 2048, 4096, 16384) for I in (1, 2, 4, 16) if C > W]
    for idx in range(240):
        S, W, C, I = grid[idx % len(grid)] if idx < len(grid) else rng.choice(grid)
        bb = C * S * rng.choice([1, 2, 3]) if idx % 5 == 0 else 256 << 20
        size = rng.choice([0, 1, S - 1, S + 1, C * S - 1, C * S, C * S + 3, rng.randrange(1, 40000)])
        kind = inputs.KINDS[idx % len(inputs.KINDS)]
        seed = 5000 + idx
        data = inputs.make(kind, size, seed, S)
        p = O.make_params(S, W, C, I, bb)
        img, st = O.ref_compress(data, p, 1, stats=True)
        case = {"id": idx, "kind": kind, "size": size, "seed": seed, "S": S, "W": W, "C": C,
                "I": I, "block_bytes": bb, "input_sha256": sha(data), "image_len": len(img),
                "image_sha256": sha(img), "pointer_tokens": st[1], "literal_tokens": st[2]}
        if len(img) <= 1536:
            case["image_hex"] = img.hex()
        cases.append(case)

    # ---- corrupted images: the reference's exact error (threads=1 schedule)
    corrupt = []
    base_specs = [("alpha", 9000, 66, 1, 255, 1024, 1, 256 << 20),
                  ("runs", 20000, 67, 2, 128, 1024, 2, 4096),
                  ("quant", 12000, 68, 4, 64, 1024, 4, 256 << 20)]
    for spec_i, (kind, size, seed, S, W, C, I, bb) in enumerate(base_specs):
        data = inputs.make(kind, size, seed, S)
        img = O.ref_compress(data, O.make_params(S, W, C, I, bb), 1)
        for it in range(60):
            bad = bytearray(img)
            flips = []
            for _ in range(rng.choice([1, 1, 2, 3])):
                at, x = rng.randrange(len(bad)), rng.randrange(1, 256)
                bad[at] ^= x
                flips.append([at, x])
            cut = len(bad) if rng.random() < 0.8 else rng.randrange(len(bad))
            bad = bytes(bad[:cut])
            entry = {"base": spec_i, "flips": flips, "cut": cut}
            try:
                out = O.ref_decompress(bad, 1)
                entry["ok_sha256"] = sha(out)
                entry["ok_len"] = len(out)
            except O.OracleError as e:
                entry["error"] = err_dict(e)
            corrupt.append(entry)

    # ---- malformed chunk slices (decompress_chunk)
    chunks = []
    for it in range(150):
        S = rng.choice([1, 2, 4])
        flags = bytes(rng.randrange(256) for _ in range(1 + rng.randrange(8)))
        payload = bytes(rng.randrange(256) for _ in range(rng.randrange(64)))
        logical = 1 + rng.randrange(200)
        p = O.make_params(S, 255, 1024, 1)
        entry = {"S": S, "flags": flags.hex(), "payload": payload.hex(), "logical": logical,
                 "chunk_index": 7}
        try:
            entry["out_hex"] = O.ref_decompress_chunk(flags, payload, logical, p, 7).hex()
        except O.OracleError as e:
            entry["error"] = err_dict(e)
        chunks.append(entry)

    # ---- validation messages (params.cpp:19-55)
    val = []
    for S, W, C, I, bb in [(3, 128, 2048, 1, 256 << 20), (2, 0, 2048, 1, 256 << 20),
                           (2, 256, 2048, 1, 256 << 20), (2, 128, 3000, 1, 256 << 20),
                           (2, 255, 1024, 3, 256 << 20), (2, 128, 2048, 1, 12345),
                           (1, 128, 1024, 16, 0), (4, 255, 16384, 1, 256 << 20),
                           (1, 4, 1024, 1, 1024)]:
        entry = {"S": S, "W": W, "C": C, "I": I, "block_bytes": bb}
        try:
            entry["min_match"] = O.ref_validate(O.make_params(S, W, C, I, bb)).min_match
        except O.OracleError as e:
            entry["error"] = err_dict(e)
        val.append(entry)

    doc = {"generator": "tests/golden/make_golden.py (reference: oracle/_ref/libplzref.so "
                        "built from /root/reference/proj/src)",
           "compress": cases, "corrupt_bases": [list(b) for b in base_specs],
           "corrupt": corrupt, "chunks": chunks, "validate": val}
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(doc, f, indent=0, separators=(",", ":"))
    print(f"wrote {len(cases)} compress, {len(corrupt)} corrupt, {len(chunks)} chunk, "
          f"{len(val)} validate cases")


if __name__ == "__main__":
    main()
