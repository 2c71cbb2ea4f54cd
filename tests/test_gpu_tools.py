"""GPU: the statistics / verification entry points of the path —
plzgpu_match_table (the matcher contract at EVERY position, matcher.cpp:113-131),
match-length histograms (corpus.cpp:75-129) and the tuner (tuner.cpp:10-45) —
against the reference, plus the CLI (tools/plz.cpp, tests/cli_test.cmake)."""
import os
import random
import subprocess

import pytest

import inputs
import oracle as O
from paper_2304_07342_b200 import plz

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2304_07342_b200", "lib", "plz_b200")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def ref_table(chunk, S, W, C, I):
    op = O.make_params(S, W, C, I)
    return (O.ref_match_chunk if O.ref_available() else O.match_chunk)(chunk, op)


def test_match_table_equals_reference_at_every_position():
    rng = random.Random(17)
    for it in range(120):
        S = rng.choice([1, 2, 4])
        W = rng.choice([4, 9, 32, 100, 128, 255])
        Cs = rng.choice([1024, 2048, 4096])
        I = rng.choice([1, 2, 4, 8, 16])
        n = 1 + rng.randrange(Cs)
        data = inputs.make(rng.choice(inputs.KINDS), n * S, it, S)
        p = plz.validate(plz.Params(S, W, Cs, I, Cs * S))
        ln, of = plz.match_table(data, p)
        rl, ro = ref_table(data, S, W, Cs, I)
        assert list(ln) == rl and list(of) == ro, f"S={S} W={W} C={Cs} I={I} n={n}"


def _ref_hist_encoded(data, p):
    """Tally pointer lengths of the reference image's tokens."""
    op = O.make_params(p.symbol_width, p.window, p.chunk_size, 1, p.block_bytes)
    img = O.ref_compress(data, op, 0) if O.ref_available() else O.compress(data, op)
    import struct

    counts = [0] * 256
    at = 0
    while at < len(img):
        n = struct.unpack_from("<I", img, at + 21)[0]
        pt = struct.unpack_from(f"<{n + 1}I", img, at + 26)
        ft = struct.unpack_from(f"<{n + 1}I", img, at + 26 + 4 * (n + 1))
        fs = at + 26 + 8 * (n + 1)
        ps = fs + ft[n]
        for k in range(n):
            fl, pl = img[fs + ft[k]:fs + ft[k + 1]], img[ps + pt[k]:ps + pt[k + 1]]
            i = 0
            for t in range(8 * len(fl)):
                if i >= len(pl):
                    break
                if (fl[t // 8] >> (7 - t % 8)) & 1:
                    counts[pl[i]] += 1
                    i += 2
                else:
                    i += p.symbol_width
        at = ps + pt[n] + img[at + 25]
    return counts


@pytest.mark.parametrize("S", [1, 2, 4])
def test_histograms_match_reference(S):
    data = inputs.make("runs", 60000, 3 + S, S)
    p = plz.validate(plz.Params(S, 255, 2048, 1))
    h = plz.match_length_histogram(data, p)
    assert h.counts == _ref_hist_encoded(data, p)
    raw = plz.match_length_histogram(data, p, raw_table=True)
    want = [0] * 256
    for k in range(0, len(data) // S, 2048):
        ln, of = ref_table(data[k * S:(k + 2048) * S], S, 255, 2048, 1)
        for l_, o_ in zip(ln, of):
            if o_ and l_:
                want[l_] += 1
    assert raw.counts == want


def test_tuner_decisions():
    # tuner.cpp:10-45 / test_tuner.cpp: noise -> S=1, quant-like u16 -> S=2, W=255
    rs = random.Random(5)
    noise = bytes(rs.randrange(256) for _ in range(1 << 18))
    base = plz.validate(plz.Params())
    assert plz.select_params([noise], 4, base).chosen.symbol_width == 1
    quant = inputs.make("quant", 1 << 18, 2, 2)
    rep = plz.select_params([quant], 2, base)
    assert (rep.chosen.symbol_width, rep.chosen.window) == (2, 255)


def _cli(*args, **kw):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, **kw)


@pytest.mark.skipif(not os.path.exists(CLI), reason="plz_b200 not built")
def test_cli_mirrors_reference_cli(tmp_path):
    # tests/cli_test.cmake, step by step
    src = tmp_path / "input.bin"
    src.write_bytes(b"0123456789abcdef0123456789abcdef" * 401)
    r = _cli("compress", "-S", 2, "-W", 128, "-C", 2048, src, tmp_path / "out.plz")
    assert r.returncode == 0 and "ratio: " in r.stdout
    if O.ref_available():  # the file is the reference's image, byte for byte
        assert (tmp_path / "out.plz").read_bytes() == O.ref_compress(
            src.read_bytes(), O.make_params(2, 128, 2048, 1), 1)
    assert _cli("decompress", tmp_path / "out.plz", tmp_path / "back.bin").returncode == 0
    assert (tmp_path / "back.bin").read_bytes() == src.read_bytes()
    r = _cli("compress", "--level", 4, src, tmp_path / "lvl.plz")
    assert r.returncode == 0 and "W: 255" in r.stdout
    assert _cli("compress", "--level", 4, "-W", 32, src, tmp_path / "x.plz").returncode == 2
    assert _cli("compress", "-W", 0, src, tmp_path / "x.plz").returncode == 2
    (tmp_path / "garbage.plz").write_bytes(b"XXXXnot a container at all")
    assert _cli("decompress", tmp_path / "garbage.plz", tmp_path / "y.bin").returncode == 3
    # --gpus: the same file from a device list (here the one GPU, three ranks)
    assert _cli("compress", "-S", 2, "-W", 128, "-C", 2048, "--block-bytes", 16384, "--gpus",
                "0,0,0", src, tmp_path / "multi.plz").returncode == 0
    assert _cli("compress", "-S", 2, "-W", 128, "-C", 2048, "--block-bytes", 16384, src,
                tmp_path / "single.plz").returncode == 0
    assert (tmp_path / "multi.plz").read_bytes() == (tmp_path / "single.plz").read_bytes()
    assert _cli("decompress", "--gpus", "0,0", tmp_path / "multi.plz",
                tmp_path / "mback.bin").returncode == 0
    assert (tmp_path / "mback.bin").read_bytes() == src.read_bytes()
    assert _cli("decompress", "--gpus", "0,0", tmp_path / "garbage.plz",
                tmp_path / "y.bin").returncode == 3
    r = _cli("stats", "-S", 1, src)
    assert r.returncode == 0 and "length,count,byte_length,fraction_gt_128,fraction_gt_256" in r.stdout
    r = _cli("tune", "--declared-width", 2, src)
    assert r.returncode == 0 and "chosen_S: " in r.stdout
    r = _cli("bench", "--kind", "runlen", "--size", 262144, "--seed", 1, "-W", "32,255",
             "--threads", 1)
    assert r.returncode == 0 and r.stdout.count("runlen,") == 2
