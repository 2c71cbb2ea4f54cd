import sys, random, struct
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import inputs, oracle as O
from paper_2304_07342_b200 import plz
from test_gpu_parity import _err, ref_decompress, P
S, C, kind = 2, 2048, "quant"
rng = random.Random(1000 * S + C)
data = inputs.make(kind, 3 * C * S + 123 * S, 77, S)
img = plz.compress(data, P(S, 255, C, 2))
n = struct.unpack_from("<I", img, 21)[0]
streams = 26 + 8 * (n + 1)
ends = (streams, len(img) - img[25])
shown = 0
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
    mine = _err(plz.decompress_bytes, bad); theirs = _err(ref_decompress, bad)
    if mine != theirs:
        print(it, mode, "GPU", mine, "REF", theirs)
        open(f"gpurun_out/bad_{it}.bin", "wb").write(bad)
        shown += 1
        if shown > 5: break
