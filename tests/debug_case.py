"""Debug aid (test infrastructure, not collected): compress one golden case on the GPU and report the first token
that differs from the C oracle (position, oracle match, GPU token)."""
import json
import sys

sys.path[:0] = [".", "oracle", "tests"]
import inputs  # noqa: E402
import oracle as O  # noqa: E402
from paper_2304_07342_b200 import plz  # noqa: E402

G = json.load(open("tests/golden/golden.json"))
case = G["compress"][int(sys.argv[1])]
print({k: v for k, v in case.items() if k not in ("image_hex",)})
data = inputs.make(case["kind"], case["size"], case["seed"], case["S"])
S, W, C, I = case["S"], case["W"], case["C"], case["I"]
p = plz.validate(plz.Params(S, W, C, I, case["block_bytes"]))
op = O.make_params(S, W, C, I, case["block_bytes"])
gpu = plz.compress(data, p)
ref = O.compress(data, op)
print("lens", len(gpu), len(ref))


def tokens(img):
    n = int.from_bytes(img[21:25], "little")
    pt = [int.from_bytes(img[26 + 4 * i:30 + 4 * i], "little") for i in range(n + 1)]
    ft = [int.from_bytes(img[26 + 4 * (n + 1) + 4 * i:30 + 4 * (n + 1) + 4 * i], "little")
          for i in range(n + 1)]
    fs = 26 + 8 * (n + 1)
    ps = fs + ft[n]
    out = []
    for k in range(n):
        fl = img[fs + ft[k]:fs + ft[k + 1]]
        pl = img[ps + pt[k]:ps + pt[k + 1]]
        i = 0
        pos = 0
        for t in range(8 * len(fl)):
            if i >= len(pl):
                break
            bit = (fl[t // 8] >> (7 - t % 8)) & 1
            if bit:
                out.append((k, pos, "P", pl[i], pl[i + 1]))
                pos += pl[i]
                i += 2
            else:
                out.append((k, pos, "L", pl[i:i + S].hex()))
                pos += 1
                i += S
    return out


tg, tr = tokens(gpu), tokens(ref)
for a, b in zip(tg, tr):
    if a != b:
        k, pos = b[0], b[1]
        chunk = data[k * C * S:(k + 1) * C * S]
        ln, of = O.match_chunk(chunk, op)
        print("first diff: gpu", a, "ref", b, "oracle match at pos", (ln[pos], of[pos]))
        print("context", chunk[max(0, (pos - 8) * S):(pos + 8) * S].hex())
        break
else:
    print("tokens identical" if len(tg) == len(tr) else "length differs")
