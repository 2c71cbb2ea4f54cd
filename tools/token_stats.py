"""Token-stream statistics behind the decode design: for the
first 4 MiB of c3 / c4 / c1, compressed by the C oracle, the share of
K-positions-per-lane waves (K = 4/S, 32K positions) that a pointer with an
offset below the wave width touches ("marked") and that truly hold a pointer
position whose source is a pointer position of the same wave ("need": the
decoder must resolve it in-wave).  CPU only; development aid."""
import struct
import sys

import numpy as np

sys.path.insert(0, "oracle")
sys.path.insert(0, ".")
import oracle as O  # noqa: E402
from paper_2304_07342_b200 import datagen  # noqa: E402


def stats(name, S, W, C, I, K):
    w = datagen.WORKLOADS[name]
    d = datagen.quant_codes(w, 42, "cpu").numpy()[:4 << 20]
    img = O.compress(d.tobytes(), O.make_params(S, W, C, I))
    n = struct.unpack_from("<I", img, 21)[0]
    pt = struct.unpack_from(f"<{n + 1}I", img, 26)
    ft = struct.unpack_from(f"<{n + 1}I", img, 26 + 4 * (n + 1))
    fs = 26 + 8 * (n + 1)
    ps = fs + ft[n]
    WV = 32 * K
    marked = need = waves = toks = 0
    for k in range(n):
        fl, pay = img[fs + ft[k]:fs + ft[k + 1]], img[ps + pt[k]:ps + pt[k + 1]]
        pos = i = t = 0
        isptr = np.zeros(C, bool)
        offpos = np.zeros(C, int)
        mk = set()
        while pos < C:
            if (fl[t >> 3] >> (7 - (t & 7))) & 1:
                ln, of = pay[i], pay[i + 1]
                i += 2
                isptr[pos:pos + ln] = True
                offpos[pos:pos + ln] = of
                if of < WV:
                    mk.update({pos // WV, (pos + ln - 1) // WV})
                pos += ln
            else:
                i += S
                pos += 1
            t += 1
        toks += t
        q = np.arange(C)
        s = q - offpos
        nd = isptr & (s // WV == q // WV) & isptr[np.clip(s, 0, C - 1)]
        need += len(set((q[nd] // WV).tolist()))
        marked += len(mk)
        waves += C // WV
    print(f"{name} K={K} waves/chunk={C // WV} tokens/chunk={toks / n:.1f} "
          f"marked={marked / waves:.3f} need={need / waves:.3f}")


if __name__ == "__main__":
    for K in (1, 2):
        stats("c3", 2, 255, 2048, 2, K)
    stats("c4", 4, 255, 1024, 4, 1)
    stats("c1", 1, 128, 4096, 1, 1)
    stats("c1", 1, 128, 4096, 1, 4)
