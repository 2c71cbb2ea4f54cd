"""e2e host-buffer compress / decompress timing on the c2 workload, for A/B
of the H2D/D2H pipeline knobs (PLZGPU_SEG_MB, PLZGPU_COPY_MB, PLZGPU_TAIL_MB,
PLZGPU_DSEG_IN_MB, PLZGPU_DSEG_OUT_MB):  TAG=x python tools/e2e_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_07342_b200 import datagen, plz  # noqa: E402

w = datagen.WORKLOADS["c2"]
d_in = datagen.quant_codes(w, 42, "cuda")
n = d_in.numel()
p = plz.validate(plz.Params(w.S, w.W, w.C, w.I))
cap = plz.compress_bound(n, p)
ctx = plz.context(0)
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_in.copy_(d_in)
h_img = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
steps = 10


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(steps):
        r = fn()
    ev[1].record()
    torch.cuda.synchronize()
    return n / (ev[0].elapsed_time(ev[1]) / steps * 1e-3) / 1e9, r


c_gbs, (n_img, _) = timed(lambda: ctx.compress_ptr(p, h_in.data_ptr(), n, h_img.data_ptr(), cap))
want = plz.compress(d_in, p)
ok_c = n_img == want.numel() and torch.equal(h_img[:n_img], want.cpu())
d_gbs, _ = timed(lambda: ctx.decompress_ptr(h_img.data_ptr(), n_img, h_out.data_ptr(), n))
print(os.environ.get("TAG", ""), "e2e compress", round(c_gbs, 2), "decompress", round(d_gbs, 2),
      "ok", ok_c and bool(torch.equal(h_out, h_in)))
