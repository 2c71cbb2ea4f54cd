"""e2e host-buffer compress/decompress timing on the c2 workload (A/B of env knobs)."""
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
n_img = ctx.compress_ptr(p, h_in.data_ptr(), n, h_img.data_ptr(), cap)[0]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(3):
    ctx.decompress_ptr(h_img.data_ptr(), n_img, h_out.data_ptr(), n)
steps = 10
ev[0].record()
for _ in range(steps):
    ctx.decompress_ptr(h_img.data_ptr(), n_img, h_out.data_ptr(), n)
ev[1].record()
torch.cuda.synchronize()
print(os.environ.get("TAG", ""), "e2e decompress GB/s", n / (ev[0].elapsed_time(ev[1]) / steps * 1e-3) / 1e9,
      "ok", bool(torch.equal(h_out, h_in)))
