"""Compress throughput vs. alphabet size per chunk (development aid): u16
quant-like codes whose per-chunk distinct-symbol count is steered by the
spread of a discretised Laplace distribution around a centre code, so the
bitmap passes (16 / 64 rows) and the wide-cell pass each get exercised."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2304_07342_b200 import plz  # noqa: E402

n = 256 << 20
g = torch.Generator(device="cuda").manual_seed(5)
p = plz.validate(plz.Params(2, 255, 2048, 2))
ctx = plz.context()
for scale in (0.5, 2.0, 6.0, 20.0, 80.0):
    u = torch.rand(n // 2, generator=g, device="cuda") - 0.5
    lap = -scale * torch.sign(u) * torch.log1p(-2 * u.abs())
    # runs: repeat each value a geometric number of times
    codes = (512 + lap.round().clamp(-511, 511)).to(torch.int16)
    rep = torch.randint(1, 6, (n // 2,), generator=g, device="cuda")
    codes = torch.repeat_interleave(codes, rep)[: n // 2].contiguous()
    d = codes.view(torch.uint8)
    sym = codes.view(-1, 2048)
    distinct = torch.tensor([torch.unique(sym[i]).numel() for i in range(0, sym.shape[0], 997)])
    cap = plz.compress_bound(d.numel(), p)
    img = torch.empty(cap, dtype=torch.uint8, device="cuda")
    ln = torch.zeros(2, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        ctx.compress_async(p, d.data_ptr(), d.numel(), img.data_ptr(), cap, ln.data_ptr(), st)
    ctx.finish(st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ctx.compress_async(p, d.data_ptr(), d.numel(), img.data_ptr(), cap, ln.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"scale {scale:5.1f}: distinct/chunk median {distinct.median().item():4d} "
          f"max {distinct.max().item():4d}  compress {d.numel() / ms / 1e6:6.1f} GB/s  "
          f"CR {d.numel() / int(ln[0].item()):.2f}", flush=True)
