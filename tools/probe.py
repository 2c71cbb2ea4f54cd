"""Quick device-resident timing probe: compress/decompress throughput of a
BASELINE workload (kernels only, CUDA events).  Development aid; bench.py is
the contract."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2304_07342_b200 import datagen, plz  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = datagen.WORKLOADS[name]
t0 = time.time()
d_in = datagen.quant_codes(w, 42, "cuda")
torch.cuda.synchronize()
print(f"{w.name}: {d_in.numel()/1e6:.1f} MB generated in {time.time()-t0:.1f}s", flush=True)
import os
W = int(os.environ.get("PROBE_W", w.W))
I = int(os.environ.get("PROBE_I", w.I))
p = plz.validate(plz.Params(w.S, W, w.C, I))
if W != w.W or I != w.I:
    print(f"override W={W} I={I}")
ctx = plz.context()
cap = plz.compress_bound(d_in.numel(), p)
img = torch.empty(cap, dtype=torch.uint8, device="cuda")
ln = torch.zeros(2, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    ctx.compress_async(p, d_in.data_ptr(), d_in.numel(), img.data_ptr(), cap, ln.data_ptr(), st)
ctx.finish(st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    ctx.compress_async(p, d_in.data_ptr(), d_in.numel(), img.data_ptr(), cap, ln.data_ptr(), st)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
n_img = int(ln[0].item())
print(f"compress: {ms:.3f} ms/step  {d_in.numel()/ms/1e6:.1f} GB/s  CR {d_in.numel()/n_img:.3f}", flush=True)
out = torch.empty(d_in.numel() + 16, dtype=torch.uint8, device="cuda")
for _ in range(2):
    ctx.decompress_async(img.data_ptr(), n_img, out.data_ptr(), out.numel(), ln.data_ptr() + 8, st)
ctx.finish(st)
e0.record()
for _ in range(iters):
    ctx.decompress_async(img.data_ptr(), n_img, out.data_ptr(), out.numel(), ln.data_ptr() + 8, st)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
ok = torch.equal(out[: d_in.numel()], d_in)
print(f"decompress: {ms:.3f} ms/step  {d_in.numel()/ms/1e6:.1f} GB/s  roundtrip={ok}", flush=True)
