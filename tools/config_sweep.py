"""Every BASELINE.json config on one B200 (bench.py's headline is c5):

    python tools/config_sweep.py [--steps 5] [--configs c1,c2,c3,c4,c5] [--cpu]

c1  u8 16 MiB, W=128, I=1           (the reference's CPU-runnable case)
c2  u16 CESM-like, W=255, I=2
c3  u16 NYX-like 512^3, W=255, I in {1,2,4,8,16}: ratio vs throughput
c4  u32 1 GiB, W=255, I=4           (decompression focus)
c5  u16 8 GiB (32 NYX-like fields), W=255, I=2, one GPU (bench.py's workload)

One JSON line per (config, I): compress / decompress GB/s of input bytes
(device-resident, CUDA events, warm-up first, inputs > L2 except c1), ratio,
round-trip check.  --cpu adds the reference library on all host threads over
the stream's first container of each config (bench.py --impl reference), for the ratio /
throughput beside it.
"""
import argparse
import json
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2304_07342_b200 import datagen, plz  # noqa: E402


def gen(name):
    w = datagen.WORKLOADS[name]
    if name != "c5":
        return w, datagen.quant_codes(w, 42, "cuda")
    # 8 GiB as 32 NYX-like 256 MiB fields with seeds 42+k
    f = datagen.Workload("nyx", (512, 512, 512), "u16", 512, 2, 255, 2048, 2, 3)
    out = torch.empty(w.n_bytes, dtype=torch.uint8, device="cuda")
    step = f.n_bytes
    for k in range(w.n_bytes // step):
        out[k * step:(k + 1) * step] = datagen.quant_codes(f, 42 + k, "cuda")
        torch.cuda.synchronize()
    return w, out


def run(ctx, d_in, params, steps):
    n = d_in.numel()
    cap = plz.compress_bound(n, params)
    img = torch.empty(cap, dtype=torch.uint8, device="cuda")
    ln = torch.zeros(2, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(2):
        ctx.compress_async(params, d_in.data_ptr(), n, img.data_ptr(), cap, ln.data_ptr(), st)
    ctx.finish(st)
    ev[0].record()
    for _ in range(steps):
        ctx.compress_async(params, d_in.data_ptr(), n, img.data_ptr(), cap, ln.data_ptr(), st)
    ev[1].record()
    torch.cuda.synchronize()
    c_ms = ev[0].elapsed_time(ev[1]) / steps
    ptr, lit = ctx.finish(st)
    n_img = int(ln[0].item())
    out = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        ctx.decompress_async(img.data_ptr(), n_img, out.data_ptr(), out.numel(), ln.data_ptr() + 8, st)
    ctx.finish(st)
    ev[0].record()
    for _ in range(steps):
        ctx.decompress_async(img.data_ptr(), n_img, out.data_ptr(), out.numel(), ln.data_ptr() + 8, st)
    ev[1].record()
    torch.cuda.synchronize()
    d_ms = ev[0].elapsed_time(ev[1]) / steps
    ctx.finish(st)
    ok = bool(torch.equal(out[:n], d_in))
    del out, img
    return {"compress_gbs": n / c_ms / 1e6, "decompress_gbs": n / d_ms / 1e6,
            "compress_ms": c_ms, "decompress_ms": d_ms, "ratio": n / n_img,
            "pointer_tokens": ptr, "literal_tokens": lit, "roundtrip_ok": ok}


def cpu_ref(name, I):
    """The reference library on all host cores over the stream's first
    container (256 MiB, or the whole input when smaller), through bench.py's
    reference arm (the one place outside tests/ that runs oracle/)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--workload", name, "--interval", str(I), "--steps", "2", "--warmup", "0"],
                       capture_output=True, text=True)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        return {"cpu_compress_gbs": d["value"], "cpu_decompress_gbs": d["decompress"]["value"],
                "cpu_ratio": d["ratio"], "cpu_cores": d["cpu_baseline"]["cores"],
                "cpu_sample_bytes": d["cpu_baseline"]["sample_bytes"]}
    except (IndexError, KeyError, ValueError):
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--cpu", action="store_true")
    args = ap.parse_args()
    ctx = plz.context(0)
    for name in args.configs.split(","):
        w, d_in = gen(name)
        intervals = (1, 2, 4, 8, 16) if name == "c3" else (w.I,)
        for I in intervals:
            params = plz.validate(plz.Params(w.S, w.W, w.C, I))
            r = run(ctx, d_in, params, args.steps)
            line = {"config": name, "workload": w.name, "bytes": d_in.numel(), "S": w.S,
                    "W": w.W, "C": w.C, "I": I, **r}
            if args.cpu:
                line.update(cpu_ref(name, I) or {})
            print(json.dumps(line), flush=True)
        del d_in
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
