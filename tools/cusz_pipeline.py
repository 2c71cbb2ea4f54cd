"""The paper's use case on B200 (Table 3): cuSZ dual quantization ->
GPULZ, device-resident, on synthetic CESM-like / NYX-like float fields.

    python tools/cusz_pipeline.py [--eb 1e-2] [--steps 5]

Prints one JSON line per field: throughput in GB/s of float32 input for the
quantizer alone, quantizer + GPULZ compress (the improved cuSZ's first two
stages; Huffman is out of scope), and the inverse path, plus the compression
ratio float bytes / (image + outlier list) and the max reconstruction error.
CUDA-event timing, warm-up first; inputs exceed L2.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2304_07342_b200 import cusz, datagen, plz  # noqa: E402

FIELDS = {"cesm-like": (26, 1800, 3600), "nyx-like": (512, 512, 512)}


def timed(fn, steps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(2):
        out = fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(steps):
        out = fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / steps, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--eb", type=float, default=1e-2, help="relative error bound")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--interval", type=int, default=1)
    args = ap.parse_args()
    params = plz.validate(plz.Params(2, 255, 2048, args.interval))
    for name, shape in FIELDS.items():
        f = datagen._field(shape, 42, "cuda")
        f += datagen.NOISE_SIGMA * torch.randn(f.shape, device="cuda",
                                               generator=torch.Generator("cuda").manual_seed(7))
        eb = args.eb * float(f.max() - f.min())
        nbytes = f.numel() * 4
        tq, q = timed(lambda: cusz.quantize(f, eb), args.steps)
        tc, cf = timed(lambda: cusz.compress_field(f, eb, params), args.steps)
        td, back = timed(lambda: cusz.decompress_field(cf), args.steps)
        err = float((back - f).abs().max())
        print(json.dumps({
            "field": name, "shape": shape, "eb_rel": args.eb, "eb_abs": eb,
            "interval": args.interval, "float_bytes": nbytes,
            "quantize_gbs": nbytes / tq / 1e6,
            "quantize_plus_gpulz_gbs": nbytes / tc / 1e6,
            "decompress_gbs": nbytes / td / 1e6,
            "code_ratio": 2 * f.numel() / int(cf.image.numel()),
            "ratio": nbytes / cf.nbytes, "outliers": int(cf.outlier_idx.numel()),
            "max_abs_error": err, "within_eb": err <= eb * (1 + 1e-4),
        }))
        del f, q, cf, back
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
