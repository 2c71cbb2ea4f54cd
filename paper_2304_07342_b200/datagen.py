"""Synthetic cuSZ-style quantization codes for the BASELINE workloads.

SURVEY.md §8d: a smooth field (sum of K=8 random separable sinusoids plus
small Gaussian noise) is pre-quantised with an error bound of 1e-3 x range
(the paper's relative bound), passed through the integer
Lorenzo predictor (1-D for c1, 3-D otherwise) and mapped to codes
``d + radius`` (|d| < radius) or 0 (outlier) — a dominant centre code with
±1..±8 neighbours and rare zeros, the shape of real dual-quant codes.

Generation runs in torch (CUDA when available) and is deterministic for a
given (shape, seed, device); the bytes handed to the CPU reference are the
same tensor copied to the host.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Tuple

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    shape: Tuple[int, ...]
    dtype: str          # "u8" | "u16" | "u32"
    radius: int
    S: int
    W: int
    C: int
    I: int
    lorenzo: int        # 1 or 3 (dimensions)
    fields: int = 1     # independent fields of `shape`, seeds seed+k, back to back

    @property
    def field_bytes(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n * {"u8": 1, "u16": 2, "u32": 4}[self.dtype]

    @property
    def n_bytes(self) -> int:
        return self.fields * self.field_bytes


# BASELINE.json configs; "window 256" runs as W=255 (params.cpp:22-23), a
# 4096-byte data block is C = 4096 / S symbols.
WORKLOADS = {
    "c1": Workload("c1-u8-quant-16MiB", (16 << 20,), "u8", 64, 1, 128, 4096, 1, 1),
    "c2": Workload("c2-u16-cesm-26x1800x3600", (26, 1800, 3600), "u16", 512, 2, 255, 2048, 2, 3),
    "c3": Workload("c3-u16-nyx-512^3", (512, 512, 512), "u16", 512, 2, 255, 2048, 1, 3),
    "c4": Workload("c4-u32-1GiB", (256, 1024, 1024), "u32", 512, 4, 255, 1024, 4, 3),
    # 8 GiB as 32 NYX-like 256 MiB fields with seeds 42+k — one
    # 256 MiB container each at the default block size, so the stream's first
    # container is exactly c3's field (seed 42)
    "c5": Workload("c5-u16-8GiB", (512, 512, 512), "u16", 512, 2, 255, 2048, 2, 3, fields=32),
}
# Field model, in units of the quantisation step 2*eb.  With a relative error
# bound of 1e-3 the value range spans 1 / (2 * 1e-3) = 500 steps: localised
# Gaussian "halos" reach that height, while the smooth background (8 separable
# sinusoids) moves by well under a step per grid point, so most Lorenzo
# residuals are 0 and the code stream is dominated by the centre code — the
# statistics of NYX/CESM quant codes (CR 5-9 at S=2, W=255).
ERROR_BOUND = 1e-3
RANGE_STEPS = 1.0 / (2 * ERROR_BOUND)
BG_AMPLITUDE = (1.0, 6.0)     # per-sinusoid amplitude, steps
BG_CYCLES = (0.3, 2.0)        # cycles per axis
N_HALOS = 24
HALO_WIDTH = (3.0, 12.0)      # grid points (std-dev)
NOISE_SIGMA = 0.12            # steps


def _field(shape, seed: int, device):
    import torch

    g = torch.Generator(device="cpu").manual_seed(seed)

    def rnd(lo, hi):
        return lo + (hi - lo) * float(torch.rand((), generator=g))

    dims = len(shape)

    def axis(d, n, fn):
        x = torch.arange(n, device=device, dtype=torch.float32)
        view = [1] * dims
        view[d] = n
        return fn(x).view(view)

    f = torch.zeros(shape, device=device, dtype=torch.float32)
    for _ in range(8):
        amp = rnd(*BG_AMPLITUDE)
        term = None
        for d, n in enumerate(shape):
            k = rnd(*BG_CYCLES) * 2 * np.pi / n
            ph = rnd(0, 2 * np.pi)
            ax = axis(d, n, lambda x: torch.sin(x * k + ph))
            term = ax if term is None else term * ax
        f += amp * term
    for h in range(N_HALOS):
        height = RANGE_STEPS * (1.0 if h == 0 else rnd(0.05, 0.8))
        term = None
        for d, n in enumerate(shape):
            c, wd = rnd(0, n), rnd(*HALO_WIDTH)
            ax = axis(d, n, lambda x: torch.exp(-0.5 * ((x - c) / wd) ** 2))
            term = ax if term is None else term * ax
        f += height * term
    return f


def quant_codes(w: Workload, seed: int = 42, device=None, fields=None):
    """Return a flat torch.uint8 tensor with the workload's code bytes.

    Multi-field workloads (c5) are the concatenation of fields k = 0..F-1,
    field k generated from seed + k; `fields` = (first, end) selects a
    contiguous run of them (a rank's share, or the reference arm's first
    container) without generating the rest."""
    import torch

    if device is None:
        device = "cuda" if torch.cuda.is_available() else "cpu"
    if w.fields > 1 or fields is not None:
        k0, k1 = fields if fields is not None else (0, w.fields)
        out = torch.empty((k1 - k0) * w.field_bytes, dtype=torch.uint8, device=device)
        for k in range(k0, k1):
            out[(k - k0) * w.field_bytes:(k - k0 + 1) * w.field_bytes] = _one_field(w, seed + k, device)
        return out
    return _one_field(w, seed, device)


def _one_field(w: Workload, seed: int, device):
    import torch

    f = _field(w.shape, seed, device)
    gen = torch.Generator(device=device).manual_seed(seed + 1000)
    f += NOISE_SIGMA * torch.randn(f.shape, generator=gen, device=device, dtype=torch.float32)
    q = torch.round(f).to(torch.int32)
    del f
    if w.lorenzo == 1:
        flat = q.reshape(-1)
        d = flat.clone()
        d[1:] -= flat[:-1]
    else:
        # 3-D Lorenzo residual = product of first differences along each axis
        d = q
        for axis in range(3):
            s = d.clone()
            hi = [slice(None)] * 3
            lo = [slice(None)] * 3
            hi[axis] = slice(1, None)
            lo[axis] = slice(None, -1)
            s[tuple(hi)] -= d[tuple(lo)]
            d = s
    codes = torch.where(d.abs() < w.radius, d + w.radius, torch.zeros_like(d))
    if w.dtype == "u8":
        codes = codes.to(torch.uint8)
    elif w.dtype == "u16":
        codes = codes.to(torch.int16)  # codes < 2 * radius <= 1024
    else:
        codes = codes.to(torch.int32)
    return codes.reshape(-1).contiguous().view(torch.uint8)


def small_quant_codes(n_symbols: int, S: int, seed: int = 42, radius: int = None) -> bytes:
    """Host-side, numpy-only 1-D variant for CPU tests and golden fixtures."""
    rs = np.random.default_rng(seed)
    x = np.arange(n_symbols, dtype=np.float64)
    f = np.zeros(n_symbols)
    for _ in range(8):
        f += (rs.random() + 0.25) * np.sin(x * (rs.random() * 5 + 0.5) * 2 * np.pi / max(1, n_symbols) * 8
                                           + rs.random() * 2 * np.pi)
    rng = float(f.max() - f.min()) or 1.0
    q = np.round(f / (2 * ERROR_BOUND * rng) + NOISE_SIGMA * rs.standard_normal(n_symbols)).astype(np.int64)
    d = np.diff(q, prepend=0)
    radius = radius or (64 if S == 1 else 512)
    codes = np.where(np.abs(d) < radius, d + radius, 0)
    return codes.astype({1: "u1", 2: "<u2", 4: "<u4"}[S]).tobytes()
