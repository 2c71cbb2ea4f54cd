"""numpy restatement of the cuSZ dual quantization — TEST INFRASTRUCTURE ONLY.

The reference library has no cuSZ code; the definition followed is the
paper's use case (PAPER.md "Use-case of gpuLZ", Table 3: cuSZ's dual-quant
codes fed to gpuLZ) as pinned in include/plzgpu.h (plzgpu_lorenzo_quantize):

  q    = rint(float32(f) * float32(1 / (2 eb)))      round half to even
  d    = Δx Δy Δz q  with q = 0 outside the field    (x fastest)
  code = d + radius if |d| < radius else 0           outliers: (index, d)
  f'   = float32(Σx Σy Σz d) * float32(2 eb)

Only tests/ import this module.
"""
import numpy as np


def lorenzo_quantize(field: np.ndarray, eb: float, radius: int):
    f = np.asarray(field, dtype=np.float32)
    if f.ndim == 1:
        f = f[None, None, :]
    elif f.ndim == 2:
        f = f[None, :, :]
    s = np.float32(1.0 / (2.0 * eb))
    q = np.rint(f * s).astype(np.int64)
    d = q
    for ax in range(3):
        d = np.diff(d, axis=ax, prepend=0)
    codes = np.where(np.abs(d) < radius, d + radius, 0).astype(np.uint16).reshape(-1)
    idx = np.flatnonzero(codes == 0).astype(np.int64)
    val = d.reshape(-1)[idx].astype(np.int32)
    return codes, idx, val


def lorenzo_reconstruct(codes, idx, val, shape, eb: float, radius: int) -> np.ndarray:
    nz, ny, nx = shape
    c = np.asarray(codes, dtype=np.int64).reshape(nz, ny, nx)
    d = np.where(c != 0, c - radius, 0)
    d.reshape(-1)[np.asarray(idx, dtype=np.int64)] = np.asarray(val, dtype=np.int64)
    q = d.cumsum(axis=2).cumsum(axis=1).cumsum(axis=0)
    return q.astype(np.float32) * np.float32(2.0 * eb)
