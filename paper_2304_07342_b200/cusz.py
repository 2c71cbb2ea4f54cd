"""cuSZ + GPULZ on the device — the paper's use case (PAPER.md "Use-case of
gpuLZ", Table 3).

cuSZ's dual quantization turns a float field into u16 quantization codes
(plus a short outlier list); the improved cuSZ of the paper runs GPULZ on
those codes (Huffman, the stage after it, is out of scope here).  Everything
stays in HBM: ``compress_field`` = quantizer kernel -> GPULZ compress of the
code bytes; ``decompress_field`` = GPULZ decompress -> inverse-Lorenzo
kernels.  The kernels live in ``csrc/cusz.cu`` behind
``plzgpu_lorenzo_quantize`` / ``plzgpu_lorenzo_reconstruct``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Tuple

from . import _lib as L
from . import plz


@dataclass
class QuantCodes:
    codes: "object"         # torch.uint16-as-int16 device tensor, nx*ny*nz codes
    outlier_idx: "object"   # int64 device tensor, increasing element indices
    outlier_val: "object"   # int32 device tensor, Lorenzo residuals of the outliers
    shape: Tuple[int, int, int]  # (nz, ny, nx), x fastest
    eb: float
    radius: int


def _dims(shape):
    if len(shape) == 1:
        return 1, 1, shape[0]
    if len(shape) == 2:
        return 1, shape[0], shape[1]
    if len(shape) == 3:
        return tuple(shape)
    raise plz.ValidationError("fields are 1-D, 2-D or 3-D")


def quantize(field, eb: float, radius: int = 512, ctx: plz.Context = None) -> QuantCodes:
    """Dual quantization of a float32 CUDA tensor (see include/plzgpu.h)."""
    import torch

    if not (field.is_cuda and field.dtype == torch.float32):
        raise plz.ValidationError("quantize takes a float32 CUDA tensor")
    field = field.contiguous()
    nz, ny, nx = _dims(tuple(field.shape))
    n = nx * ny * nz
    ctx = ctx or plz.context(field.device.index)
    dev = field.device
    codes = torch.empty(n, dtype=torch.int16, device=dev)
    cap = max(1024, n // 64)
    for _ in range(2):
        idx = torch.empty(cap, dtype=torch.int64, device=dev)
        val = torch.empty(cap, dtype=torch.int32, device=dev)
        nout, e = C.c_uint64(), L.Error()
        rc = L.lib().plzgpu_lorenzo_quantize(
            ctx.handle, C.c_void_p(field.data_ptr()), nx, ny, nz, float(eb), int(radius),
            C.c_void_p(codes.data_ptr()), C.c_void_p(idx.data_ptr()), C.c_void_p(val.data_ptr()),
            cap, C.byref(nout), C.c_void_p(torch.cuda.current_stream(dev).cuda_stream),
            C.byref(e))
        if rc == L.CAPACITY and nout.value > cap:
            cap = int(nout.value)
            continue
        plz._check(rc, e)
        break
    m = int(nout.value)
    return QuantCodes(codes, idx[:m], val[:m], (nz, ny, nx), float(eb), int(radius))


def reconstruct(q: QuantCodes, ctx: plz.Context = None):
    """Inverse of quantize: a float32 CUDA tensor of q.shape."""
    import torch

    nz, ny, nx = q.shape
    dev = q.codes.device
    ctx = ctx or plz.context(dev.index)
    out = torch.empty((nz, ny, nx), dtype=torch.float32, device=dev)
    e = L.Error()
    plz._check(L.lib().plzgpu_lorenzo_reconstruct(
        ctx.handle, C.c_void_p(q.codes.data_ptr()), C.c_void_p(q.outlier_idx.data_ptr()),
        C.c_void_p(q.outlier_val.data_ptr()), q.outlier_idx.numel(), nx, ny, nz, q.eb, q.radius,
        C.c_void_p(out.data_ptr()), C.c_void_p(torch.cuda.current_stream(dev).cuda_stream),
        C.byref(e)), e)
    return out


@dataclass
class CompressedField:
    image: "object"          # GPULZ image of the code bytes (uint8 CUDA tensor)
    outlier_idx: "object"
    outlier_val: "object"
    shape: Tuple[int, int, int]
    eb: float
    radius: int

    @property
    def nbytes(self) -> int:
        """Image + outlier list (8-byte index + 4-byte residual each)."""
        return int(self.image.numel()) + 12 * int(self.outlier_idx.numel())


def compress_field(field, eb: float, params: plz.Params = None, radius: int = 512) -> CompressedField:
    """field -> quantization codes -> GPULZ image, all on the device."""
    params = params or plz.validate(plz.Params(2, 255, 2048, 1))
    if params.symbol_width != 2:
        raise plz.ValidationError("u16 quantization codes: symbol_width must be 2")
    q = quantize(field, eb, radius)
    img = plz.compress(q.codes.view(__import__("torch").uint8), params)
    return CompressedField(img, q.outlier_idx, q.outlier_val, q.shape, q.eb, q.radius)


def decompress_field(cf: CompressedField):
    """GPULZ image -> codes -> float32 field (|f - f'| <= eb)."""
    import torch

    codes = plz.decompress_bytes(cf.image).view(torch.int16)
    return reconstruct(QuantCodes(codes, cf.outlier_idx, cf.outlier_val, cf.shape, cf.eb,
                                  cf.radius))
