"""Python face of the B200 GPULZ drop-in, mirroring the reference ``plz`` API.

Names, argument meaning and error behaviour follow the reference C++ library
(/root/reference/proj/include/plz): ``Params``/``validate``/``level_to_window``
(params.hpp), ``plan`` (partition.hpp), ``compress`` (pipeline.hpp),
``decompress_bytes``/``decompress_chunk`` (decoder.hpp), ``container_size``
(format.hpp), and the exception hierarchy of errors.hpp.  Every codec call
goes through the C-ABI (include/plzgpu.h) into the sm_100a kernels.

Data may be ``bytes``/``bytearray``/``memoryview``/numpy arrays (host) or
torch tensors (CPU or CUDA).  Host input returns ``bytes``; a CUDA tensor
input stays on the device and returns a CUDA ``uint8`` tensor.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

from . import _lib as L


# ----------------------------------------------------------------- errors
class Error(RuntimeError):
    """plz::error (errors.hpp:10)."""


class ValidationError(Error):
    """plz::validation_error (errors.hpp:15)."""


class UnsupportedFormatError(Error):
    """plz::unsupported_format_error (errors.hpp:20)."""


class CorruptionError(Error):
    """plz::corruption_error (errors.hpp:27-36): byte_offset or chunk/token."""

    def __init__(self, msg, byte_offset=0, chunk_index=None, token_index=None):
        super().__init__(msg)
        self.byte_offset = byte_offset
        self.chunk_index = chunk_index
        self.token_index = token_index


class ContractError(Error):
    """plz::contract_error (errors.hpp:39)."""


class CapacityError(Error):
    """Caller-provided output buffer too small (C-ABI only)."""


class CudaError(Error):
    """CUDA runtime failure."""


# reference spellings
error, validation_error, unsupported_format_error = Error, ValidationError, UnsupportedFormatError
corruption_error, contract_error = CorruptionError, ContractError


def _raise(e: L.Error):
    msg = e.message.decode(errors="replace")
    code = e.code
    if code == L.VALIDATION:
        raise ValidationError(msg)
    if code == L.UNSUPPORTED_FORMAT:
        raise UnsupportedFormatError(msg)
    if code == L.CORRUPTION:
        if e.chunk_index != L.NO_INDEX:
            raise CorruptionError(msg, 0, int(e.chunk_index), int(e.token_index))
        raise CorruptionError(msg, int(e.byte_offset))
    if code == L.CONTRACT:
        raise ContractError(msg)
    if code == L.CAPACITY:
        raise CapacityError(msg)
    raise CudaError(msg)


def _check(rc: int, e: L.Error):
    if rc != L.OK:
        _raise(e)


# ----------------------------------------------------------------- params
@dataclass
class Params:
    """plz::Params (params.hpp:18-25); defaults S=2, W=128, C=2048, I=1."""

    symbol_width: int = 2
    window: int = 128
    chunk_size: int = 2048
    interval: int = 1
    block_bytes: int = 256 << 20
    min_match: int = 2

    def to_c(self) -> L.Params:
        return L.Params(self.symbol_width, self.window, self.chunk_size, self.interval,
                        self.block_bytes, self.min_match, 0)


def validate(raw: Params) -> Params:
    """plz::validate (params.cpp:19-45)."""
    out, e = L.Params(), L.Error()
    _check(L.lib().plzgpu_validate(C.byref(raw.to_c()), C.byref(out), C.byref(e)), e)
    return Params(raw.symbol_width, raw.window, raw.chunk_size, raw.interval, raw.block_bytes,
                  int(out.min_match))


def level_to_window(level: int) -> int:
    """plz::level_to_window (params.cpp:47-55)."""
    w, e = C.c_int32(), L.Error()
    _check(L.lib().plzgpu_level_to_window(level, C.byref(w), C.byref(e)), e)
    return int(w.value)


def default_params() -> Params:
    return Params()


@dataclass
class BlockPlan:
    byte_start: int
    byte_len: int
    num_chunks: int
    last_chunk_len: int
    tail_len: int


def plan(total_bytes: int, params: Params) -> List[BlockPlan]:
    """plz::plan (partition.cpp:5-25)."""
    p = params.to_c()
    n = L.lib().plzgpu_plan(total_bytes, C.byref(p), None, 0)
    arr = (L.BlockPlan * max(1, n))()
    L.lib().plzgpu_plan(total_bytes, C.byref(p), arr, n)
    return [BlockPlan(b.byte_start, b.byte_len, b.num_chunks, b.last_chunk_len, b.tail_len)
            for b in arr[:n]]


def container_size(num_chunks: int, flag_total: int, payload_total: int, tail_len: int) -> int:
    """plz::container_size (format.cpp:69-73)."""
    return int(L.lib().plzgpu_container_size(num_chunks, flag_total, payload_total, tail_len))


def compress_bound(n: int, params: Params) -> int:
    return int(L.lib().plzgpu_compress_bound(n, C.byref(params.to_c())))


# ---------------------------------------------------------------- context
class Context:
    """One plzgpu_ctx (device scratch + stream).  One per host thread."""

    def __init__(self, device: int = 0):
        self.handle = C.c_void_p()
        e = L.Error()
        _check(L.lib().plzgpu_ctx_create(device, C.byref(self.handle), C.byref(e)), e)
        self.device = device

    def close(self):
        if self.handle:
            L.lib().plzgpu_ctx_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(L.lib().plzgpu_ctx_stream(self.handle) or 0)

    @property
    def last_launches(self) -> int:
        return int(L.lib().plzgpu_ctx_last_launches(self.handle))

    # ---- raw pointer entry points (bench / multi-GPU plumbing)
    def compress_ptr(self, params: Params, src: int, n: int, dst: int, cap: int,
                     stream: int = 0) -> tuple:
        out_len, st, e = C.c_uint64(), L.Stats(), L.Error()
        _check(L.lib().plzgpu_compress(self.handle, C.byref(params.to_c()), C.c_void_p(src), n,
                                       C.c_void_p(dst), cap, C.byref(out_len), C.byref(st),
                                       C.c_void_p(stream or None), C.byref(e)), e)
        return int(out_len.value), (int(st.pointer_tokens), int(st.literal_tokens))

    def compress_async(self, params: Params, d_in: int, n: int, d_out: int, cap: int,
                       d_len: int, stream: int = 0) -> None:
        e = L.Error()
        _check(L.lib().plzgpu_compress_async(self.handle, C.byref(params.to_c()), C.c_void_p(d_in),
                                             n, C.c_void_p(d_out), cap, C.c_void_p(d_len),
                                             C.c_void_p(stream or None), C.byref(e)), e)

    def decompress_ptr(self, src: int, n: int, dst: int, cap: int, stream: int = 0) -> int:
        out_len, e = C.c_uint64(), L.Error()
        _check(L.lib().plzgpu_decompress(self.handle, C.c_void_p(src), n, C.c_void_p(dst), cap,
                                         C.byref(out_len), C.c_void_p(stream or None),
                                         C.byref(e)), e)
        return int(out_len.value)

    def decompress_range(self, img: int, n: int, chunk_begin: int, chunk_end: int, out: int,
                         cap: int, stream: int = 0) -> Tuple[int, int, int]:
        """plzgpu_decompress_range: decodes global chunks [chunk_begin,
        chunk_end) into `out` (out = 0: sizes only).  Returns (out_begin,
        out_len, total_chunks)."""
        b, ln, tot, e = C.c_uint64(), C.c_uint64(), C.c_uint64(), L.Error()
        _check(L.lib().plzgpu_decompress_range(self.handle, C.c_void_p(img), n, chunk_begin,
                                               chunk_end, C.c_void_p(out or None), cap,
                                               C.byref(b), C.byref(ln), C.byref(tot),
                                               C.c_void_p(stream or None), C.byref(e)), e)
        return int(b.value), int(ln.value), int(tot.value)

    def decompressed_size(self, img: int, n: int, stream: int = 0) -> int:
        out_len, e = C.c_uint64(), L.Error()
        _check(L.lib().plzgpu_decompressed_size(self.handle, C.c_void_p(img), n, C.byref(out_len),
                                                C.c_void_p(stream or None), C.byref(e)), e)
        return int(out_len.value)

    def decompress_async(self, d_img: int, n: int, d_out: int, cap: int, d_len: int,
                         stream: int = 0) -> None:
        e = L.Error()
        _check(L.lib().plzgpu_decompress_async(self.handle, C.c_void_p(d_img), n,
                                               C.c_void_p(d_out), cap, C.c_void_p(d_len),
                                               C.c_void_p(stream or None), C.byref(e)), e)

    # ---- multi-GPU shard protocol (paper_2304_07342_b200/dist.py)
    def shard_encode(self, params: Params, src: int, n_total: int, begin: int, end: int,
                     stream: int = 0):
        maxt = 4 + (end - begin) * params.chunk_size * params.symbol_width // params.block_bytes
        tot = (C.c_uint64 * (3 * maxt))()
        nt, e = C.c_uint64(), L.Error()
        _check(L.lib().plzgpu_shard_encode(self.handle, C.byref(params.to_c()), C.c_void_p(src),
                                           n_total, begin, end, tot, maxt, C.byref(nt),
                                           C.c_void_p(stream or None), C.byref(e)), e)
        return [(tot[3 * i], tot[3 * i + 1], tot[3 * i + 2]) for i in range(nt.value)]

    def shard_assemble(self, bases, d_out: int, cap: int, stream: int = 0):
        nb = len(bases)
        b = (C.c_uint64 * max(1, 4 * nb))(*[v for row in bases for v in row])
        segs = (C.c_uint64 * max(3, 12 * nb))()
        ns, ln, e = C.c_uint64(), C.c_uint64(), L.Error()
        _check(L.lib().plzgpu_shard_assemble(self.handle, b, C.c_void_p(d_out), cap, segs, 4 * nb,
                                             C.byref(ns), C.byref(ln), C.c_void_p(stream or None),
                                             C.byref(e)), e)
        return [(segs[3 * i], segs[3 * i + 1], segs[3 * i + 2]) for i in range(ns.value)], ln.value

    def shard_headers(self, params: Params, n_total: int, totals, tail: bytes, d_img: int,
                      cap: int, stream: int = 0) -> int:
        nc = len(totals)
        t = (C.c_uint64 * max(2, 2 * nc))(*[v for row in totals for v in row])
        tb = C.create_string_buffer(bytes(tail) + b"\0" * 4, 8)
        ln, e = C.c_uint64(), L.Error()
        _check(L.lib().plzgpu_shard_headers(self.handle, C.byref(params.to_c()), n_total, t, tb,
                                            C.c_void_p(d_img), cap, C.byref(ln),
                                            C.c_void_p(stream or None), C.byref(e)), e)
        return int(ln.value)

    def encode_only(self, params: Params, d_in: int, n: int, stream: int = 0) -> None:
        """Kernel I alone (profiling hook plzgpu_profile_encode)."""
        e = L.Error()
        _check(L.lib().plzgpu_profile_encode(self.handle, C.byref(params.to_c()), C.c_void_p(d_in),
                                             n, C.c_void_p(stream or None), C.byref(e)), e)

    def profile_stages(self, params: Params, d_in: int, n: int, d_img: int, cap: int,
                       steps: int = 3, stream: int = 0):
        """CUDA-event ms of Kernel I, Kernel II and Kernel III + headers
        (plzgpu_profile_stages), each the mean over `steps` compresses."""
        ms, e = (C.c_double * 3)(), L.Error()
        _check(L.lib().plzgpu_profile_stages(self.handle, C.byref(params.to_c()), C.c_void_p(d_in),
                                             n, C.c_void_p(d_img), cap, steps, ms,
                                             C.c_void_p(stream or None), C.byref(e)), e)
        return tuple(ms)

    def finish(self, stream: int = 0):
        st, e = L.Stats(), L.Error()
        _check(L.lib().plzgpu_ctx_finish(self.handle, C.c_void_p(stream or None), C.byref(st),
                                         C.byref(e)), e)
        return int(st.pointer_tokens), int(st.literal_tokens)


_tls = threading.local()


def context(device: Optional[int] = None) -> Context:
    """The calling thread's context (created on first use)."""
    if device is None:
        try:
            import torch

            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        except Exception:
            device = 0
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


# ------------------------------------------------------------ buffer views
def _as_host(data):
    """(pointer, nbytes, keepalive) of host-resident bytes."""
    if isinstance(data, (bytes, bytearray, memoryview)):
        mv = memoryview(data).cast("B")
        buf = bytes(mv) if not isinstance(data, bytearray) else data
        if isinstance(buf, bytes):
            cbuf = C.c_char_p(buf)
            return C.cast(cbuf, C.c_void_p).value or 0, len(buf), (buf, cbuf)
        arr = (C.c_char * len(buf)).from_buffer(buf)
        return C.addressof(arr), len(buf), arr
    try:
        import numpy as np

        if isinstance(data, np.ndarray):
            a = np.ascontiguousarray(data)
            return a.ctypes.data, a.nbytes, a
    except ImportError:
        pass
    raise TypeError(f"unsupported buffer type {type(data)!r}")


def _is_torch(x) -> bool:
    try:
        import torch

        return isinstance(x, torch.Tensor)
    except ImportError:
        return False


@dataclass
class PipelineStats:
    """plz::PipelineStats (pipeline.hpp:14-18)."""

    max_cmp_per_pos: int = 0
    pointer_tokens: int = 0
    literal_tokens: int = 0


# ------------------------------------------------------------------ codec
def compress(data, params: Params, threads: int = 0, stats: Optional[PipelineStats] = None):
    """plz::compress (pipeline.cpp:88-99) on the GPU; bit-exact .plz image."""
    ctx = context()
    if _is_torch(data):
        import torch

        t = data.contiguous().view(torch.uint8).reshape(-1)
        n = t.numel()
        if t.is_cuda:
            ctx = context(t.device.index)  # the tensor's GPU, whatever the current device
            cap = compress_bound(n, params)
            out = torch.empty(max(cap, 1), dtype=torch.uint8, device=t.device)
            ln, st = ctx.compress_ptr(params, t.data_ptr(), n, out.data_ptr(), cap,
                                      torch.cuda.current_stream(t.device).cuda_stream)
            if stats is not None:
                stats.pointer_tokens += st[0]
                stats.literal_tokens += st[1]
            return out[:ln]
        data = t.numpy()
    ptr, n, keep = _as_host(data)
    cap = compress_bound(n, params)
    out = C.create_string_buffer(max(cap, 1))
    ln, st = ctx.compress_ptr(params, ptr, n, C.addressof(out), cap)
    if stats is not None:
        stats.pointer_tokens += st[0]
        stats.literal_tokens += st[1]
    return out.raw[:ln]


def decompress_bytes(img, threads: int = 0):
    """plz::decompress_bytes (decoder.cpp:129-141) on the GPU."""
    ctx = context()
    if _is_torch(img):
        import torch

        t = img.contiguous().view(torch.uint8).reshape(-1)
        if t.is_cuda:
            ctx = context(t.device.index)
            stream = torch.cuda.current_stream(t.device).cuda_stream
            cap = ctx.decompressed_size(t.data_ptr(), t.numel(), stream)  # device parse
            out = torch.empty(max(cap, 16), dtype=torch.uint8, device=t.device)
            ln = ctx.decompress_ptr(t.data_ptr(), t.numel(), out.data_ptr(), cap, stream)
            return out[:ln]
        img = t.numpy()
    ptr, n, keep = _as_host(img)
    cap = int(L.lib().plzgpu_decompressed_bound(C.c_void_p(ptr), n))
    out = C.create_string_buffer(max(cap, 1))
    ln = ctx.decompress_ptr(ptr, n, C.addressof(out), cap)
    return out.raw[:ln]


def compress_multi(data, params: Params, devices: Sequence[int],
                   stats: Optional[PipelineStats] = None):
    """plz::compress of one stream on several GPUs of this process
    (plzgpu_compress_multi): chunk-range shards, one per entry of `devices`;
    the image equals compress(data, params).  Host input -> bytes, CUDA
    tensor -> CUDA uint8 tensor on devices[0]."""
    devs = (C.c_int * len(devices))(*devices)
    e, st, ln = L.Error(), L.Stats(), C.c_uint64()
    if _is_torch(data) and data.is_cuda:
        import torch

        t = data.contiguous().view(torch.uint8).reshape(-1)
        cap = compress_bound(t.numel(), params)
        out = torch.empty(max(cap, 16), dtype=torch.uint8, device=torch.device("cuda", devices[0]))
        # the ranks run on the library's own streams: the input (and the
        # output allocation) must be complete before the call
        torch.cuda.current_stream(t.device).synchronize()
        torch.cuda.current_stream(out.device).synchronize()
        _check(L.lib().plzgpu_compress_multi(devs, len(devices), C.byref(params.to_c()),
                                             C.c_void_p(t.data_ptr()), t.numel(),
                                             C.c_void_p(out.data_ptr()), out.numel(), C.byref(ln),
                                             C.byref(st), C.byref(e)), e)
        res = out[:ln.value]
    else:
        ptr, n, keep = _as_host(data)
        cap = compress_bound(n, params)
        out = C.create_string_buffer(max(cap, 1))
        _check(L.lib().plzgpu_compress_multi(devs, len(devices), C.byref(params.to_c()),
                                             C.c_void_p(ptr), n, C.addressof(out), cap, C.byref(ln),
                                             C.byref(st), C.byref(e)), e)
        res = out.raw[:ln.value]
    if stats is not None:
        stats.pointer_tokens += st.pointer_tokens
        stats.literal_tokens += st.literal_tokens
    return res


def decompress_multi(img, devices: Sequence[int]):
    """plz::decompress_bytes on several GPUs of this process
    (plzgpu_decompress_multi): bytes in -> bytes out, CUDA tensor in -> CUDA
    uint8 tensor on devices[0]."""
    devs = (C.c_int * len(devices))(*devices)
    e, ln = L.Error(), C.c_uint64()
    if _is_torch(img) and img.is_cuda:
        import torch

        t = img.contiguous().view(torch.uint8).reshape(-1)
        cap = context(t.device.index).decompressed_size(
            t.data_ptr(), t.numel(), torch.cuda.current_stream(t.device).cuda_stream)
        out = torch.empty(max(cap, 16), dtype=torch.uint8, device=torch.device("cuda", devices[0]))
        torch.cuda.current_stream(t.device).synchronize()
        torch.cuda.current_stream(out.device).synchronize()
        _check(L.lib().plzgpu_decompress_multi(devs, len(devices), C.c_void_p(t.data_ptr()),
                                               t.numel(), C.c_void_p(out.data_ptr()), out.numel(),
                                               C.byref(ln), C.byref(e)), e)
        return out[:ln.value]
    ptr, n, keep = _as_host(img)
    cap = int(L.lib().plzgpu_decompressed_bound(C.c_void_p(ptr), n))
    out = C.create_string_buffer(max(cap, 1))
    _check(L.lib().plzgpu_decompress_multi(devs, len(devices), C.c_void_p(ptr), n,
                                           C.addressof(out), cap, C.byref(ln), C.byref(e)), e)
    return out.raw[:ln.value]


def decompress_range(img, chunk_begin: int, chunk_end: int):
    """Decodes the global chunks [chunk_begin, chunk_end) of a CUDA image
    tensor: returns (output slice tensor, its offset in the decompressed
    stream, the image's chunk count) — one rank's share of
    dist.decompress_sharded."""
    import torch

    t = img.contiguous().view(torch.uint8).reshape(-1)
    ctx = context(t.device.index)
    stream = torch.cuda.current_stream(t.device).cuda_stream
    _, ln, _ = ctx.decompress_range(t.data_ptr(), t.numel(), chunk_begin, chunk_end, 0, 0, stream)
    out = torch.empty(max(ln, 16), dtype=torch.uint8, device=t.device)
    b, ln, tot = ctx.decompress_range(t.data_ptr(), t.numel(), chunk_begin, chunk_end,
                                      out.data_ptr(), out.numel(), stream)
    return out[:ln], b, tot


def decompress_chunk(flags, payload, logical_len: int, params: Params, chunk_index: int = 0) -> bytes:
    """plz::decompress_chunk (decoder.cpp:70-90) on the GPU."""
    ctx = context()
    fp, nf, kf = _as_host(bytes(flags))
    pp, np_, kp = _as_host(bytes(payload))
    out = C.create_string_buffer(max(1, logical_len * params.symbol_width))
    e = L.Error()
    _check(L.lib().plzgpu_decompress_chunk(ctx.handle, C.c_void_p(fp), nf, C.c_void_p(pp), np_,
                                           logical_len, C.byref(params.to_c()), chunk_index,
                                           C.addressof(out), C.byref(e)), e)
    return out.raw[:logical_len * params.symbol_width]


def compression_ratio(n_in: int, n_out: int) -> float:
    """ratio = input bytes / whole-image bytes (tools/plz.cpp:79-81)."""
    return n_in / n_out if n_out else 0.0


# ------------------------------------------------- matcher / statistics / tuner
def match_table(data, params: Params):
    """plz::match_chunk over every chunk of `data` on the GPU: (length, offset)
    per symbol (matcher.cpp:113-131) as two bytes objects."""
    ptr, n, keep = _as_host(data)
    nsym = n // params.symbol_width
    ln = C.create_string_buffer(max(1, nsym))
    of = C.create_string_buffer(max(1, nsym))
    e = L.Error()
    _check(L.lib().plzgpu_match_table(context().handle, C.byref(params.to_c()), C.c_void_p(ptr), n,
                                      ln, of, None, None, C.byref(e)), e)
    return ln.raw[:nsym], of.raw[:nsym]


@dataclass
class MatchHistogram:
    """plz::MatchHistogram (corpus.hpp:33-39)."""

    counts: List[int]
    total_pointers: int
    symbol_width: int
    fraction_gt_128: float
    fraction_gt_256: float


def match_length_histogram(data, params: Params, raw_table: bool = False) -> MatchHistogram:
    """plz::match_length_histogram (corpus.cpp:75-129), interval forced to 1."""
    p = validate(Params(params.symbol_width, params.window, params.chunk_size, 1,
                        params.block_bytes))
    ptr, n, keep = _as_host(data)
    hist = (C.c_uint64 * 256)()
    e = L.Error()
    if raw_table:
        _check(L.lib().plzgpu_match_table(context().handle, C.byref(p.to_c()), C.c_void_p(ptr), n,
                                          None, None, hist, None, C.byref(e)), e)
    else:
        _check(L.lib().plzgpu_pointer_histogram(context().handle, C.byref(p.to_c()),
                                                C.c_void_p(ptr), n, hist, None, C.byref(e)), e)
    counts = [0] + [int(hist[i]) for i in range(1, 256)]
    total = sum(counts)
    s = p.symbol_width
    f128 = sum(c for l, c in enumerate(counts) if l * s > 128) / total if total else 0.0
    f256 = sum(c for l, c in enumerate(counts) if l * s > 256) / total if total else 0.0
    return MatchHistogram(counts, total, s, f128, f256)


@dataclass
class PilotReport:
    field_ratios: List[float]
    average: float
    chosen: Params


def select_params(fields, declared_width: int, base: Params, threshold: float = 1.5,
                  pilot_cap: int = 4 << 20) -> PilotReport:
    """plz::select_params (tuner.cpp:10-45): GPU pilot compressions."""
    if not fields:
        raise ValidationError("tuner requires at least one field")
    if declared_width not in (1, 2, 4):
        raise ValidationError("declared_width must be 1, 2 or 4")
    pilot = validate(Params(declared_width, base.window, base.chunk_size, base.interval,
                            base.block_bytes))
    ratios = []
    for f in fields:
        sample = bytes(f[:pilot_cap])
        img = compress(sample, pilot)
        ratios.append(len(sample) / len(img) if img else 1.0)
    avg = sum(ratios) / len(ratios)
    if avg < threshold:
        chosen = Params(1, base.window, base.chunk_size, base.interval, base.block_bytes)
    else:
        chosen = Params(declared_width, min(255, base.window * declared_width), base.chunk_size,
                        base.interval, base.block_bytes)
    return PilotReport(ratios, avg, validate(chosen))
