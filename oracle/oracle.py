"""ctypes face of the CPU checkers — TEST INFRASTRUCTURE ONLY.

Two checkers live under ``oracle/``:

* ``lib/liboracle.so`` — the plain-C restatement (``plz_oracle.c``), always
  buildable (``make -C oracle``);
* ``_ref/libplzref.so`` — the UNMODIFIED reference library compiled from
  ``/root/reference/proj/src`` (``make -C oracle ref``).  It is built in the
  development container and travels to the GPU box as a prebuilt file.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  The
product package ``paper_2304_07342_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "lib", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libplzref.so")

OK, VALIDATION, UNSUPPORTED, CORRUPTION, CONTRACT, CAPACITY = 0, 1, 2, 3, 4, 6
NO_INDEX = (1 << 64) - 1


class OParams(C.Structure):
    _fields_ = [
        ("symbol_width", C.c_int32),
        ("window", C.c_int32),
        ("chunk_size", C.c_int32),
        ("interval", C.c_int32),
        ("block_bytes", C.c_uint64),
        ("min_match", C.c_int32),
        ("reserved", C.c_int32),
    ]


class OError(C.Structure):
    _fields_ = [
        ("code", C.c_int32),
        ("reserved", C.c_int32),
        ("byte_offset", C.c_uint64),
        ("chunk_index", C.c_uint64),
        ("token_index", C.c_uint64),
        ("message", C.c_char * 240),
    ]


@dataclass(frozen=True)
class ErrorInfo:
    """Comparable summary of a plz error: (code, byte_offset, chunk, token, message)."""

    code: int
    byte_offset: int
    chunk_index: int
    token_index: int
    message: str

    @staticmethod
    def from_struct(e: OError) -> "ErrorInfo":
        return ErrorInfo(int(e.code), int(e.byte_offset), int(e.chunk_index),
                         int(e.token_index), e.message.decode(errors="replace"))


class OracleError(Exception):
    def __init__(self, info: ErrorInfo):
        super().__init__(f"[{info.code}] {info.message}")
        self.info = info


def make_params(S=2, W=128, C_=2048, I=1, block_bytes=256 << 20, min_match=None) -> OParams:
    p = OParams(S, W, C_, I, block_bytes, 0, 0)
    p.min_match = (2 // S + 1) if min_match is None else min_match
    return p


def _buf(data) -> tuple:
    try:  # contiguous numpy bytes: passed in place (no copy of GiB-sized inputs)
        import numpy as np

        if isinstance(data, np.ndarray) and data.dtype == np.uint8 and data.flags["C_CONTIGUOUS"] \
                and data.size:
            return C.cast(data.ctypes.data, C.c_char_p), data.size, data
    except ImportError:
        pass
    b = bytes(data)
    return C.c_char_p(b) if b else C.c_char_p(b"\0"), len(b), b


# --------------------------------------------------------------- C restatement
_olib = None


def olib():
    global _olib
    if _olib is None:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle`")
        lib = C.CDLL(ORACLE_SO)
        P, E, U64 = C.POINTER(OParams), C.POINTER(OError), C.c_uint64
        lib.plzo_validate.argtypes = [P, P, E]
        lib.plzo_level_to_window.argtypes = [C.c_int]
        lib.plzo_compress_bound.argtypes = [U64, P]
        lib.plzo_compress_bound.restype = U64
        lib.plzo_compress.argtypes = [C.c_char_p, U64, P, C.c_void_p, U64, C.POINTER(U64),
                                      C.POINTER(U64), E]
        lib.plzo_decompress.argtypes = [C.c_char_p, U64, C.c_void_p, U64, C.POINTER(U64), E]
        lib.plzo_decompress_chunk.argtypes = [C.c_char_p, U64, C.c_char_p, U64, U64, P, U64,
                                              C.c_void_p, E]
        lib.plzo_match_chunk.argtypes = [C.c_char_p, U64, P, C.c_void_p, C.c_void_p]
        _olib = lib
    return _olib


def validate(p: OParams) -> OParams:
    out, err = OParams(), OError()
    if olib().plzo_validate(C.byref(p), C.byref(out), C.byref(err)):
        raise OracleError(ErrorInfo.from_struct(err))
    return out


def compress(data, p: OParams) -> bytes:
    """plz::compress restated (pipeline.cpp:88-99)."""
    src, n, keep = _buf(data)
    cap = olib().plzo_compress_bound(n, C.byref(p)) + 64
    out = C.create_string_buffer(cap)
    out_len, err = C.c_uint64(), OError()
    rc = olib().plzo_compress(src, n, C.byref(p), out, cap, C.byref(out_len), None, C.byref(err))
    if rc:
        raise OracleError(ErrorInfo.from_struct(err))
    return out.raw[: out_len.value]


def compress_stats(data, p: OParams):
    src, n, keep = _buf(data)
    cap = olib().plzo_compress_bound(n, C.byref(p)) + 64
    out = C.create_string_buffer(cap)
    out_len, err = C.c_uint64(), OError()
    st = (C.c_uint64 * 3)()
    rc = olib().plzo_compress(src, n, C.byref(p), out, cap, C.byref(out_len), st, C.byref(err))
    if rc:
        raise OracleError(ErrorInfo.from_struct(err))
    return out.raw[: out_len.value], (st[0], st[1], st[2])


def decompress(img) -> bytes:
    """plz::decompress_bytes restated (decoder.cpp:129-141)."""
    src, n, keep = _buf(img)
    total, err = C.c_uint64(), OError()
    if olib().plzo_decompress(src, n, None, 0, C.byref(total), C.byref(err)):
        raise OracleError(ErrorInfo.from_struct(err))
    out = C.create_string_buffer(max(1, total.value))
    if olib().plzo_decompress(src, n, out, total.value, C.byref(total), C.byref(err)):
        raise OracleError(ErrorInfo.from_struct(err))
    return out.raw[: total.value]


def decompress_chunk(flags, payload, logical: int, p: OParams, chunk_index=0) -> bytes:
    f, nf, kf = _buf(flags)
    q, np_, kq = _buf(payload)
    out = C.create_string_buffer(max(1, logical * p.symbol_width))
    err = OError()
    if olib().plzo_decompress_chunk(f, nf, q, np_, logical, C.byref(p), chunk_index, out,
                                    C.byref(err)):
        raise OracleError(ErrorInfo.from_struct(err))
    return out.raw[: logical * p.symbol_width]


def match_chunk(chunk_bytes, p: OParams):
    src, n, keep = _buf(chunk_bytes)
    ns = n // p.symbol_width
    ln, of = (C.c_uint8 * max(1, ns))(), (C.c_uint8 * max(1, ns))()
    olib().plzo_match_chunk(src, ns, C.byref(p), ln, of)
    return list(ln)[:ns], list(of)[:ns]


# ------------------------------------------------------ reference (oracle/_ref)
_rlib = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def rlib():
    global _rlib
    if _rlib is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref` where "
                                    "/root/reference is mounted")
        lib = C.CDLL(REF_SO)
        P, E, U64 = C.POINTER(OParams), C.POINTER(OError), C.c_uint64
        PB = C.POINTER(C.c_void_p)
        lib.plzref_free.argtypes = [C.c_void_p]
        lib.plzref_validate.argtypes = [P, P, E]
        lib.plzref_compress.argtypes = [C.c_char_p, U64, P, C.c_int, PB, C.POINTER(U64),
                                        C.POINTER(U64), E]
        lib.plzref_decompress.argtypes = [C.c_char_p, U64, C.c_int, PB, C.POINTER(U64), E]
        lib.plzref_decompress_chunk.argtypes = [C.c_char_p, U64, C.c_char_p, U64, U64, P, U64,
                                                C.c_void_p, E]
        lib.plzref_match_chunk.argtypes = [C.c_char_p, U64, P, C.c_void_p, C.c_void_p]
        _rlib = lib
    return _rlib


def _take(ptr: C.c_void_p, n: int):
    """The malloc'd result as bytes (a numpy uint8 array past 1 GiB, where
    ctypes.string_at's int size overflows)."""
    try:
        if n < (1 << 30):
            return C.string_at(ptr, n) if n else b""
        import numpy as np

        out = np.empty(n, dtype=np.uint8)
        C.memmove(out.ctypes.data, ptr, n)
        return out
    finally:
        rlib().plzref_free(ptr)


def ref_validate(p: OParams) -> OParams:
    out, err = OParams(), OError()
    if rlib().plzref_validate(C.byref(p), C.byref(out), C.byref(err)):
        raise OracleError(ErrorInfo.from_struct(err))
    return out


def ref_compress(data, p: OParams, threads: int = 0, stats=False):
    """plzref::compress — the reference itself (pipeline.cpp:88-99)."""
    src, n, keep = _buf(data)
    ptr, out_len, err = C.c_void_p(), C.c_uint64(), OError()
    st = (C.c_uint64 * 3)()
    rc = rlib().plzref_compress(src, n, C.byref(p), threads, C.byref(ptr), C.byref(out_len),
                                st, C.byref(err))
    if rc:
        raise OracleError(ErrorInfo.from_struct(err))
    img = _take(ptr, out_len.value)
    return (img, (st[0], st[1], st[2])) if stats else img


def ref_compress_into(src_ptr: int, n: int, p: OParams, threads: int = 0) -> int:
    """Timed-loop variant over an existing buffer address; returns image length."""
    ptr, out_len, err = C.c_void_p(), C.c_uint64(), OError()
    rc = rlib().plzref_compress(C.cast(src_ptr, C.c_char_p), n, C.byref(p), threads,
                                C.byref(ptr), C.byref(out_len), None, C.byref(err))
    if rc:
        raise OracleError(ErrorInfo.from_struct(err))
    rlib().plzref_free(ptr)
    return out_len.value


def ref_decompress(img, threads: int = 0) -> bytes:
    src, n, keep = _buf(img)
    ptr, out_len, err = C.c_void_p(), C.c_uint64(), OError()
    if rlib().plzref_decompress(src, n, threads, C.byref(ptr), C.byref(out_len), C.byref(err)):
        raise OracleError(ErrorInfo.from_struct(err))
    return _take(ptr, out_len.value)


def ref_decompress_into(src_ptr: int, n: int, threads: int = 0) -> int:
    ptr, out_len, err = C.c_void_p(), C.c_uint64(), OError()
    if rlib().plzref_decompress(C.cast(src_ptr, C.c_char_p), n, threads, C.byref(ptr),
                                C.byref(out_len), C.byref(err)):
        raise OracleError(ErrorInfo.from_struct(err))
    rlib().plzref_free(ptr)
    return out_len.value


def ref_decompress_chunk(flags, payload, logical: int, p: OParams, chunk_index=0) -> bytes:
    f, nf, kf = _buf(flags)
    q, np_, kq = _buf(payload)
    out = C.create_string_buffer(max(1, logical * p.symbol_width))
    err = OError()
    if rlib().plzref_decompress_chunk(f, nf, q, np_, logical, C.byref(p), chunk_index, out,
                                      C.byref(err)):
        raise OracleError(ErrorInfo.from_struct(err))
    return out.raw[: logical * p.symbol_width]


def ref_match_chunk(chunk_bytes, p: OParams):
    src, n, keep = _buf(chunk_bytes)
    ns = n // p.symbol_width
    ln, of = (C.c_uint8 * max(1, ns))(), (C.c_uint8 * max(1, ns))()
    rlib().plzref_match_chunk(src, ns, C.byref(p), ln, of)
    return list(ln)[:ns], list(of)[:ns]
