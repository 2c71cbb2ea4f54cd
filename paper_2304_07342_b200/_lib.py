"""ctypes binding of libplzgpu.so (include/plzgpu.h).

The shared library is built in-tree by ``make -C paper_2304_07342_b200/csrc``
(``__graft_entry__.build()``).  There is no fallback: importing this module
without the library raises, and every codec call runs the sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PLZGPU_LIB") or os.path.join(HERE, "lib", "libplzgpu.so")

OK, VALIDATION, UNSUPPORTED_FORMAT, CORRUPTION, CONTRACT, CUDA, CAPACITY = range(7)
NO_INDEX = (1 << 64) - 1


class Params(C.Structure):
    """plzgpu_params — layout of plz::Params (params.hpp:18-25)."""

    _fields_ = [
        ("symbol_width", C.c_int32),
        ("window", C.c_int32),
        ("chunk_size", C.c_int32),
        ("interval", C.c_int32),
        ("block_bytes", C.c_uint64),
        ("min_match", C.c_int32),
        ("reserved", C.c_int32),
    ]


class Stats(C.Structure):
    _fields_ = [("max_cmp_per_pos", C.c_uint64), ("pointer_tokens", C.c_uint64),
                ("literal_tokens", C.c_uint64)]


class Error(C.Structure):
    _fields_ = [
        ("code", C.c_int32),
        ("reserved", C.c_int32),
        ("byte_offset", C.c_uint64),
        ("chunk_index", C.c_uint64),
        ("token_index", C.c_uint64),
        ("message", C.c_char * 240),
    ]


class BlockPlan(C.Structure):
    _fields_ = [("byte_start", C.c_uint64), ("byte_len", C.c_uint64), ("num_chunks", C.c_uint32),
                ("last_chunk_len", C.c_uint32), ("tail_len", C.c_uint8), ("pad", C.c_uint8 * 7)]


# (name, restype, argtypes) of every exported symbol of include/plzgpu.h
_P, _E, _U64, _VP = C.POINTER(Params), C.POINTER(Error), C.c_uint64, C.c_void_p
SIGNATURES = [  # every entry point of include/plzgpu.h
    ("plzgpu_abi_version", C.c_int, []),
    ("plzgpu_validate", C.c_int, [_P, _P, _E]),
    ("plzgpu_level_to_window", C.c_int, [C.c_int, C.POINTER(C.c_int32), _E]),
    ("plzgpu_plan", _U64, [_U64, _P, C.POINTER(BlockPlan), _U64]),
    ("plzgpu_container_size", _U64, [C.c_uint32, _U64, _U64, C.c_uint8]),
    ("plzgpu_compress_bound", _U64, [_U64, _P]),
    ("plzgpu_decompressed_bound", _U64, [_VP, _U64]),
    ("plzgpu_ctx_create", C.c_int, [C.c_int, C.POINTER(_VP), _E]),
    ("plzgpu_ctx_destroy", None, [_VP]),
    ("plzgpu_ctx_stream", _VP, [_VP]),
    ("plzgpu_ctx_last_launches", C.c_int, [_VP]),
    ("plzgpu_decompressed_size", C.c_int, [_VP, _VP, _U64, C.POINTER(_U64), _VP, _E]),
    ("plzgpu_compress", C.c_int, [_VP, _P, _VP, _U64, _VP, _U64, C.POINTER(_U64),
                                  C.POINTER(Stats), _VP, _E]),
    ("plzgpu_compress_async", C.c_int, [_VP, _P, _VP, _U64, _VP, _U64, _VP, _VP, _E]),
    ("plzgpu_decompress", C.c_int, [_VP, _VP, _U64, _VP, _U64, C.POINTER(_U64), _VP, _E]),
    ("plzgpu_decompress_async", C.c_int, [_VP, _VP, _U64, _VP, _U64, _VP, _VP, _E]),
    ("plzgpu_compress_multi", C.c_int, [C.POINTER(C.c_int), C.c_int, _P, _VP, _U64, _VP, _U64,
                                        C.POINTER(_U64), C.POINTER(Stats), _E]),
    ("plzgpu_decompress_multi", C.c_int, [C.POINTER(C.c_int), C.c_int, _VP, _U64, _VP, _U64,
                                          C.POINTER(_U64), _E]),
    ("plzgpu_decompress_range", C.c_int, [_VP, _VP, _U64, _U64, _U64, _VP, _U64, C.POINTER(_U64),
                                          C.POINTER(_U64), C.POINTER(_U64), _VP, _E]),
    ("plzgpu_ctx_finish", C.c_int, [_VP, _VP, C.POINTER(Stats), _E]),
    ("plzgpu_decompress_chunk", C.c_int, [_VP, _VP, _U64, _VP, _U64, _U64, _P, _U64, _VP, _E]),
    ("plzgpu_profile_encode", C.c_int, [_VP, _P, _VP, _U64, _VP, _E]),
    ("plzgpu_profile_stages", C.c_int, [_VP, _P, _VP, _U64, _VP, _U64, C.c_int,
                                        C.POINTER(C.c_double), _VP, _E]),
    ("plzgpu_int_peak", C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_double), _E]),
    ("plzgpu_match_table", C.c_int, [_VP, _P, _VP, _U64, _VP, _VP, C.POINTER(_U64), _VP, _E]),
    ("plzgpu_pointer_histogram", C.c_int, [_VP, _P, _VP, _U64, C.POINTER(_U64), _VP, _E]),
    ("plzgpu_num_chunks", _U64, [_U64, _P]),
    ("plzgpu_num_containers", _U64, [_U64, _P]),
    ("plzgpu_shard_encode", C.c_int, [_VP, _P, _VP, _U64, _U64, _U64, C.POINTER(_U64), _U64,
                                      C.POINTER(_U64), _VP, _E]),
    ("plzgpu_shard_segments", _U64, [_P, _U64, _U64, _U64, C.POINTER(_U64), C.POINTER(_U64), _U64,
                                     C.POINTER(_U64), _U64]),
    ("plzgpu_shard_assemble", C.c_int, [_VP, C.POINTER(_U64), _VP, _U64, C.POINTER(_U64), _U64,
                                        C.POINTER(_U64), C.POINTER(_U64), _VP, _E]),
    ("plzgpu_shard_assemble_into", C.c_int, [_VP, C.POINTER(_U64), _VP, _U64, _VP, _E]),
    ("plzgpu_shard_headers", C.c_int, [_VP, _P, _U64, C.POINTER(_U64), _VP, _VP, _U64,
                                       C.POINTER(_U64), _VP, _E]),
    ("plzgpu_lorenzo_quantize", C.c_int, [_VP, _VP, _U64, _U64, _U64, C.c_double, C.c_int32, _VP,
                                          _VP, _VP, _U64, C.POINTER(_U64), _VP, _E]),
    ("plzgpu_lorenzo_reconstruct", C.c_int, [_VP, _VP, _VP, _VP, _U64, _U64, _U64, _U64,
                                             C.c_double, C.c_int32, _VP, _VP, _E]),
]

_lib = None


def lib():
    """Load libplzgpu.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the sm_100a extension first "
                "(python -c 'import __graft_entry__ as g; g.build()' or "
                "make -C paper_2304_07342_b200/csrc)")
        handle = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib
