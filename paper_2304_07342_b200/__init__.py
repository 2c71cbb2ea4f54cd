"""B200-native GPULZ (arXiv 2304.07342): a drop-in for the reference ``plz``
compress / decompress path, built on hand-written sm_100a kernels.

    from paper_2304_07342_b200 import plz
    p = plz.validate(plz.Params(symbol_width=2, window=255, chunk_size=2048, interval=2))
    img = plz.compress(data, p)          # bit-exact with the reference's plz::compress
    assert plz.decompress_bytes(img) == data

See DESIGN.md for the kernel design and INTEGRATION.md for the C-ABI.
"""
from . import plz  # noqa: F401
from ._lib import LIB_PATH, lib  # noqa: F401

__all__ = ["plz", "lib", "LIB_PATH"]
