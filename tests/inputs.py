"""Deterministic test inputs (numpy PCG64), shared by the CPU and GPU suites
and by tests/golden/make_golden.py.  Kinds follow the reference's fuzz mix
(acceptance.cpp:46-77): uniform bytes, small alphabets, geometric runs,
adversarial periodic patterns, quant-like codes."""
import numpy as np

KINDS = ("uniform", "alpha", "runs", "periodic", "quant", "constant")


def make(kind: str, size: int, seed: int, S: int = 2) -> bytes:
    rs = np.random.default_rng(seed)
    if size == 0:
        return b""
    if kind == "uniform":
        return rs.integers(0, 256, size, dtype=np.uint8).tobytes()
    if kind == "alpha":
        a = int(rs.integers(2, 9))
        return rs.integers(0, a, size, dtype=np.uint8).tobytes()
    if kind == "runs":
        out = bytearray()
        alphabet = int(rs.integers(3, 17))
        mean = float(rs.integers(8, 513))
        while len(out) < size:
            v = int(rs.integers(0, alphabet))
            out += bytes([v]) * (1 + int(rs.geometric(1.0 / mean)))
        return bytes(out[:size])
    if kind == "periodic":
        period = int(rs.choice([1, 2, 3, 4, 5, 7, 8, 13, 16, 251]))
        pat = rs.integers(0, 256, period, dtype=np.uint8)
        return np.resize(pat, size).tobytes()
    if kind == "quant":
        n = (size + S - 1) // S
        centre = {1: 128, 2: 32768, 4: 1 << 30}[S]
        dom = rs.random(n) < (0.5 + 0.5 * rs.random())
        delta = rs.integers(1, 9, n) * np.where(rs.random(n) < 0.5, -1, 1)
        codes = np.where(dom, centre, centre + delta).astype(np.int64)
        dt = {1: np.uint8, 2: "<u2", 4: "<u4"}[S]
        return codes.astype(dt).tobytes()[:size]
    if kind == "constant":
        return bytes([int(rs.integers(0, 256))]) * size
    raise ValueError(kind)
