"""CPU, world_size 2 over gloo: the multi-GPU shard protocol's host logic
(chunk ranges, the size all-gather, offset plan, segment arithmetic of the
C-ABI, rank-0 P2P gather and header writing) run end to end with a stand-in
backend that cuts each rank's pieces out of the C oracle's image.  The
assembled image must equal the oracle's (= the reference's) image."""
import os
import struct

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
import oracle as O
from paper_2304_07342_b200 import dist as D
from paper_2304_07342_b200 import plz


def _as_plz(e: "O.OracleError") -> plz.Error:
    """The oracle's error as the plz exception of the same code."""
    cls = {1: plz.ValidationError, 2: plz.UnsupportedFormatError, 3: plz.CorruptionError,
           4: plz.ContractError}.get(e.info.code, plz.Error)
    return cls(e.info.message)


class OracleBackend:
    """Per-rank pieces taken from a reference image (test stand-in for the
    GPU kernels; the protocol code under test is dist.py + the C-ABI's
    plzgpu_shard_segments)."""

    def __init__(self, params, image):
        self.params, self.img = params, image
        self.conts = []
        at = 0
        while at < len(image):
            n = struct.unpack_from("<I", image, at + 21)[0]
            pt = struct.unpack_from(f"<{n + 1}I", image, at + 26)
            ft = struct.unpack_from(f"<{n + 1}I", image, at + 26 + 4 * (n + 1))
            fs = at + 26 + 8 * (n + 1)
            self.conts.append((n, pt, ft, fs, fs + ft[n]))
            at = fs + ft[n] + pt[n] + image[at + 25]
        self.cpb = params.block_bytes // (params.chunk_size * params.symbol_width)
        self.rank, self.fail_rank = 0, -1

    # ---- sharded decompress: the range semantics restated over the image's
    # headers and the oracle's whole-image decode
    def _starts(self):
        at, out_off, base, starts = 0, 0, 0, []
        while at < len(self.img):
            S, Cs = self.img[at + 5], struct.unpack_from("<I", self.img, at + 9)[0]
            orig = struct.unpack_from("<Q", self.img, at + 13)[0]
            n = struct.unpack_from("<I", self.img, at + 21)[0]
            starts += [out_off + k * Cs * S for k in range(n)]
            pt = struct.unpack_from("<I", self.img, at + 26 + 4 * n)[0]
            ft = struct.unpack_from("<I", self.img, at + 26 + 8 * n + 4)[0]
            at += 26 + 8 * (n + 1) + pt + ft + self.img[at + 25]
            out_off += orig
        return starts, out_off

    def total_chunks(self, img, stream=0):
        return len(self._starts()[0])

    def decode_all(self, img):
        try:
            return O.decompress(self.img)
        except O.OracleError as e:
            raise _as_plz(e) from None

    def decode_range(self, img, rng, stream=0):
        starts, total_out = self._starts()
        start = lambda g: 0 if g == 0 else (total_out if g >= len(starts) else starts[g])  # noqa: E731
        lo, hi = start(rng[0]), start(rng[1])
        if self.fail_rank == self.rank:  # a token error inside this rank's range only
            raise plz.CorruptionError("corrupt chunk (stand-in for a range decode error)", 0, 0, 0)
        full = self.decode_all(img)
        return torch.frombuffer(bytearray(full[lo:hi]) or bytearray(1), dtype=torch.uint8)[:hi - lo], lo

    def _touched(self, rng):
        b, e = rng
        out = []
        for j, (n, pt, ft, fs, ps) in enumerate(self.conts):
            g0 = j * self.cpb
            lo, hi = max(b, g0), min(e, g0 + n)
            if lo < hi:
                out.append((j, lo - g0, hi - g0))
        return out

    def encode(self, d_local, n_total, rng, stream=0):
        self.rng = rng
        res = []
        for j, klo, khi in self._touched(rng):
            n, pt, ft, _, _ = self.conts[j]
            res.append((j, pt[khi] - pt[klo], ft[khi] - ft[klo]))
        self.totals = res
        return res

    def assemble(self, bases, stream=0):
        buf = bytearray()
        for (j, klo, khi), (pb, fb, _, _) in zip(self._touched(self.rng), bases):
            n, pt, ft, fs, ps = self.conts[j]
            buf += b"".join(struct.pack("<I", pb + pt[k] - pt[klo]) for k in range(klo, khi))
            buf += b"".join(struct.pack("<I", fb + ft[k] - ft[klo]) for k in range(klo, khi))
            buf += self.img[fs + ft[klo]:fs + ft[khi]]
            buf += self.img[ps + pt[klo]:ps + pt[khi]]
        segs = D.shard_segments(self.params, self.n_total, self.rng, self.totals, bases)
        assert sum(s[2] for s in segs) == len(buf)
        return torch.frombuffer(bytearray(buf) or bytearray(1), dtype=torch.uint8), segs

    def new_image(self, n):
        return torch.zeros(max(n, 1), dtype=torch.uint8)

    def copy_into(self, img, off, src, loc, n):
        img[off:off + n].copy_(src[loc:loc + n])

    def headers(self, n_total, plan, tail, img, stream=0):
        layout = D.container_layout(n_total, self.params)
        p = self.params
        for j, ((n, blen, tl), (pt, ft)) in enumerate(zip(layout, plan.totals)):
            at = plan.img_off[j]
            hdr = b"PLZ1" + bytes([1, p.symbol_width, p.window, p.interval, 0]) + \
                struct.pack("<IQIB", p.chunk_size, blen, n, tl)
            img[at:at + 26] = torch.tensor(list(hdr), dtype=torch.uint8)
            img[at + 26 + 4 * n:at + 30 + 4 * n] = torch.tensor(list(struct.pack("<I", pt)),
                                                                dtype=torch.uint8)
            fo = at + 26 + 4 * (n + 1) + 4 * n
            img[fo:fo + 4] = torch.tensor(list(struct.pack("<I", ft)), dtype=torch.uint8)
            if tl:
                to = at + 26 + 8 * (n + 1) + pt + ft
                img[to:to + tl] = torch.tensor(list(tail[:tl]), dtype=torch.uint8)
        return plan.image_len


CASES = [(2, 255, 2048, 2, 2048 * 2 * 3, 17 * 4096 + 3), (1, 128, 1024, 1, 1024 * 2, 9 * 1024 + 5),
         (4, 64, 1024, 4, 256 << 20, 5 * 4096 + 7)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        results = []
        for S, W, Cs, I, bb, size in CASES:
            p = plz.validate(plz.Params(S, W, Cs, I, bb))
            data = inputs.make("quant", size, 7, S)
            image = O.compress(data, O.make_params(S, W, Cs, I, bb))
            be = OracleBackend(p, image)
            be.n_total = len(data)
            n_chunks, _ = D.geometry(len(data), p)
            b, e = D.chunk_ranges(n_chunks, world)[rank]
            tail = data[len(data) - len(data) % S:] if e == n_chunks else b""
            img, ln = D.compress_sharded(be, D.TorchComm("cpu"), p, len(data), None, tail)
            if rank == 0:
                results.append(bytes(img[:ln].numpy().tobytes()) == image)
        if rank == 0:
            q.put(results)
    finally:
        dist.destroy_process_group()


def _worker_dec(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        results = []
        for S, W, Cs, I, bb, size in CASES:
            p = plz.validate(plz.Params(S, W, Cs, I, bb))
            data = inputs.make("quant", size, 11, S)
            image = O.compress(data, O.make_params(S, W, Cs, I, bb))
            be = OracleBackend(p, image)
            out, local, begin = D.decompress_sharded(be, D.TorchComm("cpu"), None)
            if rank == 0:
                results.append(bytes(out.numpy().tobytes()) == data)
        if rank == 0:
            q.put(results)
    finally:
        dist.destroy_process_group()


def _spawn(target, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + 7 * world + os.getpid() % 1000 + (50 if target is _worker_dec else 0)
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
    assert all(pr.exitcode == 0 for pr in procs)
    return q.get(timeout=5)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_decompress_over_gloo(world):
    # each rank decodes its chunk range; rank 0 gathers the slices by offset
    assert _spawn(_worker_dec, world) == [True] * len(CASES)


@pytest.mark.parametrize("world", [2, 3])
def test_shard_protocol_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
    assert all(pr.exitcode == 0 for pr in procs)
    assert q.get(timeout=5) == [True] * len(CASES)


def _worker_err(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S, W, Cs, I, bb, size = CASES[0]
        p = plz.validate(plz.Params(S, W, Cs, I, bb))
        data = inputs.make("quant", size, 13, S)
        image = bytearray(O.compress(data, O.make_params(S, W, Cs, I, bb)))
        image = image[:-1]  # truncated streams in the last container
        try:
            O.decompress(bytes(image))
            want = None
        except O.OracleError as e:
            want = (e.info.code, e.info.message)
        be = OracleBackend(p, bytes(image))
        be.rank, be.fail_rank = rank, world - 1  # only the last rank's range fails
        try:
            D.decompress_sharded(be, D.TorchComm("cpu"), None)
            got = None
        except plz.Error as e:
            got = (type(e).__name__, str(e))
        q.put((rank, want, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_decompress_error_reaches_every_rank(world):
    # one rank's range fails: every rank raises the single-call error (no
    # rank waits in a collective), matching the reference decoder's message
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + world + os.getpid() % 1000
    procs = [ctx.Process(target=_worker_err, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
    assert all(pr.exitcode == 0 for pr in procs)
    res = [q.get(timeout=5) for _ in range(world)]
    for rank, want, got in res:
        assert want is not None and got is not None
        assert got == ("CorruptionError", want[1])
