"""Multi-GPU sharded compression.

Chunks are independent (no window crosses a chunk, matcher.cpp:76), so the
partition's chunk index space is split into contiguous per-rank ranges that
may cut through a container.  The only exchange is a handful of integers:

1. every rank runs Kernels I+II on its range (``plzgpu_shard_encode``) and
   gets, per container it touches, the payload / flag bytes it produced;
2. one all-gather of those triples (NCCL over NVLink on GPUs) gives every rank
   each container's stream totals, its own base offset inside each container's
   streams, and every container's offset in the final image;
3. every rank writes the table slices and stream slices it owns, rebased, into
   a local buffer (``plzgpu_shard_assemble``) — four segments per container;
4. rank 0 receives every rank's segments straight into the image at their
   offsets (P2P sends/recvs) and writes the container headers, final table
   entries and the tail (``plzgpu_shard_headers``).

The gathered image is byte-identical to a single-GPU ``compress`` of the
whole input (tests/test_gpu_shards.py) — and therefore to the reference.

The protocol is written against two small interfaces so one driver serves
NCCL ranks, gloo CPU tests and an in-process single-GPU simulation:
``Backend`` (encode / assemble / segments / headers) and ``Comm``
(all-gather of an int64 vector, point-to-point byte transfers).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Sequence, Tuple

from . import _lib as L
from . import plz

Totals = List[Tuple[int, int, int]]          # (container index, payload bytes, flag bytes)
Segment = Tuple[int, int, int]               # (image offset, local offset, length)


def chunk_ranges(n_chunks: int, world: int) -> List[Tuple[int, int]]:
    """Balanced contiguous chunk ranges, one per rank."""
    return [(n_chunks * r // world, n_chunks * (r + 1) // world) for r in range(world)]


def geometry(n_total: int, params: plz.Params):
    p = params.to_c()
    return int(L.lib().plzgpu_num_chunks(n_total, C.byref(p))), \
        int(L.lib().plzgpu_num_containers(n_total, C.byref(p)))


def container_layout(n_total: int, params: plz.Params):
    """Per container: (chunk count, byte length, tail length) — partition.cpp:5-25."""
    return [(b.num_chunks, b.byte_len, b.tail_len) for b in plz.plan(n_total, params)]


@dataclass
class Plan:
    totals: List[Tuple[int, int]]            # per container (payload total, flag total)
    img_off: List[int]                       # per container image offset
    image_len: int
    bases: List[List[Tuple[int, int, int, int]]]  # per rank, per touched container:
    # (payload_base, flag_base, container image offset, container flag total)


def plan_offsets(n_total: int, params: plz.Params, per_rank: Sequence[Totals]) -> Plan:
    """Global offsets from every rank's per-container totals (step 2)."""
    layout = container_layout(n_total, params)
    nc = len(layout)
    ptot, ftot = [0] * nc, [0] * nc
    bases = []
    for tot in per_rank:
        mine = []
        for j, pb, fb in tot:
            mine.append([j, ptot[j], ftot[j]])
            ptot[j] += pb
            ftot[j] += fb
        bases.append(mine)
    img_off, at = [], 0
    for j, (n, _, tail) in enumerate(layout):
        img_off.append(at)
        at += 26 + 8 * (n + 1) + ptot[j] + ftot[j] + tail
    rank_bases = [[(pb, fb, img_off[j], ftot[j]) for j, pb, fb in mine] for mine in bases]
    return Plan(list(zip(ptot, ftot)), img_off, at, rank_bases)


def shard_segments(params: plz.Params, n_total: int, rng: Tuple[int, int], totals: Totals,
                   bases) -> List[Segment]:
    """Image segments a shard owns (host arithmetic, plzgpu_shard_segments)."""
    nt = len(totals)
    if nt == 0:
        return []
    t = (C.c_uint64 * (3 * nt))(*[v for row in totals for v in row])
    b = (C.c_uint64 * (4 * nt))(*[v for row in bases for v in row])
    segs = (C.c_uint64 * (12 * nt))()
    ns = L.lib().plzgpu_shard_segments(C.byref(params.to_c()), n_total, rng[0], rng[1], t, b, nt,
                                       segs, 4 * nt)
    return [(segs[3 * i], segs[3 * i + 1], segs[3 * i + 2]) for i in range(ns)]


# ------------------------------------------------------------------ backend
class GpuBackend:
    """The sm_100a kernels through the C-ABI; buffers are torch CUDA tensors."""

    def __init__(self, params: plz.Params, device: int = 0, ctx: plz.Context = None):
        import torch

        self.torch = torch
        self.params = params
        self.device = torch.device("cuda", device)
        self.ctx = ctx or plz.Context(device)

    def encode(self, d_local, n_total: int, rng: Tuple[int, int], stream: int = 0) -> Totals:
        ptr = d_local.data_ptr() if d_local is not None and d_local.numel() else 0
        self._totals = self.ctx.shard_encode(self.params, ptr, n_total, rng[0], rng[1], stream)
        self._rng = rng
        return self._totals

    def assemble(self, bases, stream: int = 0):
        # local bytes = 8 table bytes per chunk + this shard's stream bytes
        cap = 8 * (self._rng[1] - self._rng[0]) + sum(p + f for _, p, f in self._totals)
        out = self.torch.empty(max(cap, 16), dtype=self.torch.uint8, device=self.device)
        segs, _ = self.ctx.shard_assemble(bases, out.data_ptr(), out.numel(), stream)
        return out, segs

    def new_image(self, n: int):
        return self.torch.empty(max(n, 16), dtype=self.torch.uint8, device=self.device)

    def total_chunks(self, img, stream: int = 0) -> int:
        return self.ctx.decompress_range(img.data_ptr(), img.numel(), 0, 0, 0, 0, stream)[2]

    def decode_range(self, img, rng: Tuple[int, int], stream: int = 0):
        b, e = rng
        _, ln, _ = self.ctx.decompress_range(img.data_ptr(), img.numel(), b, e, 0, 0, stream)
        out = self.torch.empty(max(ln, 16), dtype=self.torch.uint8, device=self.device)
        begin, ln, _ = self.ctx.decompress_range(img.data_ptr(), img.numel(), b, e,
                                                 out.data_ptr(), out.numel(), stream)
        return out[:ln], begin

    def decode_all(self, img):
        """The single-call decode of the whole image (error reporting)."""
        return plz.decompress_bytes(img)

    def headers(self, n_total: int, plan: Plan, tail: bytes, img, stream: int = 0) -> int:
        return self.ctx.shard_headers(self.params, n_total, plan.totals, tail, img.data_ptr(),
                                      img.numel(), stream)

    def copy_into(self, img, off: int, src, src_off: int, n: int):
        img[off:off + n].copy_(src[src_off:src_off + n])


# --------------------------------------------------------------------- comm
class TorchComm:
    """torch.distributed: NCCL (CUDA tensors) or gloo (CPU tensors)."""

    def __init__(self, device):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.device = torch, dist, device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def allgather(self, vec: List[int]) -> List[List[int]]:
        t = self.torch.tensor(vec, dtype=self.torch.int64, device=self.device)
        outs = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(outs, t)
        return [o.tolist() for o in outs]

    def gather_segments(self, img, local, my_segs, segs_by_rank):
        """Rank 0 receives every rank's segments into img at their offsets
        (zero-copy P2P on NCCL; host-staged when a CPU backend meets CUDA
        buffers)."""
        stage = str(self.device) == "cpu" and (
            (img is not None and img.is_cuda) or (local is not None and local.is_cuda))
        ops, landing = [], []
        if self.rank == 0:
            for r in range(1, self.world):
                for off, _, n in segs_by_rank[r]:
                    if n:
                        buf = self.torch.empty(n, dtype=self.torch.uint8) if stage else img[off:off + n]
                        landing.append((off, buf))
                        ops.append(self.dist.P2POp(self.dist.irecv, buf, r))
        else:
            src = local.cpu() if stage else local
            for _, loc, n in my_segs:
                if n:
                    ops.append(self.dist.P2POp(self.dist.isend, src[loc:loc + n].clone() if stage
                                               else src[loc:loc + n], 0))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        if stage and self.rank == 0:
            for off, buf in landing:
                img[off:off + buf.numel()].copy_(buf)


_ERR_CLASSES = {L.VALIDATION: plz.ValidationError, L.UNSUPPORTED_FORMAT: plz.UnsupportedFormatError,
                L.CORRUPTION: plz.CorruptionError, L.CONTRACT: plz.ContractError,
                L.CAPACITY: plz.CapacityError}


def _status_of(exc) -> int:
    for code, cls in _ERR_CLASSES.items():
        if type(exc) is cls:
            return code
    return L.CUDA


def _raise_remote(rank: int, status: int, own):
    """Every rank raises once any rank failed: its own error, or one of the
    failing rank's type naming it (no rank is left waiting in a collective)."""
    if own is not None:
        raise own
    raise _ERR_CLASSES.get(status, plz.CudaError)(f"rank {rank} failed (error code {status})")


def _pack(totals: Totals, tail: bytes, max_touched: int, status: int = 0) -> List[int]:
    vec = [-1] * (3 * max_touched) + [len(tail)] + list(tail) + [0] * (3 - len(tail)) + [status]
    for i, row in enumerate(totals):
        vec[3 * i:3 * i + 3] = list(row)
    return vec


def _unpack(vec: List[int], max_touched: int):
    totals = [tuple(vec[3 * i:3 * i + 3]) for i in range(max_touched) if vec[3 * i] >= 0]
    tl = vec[3 * max_touched]
    return totals, bytes(vec[3 * max_touched + 1:3 * max_touched + 1 + tl]), vec[-1]


def compress_sharded(backend, comm, params: plz.Params, n_total: int, d_local,
                     tail: bytes = b"", stream: int = 0):
    """Run the protocol on this rank; returns (image, image_len) on rank 0 and
    (None, image_len) elsewhere.  d_local holds this rank's chunk range
    (chunk_ranges(...)[rank]); the final rank also passes the input's last
    n_total % S bytes as `tail`."""
    n_chunks, _ = geometry(n_total, params)
    ranges = chunk_ranges(n_chunks, comm.world)
    rng = ranges[comm.rank]
    cpb = params.block_bytes // (params.chunk_size * params.symbol_width)
    max_touched = max((e - b + cpb - 1) // cpb + 1 for b, e in ranges)
    own = None
    try:
        mine = backend.encode(d_local, n_total, rng, stream)
    except plz.Error as e:  # reported after the exchange, on every rank
        own, mine = e, []
    gathered = [_unpack(v, max_touched)
                for v in comm.allgather(_pack(mine, tail, max_touched, _status_of(own) if own else 0))]
    for r, g in enumerate(gathered):
        if g[2]:
            _raise_remote(r, g[2], own if r == comm.rank else None)
    per_rank = [g[0] for g in gathered]
    tail_all = b"".join(g[1] for g in gathered)
    plan = plan_offsets(n_total, params, per_rank)
    if any(p > 0xFFFFFFFF or f > 0xFFFFFFFF for p, f in plan.totals):
        # scan.cpp:43-44, decided from the plan identically on every rank
        raise plz.ValidationError("block too large: offsets exceed 4-byte table range")
    local, my_segs = backend.assemble(plan.bases[comm.rank], stream)
    img = None
    if comm.rank == 0:
        img = backend.new_image(plan.image_len)
        for off, loc, n in my_segs:
            if n:
                backend.copy_into(img, off, local, loc, n)
        segs_by_rank = [shard_segments(params, n_total, ranges[r], per_rank[r], plan.bases[r])
                        for r in range(comm.world)]
    else:
        segs_by_rank = None
    comm.gather_segments(img, local, my_segs, segs_by_rank)
    if comm.rank == 0:
        backend.headers(n_total, plan, tail_all, img, stream)
    return img, plan.image_len


def decompress_sharded(backend, comm, img, gather: bool = True, stream: int = 0):
    """Sharded decompress of one image that every rank holds:
    rank r decodes the global chunk range chunk_ranges(total_chunks, world)[r]
    (``plzgpu_decompress_range``) — no exchange beyond an all-gather of each
    slice's (offset, length); with `gather`, rank 0 receives every slice at its
    offset (P2P) into the whole output.  Returns (output on rank 0 else None,
    this rank's slice, its offset in the output)."""
    own, local, begin = None, None, 0
    try:
        total = backend.total_chunks(img, stream)
        rng = chunk_ranges(total, comm.world)[comm.rank]
        local, begin = backend.decode_range(img, rng, stream)
    except plz.Error as e:
        own = e
    n_local = local.numel() if local is not None else 0
    status = [tuple(v) for v in comm.allgather([_status_of(own) if own else 0, begin, n_local])]
    if any(st for st, _, _ in status):
        # the single-call decode raises exactly the reference's error (a
        # later container's header error only after earlier containers'
        # token errors, decoder.cpp:129-141) — every rank holds the image
        backend.decode_all(img)
        r = next(i for i, (st, _, _) in enumerate(status) if st)
        _raise_remote(r, status[r][0], own if r == comm.rank else None)
    if not gather:
        return None, local, begin
    sizes = [(b, n) for _, b, n in status]
    n_out = max((b + n for b, n in sizes), default=0)
    out, segs_by_rank = None, None
    if comm.rank == 0:
        out = backend.new_image(n_out)
        if n_local:
            backend.copy_into(out, begin, local, 0, n_local)
        segs_by_rank = [[(b, 0, n)] for b, n in sizes]
    comm.gather_segments(out, local, [(begin, 0, n_local)], segs_by_rank)
    return (out[:n_out] if out is not None else None), local, begin


def simulate_sharded(params: plz.Params, data, world: int, device: int = 0):
    """Single-process run of the protocol for `world` virtual ranks on one GPU
    (one context per rank, exchanges done in memory): the per-rank C-ABI calls,
    offset plan and segment placement are exactly those of compress_sharded.
    Returns the assembled image (CUDA uint8 tensor)."""
    n_total = data.numel()
    n_chunks, _ = geometry(n_total, params)
    ranges = chunk_ranges(n_chunks, world)
    S, Cs = params.symbol_width, params.chunk_size
    backends = [GpuBackend(params, device) for _ in range(world)]
    per_rank = []
    for r, (b, e) in enumerate(ranges):
        hi = n_total if e == n_chunks else e * Cs * S
        per_rank.append(backends[r].encode(data[b * Cs * S:hi], n_total, (b, e)))
    plan = plan_offsets(n_total, params, per_rank)
    img = backends[0].new_image(plan.image_len)
    for r in range(world):
        local, segs = backends[r].assemble(plan.bases[r])
        for off, loc, n in segs:
            if n:
                backends[0].copy_into(img, off, local, loc, n)
    tail_len = n_total % S if n_total else 0
    tail = bytes(data[n_total - tail_len:].cpu().tolist()) if tail_len else b""
    backends[0].headers(n_total, plan, tail, img)
    return img[:plan.image_len]
