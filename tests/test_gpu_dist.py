"""GPU, several processes: the multi-GPU shard protocol (dist.py,
SURVEY.md §8e) run end to end by 2-3 torch.distributed ranks over gloo that
all drive the real sm_100a kernels on cuda:0 (GpuBackend) — Kernels I+II on
each rank's chunk range, the size all-gather, rebased segments, the rank-0
gather and header writing; then the sharded decompress (each rank decodes
its chunk range of the one image).  The gathered image must equal the
single-call image byte for byte (and so the reference's), and the decoded
slices must tile the input.  The one-process device-list form runs the same
protocol with host threads (plzgpu_compress_multi / _decompress_multi)."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_07342_b200 import datagen
from paper_2304_07342_b200 import dist as D
from paper_2304_07342_b200 import plz

pytestmark = pytest.mark.gpu

CASES = [(2, 255, 2048, 2, 2048 * 2 * 5, 41 * 4096 + 3),   # 9 containers, tail
         (1, 128, 4096, 1, 4096 * 7, 29 * 4096 + 100),     # cut through containers
         (4, 255, 1024, 4, 256 << 20, 64 * 4096 + 2)]      # one container, tail


def _data(S, size, seed):
    raw = datagen.small_quant_codes((size + S - 1) // S, S, seed=seed)
    return torch.frombuffer(bytearray(raw[:size]), dtype=torch.uint8).cuda()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        res = []
        for S, W, Cs, I, bb, size in CASES:
            p = plz.validate(plz.Params(S, W, Cs, I, bb))
            data = _data(S, size, 17)
            n = data.numel()
            n_chunks, _ = D.geometry(n, p)
            b, e = D.chunk_ranges(n_chunks, world)[rank]
            lo = b * Cs * S
            hi = n if e == n_chunks else e * Cs * S
            tail = bytes(data[n - n % S:].cpu().tolist()) if e == n_chunks else b""
            backend = D.GpuBackend(p, 0)
            comm = D.TorchComm("cpu")
            img, ln = D.compress_sharded(backend, comm, p, n, data[lo:hi].contiguous(), tail)
            torch.cuda.synchronize()
            want = plz.compress(data, p)
            ok_c = True if rank else bool(torch.equal(img[:ln], want))
            out, local, begin = D.decompress_sharded(backend, comm, want)
            ok_slice = bool(torch.equal(local, data[begin:begin + local.numel()]))
            ok_d = True if rank else bool(torch.equal(out, data))
            res.append((ok_c, ok_slice, ok_d, ln == want.numel()))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_protocol_over_gloo_with_gpu_backend(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + world + os.getpid() % 500
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(300)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    got = dict(q.get(timeout=10) for _ in range(world))
    for r in range(world):
        assert got[r] == [(True, True, True, True)] * len(CASES), (r, got[r])


def test_device_list_multi_matches_single_call_and_keeps_current_device():
    # plzgpu_compress_multi / _decompress_multi with pooled contexts: repeated
    # calls (warm pool), host and device inputs, the caller's device kept
    for S, W, Cs, I, bb, size in CASES:
        p = plz.validate(plz.Params(S, W, Cs, I, bb))
        data = _data(S, size, 23)
        want = plz.compress(data, p)
        for devs in ([0], [0, 0], [0, 0, 0, 0]):
            for _ in range(2):
                got = plz.compress_multi(data, p, devs)
                assert torch.equal(got, want), (S, devs)
                host = plz.compress_multi(data.cpu().numpy().tobytes(), p, devs)
                assert host == want.cpu().numpy().tobytes()
                back = plz.decompress_multi(want, devs)
                assert torch.equal(back, data)
                assert plz.decompress_multi(host, devs) == data.cpu().numpy().tobytes()
                assert torch.cuda.current_device() == 0
