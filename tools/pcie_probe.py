"""PCIe ceilings on the box: pinned H2D and D2H of the c2 input size, both
directions at once, and the decompress pattern (c2 image up while the
decoded bytes go down) — the floors the e2e paths run against."""
import torch

n = 336960000
n_img = 77938843  # the c2 image
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


for name, f in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                ("d2h", lambda: h.copy_(d, non_blocking=True))):
    print(name, round(n / timed(f) / 1e6, 1), "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)


def both(k_up, k_down):
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d[:k_up].copy_(h[:k_up], non_blocking=True)
    with torch.cuda.stream(s2):
        h2[:k_down].copy_(d2[:k_down], non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


ms = timed(lambda: both(n, n))
print("bidir", round(n / ms / 1e6, 1), "GB/s each way")
ms = timed(lambda: both(n_img, n))
print("decompress pattern (image up + output down)", round(ms, 3), "ms ->",
      round(n / ms / 1e6, 1), "GB/s of output")
