"""Host<->device copy bandwidth of the e2e state (config 2: 1.36 GB fp64), pinned memory."""
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 884736 * 192
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
h.fill_(1.0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


gb = n * 8 / 1e9
ms = t(lambda: d.copy_(h, non_blocking=True))
print(f"H2D {gb:.2f} GB {ms:.2f} ms {gb / ms * 1e3:.1f} GB/s")
ms = t(lambda: h.copy_(d, non_blocking=True))
print(f"D2H {gb:.2f} GB {ms:.2f} ms {gb / ms * 1e3:.1f} GB/s")


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


ms = t(both)
print(f"H2D||D2H {2 * gb:.2f} GB {ms:.2f} ms {2 * gb / ms * 1e3:.1f} GB/s aggregate")
for chunk_mb in (16, 64, 256):
    c = chunk_mb * 2 ** 20 // 8

    def chunked():
        for i in range(0, n, c):
            d[i:i + c].copy_(h[i:i + c], non_blocking=True)
    ms = t(chunked)
    print(f"H2D chunks {chunk_mb} MB {ms:.2f} ms {gb / ms * 1e3:.1f} GB/s")
