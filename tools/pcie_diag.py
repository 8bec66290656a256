"""Diagnostic: pinned H2D / D2H bandwidth (1 and 2 streams, chunk sizes) on this box."""
import time

import torch

n = 1 << 30  # 1 GiB
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
host2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def bw(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return nbytes / best / 1e9


print("H2D 1 stream  %.1f GB/s" % bw(lambda: dev.copy_(host, non_blocking=True), n))
h = n // 2


def two_h2d():
    with torch.cuda.stream(s1):
        dev[:h].copy_(host[:h], non_blocking=True)
    with torch.cuda.stream(s2):
        dev[h:].copy_(host[h:], non_blocking=True)


print("H2D 2 streams %.1f GB/s" % bw(two_h2d, n))
for c in (8 << 20, 64 << 20, 256 << 20):
    def chunked():
        for o in range(0, n, c):
            dev[o:o + c].copy_(host[o:o + c], non_blocking=True)
    print("H2D chunks %4d MiB %.1f GB/s" % (c >> 20, bw(chunked, n)))
print("D2H 1 stream  %.1f GB/s" % bw(lambda: host.copy_(dev, non_blocking=True), n))


def two_d2h():
    with torch.cuda.stream(s1):
        host[:h].copy_(dev[:h], non_blocking=True)
    with torch.cuda.stream(s2):
        host[h:].copy_(dev[h:], non_blocking=True)


print("D2H 2 streams %.1f GB/s" % bw(two_d2h, n))


def bidir():
    with torch.cuda.stream(s1):
        dev.copy_(host, non_blocking=True)
    with torch.cuda.stream(s2):
        host2.copy_(dev, non_blocking=True)


print("H2D+D2H concurrent %.1f GB/s (sum)" % bw(bidir, 2 * n))
