"""Diagnostic: host page-fault cost of fresh output arrays (480 MB) and THP state."""
import mmap
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

n = 480 << 20
try:
    print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
except OSError as e:
    print("THP: n/a", e)
pool = ThreadPoolExecutor(16)


def touch(a, parts):
    step = -(-a.size // parts)
    list(pool.map(lambda o: a[o:o + step].fill(1), range(0, a.size, step)))


for parts in (1, 4, 16):
    for rep in range(2):
        t0 = time.perf_counter()
        a = np.empty(n, dtype=np.uint8)
        touch(a, parts)
        print(f"np.empty + touch ({parts:2d} threads): {time.perf_counter() - t0:.4f} s")
        del a
for parts in (1, 16):
    t0 = time.perf_counter()
    mm = mmap.mmap(-1, n)
    mm.madvise(mmap.MADV_HUGEPAGE)
    a = np.frombuffer(mm, dtype=np.uint8)
    touch(a, parts)
    print(f"mmap+MADV_HUGEPAGE + touch ({parts:2d} threads): {time.perf_counter() - t0:.4f} s")
    del a
b = np.ones(n, dtype=np.uint8)
c = np.empty(n, dtype=np.uint8)
c.fill(0)
t0 = time.perf_counter()
touch_src = -(-n // 16)
list(pool.map(lambda o: np.copyto(c[o:o + touch_src], b[o:o + touch_src]), range(0, n, touch_src)))
print(f"memcpy prefaulted 16 threads: {time.perf_counter() - t0:.4f} s")
