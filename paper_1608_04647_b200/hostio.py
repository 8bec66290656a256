"""Host <-> device transfers through cached pinned staging buffers.

Pageable ``cudaMemcpy`` on this platform runs at 2-5 GB/s (the driver bounces
through its own small pinned buffer on one thread), while a copy from pinned
memory runs at PCIe speed (~55 GB/s) -- but pinning a fresh multi-GB buffer
costs more than the copy.  These helpers keep two pinned chunks per device,
pipeline chunked DMA on a side stream with multi-threaded host memcpy into
(or out of) the caller's ordinary numpy memory.  They are used for the model
read-back of ``fit`` (W, mu) and for numpy subject uploads.
"""

import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_CHUNK = 64 << 20
_SMALL = 8 << 20
_lock = threading.Lock()
_state = {}


def _torch():
    import torch

    return torch


def _get_state(device):
    torch = _torch()
    key = str(device)
    with _lock:
        st = _state.get(key)
        if st is None:
            st = {
                "bufs": [torch.empty(_CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(2)],
                "stream": torch.cuda.Stream(device=device),
                "pool": ThreadPoolExecutor(8),
            }
            _state[key] = st
    return st


def _par_copy(pool, dst, src, parts=8):
    """Copy 1-D uint8 numpy ``src`` into ``dst`` with several threads."""
    n = dst.shape[0]
    step = (n + parts - 1) // parts
    futs = [pool.submit(np.copyto, dst[a: a + step], src[a: a + step]) for a in range(0, n, step)]
    for f in futs:
        f.result()


def to_host(t):
    """Device tensor -> new numpy array (same dtype/shape)."""
    torch = _torch()
    t = t.detach().contiguous()
    nbytes = t.numel() * t.element_size()
    if not t.is_cuda or nbytes <= _SMALL:
        return t.cpu().numpy()
    out = np.empty(tuple(t.shape), dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
    dst = out.reshape(-1).view(np.uint8)
    src = t.reshape(-1).view(torch.uint8)
    st = _get_state(t.device)
    stream, pool, bufs = st["stream"], st["pool"], st["bufs"]
    stream.wait_stream(torch.cuda.current_stream(t.device))
    pending = [None, None]
    with _lock:
        for i, off in enumerate(range(0, nbytes, _CHUNK)):
            b = i % 2
            n = min(_CHUNK, nbytes - off)
            if pending[b] is not None:
                pending[b].result()
            with torch.cuda.stream(stream):
                bufs[b][:n].copy_(src[off: off + n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            ev.synchronize()
            host = bufs[b][:n].numpy()
            pending[b] = pool.submit(_par_copy, pool, dst[off: off + n], host, 4)
        for p in pending:
            if p is not None:
                p.result()
    return out


def to_pinned(t):
    """Device tensor -> numpy view of a pinned host copy (one DMA at PCIe speed).

    The pinned block comes from torch's caching host allocator and returns to
    it when the last numpy view is released, so repeated fits reuse it.
    """
    torch = _torch()
    t = t.detach().contiguous()
    host = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    host.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return host.numpy()


def to_device(arr, device, out=None):
    """numpy array -> device tensor (``out`` if given), staged through pinned chunks."""
    torch = _torch()
    arr = np.ascontiguousarray(arr)
    if out is None:
        out = torch.empty(arr.shape, dtype=torch.from_numpy(arr[:0].reshape(-1)).dtype, device=device)
    nbytes = arr.nbytes
    if nbytes <= _SMALL:
        out.copy_(torch.from_numpy(arr))
        return out
    src = arr.reshape(-1).view(np.uint8)
    dst = out.reshape(-1).view(torch.uint8)
    st = _get_state(device)
    stream, pool, bufs = st["stream"], st["pool"], st["bufs"]
    events = [None, None]
    with _lock:
        for i, off in enumerate(range(0, nbytes, _CHUNK)):
            b = i % 2
            n = min(_CHUNK, nbytes - off)
            if events[b] is not None:
                events[b].synchronize()
            _par_copy(pool, bufs[b][:n].numpy(), src[off: off + n], 4)
            with torch.cuda.stream(stream):
                dst[off: off + n].copy_(bufs[b][:n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            events[b] = ev
        for ev in events:
            if ev is not None:
                ev.synchronize()
    torch.cuda.current_stream(device).wait_stream(stream)
    return out


class PinnedRing:
    """A few reusable pinned host slots (pooled per device and slot count).

    Producers fill a slot on a worker thread after the slot's previous device
    copy has completed; the consumer issues an asynchronous copy from it and
    records an event that guards the slot's next reuse.  A ring is checked
    out by one fit at a time (:meth:`acquire` / :meth:`release`), so fits
    running concurrently (e.g. one thread per rank) never share slots, and
    :meth:`cancel` wakes producers of an abandoned fit so they return without
    writing.
    """

    _pool = {}

    def __init__(self, slot_bytes, nslots):
        torch = _torch()
        self.slots = [torch.empty(slot_bytes, dtype=torch.uint8, pin_memory=True) for _ in range(nslots)]
        self.events = [None] * nslots
        self.slot_bytes = slot_bytes
        self.issued = []
        self.cancelled = False
        self.key = None

    @classmethod
    def acquire(cls, device, slot_bytes, nslots=4, n_items=0):
        key = (str(device), nslots)
        with _lock:
            free = cls._pool.setdefault(key, [])
            ring = None
            for i, r in enumerate(free):
                if r.slot_bytes >= slot_bytes:
                    ring = free.pop(i)
                    break
        if ring is None:
            ring = cls(slot_bytes, nslots)
        ring.key = key
        ring.events = [None] * nslots
        ring.issued = [threading.Event() for _ in range(n_items)]
        ring.cancelled = False
        return ring

    def release(self):
        """Return the ring to the pool (after the fit's producers are done)."""
        with _lock:
            pool = PinnedRing._pool.setdefault(self.key, [])
            if self not in pool:
                pool.append(self)
                del pool[:-2]  # keep at most two idle rings per key

    def cancel(self):
        self.cancelled = True
        for ev in self.issued:
            ev.set()

    def view(self, i, shape, dtype=np.float64):
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        return self.slots[i % len(self.slots)][:n].numpy().view(dtype).reshape(shape)

    def tensor(self, i, nbytes):
        return self.slots[i % len(self.slots)][:nbytes]

    def wait_free(self, i):
        """Block until item i's slot is no longer read by item i - nslots's
        copy; False when the fit was cancelled."""
        prev = i - len(self.slots)
        if prev >= 0:
            self.issued[prev].wait()
            if self.cancelled:
                return False
            ev = self.events[prev % len(self.slots)]
            if ev is not None:
                ev.synchronize()
        return not self.cancelled

    def mark_used(self, i, event):
        self.events[i % len(self.slots)] = event
        if i < len(self.issued):
            self.issued[i].set()
