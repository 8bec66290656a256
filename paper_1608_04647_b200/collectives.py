"""Communicators for the SRM fit: the reference protocol on torch.distributed.

The reference fit talks to its peers only through a ``Communicator``
(``/root/reference/pkg/src/factorfit/collectives.py:94-176``): ``rank``,
``size``, ``gather(bytes)``, ``broadcast(2-D float64)``, ``barrier()`` and a
``stats`` ledger.  This module keeps that surface so the reference CLI and
tests can drive the new fit, and adds the two device collectives the B200
path actually uses per EM iteration:

* ``all_gather_into(out, mine)`` -- the ordered E-step table (every rank gets
  every subject's K x T term and sums them in ascending global subject
  order, so S is bit-identical on every rank and independent of the shard
  layout, srm.py:193-213);
* ``all_reduce_sum(buf)`` -- the unordered variant for very large subject
  counts (one K x T buffer per rank).

``TorchCommunicator`` runs them on ``torch.distributed`` (NCCL over
NVLink/NVSwitch for CUDA tensors, gloo for CPU tensors).  Any other object
with the reference protocol (e.g. factorfit's thread or socket
communicators) is accepted by ``fit`` too; its exchanges are staged through
host memory with ``gather`` + ``broadcast``.
"""

import struct
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import CollectiveContractError, ConfigError

__all__ = [
    "CollectiveStats",
    "Communicator",
    "SerialCommunicator",
    "TorchCommunicator",
    "rank_offsets",
    "rank_counts",
    "shard_bounds",
    "any_rank",
]

_LEN = struct.Struct("<Q")


@dataclass
class CollectiveStats:
    """Logical per-rank communication ledger (collectives.py:67-84 fields)."""

    reduce_calls: int = 0
    reduce_bytes: int = 0
    bcast_calls: int = 0
    bcast_bytes: int = 0
    gather_calls: int = 0
    gather_bytes: int = 0
    barrier_calls: int = 0
    allgather_calls: int = 0
    allgather_bytes: int = 0
    allreduce_calls: int = 0
    allreduce_bytes: int = 0
    alltoall_calls: int = 0
    alltoall_bytes: int = 0
    seconds: float = field(default=0.0)


def _as_payload(a, name="payload"):
    out = np.ascontiguousarray(a, dtype=np.float64)
    if out.ndim != 2:
        raise CollectiveContractError(f"{name} must be a 2-D float64 matrix")
    return out


class Communicator:
    """Rank/size handle with the reference collectives plus device collectives."""

    backend = "abstract"

    def __init__(self, rank, size):
        if size < 1 or not (0 <= rank < size):
            raise ConfigError(f"invalid rank/size ({rank}/{size})")
        self.rank = rank
        self.size = size
        self.stats = CollectiveStats()

    # -- reference protocol -------------------------------------------------
    def reduce_sum(self, local):
        local = _as_payload(local, "reduce_sum payload")
        t0 = time.perf_counter()
        try:
            out = self._reduce_sum(local)
        finally:
            self.stats.seconds += time.perf_counter() - t0
        self.stats.reduce_calls += 1
        self.stats.reduce_bytes += local.nbytes
        return out

    def broadcast(self, buf):
        if self.rank == 0:
            buf = _as_payload(buf, "broadcast payload")
        t0 = time.perf_counter()
        try:
            out = self._broadcast(buf)
        finally:
            self.stats.seconds += time.perf_counter() - t0
        self.stats.bcast_calls += 1
        self.stats.bcast_bytes += out.nbytes
        return out

    def gather(self, local):
        local = bytes(local)
        t0 = time.perf_counter()
        try:
            out = self._gather(local)
        finally:
            self.stats.seconds += time.perf_counter() - t0
        self.stats.gather_calls += 1
        self.stats.gather_bytes += len(local)
        return out

    def barrier(self):
        t0 = time.perf_counter()
        try:
            self._barrier()
        finally:
            self.stats.seconds += time.perf_counter() - t0
        self.stats.barrier_calls += 1

    # -- device collectives ---------------------------------------------------
    def all_gather_into(self, out, mine):
        """``out`` (size * n elements) <- concatenation of every rank's ``mine``."""
        t0 = time.perf_counter()
        try:
            self._all_gather_into(out, mine)
        finally:
            self.stats.seconds += time.perf_counter() - t0
        self.stats.allgather_calls += 1
        self.stats.allgather_bytes += mine.numel() * mine.element_size()

    def all_to_all_into(self, out, inp):
        """``out`` chunk r <- rank r's ``inp`` chunk for this rank (equal
        chunks of ``inp.numel() / size`` elements)."""
        t0 = time.perf_counter()
        try:
            self._all_to_all_into(out, inp)
        finally:
            self.stats.seconds += time.perf_counter() - t0
        self.stats.alltoall_calls += 1
        self.stats.alltoall_bytes += inp.numel() * inp.element_size()

    def all_reduce_sum(self, buf):
        t0 = time.perf_counter()
        try:
            self._all_reduce_sum(buf)
        finally:
            self.stats.seconds += time.perf_counter() - t0
        self.stats.allreduce_calls += 1
        self.stats.allreduce_bytes += buf.numel() * buf.element_size()

    def close(self):
        pass

    def abort(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class SerialCommunicator(Communicator):
    """Single-worker backend; all collectives are local (collectives.py:179-197)."""

    backend = "serial"

    def __init__(self):
        super().__init__(0, 1)

    def _reduce_sum(self, local):
        return local.copy()

    def _broadcast(self, buf):
        return buf.copy()

    def _gather(self, local):
        return [local]

    def _barrier(self):
        pass

    def _all_gather_into(self, out, mine):
        if out.data_ptr() != mine.data_ptr():
            out.copy_(mine.reshape(out.shape))

    def _all_reduce_sum(self, buf):
        pass

    def _all_to_all_into(self, out, inp):
        if out.data_ptr() != inp.data_ptr():
            out.copy_(inp.reshape(out.shape))


class TorchCommunicator(Communicator):
    """One rank of a ``torch.distributed`` process group.

    NCCL groups run the device collectives on CUDA tensors directly (NVLink /
    NVSwitch); gloo groups run them on CPU tensors (CUDA tensors are staged
    through host memory).  Launch one process per GPU (torchrun) and
    rendezvous on 127.0.0.1.
    """

    def __init__(self, group=None):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise ConfigError("torch.distributed is not initialised")
        self._dist = dist
        self._group = group
        super().__init__(dist.get_rank(group), dist.get_world_size(group))
        self.backend = str(dist.get_backend(group))

    @property
    def device_collectives(self):
        return self.backend == "nccl"

    def _objs(self, obj):
        out = [None] * self.size
        self._dist.all_gather_object(out, obj, group=self._group)
        return out

    def _reduce_sum(self, local):
        parts = self._objs(local)
        if self.rank != 0:
            return None
        for r, a in enumerate(parts):
            if a.shape != parts[0].shape:
                raise CollectiveContractError(
                    f"reduce_sum shape mismatch: rank {r} has {a.shape}, rank 0 has {parts[0].shape}")
        acc = parts[0].copy()
        for a in parts[1:]:
            acc += a
        return acc

    def _tensor_device(self):
        import torch

        return torch.device("cuda", torch.cuda.current_device()) if self.device_collectives else torch.device("cpu")

    def _broadcast(self, buf):
        # shape, then the raw float64 payload: two tensor broadcasts, no pickling
        import torch

        dev = self._tensor_device()
        shape = torch.zeros(2, dtype=torch.int64, device=dev)
        if self.rank == 0:
            shape[0], shape[1] = buf.shape
        self._dist.broadcast(shape, src=0, group=self._group)
        rows, cols = (int(x) for x in shape.cpu())
        if self.rank == 0:
            data = torch.from_numpy(np.ascontiguousarray(buf, dtype=np.float64)).to(dev)
        else:
            data = torch.empty((rows, cols), dtype=torch.float64, device=dev)
        self._dist.broadcast(data, src=0, group=self._group)
        return data.cpu().numpy()

    def _gather(self, local):
        parts = self._objs(local)
        return parts if self.rank == 0 else None

    def _barrier(self):
        self._dist.barrier(group=self._group)

    def _all_gather_into(self, out, mine):
        import torch

        if self.device_collectives and out.is_cuda:
            self._dist.all_gather_into_tensor(out.view(-1), mine.reshape(-1), group=self._group)
            return
        host = mine.detach().reshape(-1).cpu()
        parts = [torch.empty_like(host) for _ in range(self.size)]
        self._dist.all_gather(parts, host, group=self._group)
        out.view(-1).copy_(torch.cat(parts).to(out.device))

    def _all_to_all_into(self, out, inp):
        if self.device_collectives and out.is_cuda:
            self._dist.all_to_all_single(out.view(-1), inp.reshape(-1), group=self._group)
            return
        import torch

        host_in = inp.detach().reshape(-1).cpu()
        host_out = torch.empty_like(host_in)
        self._dist.all_to_all_single(host_out, host_in, group=self._group)
        out.view(-1).copy_(host_out.to(out.device))

    def _all_reduce_sum(self, buf):
        if self.device_collectives and buf.is_cuda:
            self._dist.all_reduce(buf, group=self._group)
            return
        host = buf.detach().cpu()
        self._dist.all_reduce(host, group=self._group)
        buf.copy_(host.to(buf.device))


def shard_bounds(n_items, workers, rank):
    """Contiguous shard [start, stop) of ``n_items`` for ``rank`` (cli.py:82-85)."""
    base, extra = divmod(n_items, workers)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def rank_counts(comm, local_count):
    """Every rank's local item count, in rank order (all ranks get the list)."""
    if comm.size == 1:
        return [int(local_count)]
    if isinstance(comm, TorchCommunicator):
        return [int(c) for c in comm._objs(int(local_count))]
    # reference protocol: gather to root, broadcast the table (collectives.py:480-494)
    blobs = comm.gather(_LEN.pack(int(local_count)))
    if comm.rank == 0:
        counts = np.array([[_LEN.unpack(b)[0] for b in blobs]], dtype=np.float64)
    else:
        counts = None
    table = comm.broadcast(counts)
    return [int(c) for c in table[0]]


def any_rank(comm, flag):
    """True on every rank when ``flag`` is true on any rank."""
    if comm.size == 1:
        return bool(flag)
    if isinstance(comm, TorchCommunicator):
        return any(bool(f) for f in comm._objs(bool(flag)))
    blobs = comm.gather(b"\x01" if flag else b"\x00")
    table = None
    if comm.rank == 0:
        table = np.array([[1.0 if any(b != b"\x00" for b in blobs) else 0.0]])
    return bool(comm.broadcast(table)[0, 0] != 0.0)


def rank_offsets(comm, local_count):
    """(this rank's first global index, total) -- collectives.py:480-494."""
    counts = rank_counts(comm, local_count)
    return int(sum(counts[: comm.rank])), int(sum(counts))
