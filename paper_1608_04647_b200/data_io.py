"""SFAB subject containers, dataset manifests and their ingestion onto the GPU.

The reference API of ``factorfit.data_io`` for the SRM path
(``/root/reference/pkg/src/factorfit/data_io.py:1-256``): the same container
layout and checks (``save_matrix``, ``read_header``, ``load_matrix``,
``load_subject``), the same manifest schema and validation
(``load_manifest``, ``write_manifest``) and the same exceptions
(``FormatError`` with ``offset``/``field``, ``DatasetConsistencyError`` with
``offenders``).  Container reads and writes go through the native library
(``srm_sfab_*`` in ``libsrm_b200.so``; host code, no GPU needed).

The ingestion path of SURVEY.md §8(f) row 1 is :func:`open_subjects` /
:func:`fit_manifest`: subject payloads are read by parallel ``pread`` calls
straight into a ring of pinned host slots, and the fit's upload pipeline
copies each slot to the device while the next files are being read.  A
subject therefore costs one pass through host memory and one H2D copy --
no intermediate numpy array.
"""

import ctypes
import json
import threading
from concurrent.futures import Future
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

import numpy as np

from . import _lib
from .data import SubjectData
from .errors import DatasetConsistencyError, InvalidInputError, ShapeError

__all__ = [
    "SubjectData",
    "ManifestEntry",
    "Manifest",
    "save_matrix",
    "load_matrix",
    "read_header",
    "save_subject",
    "load_subject",
    "load_manifest",
    "write_manifest",
    "PendingMatrix",
    "open_subjects",
    "fit_manifest",
]

MAGIC = b"SFAB"
VERSION = 1
DTYPE_F64_LE = 0
HEADER_SIZE = 28


@dataclass
class ManifestEntry:
    subject_id: str
    data_path: Path
    coords_path: Optional[Path] = None


@dataclass
class Manifest:
    name: str
    subjects: list
    grid_dims: Optional[tuple] = None
    path: Optional[Path] = None


def _path(p):
    return str(Path(p)).encode()


def save_matrix(path, X):
    """Write a 2-D float64 matrix into the SFAB container (data_io.py:130-141)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    if X.ndim != 2:
        raise ShapeError(f"container stores 2-D matrices, got ndim={X.ndim}")
    lib = _lib.load()
    ptr = X.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    _lib.check_sfab(lib.srm_sfab_write(_path(path), ptr, X.shape[0], X.shape[1]))


def read_header(path):
    """Validate a container header and return (rows, cols) (data_io.py:144-157)."""
    lib = _lib.load()
    rows, cols = ctypes.c_int64(), ctypes.c_int64()
    _lib.check_sfab(lib.srm_sfab_header(_path(path), ctypes.byref(rows), ctypes.byref(cols)))
    return int(rows.value), int(cols.value)


def _read_into(path, dst_ptr, capacity, threads=8):
    lib = _lib.load()
    _lib.check_sfab(lib.srm_sfab_read(_path(path), ctypes.c_void_p(dst_ptr), int(capacity), int(threads)))


def load_matrix(path, threads=8):
    """Read a matrix back into a fresh array, validating the header and payload length."""
    rows, cols = read_header(path)
    out = np.empty((rows, cols), dtype=np.float64)
    if out.size:
        _read_into(path, out.ctypes.data, out.nbytes, threads)
    return out


def save_subject(path, X):
    save_matrix(path, X)


def load_subject(data_path, coords_path=None, subject_id=None):
    """Load a subject matrix and, when given, its voxel coordinates (data_io.py:186-200).

    The SRM path has no use for the voxel grid; coordinates are validated as
    in the reference and kept as the raw ``V x 3`` array in ``grid``.
    """
    data_path = Path(data_path)
    X = load_matrix(data_path)
    grid = None
    if coords_path is not None:
        coords = load_matrix(coords_path)
        if coords.shape != (X.shape[0], 3):
            raise DatasetConsistencyError(
                f"coordinates {coords.shape} do not match {X.shape[0]} voxels",
                offenders=[subject_id or data_path.stem],
            )
        grid = coords
    return SubjectData(subject_id or data_path.stem, X, grid)


def load_manifest(path, model=None):
    """Parse and eagerly validate a dataset manifest (data_io.py:203-256).

    Reads every referenced subject header (not the payloads).  With
    ``model="srm"`` all subjects must share one TR count; with
    ``model="htfa"`` every subject needs coordinates.
    """
    path = Path(path)
    with open(path) as fh:
        doc = json.load(fh)
    base = path.parent
    entries = []
    seen = set()
    for item in doc.get("subjects", []):
        sid = item["id"]
        if sid in seen:
            raise DatasetConsistencyError("duplicate subject id", offenders=[sid])
        seen.add(sid)
        coords = item.get("coords_path")
        entries.append(ManifestEntry(sid, base / item["data_path"], (base / coords) if coords else None))
    if not entries:
        raise DatasetConsistencyError("manifest lists no subjects")
    dims = {}
    for e in entries:
        dims[e.subject_id] = read_header(e.data_path)
        if e.coords_path is not None:
            crows, ccols = read_header(e.coords_path)
            if ccols != 3 or crows != dims[e.subject_id][0]:
                raise DatasetConsistencyError("coordinate file does not match subject voxels",
                                              offenders=[e.subject_id])
    if model == "srm":
        ref = dims[entries[0].subject_id][1]
        offenders = [sid for sid, rc in dims.items() if rc[1] != ref]
        if offenders:
            raise DatasetConsistencyError(f"subjects disagree on TR count (expected {ref})", offenders=offenders)
    if model == "htfa":
        offenders = [e.subject_id for e in entries if e.coords_path is None]
        if offenders:
            raise DatasetConsistencyError("topographic fits need voxel coordinates for every subject",
                                          offenders=offenders)
    grid_dims = tuple(doc["grid_dims"]) if doc.get("grid_dims") else None
    return Manifest(doc.get("name", path.stem), entries, grid_dims, path)


def write_manifest(path, manifest):
    """Write ``manifest`` as JSON with paths relative to ``path``'s directory."""
    path = Path(path)
    doc = {"name": manifest.name, "subjects": []}
    for e in manifest.subjects:
        item = {"id": e.subject_id, "data_path": str(Path(e.data_path).relative_to(path.parent))}
        if e.coords_path:
            item["coords_path"] = str(Path(e.coords_path).relative_to(path.parent))
        doc["subjects"].append(item)
    if manifest.grid_dims:
        doc["grid_dims"] = list(manifest.grid_dims)
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=2)
        fh.write("\n")
    manifest.path = path
    return path


# ---------------------------------------------------------------------------
# ingestion onto the GPU
# ---------------------------------------------------------------------------

def chunk_bounds(n_items, workers, rank):
    """Contiguous shard of ``n_items`` for ``rank`` (cli.py:82-85 ``_chunk``)."""
    base, extra = divmod(n_items, workers)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


class PendingMatrix:
    """A subject payload being read into a pinned host slot.

    ``shape``/``dtype`` come from the header; :meth:`result` blocks until the
    read finished and returns the pinned ``V x T`` float64 tensor.  The fit's
    upload pipeline (``SrmEngine.load``) consumes it and calls
    :meth:`release` once its device copy is enqueued, which frees the slot for
    a later subject.
    """

    dtype = np.float64

    def __init__(self, shape, future, ring, index):
        self.shape = tuple(shape)
        self._future = future
        self._ring = ring
        self._index = index

    def result(self):
        return self._future.result()

    def release(self, event):
        self._ring.release(self._index, event)

    def numpy(self):
        """Host copy (blocks; for callers outside the GPU fit)."""
        return self.result().numpy().copy()


class _SlotRing:
    """Pinned host slots reused in order; slot i is refilled for item i + n
    only after item i's device copy (its recorded CUDA event) has completed."""

    def __init__(self, slot_bytes, n_slots, n_items):
        import torch

        self.slots = [torch.empty(slot_bytes, dtype=torch.uint8, pin_memory=True) for _ in range(n_slots)]
        self.events = [None] * n_items
        self.released = [threading.Event() for _ in range(n_items)]

    def acquire(self, i):
        prev = i - len(self.slots)
        if prev >= 0:
            self.released[prev].wait()
            if self.events[prev] is not None:
                self.events[prev].synchronize()
        return self.slots[i % len(self.slots)]

    def release(self, i, event):
        self.events[i] = event
        self.released[i].set()


def open_subjects(manifest, rank=0, size=1, threads=8, slots=3):
    """This rank's contiguous share of a manifest as ``SubjectData`` whose ``X``
    are :class:`PendingMatrix` reads into pinned slots (read-ahead ``slots``)."""
    import torch

    if not isinstance(manifest, Manifest):
        manifest = load_manifest(manifest, model="srm")
    lo, hi = chunk_bounds(len(manifest.subjects), size, rank)
    entries = manifest.subjects[lo:hi]
    if not entries:
        return []
    shapes = [read_header(e.data_path) for e in entries]
    slot_bytes = max(r * c for r, c in shapes) * 8
    ring = _SlotRing(max(slot_bytes, 8), min(slots, len(entries)), len(entries))
    futs = [Future() for _ in entries]

    def reader():  # one file at a time, each with `threads` parallel preads
        for i, e in enumerate(entries):
            try:
                buf = ring.acquire(i)
                r, c = shapes[i]
                nb = r * c * 8
                if nb:
                    _read_into(e.data_path, buf.data_ptr(), nb, threads)
                futs[i].set_result(buf[:nb].view(torch.float64).view(r, c))
            except BaseException as exc:  # noqa: BLE001 -- surfaces in PendingMatrix.result()
                for f in futs[i:]:
                    f.set_exception(exc)
                return

    # a daemon thread: a fit that stops consuming (an exception upstream) never blocks exit
    threading.Thread(target=reader, name="sfab-reader", daemon=True).start()
    return [SubjectData(e.subject_id, PendingMatrix(shapes[i], futs[i], ring, i))
            for i, e in enumerate(entries)]


def fit_manifest(manifest, config, comm=None, threads=8, **fit_kwargs):
    """``srm.fit`` over this worker's contiguous share of a manifest's subjects,
    streaming the SFAB payloads through pinned slots onto the GPU."""
    from . import srm
    from .collectives import SerialCommunicator

    comm = comm if comm is not None else SerialCommunicator()
    subjects = open_subjects(manifest, comm.rank, comm.size, threads=threads)
    if not subjects:
        raise InvalidInputError(f"rank {comm.rank} has no subjects in the manifest")
    return srm.fit(subjects, config, comm, **fit_kwargs)
