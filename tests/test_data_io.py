"""SFAB containers and manifests (data_io.py) against files written by the reference.

The fixtures under tests/golden/sfab/ were produced by the reference's own
``factorfit.data_io`` (tests/golden/make_golden_sfab.py), including the
malformed containers and the exception the reference raises for each.
Host-only: the native reader/writer needs no GPU.
"""

import json
import shutil
from pathlib import Path

import numpy as np
import pytest

from paper_1608_04647_b200 import data_io
from paper_1608_04647_b200.errors import (
    DatasetConsistencyError,
    FormatError,
    InvalidInputError,
    ShapeError,
)

GOLD = Path(__file__).resolve().parent / "golden" / "sfab"


def _golden_arrays():
    """The matrices make_golden_sfab.py drew (same generator, same order)."""
    rng = np.random.default_rng(20261020)
    out, coords = [], None
    for i, v in enumerate((37, 52, 41)):
        out.append(rng.standard_normal((v, 12)))
        if i == 1:
            coords = rng.integers(0, 9, size=(v, 3)).astype(np.float64)
    return out, coords


def test_reads_reference_containers():
    xs, coords = _golden_arrays()
    for i, x in enumerate(xs):
        p = GOLD / "subjects" / f"sub-{i:02d}.sfab"
        assert data_io.read_header(p) == x.shape
        got = data_io.load_matrix(p)
        assert got.dtype == np.float64 and np.array_equal(got, x)
    s = data_io.load_subject(GOLD / "subjects" / "sub-01.sfab", GOLD / "subjects" / "sub-01_coords.sfab", "sub-01")
    assert s.subject_id == "sub-01" and np.array_equal(s.X, xs[1]) and np.array_equal(s.grid, coords)


def test_writes_reference_bytes(tmp_path):
    xs, _ = _golden_arrays()
    for i, x in enumerate(xs):
        p = tmp_path / f"{i}.sfab"
        data_io.save_matrix(p, x)
        assert p.read_bytes() == (GOLD / "subjects" / f"sub-{i:02d}.sfab").read_bytes()


def test_large_parallel_read(tmp_path):
    x = np.random.default_rng(1).standard_normal((4096, 700))  # 23 MB: several pread workers
    p = tmp_path / "big.sfab"
    data_io.save_matrix(p, x)
    for threads in (1, 3, 8):
        assert np.array_equal(data_io.load_matrix(p, threads=threads), x)


@pytest.mark.parametrize("name", ["bad_magic", "bad_version", "bad_dtype", "short_header", "short_payload",
                                  "trailing"])
def test_malformed_containers_match_reference_errors(name):
    exp = json.loads((GOLD / "malformed" / "expected.json").read_text())[name]
    with pytest.raises(FormatError) as ei:
        data_io.load_matrix(GOLD / "malformed" / f"{name}.sfab")
    assert type(ei.value).__name__ == exp["class"]
    assert ei.value.field == exp["field"] and ei.value.offset == exp["offset"]


def test_write_rejects_bad_input(tmp_path):
    with pytest.raises(InvalidInputError):
        data_io.save_matrix(tmp_path / "nan.sfab", np.array([[1.0, np.nan]]))
    with pytest.raises(ShapeError):
        data_io.save_matrix(tmp_path / "3d.sfab", np.zeros((2, 2, 2)))
    with pytest.raises(OSError):
        data_io.load_matrix(tmp_path / "missing.sfab")


def test_manifest_round_trip(tmp_path):
    man = data_io.load_manifest(GOLD / "manifest.json", model="srm")
    assert man.name == "golden" and man.grid_dims == (9, 9, 9)
    assert [e.subject_id for e in man.subjects] == ["sub-00", "sub-01", "sub-02"]
    assert man.subjects[1].coords_path is not None and man.subjects[0].coords_path is None
    # write_manifest relative to a copy of the tree reproduces the reference's JSON
    dst = tmp_path / "ds"
    shutil.copytree(GOLD, dst)
    man2 = data_io.load_manifest(dst / "manifest.json")
    data_io.write_manifest(dst / "again.json", man2)
    assert json.loads((dst / "again.json").read_text()) == json.loads((GOLD / "manifest.json").read_text())


def test_manifest_consistency_errors(tmp_path):
    shutil.copytree(GOLD / "subjects", tmp_path / "subjects")
    data_io.save_matrix(tmp_path / "subjects" / "other_t.sfab", np.zeros((5, 7)))

    def write(doc):
        p = tmp_path / "m.json"
        p.write_text(json.dumps(doc))
        return p

    with pytest.raises(DatasetConsistencyError) as ei:
        data_io.load_manifest(write({"subjects": [{"id": "a", "data_path": "subjects/sub-00.sfab"},
                                                  {"id": "a", "data_path": "subjects/sub-02.sfab"}]}))
    assert ei.value.offenders == ["a"]
    with pytest.raises(DatasetConsistencyError) as ei:
        data_io.load_manifest(write({"subjects": [{"id": "a", "data_path": "subjects/sub-00.sfab"},
                                                  {"id": "b", "data_path": "subjects/other_t.sfab"}]}),
                              model="srm")
    assert ei.value.offenders == ["b"]
    with pytest.raises(DatasetConsistencyError):
        data_io.load_manifest(write({"subjects": []}))
    with pytest.raises(DatasetConsistencyError) as ei:
        data_io.load_manifest(write({"subjects": [{"id": "a", "data_path": "subjects/sub-00.sfab",
                                                   "coords_path": "subjects/sub-01_coords.sfab"}]}))
    assert ei.value.offenders == ["a"]
    with pytest.raises(DatasetConsistencyError):
        data_io.load_manifest(write({"subjects": [{"id": "a", "data_path": "subjects/sub-00.sfab"}]}),
                              model="htfa")


def test_chunk_bounds_match_cli():
    # cli.py:82-85: contiguous, the first `extra` ranks take one more
    assert [data_io.chunk_bounds(10, 4, r) for r in range(4)] == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert [data_io.chunk_bounds(2, 3, r) for r in range(3)] == [(0, 1), (1, 2), (2, 2)]
