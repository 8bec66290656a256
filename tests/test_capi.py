"""C ABI of libsrm_b200.so without a GPU: symbols, plan bookkeeping, errors.

srm_plan_create / srm_plan_dim / srm_plan_region are host-only calls, so the
static work decomposition and workspace layout are testable on CPU.
"""

import ctypes
import re

import pytest

from conftest import ROOT
from paper_1608_04647_b200 import _lib
from paper_1608_04647_b200.errors import (ConfigError, DeviceError, ShapeError, from_status,
                                          DefinitenessError, RankError, InvalidInputError)

HEADER = ROOT / "include" / "srm_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(srm_[a-z_0-9]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == names
    assert lib.srm_abi_version() == 1


def _plan(v, t, k, iters=3, world=1, rank=0, counts=None, flags=0):
    lib = _lib.load()
    counts = counts or [len(v)]
    p = ctypes.c_void_p()
    rc = lib.srm_plan_create(ctypes.byref(p), 0, len(v), (ctypes.c_int64 * len(v))(*v), t, k, iters,
                             world, rank, (ctypes.c_int32 * world)(*counts), flags)
    return rc, p


def test_plan_dims_and_layout():
    lib = _lib.load()
    rc, p = _plan([300, 500, 1000], 50, 5)
    assert rc == 0
    try:
        assert lib.srm_plan_dim(p, _lib.D_LDX) == 64
        assert lib.srm_plan_dim(p, _lib.D_KP) == 8
        assert lib.srm_plan_dim(p, _lib.D_ROWS) == 1800
        assert lib.srm_plan_dim(p, _lib.D_TERM_STRIDE) == 8 * 64 + 8
        assert lib.srm_plan_dim(p, _lib.D_N_SLOTS) == 3
        assert lib.srm_plan_dim(p, _lib.D_ITEMS_A) == 3 + 4 + 8
        total = lib.srm_plan_workspace_bytes(p)
        assert total > 1800 * 64 * 8
        end = 0
        for r in range(15):
            off, nb = ctypes.c_int64(), ctypes.c_int64()
            assert lib.srm_plan_region(p, r, ctypes.byref(off), ctypes.byref(nb)) == 0
            assert off.value % 256 == 0 and off.value >= end
            end = off.value + nb.value
        assert end <= total
    finally:
        lib.srm_plan_destroy(p)


def test_plan_ordered_slots_for_ranks():
    lib = _lib.load()
    # 5 subjects over 2 ranks as cli.py:_chunk splits them: [3, 2]
    rc0, p0 = _plan([40, 40, 40], 16, 3, world=2, rank=0, counts=[3, 2], flags=_lib.FLAG_ORDERED)
    rc1, p1 = _plan([40, 40], 16, 3, world=2, rank=1, counts=[3, 2], flags=_lib.FLAG_ORDERED)
    assert rc0 == 0 and rc1 == 0
    assert lib.srm_plan_dim(p0, _lib.D_N_SLOTS) == 6 and lib.srm_plan_dim(p1, _lib.D_N_SLOTS) == 6
    assert lib.srm_plan_dim(p0, _lib.D_SLOT_OFFSET) == 0
    assert lib.srm_plan_dim(p1, _lib.D_SLOT_OFFSET) == 3
    lib.srm_plan_destroy(p0)
    lib.srm_plan_destroy(p1)


@pytest.mark.parametrize("v,t,k,iters,code", [
    ([10], 8, 0, 3, _lib.load().srm_abi_version() and 1),   # k < 1 -> ConfigError
    ([10], 8, 3, 0, 1),                                      # iterations < 1
    ([2], 8, 3, 3, 2),                                       # V < k -> ShapeError
    ([500], 8, 200, 3, 7),                                   # k > 128 -> unsupported
    ([500], 8, 129, 3, 7),
])
def test_plan_errors(v, t, k, iters, code):
    rc, _ = _plan(v, t, k, iters)
    assert rc == code
    assert _lib.load().srm_last_error()


def test_status_mapping():
    assert isinstance(from_status(1), ConfigError)
    assert isinstance(from_status(2), ShapeError)
    assert isinstance(from_status(3, arg=4), InvalidInputError)
    e = from_status(4, arg=3)
    assert isinstance(e, DefinitenessError) and e.pivot == 3
    assert isinstance(from_status(5, arg=1), RankError)
    assert isinstance(from_status(6), DeviceError)
