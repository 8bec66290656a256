"""Host-side logic without a GPU: config, sharding, communicators, cost model, data."""

import numpy as np
import pytest

from paper_1608_04647_b200 import srm
from paper_1608_04647_b200.collectives import SerialCommunicator, rank_counts, rank_offsets, shard_bounds
from paper_1608_04647_b200.data import CONFIGS, recipe_numpy
from paper_1608_04647_b200.errors import CollectiveContractError, ConfigError


def test_config_validation():
    """srm.py:54-67 / test_srm.py:187-189."""
    srm.SrmConfig(k=2).validate()
    for bad in (dict(k=0), dict(k=2, iterations=0), dict(k=2, tolerance=0.0), dict(k=2, tolerance=-1.0)):
        with pytest.raises(ConfigError):
            srm.SrmConfig(**bad).validate()


def test_fit_rejects_empty_shard_without_gpu():
    with pytest.raises(ConfigError):
        srm.fit([], srm.SrmConfig(k=2))


@pytest.mark.parametrize("n,w", [(10, 3), (40, 8), (5, 2), (7, 7), (3, 4)])
def test_shard_bounds_match_reference_chunking(n, w):
    """cli.py:82-85 _chunk: contiguous, sizes differ by at most one, earlier ranks larger."""
    bounds = [shard_bounds(n, w, r) for r in range(w)]
    assert bounds[0][0] == 0 and bounds[-1][1] == n
    for (a, b), (c, _) in zip(bounds, bounds[1:]):
        assert b == c
    sizes = [b - a for a, b in bounds]
    assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)


def test_serial_communicator_protocol():
    comm = SerialCommunicator()
    assert comm.rank == 0 and comm.size == 1
    assert comm.gather(b"abc") == [b"abc"]
    a = np.arange(6.0).reshape(2, 3)
    assert np.array_equal(comm.broadcast(a), a)
    assert np.array_equal(comm.reduce_sum(a), a)
    with pytest.raises(CollectiveContractError):
        comm.broadcast(np.zeros(3))
    comm.barrier()
    assert comm.stats.gather_calls == 1 and comm.stats.bcast_calls == 1
    assert rank_counts(comm, 4) == [4]
    assert rank_offsets(comm, 4) == (0, 4)


def test_algorithm_cost_model():
    c2 = CONFIGS["cfg2"]
    assert srm.choose_algorithm([c2["n_voxels"]] * 40, c2["n_trs"], c2["k"], 20) == "gram"
    # few iterations: the one-time X^T X does not pay off
    assert srm.choose_algorithm([c2["n_voxels"]] * 40, c2["n_trs"], c2["k"], 2) == "stream"
    # T close to V: the Gram is as large as the data
    assert srm.choose_algorithm([3000] * 4, 2900, 50, 10) == "stream"
    # memory guard
    assert srm.choose_algorithm([30000] * 40, 1000, 50, 20, free_bytes=1 << 20) == "stream"


def test_recipe_is_seeded_and_row_centred():
    xs, s, rho = recipe_numpy(3, 200, 40, 5, seed=9)
    xs2, s2, rho2 = recipe_numpy(3, 200, 40, 5, seed=9)
    assert all(np.array_equal(a, b) for a, b in zip(xs, xs2)) and np.array_equal(s, s2)
    assert all(0.5 <= r <= 1.5 for r in rho)
    assert max(float(np.max(np.abs(x.mean(axis=1)))) for x in xs) < 1e-12
    sub, _, _ = recipe_numpy(3, 200, 40, 5, seed=9, first_subject=1, count=1)
    assert np.array_equal(sub[0], xs[1])
    x32, _, _ = recipe_numpy(2, 100, 20, 4, seed=1, smooth=5.0, dtype="f32")
    assert x32[0].dtype == np.float32


def _sk_ranges(count, ldx, kp, max_ctas):
    """The stream-K partition of launch_oz_sg_sk (ozaki.cu): k-blocks of all
    (subject, 128-TR block, 64-feature half) tiles end to end, CTA c taking
    [c span, (c + 1) span) with span >= the k-blocks of one tile."""
    ntb, nz, nub = -(-ldx // 128), -(-kp // 64), ldx // 32
    units = count * ntb * nz * nub
    span = max(nub, -(-units // max_ctas))
    grid = -(-units // span)
    return [(c * span, min(units, (c + 1) * span)) for c in range(grid)], nub, units


@pytest.mark.parametrize("count,ldx,kp,max_ctas", [(40, 1024, 56, 146), (10, 2016, 72, 146), (3, 96, 8, 146),
                                                   (256, 1024, 64, 146), (5, 1024, 56, 1), (7, 320, 104, 30)])
def test_stream_k_partition_joins_at_most_two_parts(count, ldx, kp, max_ctas):
    """Every tile meets at most two CTA ranges, so a cut tile has exactly one
    tail (first segment of CTA c + 1) and one head (last segment of CTA c):
    the single park slot and flag per CTA of k_oz_sg_sk suffice, and the grid
    never exceeds the co-resident CTAs it was sized for."""
    ranges, nub, units = _sk_ranges(count, ldx, kp, max_ctas)
    assert len(ranges) <= max_ctas
    assert ranges[0][0] == 0 and ranges[-1][1] == units
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    for tile in range(units // nub):
        lo, hi = tile * nub, (tile + 1) * nub
        parts = [c for c, (a, b) in enumerate(ranges) if a < hi and b > lo]
        assert 1 <= len(parts) <= 2
        if len(parts) == 2:
            c = parts[0]
            assert parts[1] == c + 1 and ranges[c][1] < hi and ranges[c + 1][0] > lo
