"""Multi-rank paths: world_size 2 over gloo (127.0.0.1).

CPU tests cover the communicator and the ordered E-step exchange layout
(the C plan's slot table), the reduction order and the final rho^2 gather.
The GPU test runs two ranks of the real fit on one GPU with gloo carrying
the exchange through host memory (no kernel waits on another rank's kernel)
and checks bit-identity with the serial fit (srm.py:193-213 contract,
test_srm.py:200-229).
"""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _comm_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from paper_1608_04647_b200 import _lib
    from paper_1608_04647_b200.collectives import TorchCommunicator, rank_counts, rank_offsets, shard_bounds

    _init(rank, world, port)
    comm = TorchCommunicator()
    n_total = 5
    a, b = shard_bounds(n_total, world, rank)
    counts = rank_counts(comm, b - a)
    off, tot = rank_offsets(comm, b - a)
    g = comm.gather(bytes([rank]) * 3)
    bc = comm.broadcast(np.full((2, 2), 7.0) if rank == 0 else None)
    rs = comm.reduce_sum(np.full((1, 3), float(rank + 1)))

    # ordered exchange with the plan's slot layout: rank r owns slots [r*m, r*m + count_r)
    lib = _lib.load()
    p = ctypes.c_void_p()
    v = (ctypes.c_int64 * (b - a))(*([40] * (b - a)))
    rc = lib.srm_plan_create(ctypes.byref(p), 0, b - a, v, 16, 3, 2, world, rank,
                             (ctypes.c_int32 * world)(*counts), _lib.FLAG_ORDERED)
    assert rc == 0
    n_slots = lib.srm_plan_dim(p, _lib.D_N_SLOTS)
    slot0 = lib.srm_plan_dim(p, _lib.D_SLOT_OFFSET)
    lib.srm_plan_destroy(p)
    m = n_slots // world
    rng = np.random.default_rng(3)
    terms = rng.standard_normal((n_total, 6))          # every subject's "E-step term"
    table = torch.zeros((n_slots, 6), dtype=torch.float64)
    for j in range(b - a):
        table[slot0 + j] = torch.from_numpy(terms[a + j])
    comm.all_gather_into(table, table[rank * m: (rank + 1) * m].clone())
    order = [r * m + j for r in range(world) for j in range(counts[r])]
    acc = table[order[0]].clone()
    for s in order[1:]:
        acc += table[s]
    serial = terms[0].copy()
    for t in terms[1:]:
        serial += t
    buf = torch.full((4,), float(rank + 1), dtype=torch.float64)
    comm.all_reduce_sum(buf)
    out.put((rank, counts, off, tot, g, bc.tolist(), None if rs is None else rs.tolist(),
             np.array_equal(acc.numpy(), serial), buf.tolist(), comm.stats.allgather_calls))
    dist.destroy_process_group()


def test_gloo_two_ranks_communicator_and_ordered_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in (0, 1):
        _, counts, off, tot, g, bc, rs, ordered_ok, buf, ag = res[rank]
        assert counts == [3, 2] and tot == 5 and off == (0 if rank == 0 else 3)
        assert bc == [[7.0, 7.0], [7.0, 7.0]]
        assert ordered_ok, "ordered all-gather sum differs from the serial ascending sum"
        assert buf == [3.0] * 4 and ag == 1
    assert res[0][4] == [b"\x00" * 3, b"\x01" * 3] and res[1][4] is None
    assert res[0][6] == [[3.0, 3.0, 3.0]] and res[1][6] is None


def _dataset(name):
    from conftest import load_golden, golden_subjects
    from paper_1608_04647_b200.data import recipe_numpy

    if name == "recipe5":  # 5 subjects over 2 ranks: shards [3, 2] (cli.py:82-85)
        xs, _, _ = recipe_numpy(5, 700, 90, 6, seed=19)
        xs = [x[: 700 - 37 * i] for i, x in enumerate(xs)]
        return xs, 6, 5, 4
    g = load_golden(name)
    return golden_subjects(g), int(g["k"]), int(g["iterations"]), int(g["seed"])


def _colblock_worker(rank, world, port, out):
    """The SRM_FLAG_COLBLOCK exchange restated on host tensors with the plan's
    own dimensions (srm_plan_dim D_XREC / D_XRED, the k_xchg_* index maps):
    pack each local record's TR block q for rank q, all-to-all, sum this
    rank's block over (rank, local j) = ascending global order as the left
    fold of k_reduce_terms (acc = t_0 / r_0, acc += t_j / r_j), all-gather,
    unpack -- equal to one rank's fold bit for bit."""
    import torch
    import torch.distributed as dist

    from paper_1608_04647_b200 import _lib
    from paper_1608_04647_b200.collectives import TorchCommunicator, rank_counts, shard_bounds

    _init(rank, world, port)
    comm = TorchCommunicator()
    n_total, K, T = 5, 3, 70
    a, b = shard_bounds(n_total, world, rank)
    counts = rank_counts(comm, b - a)
    lib = _lib.load()
    p = ctypes.c_void_p()
    v = (ctypes.c_int64 * (b - a))(*([40] * (b - a)))
    rc = lib.srm_plan_create(ctypes.byref(p), 0, b - a, v, T, K, 2, world, rank,
                             (ctypes.c_int32 * world)(*counts), _lib.FLAG_ORDERED | _lib.FLAG_COLBLOCK)
    assert rc == 0
    flags = lib.srm_plan_dim(p, _lib.D_FLAGS)
    kp, ldx = lib.srm_plan_dim(p, _lib.D_KP), lib.srm_plan_dim(p, _lib.D_LDX)
    xrec, xred = lib.srm_plan_dim(p, _lib.D_XREC), lib.srm_plan_dim(p, _lib.D_XRED)
    lib.srm_plan_destroy(p)
    assert flags & _lib.FLAG_COLBLOCK and not flags & _lib.FLAG_ORDERED
    m, xw = max(counts), (ldx + world - 1) // world
    assert xrec == kp * xw + 8 and xred == kp * xw + 8
    rng = np.random.default_rng(5)
    terms = rng.standard_normal((n_total, kp, ldx))
    rho2 = rng.uniform(0.5, 1.5, n_total)
    send = torch.zeros((world, m, xrec), dtype=torch.float64)
    for q in range(world):
        for j in range(b - a):
            for f in range(kp):
                cols = [q * xw + c for c in range(xw)]
                send[q, j, f * xw: (f + 1) * xw] = torch.tensor(
                    [terms[a + j, f, c] if c < ldx else 0.0 for c in cols])
            send[q, j, kp * xw] = rho2[a + j]
    recv = torch.empty_like(send)
    comm.all_to_all_into(recv, send)
    mine = None
    for r in range(world):
        for j in range(counts[r]):
            x = recv[r, j, : kp * xw] / recv[r, j, kp * xw]
            mine = x.clone() if mine is None else mine + x
    blocks = torch.zeros((world, xred), dtype=torch.float64)
    blocks[rank, : kp * xw] = mine
    comm.all_gather_into(blocks.view(-1), blocks[rank].clone())
    red = np.zeros((kp, ldx))
    for q in range(world):
        for f in range(kp):
            for c in range(xw):
                if q * xw + c < ldx:
                    red[f, q * xw + c] = blocks[q, f * xw + c].item()
    serial = terms[0] / rho2[0]
    for i in range(1, n_total):
        serial = serial + terms[i] / rho2[i]
    out.put((rank, np.array_equal(red, serial), comm.stats.alltoall_calls))
    dist.destroy_process_group()


def test_gloo_two_ranks_column_block_exchange():
    """Uneven shards [3, 2] of 5 subjects, T = 70 in two TR blocks: the
    column-block exchange equals the serial ascending sum bit for bit on both
    ranks (the all-to-all path of TorchCommunicator over gloo)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_colblock_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, calls in res:
        assert ok, rank
        assert calls == 1


def _fit_worker(rank, world, port, out, algorithm, data="em_ragged", ordered=None, exchange=None):
    import os

    import torch.distributed as dist

    if exchange == "gather":
        os.environ["SRM_B200_EXCHANGE"] = "gather"

    from paper_1608_04647_b200 import srm
    from paper_1608_04647_b200.collectives import TorchCommunicator, shard_bounds

    _init(rank, world, port)
    xs, k, iters, seed = _dataset(data)
    a, b = shard_bounds(len(xs), world, rank)
    engines = []
    m = srm.fit([srm.SubjectData(f"s{i}", xs[i]) for i in range(a, b)],
                srm.SrmConfig(k=k, iterations=iters, seed=seed),
                TorchCommunicator(), algorithm=algorithm, ordered=ordered, engine_out=engines)
    out.put((rank, m.S, m.W, m.rho2, m.rho0, m.sigma_s, m.rho2_all, m.subject_indices, engines[-1].ordered,
             engines[-1].colblock))
    dist.destroy_process_group()


def _two_ranks(algorithm, data="em_ragged", ordered=None, exchange=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fit_worker, args=(r, 2, port, q, algorithm, data, ordered, exchange))
             for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _serial(data, algorithm):
    from paper_1608_04647_b200 import srm

    xs, k, iters, seed = _dataset(data)
    return srm.fit([srm.SubjectData(f"s{i}", x) for i, x in enumerate(xs)],
                   srm.SrmConfig(k=k, iterations=iters, seed=seed), algorithm=algorithm)


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", ["colblock", "gather"])
@pytest.mark.parametrize("algorithm", ["stream", "gram"])
@pytest.mark.parametrize("data", ["em_ragged", "recipe5"])
def test_two_rank_fit_bit_identical_to_serial(algorithm, data, exchange):
    """Ordered exchange (srm.py:193-213), both forms bit-identical to the
    serial fit: the column-block exchange (default: all-to-all of each rank's
    terms in two TR blocks, each rank's block summed over every subject in
    ascending global order, all-gather of the K x T / 2 results) and the
    all-gathered term table (equal shards [2, 2] take the identity-order
    reduction, uneven shards [3, 2] the order table of k_reduce_terms)."""
    serial = _serial(data, algorithm)
    res = _two_ranks(algorithm, data, exchange=exchange)
    _, S0, W0, r0, rho0_0, sig0, all0, idx0, ord0, cb0 = res[0]
    _, S1, W1, r1, rho0_1, sig1, all1, idx1, ord1, cb1 = res[1]
    assert ord0 and ord1
    assert cb0 == cb1 == (exchange == "colblock")
    n0 = 2 if data == "em_ragged" else 3
    assert idx0 == list(range(n0)) and idx1 == list(range(n0, n0 + len(W1)))
    assert np.array_equal(S0, serial.S) and np.array_equal(S1, serial.S)
    for i, w in enumerate(W0 + W1):
        assert np.array_equal(w, serial.W[i])
    assert r0 + r1 == serial.rho2
    assert rho0_0 == serial.rho0 == rho0_1
    assert np.array_equal(sig0, serial.sigma_s) and sig1 is None and all1 is None
    assert np.array_equal(all0, serial.rho2_all)


@pytest.mark.gpu
@pytest.mark.parametrize("algorithm", ["stream", "gram"])
def test_two_rank_unordered_exchange_matches_serial(algorithm):
    """ordered=False (the exchange large subject counts take: each rank's
    partial sum, srm_reduce_local, then one all-reduce of [K x T | scalars]):
    the grouping changes the rounding only -- within 1e-12 of serial -- and
    both ranks hold the identical S."""
    from conftest import nrel

    serial = _serial("recipe5", algorithm)
    res = _two_ranks(algorithm, "recipe5", ordered=False)
    _, S0, W0, r0, rho0_0, sig0, all0, _, ord0, _ = res[0]
    _, S1, W1, r1, rho0_1, _, _, _, ord1, _ = res[1]
    assert not ord0 and not ord1
    assert np.array_equal(S0, S1) and rho0_0 == rho0_1
    assert nrel(S0, serial.S) <= 1e-12 and nrel(sig0, serial.sigma_s) <= 1e-12
    assert nrel(r0 + r1, serial.rho2) <= 1e-12 and nrel(all0, serial.rho2_all) <= 1e-12
    for w, ws in zip(W0 + W1, serial.W):
        assert nrel(w, ws) <= 1e-12


class _Hub:
    """In-process rendezvous of a thread group (the reference's _ThreadHub idea)."""

    def __init__(self, size):
        import threading

        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots = [None] * size


class ProtocolComm:
    """Only the reference protocol (collectives.py:94-176): rank, size,
    gather(bytes) -> list on root, broadcast(2-D float64 on root) -> array,
    barrier(), stats.  No device collectives."""

    def __init__(self, hub, rank):
        from paper_1608_04647_b200.collectives import CollectiveStats

        self.hub, self.rank, self.size = hub, rank, hub.size
        self.stats = CollectiveStats()

    def gather(self, local):
        self.hub.slots[self.rank] = bytes(local)
        self.hub.barrier.wait()
        out = list(self.hub.slots) if self.rank == 0 else None
        self.hub.barrier.wait()
        self.stats.gather_calls += 1
        return out

    def broadcast(self, buf):
        if self.rank == 0:
            self.hub.slots[0] = np.array(buf, dtype=np.float64, copy=True)
        self.hub.barrier.wait()
        out = np.array(self.hub.slots[0], copy=True)
        self.hub.barrier.wait()
        self.stats.bcast_calls += 1
        return out

    def barrier(self):
        self.hub.barrier.wait()


@pytest.mark.gpu
def test_protocol_only_communicator_fit_bit_identical():
    """Two worker threads fitting through a communicator that only speaks the
    reference protocol (gather + broadcast of host bytes, as factorfit's
    thread / socket backends): bit-identical to the serial fit."""
    import threading

    from paper_1608_04647_b200 import srm
    from paper_1608_04647_b200.collectives import shard_bounds

    xs, k, iters, seed = _dataset("recipe5")
    cfg = srm.SrmConfig(k=k, iterations=iters, seed=seed)
    serial = srm.fit([srm.SubjectData(f"s{i}", x) for i, x in enumerate(xs)], cfg, algorithm="gram")
    hub = _Hub(2)
    models, errors = [None, None], []

    def worker(rank):
        try:
            a, b = shard_bounds(len(xs), 2, rank)
            models[rank] = srm.fit([srm.SubjectData(f"s{i}", xs[i]) for i in range(a, b)], cfg,
                                   ProtocolComm(hub, rank), algorithm="gram")
        except BaseException as e:  # noqa: BLE001
            errors.append(e)
            hub.barrier.abort()

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    m0, m1 = models
    assert np.array_equal(m0.S, serial.S) and np.array_equal(m1.S, serial.S)
    for w, ws in zip(m0.W + m1.W, serial.W):
        assert np.array_equal(w, ws)
    assert m0.rho2 + m1.rho2 == serial.rho2
    assert np.array_equal(m0.sigma_s, serial.sigma_s) and m1.sigma_s is None
    assert np.array_equal(m0.rho2_all, serial.rho2_all)
