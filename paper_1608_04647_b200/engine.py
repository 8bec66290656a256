"""Device-resident SRM EM engine: one plan of libsrm_b200.so per GPU process.

``SrmEngine`` owns the plan's single HBM workspace (a torch uint8 tensor),
uploads and demeans the subjects, draws the reference initialisation,
enqueues the per-iteration phases and exposes region views as torch
tensors.  The EM loop itself is ``fit`` in :mod:`paper_1608_04647_b200.srm`;
this class is the plumbing between it and the C ABI.

Per iteration (srm.py:254-287) the device work is
``[exchange] -> srm_e_step -> srm_m_step``; with a single rank the two phase
calls are captured once into a CUDA graph and replayed (the iteration index
lives in a device counter).
"""

import ctypes
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib, hostio
from .errors import ConfigError, DeviceError, from_status

_MASK64 = 0xFFFFFFFFFFFFFFFF


def _torch():
    import torch

    return torch


def reference_gaussian(n_voxels, k, seed, subject_index):
    """The N(0,1) draw of srm.py:111 (numpy PCG64 seeded (seed, index))."""
    gen = np.random.default_rng((int(seed) & _MASK64, int(subject_index)))
    return gen.standard_normal((int(n_voxels), int(k)))


class SrmEngine:
    """Device state of one worker's subjects for an SRM fit."""

    def __init__(self, n_voxels, n_trs, k, iterations, *, storage="f64", world_size=1,
                 rank=0, counts=None, ordered=True, tolerance=False, gram=False, tc=False, gram_i8=False,
                 exact_polar=False, colblock=False, device=None):
        torch = _torch()
        self.lib = _lib.load()
        if not torch.cuda.is_available():
            raise DeviceError("the SRM engine needs a CUDA device (B200); no CPU fallback")
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        if self.device.type != "cuda":
            raise DeviceError("device must be a CUDA device")
        self.n_voxels = [int(v) for v in n_voxels]
        self.n_local = len(self.n_voxels)
        self.T = int(n_trs)
        self.K = int(k)
        self.iterations = int(iterations)
        self.world_size = int(world_size)
        self.rank = int(rank)
        self.counts = list(counts) if counts is not None else [self.n_local]
        self.storage = storage
        dt = _lib.SRM_F64 if storage == "f64" else _lib.SRM_F32
        flags = 0
        if ordered:
            flags |= _lib.FLAG_ORDERED
        if tolerance:
            flags |= _lib.FLAG_TOLERANCE
        if gram:
            flags |= _lib.FLAG_GRAM
        if tc:
            flags |= _lib.FLAG_TC
        if gram_i8:
            flags |= _lib.FLAG_GRAM_I8
        if exact_polar:
            flags |= _lib.FLAG_EXACT_POLAR
        if colblock and ordered:
            flags |= _lib.FLAG_COLBLOCK
        self.ordered = bool(ordered) or self.world_size == 1
        plan = ctypes.c_void_p()
        varr = (ctypes.c_int64 * self.n_local)(*self.n_voxels)
        carr = (ctypes.c_int32 * self.world_size)(*self.counts)
        _lib.check(self.lib.srm_plan_create(ctypes.byref(plan), dt, self.n_local, varr, self.T,
                                            self.K, self.iterations, self.world_size, self.rank,
                                            carr, flags), "plan_create")
        self.plan = plan
        nbytes = int(self.lib.srm_plan_workspace_bytes(plan))
        with torch.cuda.device(self.device):
            self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        _lib.check(self.lib.srm_plan_bind(plan, ctypes.c_void_p(self.ws.data_ptr()), nbytes), "plan_bind")
        d = lambda w: int(self.lib.srm_plan_dim(plan, w))  # noqa: E731
        self.ldx = d(_lib.D_LDX)
        self.kp = d(_lib.D_KP)
        self.rows = d(_lib.D_ROWS)
        self.term_stride = d(_lib.D_TERM_STRIDE)
        self.red_stride = d(_lib.D_RED_STRIDE)
        self.hist_stride = d(_lib.D_HIST_STRIDE)
        self.n_slots = d(_lib.D_N_SLOTS)
        self.slot0 = d(_lib.D_SLOT_OFFSET)
        self.row_off = np.concatenate([[0], np.cumsum(self.n_voxels)[:-1]]).astype(np.int64)
        eff = d(_lib.D_FLAGS)
        self.gram = bool(eff & _lib.FLAG_GRAM)
        self.tc = bool(eff & _lib.FLAG_TC)
        self.gram_i8 = bool(eff & _lib.FLAG_GRAM_I8)
        self.exact_polar = bool(eff & _lib.FLAG_EXACT_POLAR)
        # ordered accumulation by column blocks (all-to-all + all-gather of K x T / N)
        self.colblock = bool(eff & _lib.FLAG_COLBLOCK)
        if self.colblock:
            self.xrec = d(_lib.D_XREC)
            self.xred = d(_lib.D_XRED)
        self._graph = None
        self._xgraph = None  # capture_exchange (N > 1 over NCCL)
        self._staging = {}

    # ------------------------------------------------------------------ views
    def region(self, rid, dtype=None):
        torch = _torch()
        off = ctypes.c_int64()
        nb = ctypes.c_int64()
        _lib.check(self.lib.srm_plan_region(self.plan, rid, ctypes.byref(off), ctypes.byref(nb)))
        view = self.ws[off.value: off.value + nb.value]
        return view.view(dtype or torch.float64)

    @property
    def xhat(self):
        torch = _torch()
        dt = torch.float64 if self.storage == "f64" else torch.float32
        return self.region(_lib.R_XHAT, dt).view(self.rows, self.ldx)

    @property
    def amat(self):
        return self.region(_lib.R_AMAT).view(self.rows, self.kp)

    @property
    def wout(self):
        # the region also holds the init draw's int8 slices before the final W
        # (int8 Gram plans), so it may be longer than rows x K
        return self.region(_lib.R_WOUT)[: self.rows * self.K].view(self.rows, self.K)

    @property
    def mu(self):
        return self.region(_lib.R_MU)

    @property
    def terms(self):
        return self.region(_lib.R_TERMS).view(self.n_slots, self.term_stride)

    @property
    def red(self):
        return self.region(_lib.R_RED)

    @property
    def redlocal(self):
        return self.region(_lib.R_REDLOCAL)

    @property
    def S(self):
        return self.region(_lib.R_S).view(self.kp, self.ldx)[: self.K, : self.T]

    @property
    def sigma(self):
        return self.region(_lib.R_SIGMA).view(self.kp, self.kp)[: self.K, : self.K]

    @property
    def hist(self):
        return self.region(_lib.R_HIST).view(max(self.iterations, 1), self.hist_stride)

    def stream(self):
        return _torch().cuda.current_stream(self.device).cuda_stream

    # --------------------------------------------------------------- loading
    def _staging_buf(self, slot, dtype, numel):
        torch = _torch()
        key = (slot, dtype)
        buf = self._staging.get(key)
        if buf is None or buf.numel() < numel:
            buf = torch.empty(numel, dtype=dtype, device=self.device)
            self._staging[key] = buf
        return buf[:numel]

    def load(self, xs, gaussians=None, gram=False, init=False, capture=False):
        """Upload (if needed) and demean every local subject (srm.py:238-240).

        Pipelined per subject: the host-to-device copy of subject j+1 (copy
        stream) overlaps the demean -- and, with ``gram``, the one-time
        X_j^T X_j -- of subject j (compute stream).  ``gaussians`` (arrays or
        futures of the init draws) are uploaded into the A region on the way;
        with ``init`` the initial mapping (srm.py:101-118) of each batch of
        subjects runs there too, so only the iteration counter remains
        (:meth:`set_iteration`).  With ``capture`` the EM iteration graph is
        recorded while the first subject uploads (:meth:`capture`).
        """
        torch = _torch()
        if len(xs) != self.n_local:
            raise ConfigError("subject count does not match the plan")
        if init and gaussians is None:
            raise ConfigError("init needs the initial draws")
        main = torch.cuda.current_stream(self.device)
        copier = torch.cuda.Stream(device=self.device)
        gram_stream = torch.cuda.Stream(device=self.device)
        # demean gates the reuse of the staging buffers, so it runs at high priority
        # ahead of the side-stream Gram / init kernels that overlap the upload
        prep = torch.cuda.Stream(device=self.device, priority=-1)
        prep.wait_stream(main)
        n_stage = 3
        done = [None] * n_stage
        next_g = 0
        # side-stream batches: each Gram launch should fill the 148 SMs in one wave
        # (1 CTA/SM per 128 x 128 tile; cfg 2: 4 subjects x 36 tiles), which also
        # keeps the work left after the last upload to one wave; without the
        # Gram, about eight batches per load
        nt = -(-self.ldx // 128)
        batch = max(1, 148 // (nt * (nt + 1) // 2)) if (gram and self.gram) else max(1, -(-self.n_local // 8))
        init_pending = []  # (first, end, demean event) batches waiting for their draws

        def upload_ready_draws(nxt, upto):
            # draws of subjects <= upto always (they free pinned ring slots for the
            # producers); later ones only when already drawn
            while nxt < self.n_local:
                g = gaussians[nxt]
                if nxt > upto and hasattr(g, "done") and not g.done():
                    break
                with torch.cuda.stream(copier):
                    self._upload_gaussian(nxt, g, stream=copier)
                gaussians[nxt] = None
                nxt += 1
            return nxt

        def flush_init(uploaded):
            # batches whose draws are all on the device: initial mapping on the side stream
            while init_pending and init_pending[0][1] <= uploaded:
                first, end, ev_x = init_pending.pop(0)
                evd = torch.cuda.Event()
                evd.record(copier)
                gram_stream.wait_event(evd)
                gram_stream.wait_event(ev_x)
                _lib.check(self.lib.srm_init_mapping_range(self.plan, first, end - first,
                                                           ctypes.c_void_p(gram_stream.cuda_stream)),
                           "init_mapping")
        for j, x in enumerate(xs):
            v = self.n_voxels[j]
            pending = None
            if hasattr(x, "result") and not isinstance(x, (torch.Tensor, np.ndarray)):
                pending = x
                x = x.result()  # a pending read (data_io.PendingMatrix): pinned tensor
            if isinstance(x, torch.Tensor) and x.is_cuda:
                # already on a GPU: converted there (dtype, device, unit column stride) if needed
                if not (x.device == self.device and x.dim() == 2 and x.dtype in (torch.float64, torch.float32)
                        and x.stride(1) == 1):
                    dt = x.dtype if x.dtype in (torch.float64, torch.float32) else torch.float64
                    x = x.detach().to(device=self.device, dtype=dt).contiguous()
                src = x
                ld = x.stride(0) if x.dim() == 2 and x.shape[0] > 1 else self.T
            else:
                if isinstance(x, torch.Tensor):
                    host = x.detach()
                    if host.dtype not in (torch.float64, torch.float32):
                        host = host.to(torch.float64)
                    host = host.contiguous()
                else:
                    arr = np.asarray(x)
                    if arr.dtype not in (np.float64, np.float32):
                        arr = arr.astype(np.float64)
                    host = torch.from_numpy(np.ascontiguousarray(arr))
                b = j % n_stage
                buf = self._staging_buf(b, host.dtype, v * self.T).view(v, self.T)
                if done[b] is not None:
                    copier.wait_event(done[b])
                if host.is_pinned():
                    with torch.cuda.stream(copier):
                        buf.copy_(host, non_blocking=True)
                else:
                    # pageable memory: staged pinned chunks + threaded memcpy
                    done[b].synchronize() if done[b] is not None else None
                    hostio.to_device(host.numpy(), self.device, out=buf)
                ev = torch.cuda.Event()
                ev.record(copier)
                prep.wait_event(ev)
                if pending is not None:
                    pending.release(ev)  # its pinned slot is free once this copy completes
                src = buf
                ld = self.T
            if tuple(src.shape) != (v, self.T):
                raise ConfigError("subject shape does not match the plan")
            dt = _lib.SRM_F64 if src.dtype == torch.float64 else _lib.SRM_F32
            _lib.check(self.lib.srm_load_subject(self.plan, j, ctypes.c_void_p(src.data_ptr()), dt, ld,
                                                 ctypes.c_void_p(prep.cuda_stream)), "load_subject")
            ev2 = torch.cuda.Event()
            ev2.record(prep)
            done[j % n_stage] = ev2
            if (j + 1) % batch == 0 or j + 1 == self.n_local:
                # per batch of subjects, on a side stream (staging-buffer reuse only
                # waits on demean): the one-time X^T X and the initial mapping
                first = (j // batch) * batch
                gram_stream.wait_event(ev2)
                if gram and self.gram:
                    _lib.check(self.lib.srm_prepare_gram_range(self.plan, first, j + 1 - first,
                                                               ctypes.c_void_p(gram_stream.cuda_stream)),
                               "prepare_gram")
                if init:
                    init_pending.append((first, j + 1, ev2))
            if capture and j == 0:
                self.capture()  # host-side work, overlapped with the first uploads
            if gaussians is not None:
                # upload the init draws that are ready; force only those eight
                # subjects behind (the first draws take longer than an upload)
                next_g = upload_ready_draws(next_g, upto=j - 8)
                flush_init(next_g)
        if gaussians is not None:
            next_g = upload_ready_draws(next_g, upto=self.n_local)
            flush_init(next_g)
        main.wait_stream(prep)
        _lib.check(self.lib.srm_finish_load(self.plan, ctypes.c_void_p(main.cuda_stream)), "finish_load")
        main.wait_stream(gram_stream)
        main.wait_stream(copier)
        main.synchronize()
        self._staging.clear()
        self.raise_status()

    def _upload_gaussian(self, j, g, stream=None):
        """Copy subject j's init draw into its A-region rows (pad columns stay 0).

        ``g`` is an array, a tensor, a future of either, or a (ring, slot) pair
        of a PinnedRing slot filled by a worker (asynchronous copy).
        """
        torch = _torch()
        if hasattr(g, "result"):
            g = g.result()
        r0 = int(self.row_off[j])
        rows = self.amat[r0: r0 + self.n_voxels[j]]
        if isinstance(g, tuple):
            ring, slot = g
            nbytes = self.n_voxels[j] * self.K * 8
            src = ring.tensor(slot, nbytes).view(torch.float64).view(self.n_voxels[j], self.K)
            st = stream or torch.cuda.current_stream(self.device)
            with torch.cuda.stream(st):
                tmp = torch.empty((self.n_voxels[j], self.K), dtype=torch.float64, device=self.device)
                tmp.copy_(src, non_blocking=True)
                rows[:, : self.K].copy_(tmp)
                ev = torch.cuda.Event()
                ev.record(st)
            ring.mark_used(slot, ev)
            return
        if isinstance(g, torch.Tensor):
            rows[:, : self.K].copy_(g)
            return
        tmp = hostio.to_device(np.ascontiguousarray(g, dtype=np.float64), self.device)
        rows[:, : self.K].copy_(tmp)

    def init_kernels(self):
        """The device part of init_subject once the draws are in the A region."""
        _lib.check(self.lib.srm_init_mapping(self.plan, ctypes.c_void_p(self.stream())), "init_mapping")

    def init_mapping(self, seed, global_offset, gaussians=None, threads=8):
        """init_subject (srm.py:101-113): host PCG64 draws, device polar + first E-step."""
        torch = _torch()
        amat = self.amat
        if gaussians is None:
            def draw(j):
                return reference_gaussian(self.n_voxels[j], self.K, seed, global_offset + j)

            with ThreadPoolExecutor(max(1, min(threads, self.n_local))) as pool:
                futures = [pool.submit(draw, j) for j in range(self.n_local)]
                for j, fut in enumerate(futures):
                    g = fut.result()
                    r0 = int(self.row_off[j])
                    amat[r0: r0 + self.n_voxels[j], : self.K].copy_(torch.from_numpy(g))
                    futures[j] = None
        else:
            for j, g in enumerate(gaussians):
                if hasattr(g, "result"):
                    g = g.result()
                r0 = int(self.row_off[j])
                src = g if isinstance(g, torch.Tensor) else torch.from_numpy(np.asarray(g, np.float64))
                amat[r0: r0 + self.n_voxels[j], : self.K].copy_(src)
                gaussians[j] = None
        _lib.check(self.lib.srm_init_mapping(self.plan, ctypes.c_void_p(self.stream())), "init_mapping")

    # ------------------------------------------------------------- iteration
    def exchange(self, comm, force=False):
        """Make every subject's E-step term visible to this rank (srm.py:259-269).
        ``force`` runs the device collective even on one rank (an in-place
        one-rank all-gather: the graph-capture test of :meth:`capture_exchange`)."""
        torch = _torch()
        if self.world_size == 1 and not (force and hasattr(comm, "all_gather_into")):
            return
        if self.colblock:
            # srm.py:193-213 by column blocks: pack -> all-to-all -> ordered
            # block sums -> all-gather of the K x T / N blocks -> unpack
            st = ctypes.c_void_p(self.stream())
            _lib.check(self.lib.srm_xchg_pack(self.plan, st), "xchg_pack")
            comm.all_to_all_into(self.region(_lib.R_XRECV), self.region(_lib.R_XSEND))
            _lib.check(self.lib.srm_xchg_reduce(self.plan, st), "xchg_reduce")
            blocks = self.region(_lib.R_XRED)
            comm.all_gather_into(blocks, blocks[self.rank * self.xred: (self.rank + 1) * self.xred])
            _lib.check(self.lib.srm_xchg_unpack(self.plan, st), "xchg_unpack")
            return
        if hasattr(comm, "all_gather_into"):
            if self.ordered:
                m = self.n_slots // self.world_size
                mine = self.terms[self.rank * m: (self.rank + 1) * m]
                comm.all_gather_into(self.terms, mine)
            else:
                _lib.check(self.lib.srm_reduce_local(self.plan, ctypes.c_void_p(self.stream())))
                self.red.copy_(self.redlocal)
                comm.all_reduce_sum(self.red)
            return
        # reference protocol (gather + broadcast of host bytes)
        if not self.ordered:
            raise ConfigError("reference-protocol communicators need ordered exchange")
        m = self.n_slots // self.world_size
        mine = self.terms[self.rank * m: (self.rank + 1) * m].cpu().numpy()
        blobs = comm.gather(mine.tobytes())
        table = None
        if comm.rank == 0:
            table = np.concatenate([np.frombuffer(b, dtype=np.float64) for b in blobs]).reshape(
                self.n_slots, self.term_stride)
        table = comm.broadcast(table)
        self.terms.copy_(torch.from_numpy(np.ascontiguousarray(table)).to(self.device))

    def step(self, comm=None):
        """One EM iteration: [exchange] -> E-step tail -> M-step."""
        if comm is not None and self.world_size > 1:
            self.exchange(comm)
        st = ctypes.c_void_p(self.stream())
        _lib.check(self.lib.srm_e_step(self.plan, st), "e_step")
        _lib.check(self.lib.srm_m_step(self.plan, st), "m_step")

    def capture(self):
        """Record {e_step, m_step} as a native CUDA graph (single rank only)."""
        if self.world_size != 1:
            raise ConfigError("graph capture is for single-rank plans")
        _lib.check(self.lib.srm_graph_capture(self.plan), "graph_capture")
        self._graph = True

    def replay(self):
        _lib.check(self.lib.srm_graph_launch(self.plan, ctypes.c_void_p(self.stream())), "graph_launch")

    def exchange_capturable(self, comm):
        """True when {exchange, E-step, M-step} can be one CUDA graph: the
        exchange is a device collective on this GPU (NCCL), not host staging."""
        return (bool(getattr(comm, "device_collectives", False)) and hasattr(comm, "all_gather_into")
                and (not self.colblock or hasattr(comm, "all_to_all_into")))

    def capture_exchange(self, comm, force=False):
        """Record one multi-rank EM iteration -- the NCCL all-gather (ordered)
        or all-reduce (unordered) of the E-step terms, then the E-step tail and
        the M-step with their side lanes -- as one CUDA graph on this rank.
        Each rank captures its own graph; the collective's communicator must
        have run once eagerly first (NCCL sets up its channels outside
        capture).  Replaces the reference's per-iteration gather + broadcast
        (srm.py:259-269) and the eager launch sequence of :meth:`step`."""
        torch = _torch()
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(self.device)
        cap.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
            self.exchange(comm, force=force)
            st = ctypes.c_void_p(cap.cuda_stream)
            _lib.check(self.lib.srm_e_step(self.plan, st), "e_step")
            _lib.check(self.lib.srm_m_step(self.plan, st), "m_step")
        torch.cuda.current_stream(self.device).wait_stream(cap)
        self._xgraph = g

    def replay_exchange(self):
        """One EM iteration of the :meth:`capture_exchange` graph on the current stream."""
        torch = _torch()
        cur = torch.cuda.current_stream(self.device)
        # CUDAGraph.replay launches on torch's current stream
        with torch.cuda.stream(cur):
            self._xgraph.replay()

    def prepare_gram(self):
        """One-time X_i^T X_i for the Gram path (no-op on streaming plans)."""
        _lib.check(self.lib.srm_prepare_gram(self.plan, ctypes.c_void_p(self.stream())), "prepare_gram")

    def reset(self):
        _lib.check(self.lib.srm_reset(self.plan, ctypes.c_void_p(self.stream())), "reset")

    def set_iteration(self, it):
        _lib.check(self.lib.srm_set_iteration(self.plan, int(it), ctypes.c_void_p(self.stream())))

    def profile_iteration(self):
        """One eager iteration with an event between kernels -> [(name, ms)]."""
        cap = 64
        ms = (ctypes.c_float * cap)()
        n = ctypes.c_int32()
        _lib.check(self.lib.srm_profile_iteration(self.plan, ms, cap, ctypes.byref(n),
                                                  ctypes.c_void_p(self.stream())), "profile")
        return [(self.lib.srm_profile_name(i).decode(), float(ms[i])) for i in range(n.value)]

    def _profile(self, fn, what):
        cap = 16
        ms = (ctypes.c_float * cap)()
        n = ctypes.c_int32()
        _lib.check(fn(self.plan, ms, cap, ctypes.byref(n), ctypes.c_void_p(self.stream())), what)
        return [(self.lib.srm_profile_name(i).decode(), float(ms[i])) for i in range(n.value)]

    def profile_gram(self):
        """The one-time X^T X stages, eagerly, with an event between kernels -> [(name, ms)]."""
        return self._profile(self.lib.srm_profile_gram, "profile_gram")

    def profile_finalize(self):
        """The final W stages, eagerly, with an event between kernels -> [(name, ms)]."""
        return self._profile(self.lib.srm_profile_finalize, "profile_finalize")

    @property
    def launches_per_iteration(self):
        return int(self.lib.srm_plan_dim(self.plan, _lib.D_LAUNCHES))

    def finalize(self):
        _lib.check(self.lib.srm_finalize(self.plan, ctypes.c_void_p(self.stream())), "finalize")

    def finalize_to_host(self, n_batches=4):
        """srm_finalize in subject batches, each batch's W_i rows copied into
        one pinned host array on a side stream while the next batch is
        formed.  Returns the numpy view (rows of all local subjects)."""
        torch = _torch()
        host = torch.empty(tuple(self.wout.shape), dtype=self.wout.dtype, pin_memory=True)
        main = torch.cuda.current_stream(self.device)
        side = self._side_stream()
        nb = max(1, min(int(n_batches), self.n_local))
        bounds = [self.n_local * b // nb for b in range(nb + 1)]
        for b in range(nb):
            first, last = bounds[b], bounds[b + 1]
            _lib.check(self.lib.srm_finalize_range(self.plan, first, last - first,
                                                   ctypes.c_void_p(main.cuda_stream)), "finalize_range")
            r0 = int(self.row_off[first])
            r1 = int(self.row_off[last]) if last < self.n_local else int(sum(self.n_voxels))
            ev = torch.cuda.Event()
            ev.record(main)
            side.wait_event(ev)
            with torch.cuda.stream(side):
                host[r0:r1].copy_(self.wout[r0:r1], non_blocking=True)
        side.synchronize()
        return host.numpy()

    def start_mu_readback(self):
        """Copy model.mu (final once the upload and demean are done) into
        pinned memory on the side stream while the EM runs."""
        torch = _torch()
        main = torch.cuda.current_stream(self.device)
        side = self._side_stream()
        self._mu_host = torch.empty(tuple(self.mu.shape), dtype=self.mu.dtype, pin_memory=True)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            self._mu_host.copy_(self.mu, non_blocking=True)
        self._mu_event = torch.cuda.Event()
        self._mu_event.record(side)

    def mu_host(self):
        """numpy model.mu from start_mu_readback (or a synchronous copy)."""
        if getattr(self, "_mu_host", None) is None:
            return hostio.to_host(self.mu)
        self._mu_event.synchronize()
        return self._mu_host.numpy()

    def small_results_to_host(self, n_done):
        """rho^2 of the local subjects, the history rows, S and Sigma_s in one
        batch of asynchronous copies to pinned memory and one synchronise."""
        torch = _torch()
        srcs = [self.local_rho2(), self.hist[:n_done], self.S.contiguous(), self.sigma.contiguous()]
        outs = [torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True) for t in srcs]
        for o, t in zip(outs, srcs):
            o.copy_(t, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return [o.numpy() for o in outs]

    def _side_stream(self):
        torch = _torch()
        if getattr(self, "_d2h_stream", None) is None:
            self._d2h_stream = torch.cuda.Stream(self.device)
        return self._d2h_stream

    # --------------------------------------------------------------- results
    def status(self):
        out = (ctypes.c_int32 * 4)()
        _lib.check(self.lib.srm_read_status(self.plan, out), "read_status")
        return list(out)

    def raise_status(self):
        code, arg, it, _ = self.status()
        if code:
            raise from_status(code, arg=arg)

    def poll(self, it):
        """(code, arg, warnings, |S - S_prev|, |S_prev|) after iteration ``it``:
        the status word and the tolerance statistics in one asynchronous copy
        to pinned memory and one stream synchronisation (the tolerance stop,
        srm.py:275-287)."""
        torch = _torch()
        if getattr(self, "_poll_buf", None) is None:
            self._poll_buf = torch.empty(32, dtype=torch.uint8, pin_memory=True)
        buf = self._poll_buf
        status = self.region(_lib.R_STATUS, torch.uint8)[:16]
        row = self.hist[it % self.iterations][_lib.H_SDIFF: _lib.H_SPREV + 1].contiguous().view(torch.uint8)
        buf[:16].copy_(status, non_blocking=True)
        buf[16:].copy_(row, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        st = buf[:16].view(torch.int32).tolist()
        sdiff, sprev = buf[16:].view(torch.float64).tolist()
        return st[0], st[1], st[3], sdiff, sprev

    @property
    def warnings(self):
        """SRM_WARN_* bits raised so far (synchronises)."""
        return self.status()[3]

    def local_rho2(self):
        col = self.kp * self.ldx + _lib.REC_RHO2
        return self.terms[self.slot0: self.slot0 + self.n_local, col]

    def subject_rows(self, j):
        r0 = int(self.row_off[j])
        return slice(r0, r0 + self.n_voxels[j])

    def close(self):
        if getattr(self, "plan", None) is not None and self.lib is not None:
            self.lib.srm_plan_destroy(self.plan)
            self.plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
