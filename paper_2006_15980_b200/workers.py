"""Batch workers on B200: the reference's accelerator seam, real.

Mirrors hetmf/workers.py's batch half (workers.py:45-369, 408-514):
BatchWorkerConfig, block_order_seed, BatchEngine (stage_rows / flush_rows /
stage_in / stage_in_async / stage_out / compute / close, `resident`,
`staged`), BatchWorker (lease loop with P-band residency and a staged-ahead
unit), time_batch_prefixes and throughput_sweep.  The reference emulates the
GPU with sleeps and CPU lanes; here:

* factors live in HBM.  A FactorStore shared by the engines of one run keeps a
  full-size replica of P and Q per device and records, per user and per
  item, which device holds the freshest copy and the CUDA event that
  completes it.  Staging a band brings it from that home: nothing if it is
  already local, a peer copy over NVLink (cudaMemcpyPeerAsync on the copy
  stream) from another GPU, or an H2D copy from the host model.  The copy is
  ordered before compute by a stream wait on the home's event — no host
  round trip.  stage_out / flush_rows only move the home; the host model is
  refreshed at barriers and at the end (FactorStore.sync_host), invisible to
  callers that read the model afterwards (SURVEY §7 hard part 6);
* triples are resident too: each device keeps one block-major copy of the
  grid (f32 ratings), Q-band sub-bucketed for the shared-memory kernel;
* compute launches one kernel per sub-block with the reference's seeds
  (block_order_seed(unit_seed, i), workers.py:77-83 / 234-237).  Lanes are a
  CPU notion: `lanes`, `launch_overhead` and `bandwidth` are accepted and
  ignored.  `mode="exact"` runs the reference's visit order and arithmetic, so
  a CUDA batch worker equals a reference stream worker bit for bit over the
  same lease sequence (the reference's own degenerate-equivalence property,
  workers.py:19-21);
* stage methods return CUDA-event-timed seconds, which calibration fits.
"""

from __future__ import annotations

import ctypes
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, kernels
from .data import BlockGrid, DeviceGrid, bucket_qbands
from .scheduler import CLASS_BATCH, GridScheduler, Unit
from .sgd import FactorModel, Hyperparams, init_model

TRIPLE_BYTES = 12  # int32 row + int32 col + f32 rating on device (the reference: 16)
HOST = -1


def _torch():
    import torch
    return torch


@dataclass
class BatchWorkerConfig:
    """workers.py:45-58, plus the B200 knobs."""

    lanes: int = 4                  # accepted for compatibility; no CPU lanes on B200
    launch_overhead: float = 0.002  # accepted; the real overhead is measured
    bandwidth: float = 4e9          # accepted; the real copies are measured
    pipeline_depth: int = 3
    device: int | None = None       # CUDA device index (None: current device)
    precision: str = "f32"          # factor storage on device: f32 | f16 | f64
    kernel: str = "qband"           # qband (Q band in shared memory) | range (hmf_sgd_range)
    mode: str = "hogwild"           # for kernel="range": hogwild | hogwild_lww | ordered | exact

    def validate(self) -> None:
        if self.lanes < 1:
            raise ValueError("lanes must be >= 1")
        if self.launch_overhead < 0:
            raise ValueError("launch_overhead must be >= 0")
        if self.bandwidth <= 0:
            raise ValueError("bandwidth must be > 0")
        if self.precision not in ("f32", "f16", "f64"):
            raise ValueError(f"unknown precision {self.precision!r}")
        if self.kernel not in ("qband", "range"):
            raise ValueError(f"unknown kernel {self.kernel!r}")
        if self.mode not in _lib.MODES:
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.kernel == "qband" and self.precision == "f64":
            raise ValueError("the Q-band kernel stores f32 or f16 factors")

    def device_name(self) -> str:
        torch = _torch()
        d = torch.cuda.current_device() if self.device is None else self.device
        return torch.cuda.get_device_name(d).replace(" ", "_")


def block_order_seed(unit_seed: int, index: int) -> int:
    """Visit-order seed of sub-block `index` of a unit (workers.py:77-83)."""
    return kernels.mix64(unit_seed, index)


_DTYPES = {"f32": "float32", "f16": "float16", "f64": "float64"}


class FactorStore:
    """Per-device factor replicas and the home of every user / item row.

    home_p[u] / home_q[v] is HOST or the device index holding the freshest
    copy; ready_* maps a device to the CUDA event after which its copy is
    complete.  All methods are called with the band leased to the caller, so
    the rows they touch are not moving concurrently (the lease protocol's
    conflict freedom); the lock only guards the bookkeeping itself.
    """

    def __init__(self, model: FactorModel, precision: str = "f32", grid=None):
        self.model = model
        self.precision = precision
        self.k = model.n_factors
        self.home_p = np.full(model.n_users, HOST, dtype=np.int16)
        self.home_q = np.full(model.n_items, HOST, dtype=np.int16)
        self.replicas: dict[int, tuple] = {}
        self.events: dict[int, object] = {}
        # engines per device: with one, every recorded event is on that
        # engine's stream (or a gather's), so a device's latest event covers
        # all of its earlier work
        self.engines_on: dict[int, int] = {}
        self.grids: dict[int, DeviceGrid] = {}
        self.host_grid = grid
        self.copy_streams: dict[int, object] = {}
        self.lock = threading.RLock()

    # -- device resources -----------------------------------------------------
    def replica(self, dev: int):
        torch = _torch()
        with self.lock:
            if dev not in self.replicas:
                dt = getattr(torch, _DTYPES[self.precision])
                d = torch.device("cuda", dev)
                self.replicas[dev] = (torch.empty((self.model.n_users, self.k), dtype=dt, device=d),
                                      torch.empty((self.model.n_items, self.k), dtype=dt, device=d))
                self.copy_streams[dev] = torch.cuda.Stream(device=d)
            return self.replicas[dev]

    def copy_stream(self, dev: int):
        self.replica(dev)
        return self.copy_streams[dev]

    def device_grid(self, dev: int, grid: BlockGrid, kernel: str) -> DeviceGrid:
        torch = _torch()
        with self.lock:
            g = self.grids.get(dev)
            if g is None or self.host_grid is not grid:
                rd = "float64" if self.precision == "f64" else "float32"
                with torch.cuda.device(dev):
                    g = DeviceGrid.from_host(grid, torch.device("cuda", dev), rd)
                    if kernel == "qband":
                        bucket_qbands(g, self.k,
                                      elem_bytes=2 if self.precision == "f16" else 4)
                    # built on the current stream, read by the engines' own
                    # streams: finish it before anyone launches on it
                    torch.cuda.current_stream(dev).synchronize()
                self.grids[dev] = g
                self.host_grid = grid
            return g

    # -- moving rows to a device ------------------------------------------------
    def _runs(self, home: np.ndarray, lo: int, hi: int):
        """Maximal [a, b) runs of equal home inside [lo, hi)."""
        seg = home[lo:hi]
        if len(seg) == 0:
            return []
        edges = np.flatnonzero(np.diff(seg)) + 1
        starts = np.concatenate([[0], edges])
        ends = np.concatenate([edges, [len(seg)]])
        return [(lo + int(a), lo + int(b), int(seg[a])) for a, b in zip(starts, ends)]

    def bring(self, which: str, dev: int, lo: int, hi: int, stream) -> int:
        """Make rows [lo, hi) of P ('p') or Q ('q') fresh on `dev`, enqueued on
        `stream`; returns bytes moved."""
        torch = _torch()
        P, Q = self.replica(dev)
        dst = P if which == "p" else Q
        home = self.home_p if which == "p" else self.home_q
        host = self.model.user_factors if which == "p" else self.model.item_factors
        moved = 0
        with self.lock:
            runs = self._runs(home, lo, hi)
            mine = self.events.get(dev)
        # work already recorded on dev's rows (a gather on the copy stream,
        # another engine's compute) completes before `stream` touches them
        if mine is not None:
            stream.wait_event(mine)
        for a, b, h in runs:
            if h == dev:
                continue
            with torch.cuda.stream(stream):
                if h == HOST:
                    src = torch.from_numpy(np.ascontiguousarray(host[a:b]))
                    dst[a:b].copy_(src.to(dst.dtype), non_blocking=False)
                else:
                    ev = self.events.get(h)
                    if ev is not None:
                        stream.wait_event(ev)
                    sp, sq = self.replicas[h]
                    src = sp if which == "p" else sq
                    _lib.check(_lib.load().hmf_memcpy_peer_async(
                        dst[a:b].data_ptr(), dev, src[a:b].data_ptr(), h,
                        (b - a) * self.k * dst.element_size(), stream.cuda_stream),
                        "hmf_memcpy_peer_async")
            moved += (b - a) * self.k * dst.element_size()
            with self.lock:
                home[a:b] = dev
        return moved

    def claim(self, which: str, dev: int, lo: int, hi: int, event) -> None:
        """Record that `dev` holds the freshest rows [lo, hi), complete at `event`."""
        with self.lock:
            (self.home_p if which == "p" else self.home_q)[lo:hi] = dev
            self.events[dev] = event

    def sync_host(self) -> None:
        """Copy every device-homed row back into the host model (f64)."""
        torch = _torch()
        for which in ("p", "q"):
            home = self.home_p if which == "p" else self.home_q
            host = self.model.user_factors if which == "p" else self.model.item_factors
            with self.lock:
                runs = self._runs(home, 0, len(home))
            for a, b, h in runs:
                if h == HOST:
                    continue
                torch.cuda.synchronize(h)
                src = self.replicas[h][0 if which == "p" else 1]
                host[a:b] = src[a:b].to(torch.float64).cpu().numpy()

    def gather_on(self, dev: int):
        """Bring every row to `dev` (for metrics at a barrier); returns (P, Q)."""
        torch = _torch()
        s = self.copy_stream(dev)
        self.bring("p", dev, 0, self.model.n_users, s)
        self.bring("q", dev, 0, self.model.n_items, s)
        # every row is now homed on dev and complete at this event: other
        # devices' pulls from dev and dev's own engine stream order on it
        # (through events[dev]), not only the caller's current stream
        ev = torch.cuda.Event()
        ev.record(s)
        with self.lock:
            self.events[dev] = ev
        torch.cuda.current_stream(dev).wait_stream(s)
        return self.replicas[dev]


class StagedBlock:
    """A staged unit: its device grid, item span and sub-block count."""

    __slots__ = ("unit", "grid", "col_lo", "col_hi", "offsets", "items")

    def __init__(self, unit, grid, col_lo, col_hi, offsets, items=None):
        self.unit = unit
        self.grid = grid
        self.col_lo = col_lo
        self.col_hi = col_hi
        self.offsets = offsets
        self.items = items


class BatchEngine:
    """CUDA batch engine with the reference's method surface (workers.py:144-266)."""

    def __init__(self, config: BatchWorkerConfig, model: FactorModel, hparams: Hyperparams,
                 store: FactorStore | None = None):
        torch = _torch()
        if not isinstance(config, BatchWorkerConfig):
            # the reference's BatchWorkerConfig (lanes, launch_overhead,
            # bandwidth; workers.py:45-58): the drop-in binding
            # `hetmf.workers.BatchEngine = paper_2006_15980_b200.workers.BatchEngine`
            # hands those to the reference's own BatchWorker (workers.py:315)
            config = BatchWorkerConfig(lanes=config.lanes, launch_overhead=config.launch_overhead,
                                       bandwidth=config.bandwidth)
        config.validate()
        _lib.load()
        if not torch.cuda.is_available():
            raise _lib.HmfError("no CUDA device: the B200 engine has no CPU fallback")
        self.config = config
        self.model = model
        self.hparams = hparams
        self.dev = torch.cuda.current_device() if config.device is None else int(config.device)
        self.store = store if store is not None else FactorStore(model, config.precision)
        self.stream = torch.cuda.Stream(device=torch.device("cuda", self.dev))
        self.resident = None
        self.staged: dict = {}
        self._owns_store = store is None
        with self.store.lock:
            self.store.engines_on[self.dev] = self.store.engines_on.get(self.dev, 0) + 1

    def close(self):
        if self._owns_store:
            self.store.sync_host()

    def _timed(self, fn, stream):
        torch = _torch()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(self.dev):
            e0.record(stream)
            out = fn()
            e1.record(stream)
            e1.synchronize()
        return out, e0.elapsed_time(e1) / 1e3

    # -- staging ---------------------------------------------------------------
    def stage_rows(self, row_lo: int, row_hi: int) -> float:
        """Make a P band resident on this GPU (from host or a peer)."""
        _, secs = self._timed(lambda: self.store.bring("p", self.dev, row_lo, row_hi, self.stream),
                              self.stream)
        P, _ = self.store.replica(self.dev)
        self.resident = (row_lo, row_hi, P[row_lo:row_hi])
        return secs

    def flush_rows(self) -> float:
        """Release the resident band: its home stays on this GPU; the host
        copy is refreshed at barriers / close (sync_host)."""
        if self.resident is None:
            return 0.0
        torch = _torch()
        lo, hi, _ = self.resident
        ev = torch.cuda.Event()
        ev.record(self.stream)
        self.store.claim("p", self.dev, lo, hi, ev)
        if self._owns_store:
            self.store.sync_host()
        self.resident = None
        return 0.0

    def _stage(self, key, grid, unit: Unit, stream) -> int:
        g = self.store.device_grid(self.dev, grid, self.config.kernel)
        col_lo, col_hi = grid.col_span(unit.col)
        moved = self.store.bring("q", self.dev, col_lo, col_hi, stream)
        spans = [grid.block_range(b) for b in unit.blocks]
        offsets = np.concatenate([[0], np.cumsum([hi - lo for lo, hi in spans])])
        _, Q = self.store.replica(self.dev)
        self.staged[key] = StagedBlock(unit, g, col_lo, col_hi, offsets, Q[col_lo:col_hi])
        return moved

    def stage_in(self, key, grid, unit: Unit) -> float:
        """Stage a unit: device triples (resident) plus its Q band."""
        _, secs = self._timed(lambda: self._stage(key, grid, unit, self.stream), self.stream)
        return secs

    def stage_in_async(self, key, grid, unit: Unit):
        """Stage on the copy stream; the returned join makes compute wait for it."""
        torch = _torch()
        cs = self.store.copy_stream(self.dev)
        self._stage(key, grid, unit, cs)
        ev = torch.cuda.Event()
        ev.record(cs)

        def join():
            self.stream.wait_event(ev)
        return join

    def stage_out(self, key) -> float:
        """The Q band stays here; record the home (the host copy is refreshed
        at barriers / close)."""
        torch = _torch()
        st = self.staged.pop(key)
        ev = torch.cuda.Event()
        ev.record(self.stream)
        self.store.claim("q", self.dev, st.col_lo, st.col_hi, ev)
        if self._owns_store:
            self.store.sync_host()
        return 0.0

    # -- compute ---------------------------------------------------------------
    def compute(self, key, unit_seed: int) -> int:
        """Run every staged block once, sub-blocks in order with the
        reference's seeds (workers.py:222-255)."""
        st = self.staged[key]
        hp = self.hparams
        P, Q = self.store.replica(self.dev)
        g = st.grid
        done = 0
        for i, b in enumerate(st.unit.blocks):
            seed = block_order_seed(unit_seed, i)
            if self.config.kernel == "qband":
                done += kernels.launch_block_qband(P, Q, g, b, hp.learning_rate, hp.reg_user,
                                                   hp.reg_item, seed,
                                                   stream=self.stream.cuda_stream)
            else:
                lo, hi = g.block_range(b)
                done += kernels.launch_sgd_range(P, Q, g.users, g.items, g.ratings, lo, hi,
                                                 hp.learning_rate, hp.reg_user, hp.reg_item, seed,
                                                 0, 0, self.config.mode, self.stream.cuda_stream)
        return done

    def synchronize(self) -> None:
        self.stream.synchronize()


class BatchWorker(threading.Thread):
    """Lease loop of one GPU (workers.py:305-369)."""

    def __init__(self, worker_id: int, scheduler: GridScheduler, model: FactorModel,
                 grid: BlockGrid, hparams: Hyperparams, config: BatchWorkerConfig,
                 store: FactorStore | None = None):
        super().__init__(name=f"batch-{worker_id}", daemon=True)
        self.worker_id = worker_id
        self.scheduler = scheduler
        self.grid = grid
        self.config = config
        self.engine = None
        self._model, self._hp, self._store = model, hparams, store
        self.blocks_done = 0
        self.error = None
        self.kernel_seconds = 0.0

    def _row_span(self, unit: Unit):
        return self.grid.row_span(unit.rows[0])[0], self.grid.row_span(unit.rows[-1])[1]

    def _ensure_resident(self, unit: Unit) -> None:
        span = self._row_span(unit)
        if self.engine.resident is None or self.engine.resident[:2] != span:
            self.engine.flush_rows()
            self.engine.stage_rows(*span)

    def run(self):
        torch = _torch()
        try:
            dev = self.config.device if self.config.device is not None else 0
            torch.cuda.set_device(dev)
            self.engine = BatchEngine(self.config, self._model, self._hp, self._store)
            engine = self.engine
            lease = self.scheduler.acquire(self.worker_id, CLASS_BATCH)
            if lease is None:
                return
            self._ensure_resident(lease.unit)
            engine.stage_in(id(lease.unit), self.grid, lease.unit)
            while True:
                unit = lease.unit
                join = None
                if lease.prefetch is not None and id(lease.prefetch) not in engine.staged:
                    join = engine.stage_in_async(id(lease.prefetch), self.grid, lease.prefetch)
                done = engine.compute(id(unit), unit.order_seed)
                if join is not None:
                    join()
                engine.stage_out(id(unit))
                self.blocks_done += len(unit.blocks)
                if lease.prefetch is None:
                    engine.flush_rows()
                # the next owner of this unit's bands must see finished data:
                # homes carry the completion event (stage_out / flush_rows),
                # and a puller's stream waits on it.  That event is the
                # device's latest only while one engine runs there; with
                # several on one device the release waits for the kernel.
                if engine.store.engines_on.get(engine.dev, 0) > 1:
                    engine.synchronize()
                nxt = self.scheduler.release(lease, done)
                if nxt is None:
                    engine.staged.clear()
                    nxt = self.scheduler.acquire(self.worker_id, CLASS_BATCH)
                    if nxt is None:
                        break
                self._ensure_resident(nxt.unit)
                if id(nxt.unit) not in engine.staged:
                    engine.stage_in(id(nxt.unit), self.grid, nxt.unit)
                lease = nxt
        except BaseException as exc:  # re-raised by the driver (engine.py)
            self.error = exc
            self.scheduler.abort("worker error")
        finally:
            if self.engine is not None:
                try:
                    self.engine.flush_rows()
                    self.engine.synchronize()
                finally:
                    self.engine.close()


def chunk_cuts(n_tiles: int, tiles_per_chunk: int, last_chunk_tiles: int = 0) -> list:
    """Tile cuts of a block's streamed chunks: runs of tiles_per_chunk tiles,
    the last chunk last_chunk_tiles long when 0 < last_chunk_tiles < n_tiles
    (e.g. 8 tiles, 4 per chunk, last 1 -> [0, 4, 7, 8])."""
    g = max(1, int(tiles_per_chunk))
    head = n_tiles - last_chunk_tiles if 0 < last_chunk_tiles < n_tiles else n_tiles
    cuts = [0]
    while cuts[-1] < head:
        cuts.append(min(head, cuts[-1] + g))
    if head < n_tiles:
        cuts.append(n_tiles)
    return cuts


class StreamingEpoch:
    """Epochs whose rating triples stream from pinned host memory.

    The reference stages a unit's triples into the accelerator for every
    lease (BatchEngine.stage_in, workers.py:186-202).  This is that pipeline
    for data that is not kept resident.  P and Q stay on the device; every
    epoch uploads chunk c+1 on a copy stream while the Q-band kernel updates
    chunk c (a ring of device staging buffers, ordered by CUDA events).

    Chunks are runs of `tiles_per_chunk` row tiles of each block
    (data.bucket_qbands), the last one `last_chunk_tiles` long if set: once
    the copy engine has uploaded an epoch, only that short launch remains
    (uploads are the bound: an epoch takes its upload time plus the training
    of its last chunk).  Chunk (b, c) holds block b's triples of those tiles,
    item runs inside each.  One launch trains a chunk, walking its tiles as
    the resident kernel walks a block's (each tile's P rows sit in L2 while
    its bins run); the epoch walks each block's chunks in a seeded rotation.

    Bytes per rating on the host stream (the chained kernel, one item per
    sub-band, every tile at most 65536 rows): a 2-byte user id relative to
    the tile plus the 4-byte rating — the item is implicit in the sub-band
    (hmf_sgd_block_qband_u16_*, cols = NULL).  Otherwise 8 (4-byte user ids,
    implicit items) or 12.
    """

    def __init__(self, grid: DeviceGrid, k: int, tile_bytes=None, n_buffers: int = 3,
                 elem_bytes: int = 4, compact: bool = True, tiles_per_chunk: int = 4,
                 last_chunk_tiles: int = 0, reuse: bool = False, opts=None, impl=None,
                 runs_chunks_per_block: int = 2):
        torch = _torch()
        self.dev = grid.device
        # a grid the caller already laid out for the Q-band kernel is used as is
        sg = grid if grid.sub_ptr is not None else bucket_qbands(
            grid, k, tile_bytes=tile_bytes, elem_bytes=elem_bytes, impl=impl)
        self.k = k
        self.nnz = sg.nnz
        self.sub_impl = sg.sub_impl
        self.qsync = sg.sub_qsync
        self.sub_pstore = sg.sub_pstore
        # the launch options of this layout (plus explicit overrides), passed
        # with every launch (ABI 4: nothing process-wide)
        self.opts = kernels.qband_opts(sg, **dict(opts or {}))
        self.reuse = bool(reuse)
        # implementation 8 (run groups): the item of a rating is its run's,
        # and its tiles hold at most hmf_ptile_max_rows users, so the stream
        # is always the compact one (uint16 tile-relative user + rating)
        self.runs = int(sg.sub_impl) == 8
        # every sub-band a single item (or a part of one): the item is implicit
        self.implicit_items = self.runs or (compact and sg.sub_impl >= 4 and all(
            bool(torch.all(c[1:] - c[:-1] <= 1)) for c in sg.sub_cuts))
        self.u16 = self.implicit_items and all(
            int(np.max(np.diff(r))) <= 65536 for r in sg.sub_tile_rows)
        # run groups over tiles of at most 256 rows: one byte per user id
        self.u8 = self.runs and int(sg.sub_max_rows) <= 256
        # chunks: G consecutive row tiles of a block -> [lo, hi) of the
        # bucketed arrays, the number of tiles, their sub-band offsets relative
        # to lo, their first rows (device int32, uint16 ids only)
        self.tiles_per_chunk = max(1, int(tiles_per_chunk))
        self.last_chunk_tiles = max(0, int(last_chunk_tiles))
        self.blocks = []
        users = sg.users
        if self.u16:
            users = torch.empty(sg.nnz, dtype=torch.uint8 if self.u8 else torch.int16,
                                device=self.dev)
        if self.runs:
            self._init_runs(sg, users, runs_chunks_per_block)
        for b in range(0 if self.runs else sg.n_blocks):
            sp = sg.sub_ptr[b].cpu().numpy()
            T = sg.sub_tiles[b]
            S = (len(sp) - 1) // T
            cuts = chunk_cuts(T, self.tiles_per_chunk, self.last_chunk_tiles)
            chunks = []
            for t0, t1 in zip(cuts, cuts[1:]):
                lo, hi = int(sp[t0 * S]), int(sp[t1 * S])
                rows0 = [int(r) for r in sg.sub_tile_rows[b][t0:t1]]
                rel = (sg.sub_ptr[b][t0 * S:t1 * S + 1] - lo).contiguous()
                trow = torch.tensor(rows0, dtype=torch.int32, device=self.dev)
                chunks.append((lo, hi, t1 - t0, rel, trow))
                if self.u16:
                    for t in range(t0, t1):
                        a, z = int(sp[t * S]), int(sp[(t + 1) * S])
                        if z > a:
                            # uint16 bit pattern of (user - tile's first row)
                            users[a:z] = (sg.users[a:z] - rows0[t - t0]).to(torch.int32).to(
                                torch.int16)
            self.blocks.append((chunks, sg.sub_cuts[b]))
        arrays = [users] + ([] if self.implicit_items else [sg.items]) + [sg.ratings]
        self.host = [a.cpu().pin_memory() for a in arrays]
        cap = max([c[1] - c[0] for chunks, _ in self.blocks for c in chunks] + [0]) + 8
        self.n_buffers = max(2, int(n_buffers))
        self.bufs = [tuple(torch.empty(cap, dtype=a.dtype, device=self.dev) for a in arrays)
                     for _ in range(self.n_buffers)]
        self.copy_stream = torch.cuda.Stream(device=self.dev)
        self.freed = [None] * self.n_buffers
        self.lru = [None] * self.n_buffers            # chunk (block, index) held by each buffer
        self.lru_order = list(range(self.n_buffers))  # buffers, least recently used first
        self.n_chunks = sum(len(c) for c, _ in self.blocks)
        self.last_h2d = 0
        self.trace = None     # set to a list to record per-chunk CUDA events
        del users

    def _init_runs(self, sg, users, chunks_per_block: int) -> None:
        """Chunks of implementation 8: each block's row tiles cut into
        `chunks_per_block` runs of consecutive tiles (a launch needs at least
        one tile per SM to fill the GPU, so chunks are whole fractions of a
        block, not a few tiles); a chunk is the ratings of its tiles' runs,
        contiguous in the layout.  Users go out as uint16 offsets from their
        tile's first row; the run descriptors (items, lengths) stay resident."""
        torch = _torch()
        self.sg = sg
        for b in range(sg.n_blocks):
            blo, bhi = sg.block_range(b)
            T = sg.sub_tiles[b]
            trun = sg.sub_tile_run[b].cpu().numpy().astype(np.int64)
            runs = sg.sub_ptr[b].cpu().numpy().astype(np.int64)
            starts = np.concatenate([runs[:, 0], [bhi - blo]]) if len(runs) else \
                np.array([bhi - blo], dtype=np.int64)
            tiles = sg.sub_tile_rows[b]
            if bhi > blo:
                d_tiles = torch.from_numpy(tiles).to(self.dev)
                tile_of = torch.bucketize(sg.users[blo:bhi], d_tiles[1:-1].to(torch.int32),
                                          right=True)
                users[blo:bhi] = (sg.users[blo:bhi] - d_tiles[tile_of]).to(torch.int32).to(
                    users.dtype)
            per = -(-T // max(1, int(chunks_per_block)))
            cuts = list(range(0, T, per)) + [T]
            chunks = []
            for t0, t1 in zip(cuts, cuts[1:]):
                off = int(starts[trun[t0]])
                end = int(starts[trun[t1]])
                chunks.append((blo + off, blo + end, t1 - t0, off, t0))
            self.blocks.append((chunks, b))

    def _launch_runs(self, P, Q, hparams, b, chunk, buf, tseed, stream) -> None:
        sg = self.sg
        lo, hi, n_tiles, off, t0 = chunk
        st = "f16" if P.dtype == _torch().float16 else "f32"
        idb = 1 if self.u8 else 2           # bytes per user id
        fn = getattr(_lib.load(), f"hmf_sgd_block_runs_u{8 * idb}_{st}")
        # run descriptors count from the block's first rating; the staging
        # buffer starts at the chunk's
        _lib.check(fn(P.data_ptr(), Q.data_ptr(), self.k, buf[0].data_ptr() - idb * off,
                      buf[-1].data_ptr() - 4 * off, sg.sub_ptr[b].data_ptr(),
                      sg.sub_tile_run[b].data_ptr() + 4 * t0,
                      sg.sub_tile_cuts[b].data_ptr() + 4 * t0, n_tiles, int(sg.sub_max_rows),
                      ctypes.byref(self.opts), hparams.learning_rate, hparams.reg_user,
                      hparams.reg_item, tseed, 0, 0, stream.cuda_stream),
                   "hmf_sgd_block_runs_u8/u16")

    @property
    def bytes_per_rating(self) -> int:
        if self.u8:
            return 5
        return 6 if self.u16 else (8 if self.implicit_items else 12)

    @property
    def h2d_bytes(self) -> int:
        """Bytes of triples one epoch uploads (all chunks; an epoch that
        starts on chunks still resident from the previous one uploads
        less — see h2d_bytes_last)."""
        return self.bytes_per_rating * self.nnz

    def h2d_bytes_last(self) -> int:
        """Bytes the last run() uploaded."""
        return self.last_h2d

    def run(self, P, Q, hparams: Hyperparams, seed: int, stream=None) -> int:
        """One epoch over every block; returns triples processed (async).

        With `reuse`, chunks still in a staging buffer from the previous epoch
        are trained first and not uploaded again (the tail of epoch e is the
        head of epoch e+1); the rest follow block by block, each block's
        chunks in a seeded rotation.  Without it every chunk is uploaded every
        epoch."""
        torch = _torch()
        comp = torch.cuda.current_stream(self.dev) if stream is None else stream
        st = "f16" if P.dtype == torch.float16 else "f32"
        lib = _lib.load()
        fn = getattr(lib, f"hmf_sgd_block_qband_u16_tiles_{st}" if self.u16
                     else f"hmf_sgd_block_qband_{st}")
        order = []
        for b, (chunks, _) in enumerate(self.blocks):
            bseed = kernels.mix64(seed, b) & 0xFFFFFFFFFFFFFFFF
            # a short last chunk (last_chunk_tiles) stays last: after the
            # epoch's final upload only a short launch remains
            t = 1 if self.last_chunk_tiles and len(chunks) > 1 else 0
            n = len(chunks) - t
            rot = bseed % n if n else 0
            order += [(b, (i + rot) % n, bseed) for i in range(n)]
            order += [(b, n + c, bseed) for c in range(t)]
        if self.reuse:
            resident = [ch for ch in reversed(self.lru) if ch is not None]
            head = [o for ch in resident for o in order if (o[0], o[1]) == ch]
            order = head + [o for o in order if (o[0], o[1]) not in resident]
        done, uploaded = 0, 0
        for b, t, bseed in order:
            chunks, sc = self.blocks[b]
            lo, hi, n_tiles, rel, trow = chunks[t]
            if hi <= lo:
                continue
            tr = None if self.trace is None else {"chunk": (b, t), "copied": False}
            if self.reuse and (b, t) in self.lru:
                slot = self.lru.index((b, t))        # already on the device
                buf = self.bufs[slot]
            else:
                slot = self.lru_order[0]             # least recently used buffer
                buf = self.bufs[slot]
                with torch.cuda.stream(self.copy_stream):
                    if self.freed[slot] is not None:
                        self.copy_stream.wait_event(self.freed[slot])
                    if tr is not None:
                        tr["copied"] = True
                        tr["c0"] = torch.cuda.Event(enable_timing=True)
                        tr["c0"].record(self.copy_stream)
                    for dst, src in zip(buf, self.host):
                        dst[:hi - lo].copy_(src[lo:hi], non_blocking=True)
                    up = torch.cuda.Event(enable_timing=tr is not None)
                    up.record(self.copy_stream)
                    if tr is not None:
                        tr["c1"] = up
                comp.wait_event(up)
                self.lru[slot] = (b, t)
                uploaded += hi - lo
            self.lru_order.remove(slot)
            self.lru_order.append(slot)
            tseed = kernels.mix64(bseed, t) & 0xFFFFFFFFFFFFFFFF
            if self.runs:
                if tr is not None:
                    tr["k0"] = torch.cuda.Event(enable_timing=True)
                    tr["k0"].record(comp)
                self._launch_runs(P, Q, hparams, sc, chunks[t], buf, tseed, comp)
                ev = torch.cuda.Event(enable_timing=tr is not None)
                ev.record(comp)
                self.freed[slot] = ev
                if tr is not None:
                    tr["k1"] = ev
                    self.trace.append(tr)
                done += hi - lo
                continue
            items = 0 if self.implicit_items else buf[1].data_ptr()
            args = (P.data_ptr(), Q.data_ptr(), self.k, buf[0].data_ptr(), items,
                    buf[-1].data_ptr(), rel.data_ptr(), sc.data_ptr(), int(sc.numel()) - 1,
                    n_tiles)
            if self.u16:        # tile-relative uint16 ids, first rows per tile
                args += (trow.data_ptr(), ctypes.byref(self.opts), hparams.learning_rate,
                         hparams.reg_user, hparams.reg_item, tseed, 0, comp.cuda_stream)
            else:
                args += (ctypes.byref(self.opts), hparams.learning_rate, hparams.reg_user,
                         hparams.reg_item, tseed, 0, 0, comp.cuda_stream)
            if tr is not None:
                tr["k0"] = torch.cuda.Event(enable_timing=True)
                tr["k0"].record(comp)
            _lib.check(fn(*args), "hmf_sgd_block_qband")
            ev = torch.cuda.Event(enable_timing=tr is not None)
            ev.record(comp)
            self.freed[slot] = ev
            if tr is not None:
                tr["k1"] = ev
                self.trace.append(tr)
            done += hi - lo
        self.last_h2d = uploaded * self.bytes_per_rating
        return done


# -- calibration / benchmarking helpers ----------------------------------------


class _PrefixWork:
    """A triple prefix as a one-block grid (workers.py:396-405)."""

    def __init__(self, matrix, size):
        from .data import RatingMatrix, build_grid
        sub = RatingMatrix(matrix.n_users, matrix.n_items, matrix.users[:size],
                           matrix.items[:size], matrix.ratings[:size])
        self.grid = build_grid(sub, [0, matrix.n_users], [0, matrix.n_items])
        self.unit = Unit(blocks=(0,), rows=(0,), col=0, size=size)


def time_batch_prefixes(matrix, prefixes, repeats, hparams: Hyperparams,
                        config: BatchWorkerConfig, seed: int):
    """Per-stage mean seconds of the CUDA engine on each prefix
    (workers.py:408-444): transfer_in = stage_rows + stage_in (H2D of P, Q
    band and triples), kernel = compute, transfer_out = stage_out + flush_rows
    + the D2H write-back; CUDA events, stages timed separately."""
    torch = _torch()
    out = {"transfer_in": [], "kernel": [], "transfer_out": []}
    for size in prefixes:
        work = _PrefixWork(matrix, size)
        t_in = t_k = t_out = 0.0
        for rep in range(repeats):
            model = init_model(matrix.n_users, matrix.n_items, hparams,
                               kernels.mix64(seed, size, rep, 2))
            store = FactorStore(model, config.precision)
            eng = BatchEngine(config, model, hparams, store)
            t0 = time.perf_counter()
            eng.stage_rows(0, matrix.n_users)
            eng.stage_in("cal", work.grid, work.unit)
            torch.cuda.synchronize(eng.dev)
            t_in += time.perf_counter() - t0
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream)
            eng.compute("cal", kernels.mix64(seed, size, rep, 3))
            e1.record(eng.stream)
            e1.synchronize()
            t_k += e0.elapsed_time(e1) / 1e3
            t0 = time.perf_counter()
            eng.stage_out("cal")
            eng.flush_rows()
            store.sync_host()
            t_out += time.perf_counter() - t0
        out["transfer_in"].append(t_in / repeats)
        out["kernel"].append(t_k / repeats)
        out["transfer_out"].append(t_out / repeats)
    return out


def throughput_sweep(worker_class: str, sizes, repeats: int = 3, *,
                     hparams: Hyperparams | None = None,
                     batch_config: BatchWorkerConfig | None = None, n_rows: int = 4096,
                     n_cols: int = 4096, seed: int = 0):
    """Elements/second per workload size of the CUDA batch worker
    (workers.py:447-514, batch branch); the fastest of `repeats`."""
    from .data import RatingMatrix
    if list(sizes) != sorted(sizes):
        raise ValueError("sizes must be ascending")
    if worker_class != CLASS_BATCH:
        raise ValueError("the B200 engine provides batch workers only; stream workers are "
                         "the reference's CPU path")
    if batch_config is None:
        raise ValueError("batch sweeps need a BatchWorkerConfig")
    hparams = hparams or Hyperparams()
    torch = _torch()
    rng = np.random.default_rng(seed)
    res = []
    for size in sizes:
        m = RatingMatrix(n_rows, n_cols, rng.integers(0, n_rows, size=size).astype(np.int32),
                         rng.integers(0, n_cols, size=size).astype(np.int32),
                         rng.normal(size=size))
        work = _PrefixWork(m, size)
        best = None
        for rep in range(repeats):
            model = init_model(n_rows, n_cols, hparams, kernels.mix64(seed, size, rep, 4))
            eng = BatchEngine(batch_config, model, hparams, FactorStore(model, batch_config.precision))
            t0 = time.perf_counter()
            t_in = eng.stage_rows(0, n_rows) + eng.stage_in("s", work.grid, work.unit)
            t1 = time.perf_counter()
            eng.compute("s", kernels.mix64(rep, size, 5))
            eng.synchronize()
            t_kernel = time.perf_counter() - t1
            t2 = time.perf_counter()
            eng.stage_out("s")
            eng.flush_rows()
            eng.store.sync_host()
            t_out = time.perf_counter() - t2
            total = time.perf_counter() - t0
            entry = {"size": size, "seconds": total, "elements_per_second": size / total,
                     "stage_in_seconds": t_in, "kernel_seconds": t_kernel,
                     "stage_out_seconds": t_out}
            if best is None or total < best["seconds"]:
                best = entry
        res.append(best)
    torch.cuda.synchronize()
    return res
