"""Multi-GPU block scheduling across processes: one process per GPU.

The reference runs its workers as threads around one GridScheduler
(scheduler.py:333-409) and moves item columns through shared host arrays
(workers.py:186-218).  Across B200 processes the same protocol becomes:

* rows are banded one band per GPU (partition.gpu_plan: mass proportional to
  each GPU's fitted throughput) and each P band stays resident on its GPU —
  the reference's P-band residency (workers.py:13-17, 324-328);
* columns are 2*N+1 bands (a primary and a staged-ahead column per GPU plus a
  spare, the reference's column rule for batch workers);
* a column lease is a compare-and-set on a lock-free table in node-local
  shared memory (ShmLeaseTable, csrc/lease.cu; or, portably, on a key of the
  torch.distributed store, LeaseTable): at most one GPU holds a column band,
  so Q bands have a single owner at a time, exactly the scheduler's
  independence rule;
* each GPU pulls (RowBandTrainer) its undone blocks dynamically, least-updated
  first with a seeded tie break, and keeps a staged-ahead column: while the
  kernel runs on column c it tries to lease the next column and starts
  pulling that Q band from its last owner on a copy stream (CUDA IPC +
  cudaMemcpyPeerAsync over NVLink), the reference's prefetch unit
  (scheduler.py:280-304, workers.py:338-361);
* an epoch is the reference's quota epoch: every block once, then a barrier
  where metrics are reduced (all_reduce of the residual sums).

No process ever holds a column while waiting for another one, so the
protocol cannot deadlock.  The transport and the compute are pluggable: the
GPU implementation lives in CudaRowBand; tests drive the same trainer with a
CPU transport over gloo (world size 2).
"""

from __future__ import annotations

import ctypes
import time
import uuid

import numpy as np

from .kernels import mix64

FREE = b"free"


class LeaseTable:
    """Column-band leases over a torch.distributed Store (compare-and-set):
    portable (any backend, any number of nodes), one TCP round trip per
    operation.  `ops` / `seconds` count the store operations and the host
    time spent in them."""

    kind = "store"

    def __init__(self, store, n_cols: int, rank: int, run_id: str):
        self.store = store
        self.n_cols = n_cols
        self.rank = rank
        self.prefix = f"hmf/{run_id}"
        self._me = str(rank).encode()
        self.ops = 0
        self.seconds = 0.0

    def _key(self, kind: str, c: int) -> str:
        return f"{self.prefix}/{kind}/{c}"

    def initialize(self) -> None:
        """Rank 0, before the first barrier: every column free, no owner yet
        (every replica of Q starts from the same seeded init)."""
        for c in range(self.n_cols):
            self.store.set(self._key("lease", c), FREE)
            self.store.set(self._key("owner", c), b"-1")

    def try_acquire(self, c: int) -> bool:
        t0 = time.perf_counter()
        got = self.store.compare_set(self._key("lease", c), FREE, self._me)
        self.ops += 1
        self.seconds += time.perf_counter() - t0
        return bytes(got) == self._me

    def owner(self, c: int) -> int:
        t0 = time.perf_counter()
        o = int(bytes(self.store.get(self._key("owner", c))))
        self.ops += 1
        self.seconds += time.perf_counter() - t0
        return o

    def release(self, c: int) -> None:
        t0 = time.perf_counter()
        # publish the new owner first: whoever leases c next pulls from us
        self.store.set(self._key("owner", c), self._me)
        got = self.store.compare_set(self._key("lease", c), self._me, FREE)
        self.ops += 2
        self.seconds += time.perf_counter() - t0
        if bytes(got) != FREE:
            raise RuntimeError(f"rank {self.rank} released column {c} it did not hold")

    def ticket(self) -> int:
        """A global sequence number (lease order, for traces and tests)."""
        t0 = time.perf_counter()
        n = int(self.store.add(f"{self.prefix}/seq", 1))
        self.ops += 1
        self.seconds += time.perf_counter() - t0
        return n

    def abort(self) -> None:
        """Mark the run aborted by this rank (a store key every acquire checks)."""
        self.store.compare_set(f"{self.prefix}/aborted", b"", str(self.rank).encode())

    def claim(self, target: int) -> int:
        """The free policy's job-wide block count: the ordinal of the claimed
        block update, or 0 once `target` are claimed (an over-claim is given
        back, so the count stops at the target)."""
        t0 = time.perf_counter()
        n = int(self.store.add(f"{self.prefix}/work", 1))
        self.ops += 1
        if n > target:
            self.store.add(f"{self.prefix}/work", -1)
            self.ops += 1
            n = 0
        self.seconds += time.perf_counter() - t0
        return n

    def aborted_by(self) -> int:
        if not self.store.check([f"{self.prefix}/aborted"]):
            return -1
        return int(bytes(self.store.get(f"{self.prefix}/aborted")))

    def close(self, unlink: bool = False) -> None:
        pass


class LeaseAborted(RuntimeError):
    """Another rank aborted the run (its lease loop raised); the reference
    re-raises a worker's exception after scheduler.abort (workers.py:300-302,
    engine.py:255-258)."""


class ShmLeaseTable:
    """Column-band leases in node-local shared memory (csrc/lease.cu): the
    same protocol as LeaseTable — holder compare-and-set, owner published
    before the release — as lock-free atomics on a POSIX shared-memory
    segment that every GPU process of the node maps.  An operation costs
    ~0.1-1 us instead of a TCP round trip, and acquire_first tries a whole
    candidate list in one call.  Rank 0 creates the segment in initialize()
    (before the first barrier, as LeaseTable); the others map it on first
    use.  Host code only: works without a GPU (the gloo tests)."""

    kind = "shm"

    def __init__(self, n_cols: int, rank: int, run_id: str):
        self.n_cols = n_cols
        self.rank = rank
        self.name = f"/hmf_lease_{run_id}".encode()
        self._t = None
        self._lib = None
        self.ops = 0
        self.seconds = 0.0

    def _open(self, create: bool) -> None:
        from . import _lib
        lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(lib.hmf_lease_open(self.name, self.n_cols, 1 if create else 0,
                                      ctypes.byref(h)), "hmf_lease_open")
        self._t, self._lib = h, lib

    def _table(self):
        if self._t is None:
            self._open(create=False)
        return self._t

    def initialize(self) -> None:
        self._open(create=True)

    def try_acquire(self, c: int) -> bool:
        t = self._table()
        t0 = time.perf_counter()
        rc = self._lib.hmf_lease_try_acquire(t, int(c), self.rank)
        self.ops += 1
        self.seconds += time.perf_counter() - t0
        return self._check(rc, "hmf_lease_try_acquire") == 1

    def acquire_first(self, cands) -> int | None:
        """The first candidate column granted (in list order), or None."""
        t = self._table()
        arr = (ctypes.c_int32 * len(cands))(*[int(c) for c in cands])
        got = ctypes.c_int32(-1)
        t0 = time.perf_counter()
        rc = self._lib.hmf_lease_acquire_first(t, arr, len(cands), self.rank, ctypes.byref(got))
        self.ops += 1
        self.seconds += time.perf_counter() - t0
        self._check(rc, "hmf_lease_acquire_first")
        return None if got.value < 0 else int(got.value)

    def owner(self, c: int) -> int:
        t = self._table()
        o = ctypes.c_int32()
        t0 = time.perf_counter()
        rc = self._lib.hmf_lease_owner(t, int(c), ctypes.byref(o))
        self.ops += 1
        self.seconds += time.perf_counter() - t0
        self._check(rc, "hmf_lease_owner")
        return int(o.value)

    def holder(self, c: int) -> int:
        o = ctypes.c_int32()
        t = self._table()
        self._check(self._lib.hmf_lease_holder(t, int(c), ctypes.byref(o)), "hmf_lease_holder")
        return int(o.value)

    def release(self, c: int) -> None:
        t = self._table()
        t0 = time.perf_counter()
        rc = self._lib.hmf_lease_release(t, int(c), self.rank)
        self.ops += 1
        self.seconds += time.perf_counter() - t0
        if rc < 0:
            raise RuntimeError(f"rank {self.rank} released column {c} it did not hold")

    def ticket(self) -> int:
        t = self._table()
        t0 = time.perf_counter()
        n = self._lib.hmf_lease_ticket(t)
        self.ops += 1
        self.seconds += time.perf_counter() - t0
        return int(self._check(n, "hmf_lease_ticket"))

    def total_ops(self) -> int:
        """Operations served by the segment, all processes."""
        t = self._table()            # maps the segment (and binds the library) first
        return int(self._lib.hmf_lease_ops(t))

    def abort(self) -> None:
        """Mark the run aborted by this rank: every later acquire, on every
        rank, raises LeaseAborted (scheduler.abort, scheduler.py:415-423)."""
        t = self._table()
        self._check(self._lib.hmf_lease_abort(t, self.rank), "hmf_lease_abort")

    def aborted_by(self) -> int:
        """The rank that aborted the run, or -1."""
        t = self._table()
        return int(self._lib.hmf_lease_aborted(t))

    def claim(self, target: int) -> int:
        """The free policy's job-wide block count (hmf_lease_claim): the
        ordinal of the claimed block update, or 0 once `target` are claimed."""
        t = self._table()
        t0 = time.perf_counter()
        n = self._lib.hmf_lease_claim(t, int(target))
        self.ops += 1
        self.seconds += time.perf_counter() - t0
        return int(self._check(n, "hmf_lease_claim"))

    def _check(self, rc: int, what: str) -> int:
        from . import _lib
        if rc == _lib.HMF_ERR_ABORTED:
            raise LeaseAborted(_lib.last_error())
        if rc < 0:
            raise _lib.HmfError(f"{what} failed ({rc}): {_lib.last_error()}")
        return rc

    def close(self, unlink: bool = False) -> None:
        if self._t is not None:
            self._lib.hmf_lease_close(self._t, 1 if unlink else 0)
            self._t = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_lease_table(kind: str, store, n_cols: int, rank: int, run_id: str):
    """kind "shm" (one node, the default) or "store" (the torch.distributed
    store: portable across nodes)."""
    if kind == "shm":
        return ShmLeaseTable(n_cols, rank, run_id)
    if kind == "store":
        return LeaseTable(store, n_cols, rank, run_id)
    raise ValueError(f"lease table kind must be 'shm' or 'store', not {kind!r}")


def new_run_id() -> str:
    return uuid.uuid4().hex[:12]


class RowBandTrainer:
    """One GPU's lease loop over the blocks of its row band.

    backend must provide:
      n_cols                        column bands
      pull(c, owner)                enqueue the Q band c copy from `owner`'s
                                    replica (no-op when owner is self or -1)
      compute(c, seed) -> int       enqueue the block's update; returns triples
      finish(c)                     block until the compute of c completed
    """

    def __init__(self, backend, table: LeaseTable, rank: int, seed: int = 0,
                 prefetch: bool = True, record: bool = False, policy: str = "quota",
                 world: int = 1):
        self.backend = backend
        self.table = table
        self.rank = rank
        self.seed = seed
        self.prefetch = prefetch
        self.n_cols = backend.n_cols
        self.counts = np.zeros(self.n_cols, dtype=np.int64)
        self._rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(0xC1, rank)))
        self.record = record
        self.log = []            # (ticket, column, seed) per granted block
        self.total_updates = 0
        self.wait_seconds = 0.0
        # the reference's scheduling policies (scheduler.py:41-43, 255-304,
        # 411-429): "quota" — every rank trains each of its blocks once per
        # epoch (batch-only, stream-only); "free" — any free column, least
        # updated first, an epoch being world x n_cols block updates claimed
        # job-wide by whoever is free (the hsgd schedule's POLICY_FREE)
        if policy not in ("quota", "free"):
            raise ValueError(f"policy must be 'quota' or 'free', not {policy!r}")
        self.policy = policy
        self.world = max(1, int(world))
        self.epochs_done = 0

    def _candidates(self, todo: set) -> list:
        cols = sorted(todo)
        ties = self._rng.permutation(len(cols))
        return [c for _, _, c in sorted(zip((self.counts[c] for c in cols), ties, cols))]

    def _grab(self, todo: set, blocking: bool):
        delay = 2e-6 if hasattr(self.table, "acquire_first") else 2e-5
        t0 = time.perf_counter()
        while todo:
            cands = self._candidates(todo)
            if hasattr(self.table, "acquire_first"):
                c = self.table.acquire_first(cands)
                if c is not None:
                    self.wait_seconds += time.perf_counter() - t0
                    return c
            else:
                for c in cands:
                    if self.table.try_acquire(c):
                        self.wait_seconds += time.perf_counter() - t0
                        return c
            if not blocking:
                return None
            if not hasattr(self.table, "acquire_first") and self.table.aborted_by() >= 0:
                raise LeaseAborted(f"the run was aborted by rank {self.table.aborted_by()}")
            time.sleep(delay)
            delay = min(delay * 2, 1e-3)
        return None

    def lease_stats(self) -> dict:
        """Lease-table cost on this rank: operations and host seconds spent
        in them, per granted lease."""
        n = max(1, int(self.counts.sum()))
        return {"table": getattr(self.table, "kind", "?"), "leases": int(self.counts.sum()),
                "ops": int(self.table.ops), "ops_per_lease": self.table.ops / n,
                "seconds": float(self.table.seconds),
                "us_per_lease": 1e6 * self.table.seconds / n,
                "wait_seconds": float(self.wait_seconds)}

    def _start(self, c: int) -> None:
        """Lease granted: stamp the seed, pull the band, enqueue compute."""
        block = self.rank * self.n_cols + c
        unit_seed = mix64(self.seed, block, int(self.counts[c]))
        if self.record:
            self.log.append((self.table.ticket(), c, unit_seed))
        self.backend.pull(c, self.table.owner(c))
        self.total_updates += self.backend.compute(c, mix64(unit_seed, 0))

    def run_epoch(self) -> None:
        """One quota epoch of this rank's blocks.  A failure here aborts the
        whole run: the lease table is marked, every other rank's next acquire
        raises LeaseAborted instead of waiting for a column this rank may
        hold (workers.py:300-302)."""
        try:
            self._run_epoch()
        except LeaseAborted:
            raise
        except BaseException:
            try:
                self.table.abort()
            finally:
                raise

    def _run_epoch(self) -> None:
        if self.policy == "free":
            self._run_epoch_free()
        else:
            self._run_epoch_quota()
        self.epochs_done += 1

    def _run_epoch_free(self) -> None:
        """POLICY_FREE: lease any column this rank does not hold, least
        updated first; a block runs only if it claims one of the epoch's
        world x n_cols job-wide block updates (hmf_lease_claim), so ranks that
        are free keep working until the epoch's quota is spent, with no rank
        waiting on a particular column at the epoch's end."""
        target = (self.epochs_done + 1) * self.world * self.n_cols
        everything = set(range(self.n_cols))
        pending = False          # an update claimed but not yet bound to a column

        def take(held, blocking):
            # claim first, lease second: a lease taken and handed back unused
            # would publish this rank as the band's owner without its update
            nonlocal pending
            if not pending:
                if self.table.claim(target) <= 0:     # the epoch's updates are spent
                    return None, True
                pending = True
            c = self._grab(everything - held, blocking)
            if c is None:        # keep the claim for the blocking grab after finish
                return None, False
            pending = False
            self._start(c)
            return c, False

        cur, spent = take(set(), True)
        while cur is not None:
            nxt = None
            if self.prefetch and not spent:
                nxt, spent = take({cur}, False)
            self.backend.finish(cur)
            self.table.release(cur)
            self.counts[cur] += 1
            if nxt is None and not spent:
                nxt, spent = take(set(), True)
            cur = nxt

    def _run_epoch_quota(self) -> None:
        todo = set(range(self.n_cols))
        cur = self._grab(todo, blocking=True)
        todo.discard(cur)
        self._start(cur)
        while cur is not None:
            nxt = None
            if self.prefetch and todo:
                nxt = self._grab(todo, blocking=False)
                if nxt is not None:
                    todo.discard(nxt)
                    self._start(nxt)          # queued behind cur on the device
            self.backend.finish(cur)
            self.table.release(cur)
            self.counts[cur] += 1
            if nxt is None and todo:
                nxt = self._grab(todo, blocking=True)
                todo.discard(nxt)
                self._start(nxt)
            cur = nxt


# ---------------------------------------------------------------------------
# GPU backend
# ---------------------------------------------------------------------------
class CudaRowBand:
    """One rank's device state: its P band, a full Q replica, its triples.

    Q replicas of all ranks are mapped into every process with CUDA IPC, so a
    pull is a one-sided peer copy from the band's last owner — the owner does
    not participate.  Blocks use the Q-band layout and kernel (row tiles of
    this band, item runs split over the chains when the band is narrow), or
    the global-Q HOGWILD / EXACT range kernels.
    """

    def __init__(self, dist, rank: int, world: int, device, triples, row_lo: int, row_hi: int,
                 col_cuts, k: int, lr: float, reg_user: float, reg_item: float,
                 init_seed: int = 0, kernel: str = "auto", init=None, concurrency: int = 1,
                 split: int | None = None, impl: int | None = None):
        import torch
        from . import _lib
        from .data import DeviceTriples, bucket_qbands, build_device_grid, resident_warps
        self.torch = torch
        self.lib = _lib
        self.dev = torch.device(device)
        self.rank, self.world = rank, world
        self.k = k
        self.lr, self.ru, self.ri = lr, reg_user, reg_item
        self.row_lo, self.row_hi = row_lo, row_hi
        self.col_cuts = np.asarray(col_cuts, dtype=np.int64)
        self.n_cols = len(self.col_cuts) - 1
        n_items = int(self.col_cuts[-1])
        # P band (rows of this rank) and a full Q replica, same init law on
        # every rank for Q (so owner -1 = "any replica is current")
        if init is not None:   # explicit starting factors (host arrays: P band, Q)
            self.P = torch.from_numpy(np.ascontiguousarray(init[0], dtype=np.float32)).to(self.dev)
            self.Q = torch.from_numpy(np.ascontiguousarray(init[1], dtype=np.float32)).to(self.dev)
        else:
            g = torch.Generator(device=self.dev)
            g.manual_seed(init_seed * 1_000_003 + rank + 1)
            top = 1.0 / float(np.sqrt(k))
            self.P = (torch.rand((row_hi - row_lo, k), generator=g, device=self.dev)
                      * top).contiguous()
            gq = torch.Generator(device=self.dev)
            gq.manual_seed(init_seed * 1_000_003)
            self.Q = (torch.rand((n_items, k), generator=gq, device=self.dev) * top).contiguous()
        # local triples (users already global ids within [row_lo, row_hi))
        local = DeviceTriples(row_hi, n_items, triples.users, triples.items, triples.ratings)
        # row bands [0, row_lo) (empty) and [row_lo, row_hi): row tiles of the
        # Q-band layout then cover this rank's band only
        rows = [0, row_hi] if row_lo == 0 else [0, row_lo, row_hi]
        self.grid = build_device_grid(local, rows, self.col_cuts)
        first = 0 if row_lo == 0 else self.n_cols
        self.block_of = [first + c for c in range(self.n_cols)]   # block of column c
        # the Q-band layout (row tiles: this band's P rows in L2) also wins for
        # narrow column bands once two of them run side by side: projected
        # 6.5 vs 4.0 G upd/s per GPU for the global-Q kernel at the 8-GPU
        # geometry (bench.py --sim-world 8, profiles/r02/sim_world8_*.json)
        self.kernel = kernel if kernel != "auto" else (
            "qband" if k in (32, 64, 128, 256) else "range")
        if self.kernel == "qband":
            # narrow column bands split their item runs over the chains
            # (data.qband_split_for, implementation 5)
            if split:
                bucket_qbands(self.grid, k, impl=5, split=int(split))
            elif concurrency > 1:
                slots = resident_warps(self.dev, k, False, 4) // int(concurrency)
                widest = int(np.max(np.diff(self.col_cuts)))
                bucket_qbands(self.grid, k, impl=5, split=max(1, min(16, slots // widest)))
            else:
                # the automatic layout (data.tile_resident_impl: a Netflix-
                # density band picks run groups over a shared-memory P tile)
                bucket_qbands(self.grid, k, impl=impl)
        # column blocks in flight at once, each on its own stream with a
        # 1/concurrency share of the GPU.  Default 1: with item runs split
        # over chains (implementation 5) one narrow block fills the GPU, and
        # a single full-GPU launch has no tail (bench.py --sim-world 8:
        # 8.85 vs 8.05 G upd/s per GPU with two half-GPU launches)
        self.concurrency = max(1, int(concurrency)) if self.kernel == "qband" else 1
        self.streams = [torch.cuda.Stream(device=self.dev) for _ in range(self.concurrency)]
        self.stream = self.streams[0]
        self._next_stream = 0
        self.stream_of = {}
        self.copy_stream = torch.cuda.Stream(device=self.dev)
        self.done_events = {}
        # host staging (stage_from_host): every granted block's triples are
        # uploaded from pinned host copies on its stream before the launch,
        # as BatchEngine.stage_in does per lease (workers.py:186-202)
        self.host = None
        self.compact = None      # block -> its tiles' first rows (compact stream)
        self.staged_bytes = 0
        # P, Q and the grid were produced on the current stream; the band's
        # own compute / copy streams must not start before they exist
        torch.cuda.current_stream(self.dev).synchronize()
        # exchange IPC handles of the Q replicas
        import ctypes
        handle = (ctypes.c_uint8 * 64)()
        off = ctypes.c_int64(0)
        _lib.check(_lib.load().hmf_ipc_get_handle(self.Q.data_ptr(), handle, ctypes.byref(off)),
                   "hmf_ipc_get_handle")
        mine = (bytes(handle), int(off.value), self.dev.index)
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        self.peer_q = {}
        for r, (hb, offset, pdev) in enumerate(allh):
            if r == rank:
                continue
            buf = (ctypes.c_uint8 * 64).from_buffer_copy(hb)
            ptr = ctypes.c_void_p()
            _lib.check(_lib.load().hmf_ipc_open_handle(buf, ctypes.byref(ptr)),
                       "hmf_ipc_open_handle")
            self.peer_q[r] = (ptr.value + offset, pdev)

    # -- backend protocol ------------------------------------------------------
    def _stream_for(self, c: int):
        """The compute stream column c's block runs on (assigned at its pull)."""
        if c not in self.stream_of:
            self.stream_of[c] = self.streams[self._next_stream]
            self._next_stream = (self._next_stream + 1) % len(self.streams)
        return self.stream_of[c]

    def pull(self, c: int, owner: int) -> None:
        stream = self._stream_for(c)
        if owner < 0 or owner == self.rank:
            return
        lo, hi = int(self.col_cuts[c]), int(self.col_cuts[c + 1])
        nbytes = (hi - lo) * self.k * 4
        src, _ = self.peer_q[owner]
        _lib = self.lib
        # IPC-mapped peer pointer: a UVA copy (device -1) over NVLink
        _lib.check(_lib.load().hmf_memcpy_peer_async(
            self.Q.data_ptr() + lo * self.k * 4, -1, src + lo * self.k * 4, -1,
            nbytes, self.copy_stream.cuda_stream), "hmf_memcpy_peer_async")
        ev = self.torch.cuda.Event()
        ev.record(self.copy_stream)
        stream.wait_event(ev)

    def stage_from_host(self, on: bool = True) -> None:
        """Upload each granted block's triples from pinned host memory before
        its launch (the end-to-end path); training is unchanged.  With the
        chained kernel on single-item sub-bands and row tiles of at most
        65 536 users the stream is compact, as in workers.StreamingEpoch:
        uint16 user ids relative to the tile plus the rating, 6 bytes per
        rating (hmf_sgd_block_qband_u16_tiles_*); otherwise the triples, 12."""
        torch = self.torch
        if on and self.host is None:
            g = self.grid
            runs = self.kernel == "qband" and g.sub_impl == 8
            compact = runs or (self.kernel == "qband" and (g.sub_impl or 0) in (4, 5, 6)
                               and all(bool(torch.all(sc[1:] - sc[:-1] <= 1))
                                       for sc in g.sub_cuts)
                               and all(len(r) < 2 or int(np.max(np.diff(r))) <= 65536
                                       for r in g.sub_tile_rows))
            self.compact = {} if compact else None
            if runs:
                # implementation 8: users relative to their (shared-memory) row
                # tile, items in the resident run descriptors
                rel = torch.empty(g.nnz, dtype=torch.int16, device=self.dev)
                for c in range(self.n_cols):
                    b = self.block_of[c]
                    lo, hi = g.block_range(b)
                    if hi > lo:
                        d_tiles = torch.from_numpy(g.sub_tile_rows[b]).to(self.dev)
                        tile_of = torch.bucketize(g.users[lo:hi],
                                                  d_tiles[1:-1].to(torch.int32), right=True)
                        rel[lo:hi] = (g.users[lo:hi] - d_tiles[tile_of]).to(torch.int32).to(
                            torch.int16)
                    self.compact[b] = None
                self.host = [rel.cpu().pin_memory(), g.ratings.cpu().pin_memory()]
                self.dev_rel = rel
            elif compact:
                rel = torch.empty(g.nnz, dtype=torch.int16, device=self.dev)
                for c in range(self.n_cols):
                    b = self.block_of[c]
                    sp = g.sub_ptr[b].cpu().numpy()
                    T = g.sub_tiles[b]
                    S = (len(sp) - 1) // T
                    rows0 = [int(r) for r in g.sub_tile_rows[b][:T]]
                    for t in range(T):
                        a, z = int(sp[t * S]), int(sp[(t + 1) * S])
                        if z > a:
                            rel[a:z] = (g.users[a:z] - rows0[t]).to(torch.int32).to(torch.int16)
                    # first rows relative to this band's P (row_lo)
                    self.compact[b] = torch.tensor([r - self.row_lo for r in rows0],
                                                   dtype=torch.int32, device=self.dev)
                self.host = [rel.cpu().pin_memory(), g.ratings.cpu().pin_memory()]
                self.dev_rel = rel
            else:
                self.host = [a.cpu().pin_memory() for a in (g.users, g.items, g.ratings)]
        self._staging = bool(on)

    def _launch_compact(self, b: int, seed: int, stream) -> int:
        from . import kernels
        g = self.grid
        lo, hi = g.block_range(b)
        sp, sc = g.sub_ptr[b], g.sub_cuts[b]
        opts = kernels.qband_opts(g, grid_share=self.concurrency)
        lib = self.lib.load()
        st = "f16" if self.P.dtype == self.torch.float16 else "f32"
        if g.sub_impl == 8:
            fn = getattr(lib, f"hmf_sgd_block_runs_u16_{st}")
            self.lib.check(fn(self.P.data_ptr(), self.Q.data_ptr(), self.k,
                              self.dev_rel.data_ptr() + 2 * lo, g.ratings.data_ptr() + 4 * lo,
                              sp.data_ptr(), g.sub_tile_run[b].data_ptr(),
                              g.sub_tile_cuts[b].data_ptr(), int(g.sub_tiles[b]),
                              int(g.sub_max_rows), ctypes.byref(opts), float(self.lr),
                              float(self.ru), float(self.ri), int(seed) & kernels._MASK64,
                              self.row_lo, 0, stream.cuda_stream), "hmf_sgd_block_runs_u16")
            return hi - lo
        fn = getattr(lib, f"hmf_sgd_block_qband_u16_tiles_{st}")
        self.lib.check(fn(self.P.data_ptr(), self.Q.data_ptr(), self.k, self.dev_rel.data_ptr(),
                          0, g.ratings.data_ptr(), sp.data_ptr(), sc.data_ptr(),
                          int(sc.numel()) - 1, int(g.sub_tiles[b]),
                          self.compact[b].data_ptr(), ctypes.byref(opts), float(self.lr),
                          float(self.ru), float(self.ri), int(seed) & kernels._MASK64, 0,
                          stream.cuda_stream), "hmf_sgd_block_qband_u16_tiles")
        return hi - lo

    def compute(self, c: int, seed: int) -> int:
        from . import kernels
        b = self.block_of[c]
        lo, hi = self.grid.block_range(b)
        stream = self._stream_for(c)
        staging = getattr(self, "_staging", False) and hi > lo
        if staging:
            # on the copy stream: a block granted ahead (the trainer's
            # prefetch) uploads while the current block's kernel runs; its
            # range is disjoint from every block in flight, and its previous
            # launch finished before the lease was released
            dsts = ((self.dev_rel, self.grid.ratings) if self.compact is not None
                    else (self.grid.users, self.grid.items, self.grid.ratings))
            with self.torch.cuda.stream(self.copy_stream):
                for dst, src in zip(dsts, self.host):
                    dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
                    self.staged_bytes += (hi - lo) * dst.element_size()
                up = self.torch.cuda.Event()
                up.record(self.copy_stream)
            stream.wait_event(up)
        if staging and self.compact is not None:
            n = self._launch_compact(b, seed, stream)
            ev = self.torch.cuda.Event()
            ev.record(stream)
            self.done_events[c] = ev
            return n
        if self.kernel == "qband":
            # several column blocks in flight: each launch fills 1/concurrency
            # of the GPU (a per-launch option, ABI 4)
            n = kernels.launch_block_qband(self.P, self.Q, self.grid, b, self.lr, self.ru,
                                           self.ri, seed, row_base=self.row_lo,
                                           stream=stream.cuda_stream,
                                           opts={"grid_share": self.concurrency})
        else:   # "range" (HOGWILD) or "exact" (reference order and arithmetic)
            n = kernels.launch_sgd_range(self.P, self.Q, self.grid.users, self.grid.items,
                                         self.grid.ratings, lo, hi, self.lr, self.ru, self.ri,
                                         seed, self.row_lo, 0,
                                         "exact" if self.kernel == "exact" else "hogwild",
                                         stream.cuda_stream)
        ev = self.torch.cuda.Event()
        ev.record(stream)
        self.done_events[c] = ev
        return n

    def finish(self, c: int) -> None:
        ev = self.done_events.pop(c, None)
        self.stream_of.pop(c, None)
        if ev is not None:
            ev.synchronize()

    def refresh_q(self, table: LeaseTable) -> None:
        """Pull every band from its owner (metrics / end of run)."""
        for c in range(self.n_cols):
            self.pull(c, table.owner(c))
            self.stream_of.pop(c, None)
        for s in self.streams:
            s.synchronize()
