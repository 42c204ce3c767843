"""The node-local lease table (csrc/lease.cu, distributed.ShmLeaseTable): the
column-lease half of the reference's GridScheduler.acquire/release
(scheduler.py:333-409) across the processes of one node.  Host code only —
these run without a GPU.

* the single-process contract: a column has at most one holder, a release
  by a non-holder fails and leaves the owner alone, the owner is published
  by the release, tickets count up, acquire_first honours the candidate
  order;
* mutual exclusion under contention: four processes lease and release
  random columns thousands of times, each checking a shared occupancy word
  inside its critical section;
* the cost: an operation is a few microseconds at most from Python (the
  torch.distributed store needs a TCP round trip per operation).
"""

import os
import time
import uuid

import numpy as np
import pytest
import torch.multiprocessing as mp


def _table(n_cols, rank, run_id):
    from paper_2006_15980_b200.distributed import ShmLeaseTable
    return ShmLeaseTable(n_cols, rank, run_id)


def test_single_process_contract():
    from paper_2006_15980_b200 import _lib
    run = uuid.uuid4().hex[:10]
    a = _table(5, 0, run)
    a.initialize()
    b = _table(5, 1, run)
    try:
        assert [a.owner(c) for c in range(5)] == [-1] * 5
        assert [a.holder(c) for c in range(5)] == [-1] * 5
        assert a.try_acquire(2)
        assert not b.try_acquire(2)
        assert a.holder(2) == 0 and b.holder(2) == 0
        with pytest.raises(RuntimeError, match="did not hold"):
            b.release(2)
        assert a.owner(2) == -1            # a bad release does not publish an owner
        a.release(2)
        assert a.owner(2) == 0 and a.holder(2) == -1
        # acquire_first: the first free candidate in list order
        assert a.try_acquire(4)
        assert b.acquire_first([4, 1, 3]) == 1
        assert b.acquire_first([4, 1]) is None
        b.release(1)
        assert a.owner(1) == 1
        a.release(4)
        assert [a.ticket() for _ in range(3)] == [1, 2, 3]
        assert b.ticket() == 4
        assert a.total_ops() >= 12
        # argument checks
        with pytest.raises(_lib.HmfError, match="out of range"):
            a.try_acquire(5)
        with pytest.raises(_lib.HmfError, match="out of range"):
            a.acquire_first([0, 7])
    finally:
        b.close()
        a.close(unlink=True)


def test_claim_counts_to_the_target():
    """hmf_lease_claim, the free policy's job-wide update counter: ordinals
    1..target across processes' tables, then 0 (never past the target); the
    next epoch raises the target; an aborted run raises."""
    from paper_2006_15980_b200.distributed import LeaseAborted
    run = uuid.uuid4().hex[:10]
    a = _table(3, 0, run)
    a.initialize()
    b = _table(3, 1, run)
    try:
        got = [a.claim(5), b.claim(5), a.claim(5), b.claim(5), a.claim(5)]
        assert got == [1, 2, 3, 4, 5]
        assert a.claim(5) == 0 and b.claim(5) == 0 and a.claim(5) == 0
        assert b.claim(10) == 6
        b.abort()
        with pytest.raises(LeaseAborted, match="rank 1"):
            a.claim(10)
    finally:
        b.close()
        a.close(unlink=True)


def test_store_claim_counts_to_the_target():
    import datetime

    import torch.distributed as dist
    from paper_2006_15980_b200.distributed import LeaseTable
    from test_distributed import _free_port
    store = dist.TCPStore("127.0.0.1", _free_port(), 1, True,
                          timeout=datetime.timedelta(seconds=30))
    a, b = LeaseTable(store, 3, 0, "claim"), LeaseTable(store, 3, 1, "claim")
    a.initialize()
    assert [a.claim(3), b.claim(3), a.claim(3), b.claim(3), a.claim(3)] == [1, 2, 3, 0, 0]
    assert b.claim(6) == 4                 # over-claims were given back


def test_open_errors():
    from paper_2006_15980_b200 import _lib
    run = uuid.uuid4().hex[:10]
    with pytest.raises(_lib.HmfError, match="shm_open"):
        _table(3, 1, run).try_acquire(0)          # nobody created it
    a = _table(3, 0, run)
    a.initialize()
    try:
        with pytest.raises(_lib.HmfError, match="column count|too small"):
            _table(4, 1, run).try_acquire(0)
    finally:
        a.close(unlink=True)


ROUNDS = 3000


def _hammer(rank, world, run_id, occ_path, n_cols):
    from paper_2006_15980_b200.distributed import ShmLeaseTable
    occ = np.memmap(occ_path, dtype=np.int32, mode="r+", shape=(n_cols + 1 + world,))
    t = ShmLeaseTable(n_cols, rank, run_id)
    rng = np.random.default_rng(rank)
    grants = bad = 0
    while grants < ROUNDS:
        c = t.acquire_first(rng.permutation(n_cols).tolist())
        if c is None:
            continue
        grants += 1
        if occ[c] != 0:
            bad += 1
        occ[c] = rank + 1
        for _ in range(int(rng.integers(0, 20))):
            pass
        if occ[c] != rank + 1:
            bad += 1
        occ[c] = 0
        t.release(c)
    occ[n_cols + 1 + rank] = bad
    occ.flush()
    t.close()


def test_mutual_exclusion_under_contention(tmp_path):
    world, n_cols = 4, 3          # fewer columns than processes: constant contention
    run = uuid.uuid4().hex[:10]
    occ_path = str(tmp_path / "occ.bin")
    occ = np.memmap(occ_path, dtype=np.int32, mode="w+", shape=(n_cols + 1 + world,))
    occ[:] = 0
    occ.flush()
    owner = _table(n_cols, 0, run)
    owner.initialize()
    try:
        ctx = mp.get_context("spawn")
        procs = [ctx.Process(target=_hammer, args=(r, world, run, occ_path, n_cols))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        occ = np.memmap(occ_path, dtype=np.int32, mode="r", shape=(n_cols + 1 + world,))
        assert occ[n_cols + 1:].tolist() == [0] * world, "two holders seen in a critical section"
        assert [owner.holder(c) for c in range(n_cols)] == [-1] * n_cols
        assert owner.total_ops() >= world * ROUNDS * 2
    finally:
        owner.close(unlink=True)


def test_operation_cost_is_microseconds():
    run = uuid.uuid4().hex[:10]
    t = _table(17, 0, run)
    t.initialize()
    try:
        n = 2000
        t0 = time.perf_counter()
        for i in range(n):
            c = t.acquire_first([i % 17])
            t.owner(c)
            t.release(c)
        per_lease = (time.perf_counter() - t0) / n
        assert t.ops == 3 * n
        # three ctypes calls per lease; a TCPStore round trip alone is ~50-100 us
        assert per_lease < 200e-6, per_lease
    finally:
        t.close(unlink=True)


def _abort_rank(rank, run_id, n_cols, out_path):
    """Rank 1 holds a column and fails; rank 0 waits for that column and
    must get LeaseAborted instead of waiting forever."""
    import time as _t

    from paper_2006_15980_b200.distributed import LeaseAborted, RowBandTrainer, ShmLeaseTable

    class Band:
        def __init__(self):
            self.n_cols = n_cols

        def pull(self, c, owner):
            pass

        def compute(self, c, seed):
            if rank == 1:
                _t.sleep(0.5)
                raise RuntimeError("device failure on rank 1")
            return 1

        def finish(self, c):
            pass

    table = ShmLeaseTable(n_cols, rank, run_id)
    trainer = RowBandTrainer(Band(), table, rank, seed=0)
    try:
        if rank == 0:              # start once rank 1 holds column 0
            deadline = _t.time() + 30
            while table.holder(0) != 1 and _t.time() < deadline:
                _t.sleep(0.005)
        trainer.run_epoch()
        result = "finished"
    except LeaseAborted as exc:
        result = f"aborted: {exc}"
    except RuntimeError as exc:
        result = f"failed: {exc}"
    with open(out_path + f".{rank}", "w") as fh:
        fh.write(result)
    table.close()


def test_abort_releases_waiting_ranks(tmp_path):
    """A rank whose lease loop raises marks the run aborted (hmf_lease_abort,
    the reference's scheduler.abort on a worker error, workers.py:300-302):
    a rank blocked waiting for a column gets LeaseAborted, and nobody hangs."""
    run = uuid.uuid4().hex[:10]
    n_cols = 1                           # both ranks need the same column
    owner = _table(n_cols, 0, run)
    owner.initialize()
    try:
        ctx = mp.get_context("spawn")
        out = str(tmp_path / "res")
        procs = [ctx.Process(target=_abort_rank, args=(r, run, n_cols, out)) for r in (1, 0)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(60)
            assert p.exitcode == 0
        assert open(out + ".1").read() == "failed: device failure on rank 1"
        r0 = open(out + ".0").read()
        assert r0.startswith("aborted") and "rank 1" in r0, r0
        assert owner.aborted_by() == 1
        from paper_2006_15980_b200.distributed import LeaseAborted
        with pytest.raises(LeaseAborted):
            owner.try_acquire(0)
    finally:
        owner.close(unlink=True)


@pytest.mark.parametrize("policy", ["quota", "free"])
def test_lease_sim_runs(policy):
    """scripts/lease_sim.py (the protocol-efficiency simulation DESIGN §6
    quotes) runs end to end on the host: 2 simulated GPUs, both policies."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(root / "scripts" / "lease_sim.py"), "--gpus", "2",
                          "--epochs", "2", "--policy", policy, "--ratings-per-gpu", "2e8"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["policy"] == policy and line["gpus"] == 2 and line["column_bands"] == 5
    assert sum(line["blocks_per_rank"]) == 2 * 2 * 5
    assert 0.5 < line["throughput_efficiency"] <= 1.05
