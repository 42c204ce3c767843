"""The multi-GPU lease protocol on CPU: world size 2 over gloo.

Each process plays one GPU: a resident P row band, its own Q replica (a
shared memory-mapped file standing in for the device allocation peers map
with CUDA IPC), the oracle kernel as the compute.  Columns are leased
through the node-local shared-memory lease table (csrc/lease.cu) or the
torch.distributed store, exactly as on the GPU path, Q bands are
pulled from their last owner, and the result must equal a serial replay of
the recorded lease order bit for bit — the reference's own check for its
threaded workers (tests/test_workers.py:43-70).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp




def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


N_USERS, N_ITEMS, K, NNZ = 80, 70, 4, 2400
EPOCHS, SEED, LR, REG = 3, 5, 0.02, 0.01


def _problem():
    rng = np.random.default_rng(11)
    cells = rng.permutation(N_USERS * N_ITEMS)[:NNZ]
    users = (cells // N_ITEMS).astype(np.int32)
    items = (cells % N_ITEMS).astype(np.int32)
    vals = rng.uniform(0, 1, NNZ)
    P0 = rng.uniform(0, 0.5, size=(N_USERS, K))
    Q0 = rng.uniform(0, 0.5, size=(N_ITEMS, K))
    return users, items, vals, P0, Q0


class CpuBand:
    """CPU stand-in for CudaRowBand (same backend protocol)."""

    def __init__(self, rank, world, tmp, row_cuts, col_cuts, users, items, vals, P0, Q0):
        import oracle
        from paper_2006_15980_b200.data import RatingMatrix, build_grid
        self.oracle = oracle
        self.rank = rank
        self.col_cuts = col_cuts
        self.n_cols = len(col_cuts) - 1
        self.lo, self.hi = int(row_cuts[rank]), int(row_cuts[rank + 1])
        keep = (users >= self.lo) & (users < self.hi)
        m = RatingMatrix(self.hi, N_ITEMS, users[keep], items[keep], vals[keep])
        self.grid = build_grid(m, [0, self.hi], col_cuts)
        self.P = P0[self.lo:self.hi].copy()
        self.Q = {r: np.memmap(os.path.join(tmp, f"q{r}.bin"), dtype=np.float64, mode="r+",
                               shape=(N_ITEMS, K)) for r in range(world)}
        self.pulls = 0

    def pull(self, c, owner):
        if owner < 0 or owner == self.rank:
            return
        a, b = int(self.col_cuts[c]), int(self.col_cuts[c + 1])
        self.Q[self.rank][a:b] = self.Q[owner][a:b]
        self.pulls += 1

    def compute(self, c, seed):
        lo, hi = self.grid.block_range(c)
        q = self.Q[self.rank]
        Qa = np.ascontiguousarray(q)
        n = self.oracle.sgd_range(self.P, Qa, self.grid.users, self.grid.items, self.grid.ratings,
                                  lo, hi, LR, REG, REG, seed, self.lo, 0)
        a, b = int(self.col_cuts[c]), int(self.col_cuts[c + 1])
        q[a:b] = Qa[a:b]
        q.flush()
        return n

    def finish(self, c):
        pass


def _worker(rank, world, port, tmp, kind="store", policy="quota"):
    import torch.distributed as dist
    from paper_2006_15980_b200.distributed import RowBandTrainer, make_lease_table
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    users, items, vals, P0, Q0 = _problem()
    row_cuts = np.array([0, 41, N_USERS])
    col_cuts = np.array([0, 14, 28, 42, 56, N_ITEMS])       # 2N+1 column bands
    band = CpuBand(rank, world, tmp, row_cuts, col_cuts, users, items, vals, P0, Q0)
    store = dist.distributed_c10d._get_default_store()
    table = make_lease_table(kind, store, band.n_cols, rank, f"test{port}")
    if rank == 0:
        table.initialize()
    dist.barrier()
    trainer = RowBandTrainer(band, table, rank, seed=SEED, record=True, policy=policy,
                             world=world)
    for _ in range(EPOCHS):
        trainer.run_epoch()
        dist.barrier()
    logs = [None] * world
    dist.all_gather_object(logs, (trainer.log, band.P, band.pulls, trainer.total_updates,
                                  trainer.counts.tolist()))
    # the final Q: every band from its owner
    for c in range(band.n_cols):
        band.pull(c, table.owner(c))
    if rank == 0:
        np.save(os.path.join(tmp, "Q_final.npy"), np.asarray(band.Q[0]))
        import pickle
        with open(os.path.join(tmp, "logs.pkl"), "wb") as fh:
            pickle.dump(logs, fh)
    dist.barrier()
    table.close(unlink=rank == 0)
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,policy", [("store", "quota"), ("shm", "quota"),
                                         ("store", "free"), ("shm", "free")])
def test_two_rank_lease_protocol_equals_serial_replay(tmp_path, kind, policy):
    import pickle

    import oracle
    from paper_2006_15980_b200.data import RatingMatrix, build_grid
    oracle.build()
    users, items, vals, P0, Q0 = _problem()
    for r in range(2):
        mm = np.memmap(tmp_path / f"q{r}.bin", dtype=np.float64, mode="w+", shape=(N_ITEMS, K))
        mm[:] = Q0
        mm.flush()
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), kind, policy), nprocs=2, join=True)
    logs = pickle.loads((tmp_path / "logs.pkl").read_bytes())
    row_cuts = np.array([0, 41, N_USERS])
    col_cuts = np.array([0, 14, 28, 42, 56, N_ITEMS])
    if policy == "quota":
        # every rank did every block of its band once per epoch
        for rank, (log, Pb, pulls, updates, counts) in enumerate(logs):
            assert counts == [EPOCHS] * 5
            assert len(log) == EPOCHS * 5
        assert sum(x[3] for x in logs) == EPOCHS * NNZ
    else:
        # POLICY_FREE: the job did world x n_cols block updates per epoch, by
        # whoever was free; a rank spreads its own updates over its columns
        # (least updated first)
        assert sum(sum(x[4]) for x in logs) == EPOCHS * 2 * 5
        for rank, (log, Pb, pulls, updates, counts) in enumerate(logs):
            assert len(log) == sum(counts)
            assert max(counts) - min(counts) <= 1 + max(counts) // 2
    assert sum(x[2] for x in logs) > 0, "no Q band ever moved between ranks"
    # serial replay in global lease order
    events = sorted((t, rank, c, s) for rank, (log, *_rest) in enumerate(logs) for t, c, s in log)
    m = RatingMatrix(N_USERS, N_ITEMS, users, items, vals)
    g = build_grid(m, row_cuts, col_cuts)
    P, Q = P0.copy(), Q0.copy()
    for _, rank, c, unit_seed in events:
        lo, hi = g.block_range(rank * 5 + c)
        oracle.sgd_range(P, Q, g.users, g.items, g.ratings, lo, hi, LR, REG, REG,
                         oracle.mix64(unit_seed, 0), 0, 0)
    got_P = np.concatenate([logs[0][1], logs[1][1]])
    assert np.array_equal(got_P, P)
    assert np.array_equal(np.load(tmp_path / "Q_final.npy"), Q)


def test_store_table_abort():
    """The portable (TCPStore) table aborts like the shared-memory one: the
    first abort wins and a blocked acquire raises LeaseAborted."""
    import datetime

    import torch.distributed as dist
    from paper_2006_15980_b200.distributed import LeaseAborted, LeaseTable, RowBandTrainer
    store = dist.TCPStore("127.0.0.1", _free_port(), 1, True,
                          timeout=datetime.timedelta(seconds=30))
    a = LeaseTable(store, 2, 0, "abort")
    a.initialize()
    b = LeaseTable(store, 2, 1, "abort")
    assert a.aborted_by() == -1
    assert a.try_acquire(0) and a.try_acquire(1)        # rank 0 holds everything
    b.abort()
    a.abort()                                           # the first abort wins
    assert a.aborted_by() == b.aborted_by() == 1

    class Band:
        n_cols = 2

    with pytest.raises(LeaseAborted, match="rank 1"):
        RowBandTrainer(Band(), b, 1)._grab({0, 1}, blocking=True)
