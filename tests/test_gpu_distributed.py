"""Multi-process GPU path on real device memory: 2 ranks (sharing one GPU when
only one is visible), Q bands exchanged by CUDA IPC peer copies, columns
leased through the store.  EXACT-mode kernels make the run deterministic
given the lease order, so it must equal the reference algorithm replayed
serially in that order, bit for bit (f32 storage, reference arithmetic)."""

import pickle
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("policy", ["quota", "free"])
def test_two_ranks_ipc_lease_protocol_equals_serial_replay(tmp_path, policy):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    sys.path.insert(0, str(ROOT / "tests"))
    import dist_gpu_worker as W
    from paper_2006_15980_b200.data import RatingMatrix, build_grid
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           str(ROOT / "tests" / "dist_gpu_worker.py"), str(tmp_path), "exact", policy]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res, Q_final, row_cuts, col_cuts = pickle.loads((tmp_path / "result.pkl").read_bytes())
    n_cols = len(col_cuts) - 1
    if policy == "quota":
        for log, Pb, counts in res:
            assert counts == [W.EPOCHS] * n_cols
    else:      # POLICY_FREE: world x n_cols block updates per epoch, job-wide
        assert sum(sum(c) for _l, _p, c in res) == W.EPOCHS * 2 * n_cols
    users, items, vals, P0, Q0 = W.problem()
    g = build_grid(RatingMatrix(W.N_USERS, W.N_ITEMS, users, items, vals), row_cuts, col_cuts)
    events = sorted((t, rank, c, s) for rank, (log, *_r) in enumerate(res) for t, c, s in log)
    P, Q = P0.copy(), Q0.copy()
    for _, rank, c, unit_seed in events:
        lo, hi = g.block_range(rank * n_cols + c)
        oracle.sgd_range(P, Q, g.users, g.items, g.ratings, lo, hi, W.LR, W.REG, W.REG,
                         oracle.mix64(unit_seed, 0), 0, 0)
    assert np.array_equal(np.concatenate([x[1] for x in res]), P)
    assert np.array_equal(Q_final, Q)


@pytest.mark.parametrize("layout", ["qband", "qband8"], ids=["auto", "run_groups"])
@pytest.mark.parametrize("stage", [False, True], ids=["resident", "host_staged"])
def test_two_ranks_qband_path_applies_every_triple(tmp_path, stage, layout):
    """The default multi-GPU kernel path (Q-band layout of each rank's band,
    narrow column bands split over the chains) on conflict-free triples:
    order-free, so after the epochs P and Q equal the reference update of
    every triple once per epoch (oracle, f64) within fp32 rounding — with the
    triples resident, and uploaded from pinned host memory per lease (the
    N>1 e2e path, CudaRowBand.stage_from_host)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    sys.path.insert(0, str(ROOT / "tests"))
    import dist_gpu_worker as W
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           str(ROOT / "tests" / "dist_gpu_worker.py"), str(tmp_path), layout]
    if stage:
        cmd.append("stage")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res, Q_final, row_cuts, col_cuts = pickle.loads((tmp_path / "result.pkl").read_bytes())
    for log, Pb, counts in res:
        assert counts == [W.EPOCHS] * (len(col_cuts) - 1)
    if stage:
        # the compact 6-byte stream (uint16 tile-relative ids, implicit items) ran
        assert (tmp_path / "staged.txt").read_text() == "compact"
    users, items, vals, P0, Q0 = W.problem(conflict_free=True)
    P, Q = P0.astype(np.float64), Q0.astype(np.float64)
    for e in range(W.EPOCHS):
        oracle.sgd_range(P, Q, users, items, vals, 0, len(users), W.LR, W.REG, W.REG, e, 0, 0)
    got_P = np.concatenate([x[1] for x in res]).astype(np.float64)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    assert rel(got_P, P) < 1e-5
    assert rel(Q_final.astype(np.float64), Q) < 1e-5
