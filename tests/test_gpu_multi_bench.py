"""N > 1 runs on ONE matrix, gated against the 1-rank run (B200).

* data.synthetic_band: the bands of any row partition are exactly the pieces
  of the whole matrix — same cells, same values, same held-out cells — so N
  ranks each generating their own band train on the matrix one GPU trains on.
* `python bench.py --gpus 2 --workload yahoo --scaling strong` (two ranks on
  the box's GPU, self-launched, CUDA IPC between them) reports a test RMSE
  within 0.005 of `python bench.py --gpus 1 --workload yahoo` after the same
  epochs, on the same training and test sets (north star: test RMSE within
  0.005; reference lease protocol scheduler.py:333-409, uniform g x (g+1)
  plan partition.py:89-107).
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _cells(t):
    u = t.users.cpu().numpy().astype(np.int64)
    i = t.items.cpu().numpy().astype(np.int64)
    r = t.ratings.cpu().numpy()
    order = np.argsort(u * 1_000_003 + i, kind="stable")
    return u[order], i[order], r[order]


@pytest.mark.parametrize("cuts", [[0, 7000], [0, 2500, 7000], [0, 1, 3333, 5000, 7000]])
def test_synthetic_bands_are_pieces_of_one_matrix(cuts):
    from paper_2006_15980_b200.data import synthetic_band
    d = torch.device("cuda", 0)
    n_users, n_items, nnz = 7000, 900, 400_000
    whole_tr, whole_te = synthetic_band(n_users, n_items, nnz, seed=4, device=d)
    parts = [synthetic_band(n_users, n_items, nnz, lo, hi, seed=4, device=d)
             for lo, hi in zip(cuts, cuts[1:])]
    for which in (0, 1):
        whole = _cells((whole_tr, whole_te)[which])
        got = [_cells(p[which]) for p in parts]
        got = tuple(np.concatenate([g[j] for g in got]) for j in range(3))
        order = np.argsort(got[0] * 1_000_003 + got[1], kind="stable")
        for j in range(3):
            assert np.array_equal(got[j][order], whole[j])
    n_tr, n_te = whole_tr.nnz, whole_te.nnz
    assert abs(n_tr + n_te - nnz) < 6 * np.sqrt(nnz)          # Bernoulli count
    assert abs(n_te / (n_tr + n_te) - 0.05) < 0.005
    # every band's users are global ids inside the band
    for (lo, hi), (tr, te) in zip(zip(cuts, cuts[1:]), parts):
        for t in (tr, te):
            if t.nnz:
                assert int(t.users.min()) >= lo and int(t.users.max()) < hi
    # the law: mean rating ~ rank * (1/(2 sqrt 8))^2 * ... as the reference's (data.py:311-336)
    r = whole_tr.ratings.double()
    assert 0.2 < float(r.mean()) < 0.3 and 0.1 < float(r.std()) < 0.16


def _bench(*args, timeout=900):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return lines[0], out.stderr


def test_two_ranks_strong_yahoo_matches_one_rank_rmse():
    common = ["--workload", "yahoo", "--steps", "4", "--warmup", "3", "--no-e2e", "--no-cpu"]
    one, _ = _bench("--gpus", "1", *common)
    two, err = _bench("--gpus", "2", "--scaling", "strong", *common)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    # the same matrix: same training and test cells
    assert two["counts"]["train_ratings"] == one["counts"]["train_ratings"]
    assert two["counts"]["test_ratings"] == one["counts"]["test_ratings"]
    assert one["rmse"]["epochs"] == two["rmse"]["epochs"] == 7
    assert abs(two["rmse"]["test"] - one["rmse"]["test"]) <= 0.005, (one["rmse"], two["rmse"])
    assert two["value"] > 0 and two["gpu_launches"] == 2 * 5 * 4   # 2 ranks x 5 columns x steps
    # leases through the node-local table: a few atomics per lease, a
    # negligible share of the step (the TCPStore cost was unmeasured)
    assert two["leases"]["table"] == "shm"
    assert two["leases"]["share_of_step_max_rank"] < 0.02, two["leases"]
