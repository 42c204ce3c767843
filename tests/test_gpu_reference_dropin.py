"""The drop-in, proven against the unmodified reference (B200).

The reference package (`hetmf`, installed under oracle/_ref by
oracle/reference.py) runs its OWN training driver — run_training, its
GridScheduler, its BatchWorker lease loop (engine.py:190-268,
workers.py:305-369) — with one seam swapped for the B200 build, exactly the
binding INTEGRATION.md shows a maintainer adding:

* `hetmf.kernels.sgd_range` -> `paper_2006_15980_b200.kernels.sgd_range`
  (the C-ABI kernel on the reference's numpy buffers; the reference's four
  BatchEngine lanes call it concurrently on the same staged buffers);
* `hetmf.workers.BatchEngine` -> `paper_2006_15980_b200.workers.BatchEngine`
  (device-resident factors, CUDA staging, the Q-band kernel).

Both must train ML-1M-shaped data (k = 32, 20 epochs) to the reference's own
test RMSE within 0.005 (north star; tests/golden/training.json holds the
reference's stream-only trajectory on the same split).  The reference's
single-update pins (tests/test_sgd.py:91-113) run through sgd.sgd_update.
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hetmf():
    from oracle import reference
    if not reference.installed():
        pytest.skip("reference not installed under oracle/_ref (__graft_entry__.build())")
    return reference.hetmf()


@pytest.fixture(scope="module")
def ml1m(hetmf):
    """The golden split (tests/golden/make_golden.py training_cases)."""
    full = hetmf.synthetic_ratings(6040, 3706, rank=8, density=1.05e6 / (6040 * 3706),
                                   noise=0.1, seed=0)
    perm = np.random.default_rng(1).permutation(full.nnz)
    n_test = full.nnz // 21
    te, tr = perm[:n_test], perm[n_test:]
    M = hetmf.RatingMatrix
    train = M(full.n_users, full.n_items, full.users[tr], full.items[tr], full.ratings[tr])
    test = M(full.n_users, full.n_items, full.users[te], full.items[te], full.ratings[te])
    return train, test


def _ref_config(hetmf, epochs):
    return hetmf.RunConfig(schedule="batch-only", n_stream=0, n_batch=1, n_factors=32,
                           learning_rate=0.01, reg_user=0.01, reg_item=0.01, epochs=epochs,
                           seed=0, batch_overhead_ms=0.0, batch_bandwidth_mb=1e9,
                           log_train_loss=False)


def _golden_rmse(label):
    return json.loads((GOLDEN / "training.json").read_text())[label]["test_rmse"]


def test_reference_run_training_with_b200_sgd_range(hetmf, ml1m, monkeypatch):
    from paper_2006_15980_b200 import kernels as ours
    import hetmf.workers as ref_workers
    calls = {"n": 0}

    def sgd_range(*args):
        calls["n"] += 1
        return ours.sgd_range(*args)

    monkeypatch.setattr(ref_workers.kernels, "sgd_range", sgd_range)
    train, test = ml1m
    res = hetmf.run_training(_ref_config(hetmf, 20), matrix=train)
    got = hetmf.rmse(test, res.model).value
    assert calls["n"] > 0 and res.scheduler.total_updates == 20 * train.nnz
    assert abs(got - _golden_rmse("e20")) <= 0.005, (got, _golden_rmse("e20"))


def test_reference_run_training_with_b200_engine(hetmf, ml1m, monkeypatch):
    from paper_2006_15980_b200 import workers as ours
    import hetmf.workers as ref_workers
    made = []

    class Engine(ours.BatchEngine):
        def __init__(self, *a, **kw):
            super().__init__(*a, **kw)
            made.append(self)

    monkeypatch.setattr(ref_workers, "BatchEngine", Engine)
    train, test = ml1m
    for epochs, label in ((1, "e1"), (20, "e20")):
        res = hetmf.run_training(_ref_config(hetmf, epochs), matrix=train)
        got = hetmf.rmse(test, res.model).value
        assert res.scheduler.total_updates == epochs * train.nnz
        assert abs(got - _golden_rmse(label)) <= 0.005, (label, got, _golden_rmse(label))
    assert made and all(isinstance(e, ours.BatchEngine) for e in made)


def test_reference_sgd_update_pins(hetmf):
    """tests/test_sgd.py:91-98 and :100-113 of the reference, through the
    B200 sgd_update (EXACT mode on the device), and against the reference's
    own sgd_update on the same inputs."""
    from paper_2006_15980_b200 import sgd
    m = sgd.FactorModel(np.array([[1.0]]), np.array([[1.0]]))
    tr = sgd.sgd_update(m, 0, 0, 2.0, sgd.Hyperparams(1, 0.0, 0.0, 0.1))
    assert tr.residual == pytest.approx(1.0)
    assert m.user_factors[0, 0] == pytest.approx(1.1)
    assert m.item_factors[0, 0] == pytest.approx(1.1)
    rng = np.random.default_rng(4)
    for _ in range(20):
        p, q, r = rng.normal(size=2), rng.normal(size=2), float(rng.normal())
        lr, ru, ri = 0.05, 0.02, 0.03
        e = r - float(p @ q)
        exp_p, exp_q = p + lr * (e * q - ru * p), q + lr * (e * p - ri * q)
        ours = sgd.FactorModel(p.reshape(1, -1).copy(), q.reshape(1, -1).copy())
        t = sgd.sgd_update(ours, 0, 0, r, sgd.Hyperparams(2, ru, ri, lr))
        assert t.residual == pytest.approx(e, rel=1e-12)
        assert ours.user_factors[0] == pytest.approx(exp_p, rel=1e-12)
        assert ours.item_factors[0] == pytest.approx(exp_q, rel=1e-12)
        ref = hetmf.FactorModel(p.reshape(1, -1).copy(), q.reshape(1, -1).copy())
        hetmf.sgd_update(ref, 0, 0, r, hetmf.Hyperparams(2, ru, ri, lr))
        # the reference's own kernel-vs-sgd_update pin is rtol 1e-15
        # (tests/test_sgd.py:195-205)
        np.testing.assert_allclose(ours.user_factors, ref.user_factors, rtol=1e-15, atol=0)
        np.testing.assert_allclose(ours.item_factors, ref.item_factors, rtol=1e-15, atol=0)
