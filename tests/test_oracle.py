"""The CPU oracle against the reference's own outputs (tests/golden/).

Pins oracle/hmf_oracle.c bit for bit to hetmf (the vectors were produced by
tests/golden/make_golden.py from the unmodified reference), so the GPU parity
tests can use the oracle as the checker at sizes no fixture covers.
"""

import json

import numpy as np
import pytest

import oracle
from conftest import GOLDEN


@pytest.fixture(scope="module", autouse=True)
def built():
    oracle.build()


def test_mix64_matches_reference():
    meta = json.loads((GOLDEN / "golden.json").read_text())["mix64"]
    for parts, value in zip(meta["parts"], meta["values"]):
        assert oracle.mix64(*parts) == value


def test_visit_order_matches_reference():
    orders = np.load(GOLDEN / "visit_order.npz")
    for key in orders.files:
        n = int(key.split("_")[0][1:])
        seed = int(key.split("_s")[1])
        assert np.array_equal(oracle.visit_order(n, seed), orders[key]), key


def test_visit_order_is_a_permutation_in_windows():
    perm = oracle.visit_order(10_000, 3)
    assert np.array_equal(np.sort(perm), np.arange(10_000))
    # every block of consecutive updates of a full window stays inside one window
    w = perm[:4096] // 4096
    assert len(np.unique(w)) == 1 or len(np.unique(perm[:4096 - (10_000 % 4096)] // 4096)) == 1


def test_sgd_range_bitwise(golden_sgd):
    for name, c in golden_sgd.items():
        P, Q = c["P0"].copy(), c["Q0"].copy()
        start, stop, seed, rb, cb, got = (int(x) for x in c["meta"])
        lr, ru, ri = c["hyper"]
        n = oracle.sgd_range(P, Q, c["rows"], c["cols"], c["vals"], start, stop, lr, ru, ri,
                             seed, rb, cb)
        assert n == got, name
        assert np.array_equal(P, c["P1"]), name
        assert np.array_equal(Q, c["Q1"]), name


def test_sgd_range_empty_range_is_noop():
    P = np.ones((2, 3))
    Q = np.ones((2, 3))
    z = np.zeros(2, np.int32)
    assert oracle.sgd_range(P, Q, z, z, np.ones(2), 1, 1, 0.1, 0, 0, 1, 0, 0) == 0
    assert np.all(P == 1) and np.all(Q == 1)


def test_residual_sums_match_reference_metrics():
    m = np.load(GOLDEN / "metrics.npz")
    sq, pp, qq = oracle.residual_sums(m["P"], m["Q"], m["rows"], m["cols"], m["vals"])
    n = len(m["vals"])
    assert np.sqrt(sq / n) == pytest.approx(float(m["rmse"][0]), rel=1e-12)
    assert sq + 0.3 * pp + 0.7 * qq == pytest.approx(float(m["loss"][0]), rel=1e-12)


def test_stream_train_matches_serial_replay():
    """Two threads on a 2x3 grid equal a serial replay of the recorded lease
    order: disjoint blocks commute (reference tests/test_workers.py:43-70)."""
    from conftest import random_matrix
    from paper_2006_15980_b200.data import build_grid
    m = random_matrix(60, 60, 1200, 2)
    g = build_grid(m, [0, 30, 60], [0, 20, 40, 60])
    rng = np.random.default_rng(2)
    P = rng.uniform(0, 0.5, size=(60, 4))
    Q = rng.uniform(0, 0.5, size=(60, 4))
    P1, Q1 = P.copy(), Q.copy()
    got, counts, order = oracle.stream_train(P1, Q1, g.users, g.items, g.ratings, g.block_ptr,
                                             2, 3, 0.02, 0.01, 0.01, 7, 3, 2, trace=True)
    assert got == 3 * m.nnz
    assert np.all(counts == 3)
    P2, Q2 = P.copy(), Q.copy()
    seen = np.zeros(6, dtype=np.int64)
    for b in order:
        lo, hi = g.block_range(int(b))
        unit = oracle.mix64(7, int(b), int(seen[b]))
        oracle.sgd_range(P2, Q2, g.users, g.items, g.ratings, lo, hi, 0.02, 0.01, 0.01,
                         oracle.mix64(unit, 0), 0, 0)
        seen[b] += 1
    assert np.array_equal(P1, P2) and np.array_equal(Q1, Q2)
