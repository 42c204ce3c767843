"""Host logic on CPU: division plans, the lease scheduler and the cost model,
checked against the reference's own outputs (tests/golden/) and the
reference test suite's properties (tests/test_partition.py,
test_scheduler.py, test_costmodel.py in the reference)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN

from paper_2006_15980_b200.costmodel import (FAMILY_LINEAR, FAMILY_LOG, FAMILY_SQRT_LOG,
                                             CalibrationProfile, CalibrationSample,
                                             DeviceTopology, PiecewiseCostModel,
                                             detect_threshold, fit_linear, fit_piecewise,
                                             gpu_shares, load_profile, predicted_makespan,
                                             save_profile, solve_alpha)
from paper_2006_15980_b200.data import RatingMatrix, build_grid
from paper_2006_15980_b200.partition import (gpu_plan, nonuniform_plan, uniform_plan,
                                             validate_plan)
from paper_2006_15980_b200.scheduler import (CLASS_BATCH, CLASS_STREAM, POLICY_FREE,
                                             POLICY_QUOTA, POLICY_REGIONS, GridScheduler)


@pytest.fixture(scope="module")
def meta():
    return json.loads((GOLDEN / "golden.json").read_text())


# -- plans ---------------------------------------------------------------------
def test_plans_match_reference(meta):
    mm = np.load(GOLDEN / "plan_matrix.npz")
    shape = meta["plans"]["matrix"]
    m = RatingMatrix(shape["n_users"], shape["n_items"], mm["users"], mm["items"],
                     np.zeros(len(mm["users"])))
    for case in meta["plans"]["cases"]:
        topo = DeviceTopology(case["n_stream"], case["n_batch"])
        if case["kind"] == "uniform":
            p = uniform_plan(topo, shape=(m.n_users, m.n_items))
        else:
            p = nonuniform_plan(topo, case["alpha"], m)
            assert p.region_of_row.tolist() == case["region_of_row"]
            assert p.sub_row_parent.tolist() == case["sub_row_parent"]
            assert p.region_boundary_row == case["boundary"]
        assert p.row_cuts.tolist() == case["row_cuts"], case
        assert p.col_cuts.tolist() == case["col_cuts"], case
        assert validate_plan(p, topo) == []


def test_uniform_rule_1():
    p = uniform_plan(DeviceTopology(16, 1))
    assert (p.row_band_count, p.col_count) == (17, 18)


def test_gpu_plan_shares_and_validation():
    rng = np.random.default_rng(0)
    m = RatingMatrix(1000, 400, rng.integers(0, 1000, 50_000).astype(np.int32),
                     rng.integers(0, 400, 50_000).astype(np.int32), np.zeros(50_000))
    p = gpu_plan(4, m, shares=[1, 1, 2, 4])
    assert validate_plan(p, DeviceTopology(0, 4)) == []
    assert p.col_count == 9 and len(p.row_cuts) == 5
    mass = np.diff(np.searchsorted(np.sort(m.users), p.row_cuts))
    assert mass[3] / mass[0] == pytest.approx(4.0, rel=0.05)
    with pytest.raises(ValueError):
        gpu_plan(2, m, shares=[1, 0])


# -- scheduler: the reference's lease sequence ------------------------------------
def _replay(policy, grid, classes, seed, steps, rng_seed, prefetch=True):
    sched = GridScheduler(grid, policy, max_epochs=10 ** 6, seed=seed, batch_prefetch=prefetch)
    rng = np.random.default_rng(rng_seed)
    held, events = {}, []
    for _ in range(steps):
        if held and rng.random() < 0.5:
            wid = sorted(held)[int(rng.integers(len(held)))]
            nxt = sched.release(held.pop(wid), 1)
            events.append(["release", wid])
            if nxt is not None:
                held[wid] = nxt
                events.append(["promote", wid, list(nxt.unit.blocks), nxt.unit.order_seed,
                               list(nxt.prefetch.blocks) if nxt.prefetch else None])
        else:
            free = [w for w in sorted(classes) if w not in held]
            if free:
                wid = free[int(rng.integers(len(free)))]
                lease = sched.acquire(wid, classes[wid], blocking=False)
                if lease is not None:
                    held[wid] = lease
                    events.append(["grant", wid, list(lease.unit.blocks), lease.unit.order_seed,
                                   list(lease.prefetch.blocks) if lease.prefetch else None])
                else:
                    events.append(["none", wid])
    return dict(events=events, counts=sched.counts.tolist(), epoch=sched.epoch, phase=sched.phase)


def test_scheduler_matches_reference_lease_sequences(meta):
    sm = np.load(GOLDEN / "sched_matrix.npz")
    m = RatingMatrix(150, 150, sm["users"], sm["items"], sm["ratings"])
    g = build_grid(m, np.linspace(0, 150, 4, dtype=int), np.linspace(0, 150, 5, dtype=int))
    gold = meta["scheduler"]
    got = _replay(POLICY_QUOTA, g, {0: CLASS_BATCH, 1: CLASS_BATCH, 2: CLASS_BATCH}, 5, 400, 6)
    assert got == gold["quota_3x4"]
    got = _replay(POLICY_FREE, g, {0: CLASS_STREAM, 1: CLASS_STREAM}, 7, 300, 8)
    assert got == gold["free_3x4"]
    geo = gold["regions_geometry"]
    g2 = build_grid(m, geo["row_cuts"], geo["col_cuts"], geo["region_of_row"], geo["sub_row_parent"])
    got = _replay(POLICY_REGIONS, g2, {0: CLASS_STREAM, 1: CLASS_STREAM, 2: CLASS_STREAM,
                                        3: CLASS_BATCH}, 32, 600, 33)
    assert got == gold["regions_3p1"]


def _conflicts(leases):
    """Independent check: live units of different workers share no band."""
    seen_rows, seen_cols = {}, {}
    for lease in leases:
        units = [lease.unit] + ([lease.prefetch] if lease.prefetch else [])
        for u in units:
            for r in u.rows:
                if seen_rows.setdefault(r, lease.worker) != lease.worker:
                    return True
            if seen_cols.setdefault(u.col, lease.worker) != lease.worker:
                return True
    return False


def test_scheduler_conflict_free_under_random_interleavings():
    rng = np.random.default_rng(1)
    m = RatingMatrix(120, 120, rng.integers(0, 120, 5000).astype(np.int32),
                     rng.integers(0, 120, 5000).astype(np.int32), np.zeros(5000))
    p = gpu_plan(4, m)
    g = build_grid(m, p.row_cuts, p.col_cuts, p.region_of_row, p.sub_row_parent)
    sched = GridScheduler(g, POLICY_QUOTA, max_epochs=10 ** 9, seed=2)
    held = {}
    for _ in range(4000):
        if held and rng.random() < 0.5:
            wid = int(rng.choice(list(held)))
            nxt = sched.release(held.pop(wid), 1)
            if nxt is not None:
                held[wid] = nxt
        else:
            free = [w for w in range(4) if w not in held]
            if free:
                wid = int(rng.choice(free))
                lease = sched.acquire(wid, CLASS_BATCH, blocking=False)
                if lease is not None:
                    held[wid] = lease
        assert not _conflicts(held.values())
    assert sched.counts.max() - sched.counts.min() <= 1


def test_quota_epochs_count_every_block_once():
    rng = np.random.default_rng(3)
    m = RatingMatrix(60, 60, rng.integers(0, 60, 900).astype(np.int32),
                     rng.integers(0, 60, 900).astype(np.int32), np.zeros(900))
    g = build_grid(m, [0, 20, 40, 60], [0, 15, 30, 45, 60])
    sched = GridScheduler(g, POLICY_QUOTA, max_epochs=3, seed=1)
    while True:
        lease = sched.acquire(0, CLASS_BATCH, blocking=False)
        if lease is None:
            break
        while lease is not None:
            lease = sched.release(lease, 1)
    assert sched.epoch == 3 and sched.terminated
    assert np.all(sched.counts == 3)


# -- cost model ----------------------------------------------------------------------
def _samples(sizes, fn):
    return [CalibrationSample(int(s), float(fn(s))) for s in sizes]


def test_fit_linear_exact():
    a2, b2 = fit_linear(_samples([1000, 2000, 4000, 8000], lambda s: 2e-6 * s + 1e-3))
    assert a2 == pytest.approx(2e-6) and b2 == pytest.approx(1e-3)


def test_detect_threshold_two_percent_rule():
    sizes = [1000, 2000, 4000, 8000, 16000, 32000]
    speeds = [1e5, 2e5, 3e5, 3.02e5, 3.03e5, 3.04e5]
    s = [CalibrationSample(n, n / v) for n, v in zip(sizes, speeds)]
    assert detect_threshold(s) == 4000


def test_fit_piecewise_recovers_log_regime():
    sizes = [2 ** i * 1000 for i in range(10)]

    def elapsed(n):
        plateau = 2 ** 6 * 1000
        speed = 1e5 * np.log(min(n, plateau)) - 3e5
        return n / speed
    m = fit_piecewise(_samples(sizes, elapsed), FAMILY_LOG)
    assert m.family == FAMILY_LOG
    for n in (3000, 50_000, 300_000):
        assert m.eval(n) == pytest.approx(elapsed(n), rel=0.05)


def test_solve_alpha_closed_forms():
    lin = lambda a: PiecewiseCostModel(family=FAMILY_LINEAR, a2=a, b2=0.0)  # noqa: E731
    prof = CalibrationProfile(stream=lin(3e-6), transfer_in=lin(1e-7), transfer_out=lin(1e-7),
                              kernel=lin(1e-6))
    # equal devices, batch 3x faster: alpha = 3/4
    a = solve_alpha(prof, DeviceTopology(1, 1), 10 ** 6)
    assert a == pytest.approx(0.75, abs=0.005)
    # 2 stream workers vs 1 batch worker with the same speed ratio: alpha = 3/5
    a = solve_alpha(prof, DeviceTopology(2, 1), 10 ** 6)
    assert a == pytest.approx(0.6, abs=0.005)
    assert solve_alpha(prof, DeviceTopology(0, 4), 10 ** 6) == 1.0
    mk = predicted_makespan(prof, DeviceTopology(1, 1), 10 ** 6, 0.75)
    assert mk == pytest.approx(0.75, rel=0.01)


def test_profile_round_trip(tmp_path):
    prof = CalibrationProfile(
        stream=PiecewiseCostModel(family=FAMILY_LINEAR, a2=1e-6, b2=1e-4),
        transfer_in=PiecewiseCostModel(family=FAMILY_SQRT_LOG, a1=1.0, b1=2.0, plateau=100,
                                       a2=3e-9, b2=4e-5, floor=10),
        transfer_out=PiecewiseCostModel(family=FAMILY_LINEAR, a2=1e-9, b2=1e-5),
        kernel=PiecewiseCostModel(family=FAMILY_LOG, a1=5.0, b1=6.0, plateau=1000, a2=7e-10,
                                  b2=8e-6, floor=100),
        fingerprint={"n_stream": 0, "n_batch": 2, "device": "NVIDIA_B200"})
    save_profile(tmp_path / "p.txt", prof)
    back = load_profile(tmp_path / "p.txt", DeviceTopology(0, 2))
    assert back.kernel == prof.kernel and back.transfer_in == prof.transfer_in
    assert back.fingerprint == prof.fingerprint and not back.stale
    assert load_profile(tmp_path / "p.txt", DeviceTopology(0, 3)).stale


def test_gpu_shares_homogeneous_and_skewed():
    fast = PiecewiseCostModel(family=FAMILY_LINEAR, a2=1e-9, b2=0.0)
    slow = PiecewiseCostModel(family=FAMILY_LINEAR, a2=2e-9, b2=0.0)
    assert np.allclose(gpu_shares([fast] * 4, 1e6), 0.25)
    s = gpu_shares([fast, slow], 1e6)
    assert s[0] == pytest.approx(2 / 3)
