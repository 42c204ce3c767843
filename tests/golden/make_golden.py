"""Generate the golden fixtures in tests/golden/ from the reference itself.

Run in the dev container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the unmodified reference package (hetmf, /root/reference/pkg/src)
and records its outputs on small seeded inputs.  The fixtures are committed;
the GPU box never needs /root/reference.  Everything here is the reference's
behaviour, captured: nothing in this script reimplements the algorithm.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = os.environ.get("HMF_REFERENCE_SRC", "/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF_SRC)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from hetmf import kernels  # noqa: E402
from hetmf.costmodel import DeviceTopology  # noqa: E402
from hetmf.data import (RatingMatrix, build_grid, shuffle_triples,  # noqa: E402
                        synthetic_ratings)
from hetmf.engine import RunConfig, run_training  # noqa: E402
from hetmf.partition import nonuniform_plan, uniform_plan  # noqa: E402
from hetmf.scheduler import (CLASS_BATCH, CLASS_STREAM, POLICY_FREE,  # noqa: E402
                             POLICY_QUOTA, POLICY_REGIONS, GridScheduler)
from hetmf.sgd import (FactorModel, Hyperparams, init_model,  # noqa: E402
                       regularized_loss, rmse)


def random_matrix(n_users, n_items, nnz, seed, lo=1.0, hi=5.0):
    # same construction as the reference tests' conftest.random_matrix
    rng = np.random.default_rng(seed)
    chosen = rng.permutation(n_users * n_items)[:nnz]
    return RatingMatrix(n_users, n_items, (chosen // n_items).astype(np.int32),
                        (chosen % n_items).astype(np.int32), rng.uniform(lo, hi, size=nnz))


def mix64_cases():
    cases = [(0,), (1,), (0, 0), (7, 3, 1), (2 ** 63 - 1, 5), (123456789, 42, 17, 3),
             (2, 11, 0), (9, 1), (0xC0, 2 ** 40)]
    return {"parts": [list(c) for c in cases], "values": [kernels.mix64(*c) for c in cases]}


def visit_order(n, seed):
    """Recover sgd_range's visit order from its own output.

    Triple i has its own row i and all triples share item 0.  With p_i = 1,
    q = 10, r = 1, lr = 1, reg_user = 0, reg_item = -1 the item value before
    the t-th update is exactly 10 + t, and row i ends at 1 - (9+t)(10+t), so
    the position t of every triple is read back exactly (integers < 2^53)."""
    user_f = np.ones((n, 1))
    item_f = np.full((1, 1), 10.0)
    rows = np.arange(n, dtype=np.int32)
    cols = np.zeros(n, dtype=np.int32)
    vals = np.ones(n)
    kernels.sgd_range(user_f, item_f, rows, cols, vals, 0, n, 1.0, 0.0, -1.0, seed, 0, 0)
    p = user_f[:, 0]
    # solve (9+t)(10+t) = 1 - p for t >= 0
    c = 1.0 - p
    t = np.rint((-19.0 + np.sqrt(1.0 + 4.0 * c)) / 2.0).astype(np.int64)
    assert np.array_equal(np.sort(t), np.arange(n)), "order recovery failed"
    perm = np.empty(n, dtype=np.int64)
    perm[t] = np.arange(n)
    return perm


def sgd_cases():
    """sgd_range on random inputs: f64 and f32 arrays, offsets and bases."""
    out = {}
    specs = [
        # name, n_users, n_items, nnz, k, start, stop, seed, dtype, row_base, col_base, lr, reg
        ("tiny_k1", 4, 4, 1, 1, 0, 1, 77, np.float64, 0, 0, 0.1, 0.02),
        ("k2_30", 12, 12, 30, 2, 0, 30, 99, np.float64, 0, 0, 0.05, 0.01),
        ("k3_offset", 20, 20, 120, 3, 17, 101, 1001, np.float64, 0, 0, 0.02, 0.01),
        ("k8_5000", 300, 200, 5000, 8, 0, 5000, 12345, np.float64, 0, 0, 0.01, 0.05),
        ("k16_9753", 400, 300, 9753, 16, 3, 9753, 2 ** 40 + 7, np.float64, 0, 0, 0.005, 0.05),
        ("k32_staged", 500, 400, 6000, 32, 0, 6000, 31337, np.float64, 100, 50, 0.01, 0.02),
        ("k128_2000", 300, 200, 2000, 128, 0, 2000, 555, np.float64, 0, 0, 0.005, 0.05),
        ("f32_k32", 500, 400, 6000, 32, 5, 5990, 4242, np.float32, 0, 0, 0.01, 0.02),
        ("f32_k128", 300, 200, 3000, 128, 0, 3000, 777, np.float32, 0, 0, 0.005, 0.05),
        ("f32_k5_staged", 60, 50, 900, 5, 0, 900, 8, np.float32, 10, 20, 0.02, 0.01),
    ]
    for (name, nu, ni, nnz, k, start, stop, seed, dt, rb, cb, lr, reg) in specs:
        m = random_matrix(nu, ni, nnz, seed % 1000)
        rng = np.random.default_rng(seed % 997)
        if rb or cb:
            # staged sub-buffers: triples restricted to rows >= rb, cols >= cb
            keep = (m.users >= rb) & (m.items >= cb)
            m = RatingMatrix(nu, ni, m.users[keep], m.items[keep], m.ratings[keep])
            stop = min(stop, m.nnz)
            P = rng.uniform(0, 1 / np.sqrt(k), size=(nu - rb, k)).astype(dt)
            Q = rng.uniform(0, 1 / np.sqrt(k), size=(ni - cb, k)).astype(dt)
        else:
            P = rng.uniform(0, 1 / np.sqrt(k), size=(nu, k)).astype(dt)
            Q = rng.uniform(0, 1 / np.sqrt(k), size=(ni, k)).astype(dt)
        vals = m.ratings / 5.0
        if dt == np.float32:
            vals = vals.astype(np.float32).astype(np.float64)  # f32-representable ratings
        P0, Q0 = P.copy(), Q.copy()
        got = kernels.sgd_range(P, Q, m.users, m.items, vals, start, stop, lr, reg, reg * 1.5,
                                seed, rb, cb)
        out[name] = dict(P0=P0, Q0=Q0, P1=P, Q1=Q, rows=m.users, cols=m.items, vals=vals,
                         meta=np.array([start, stop, seed, rb, cb, got], dtype=np.int64),
                         hyper=np.array([lr, reg, reg * 1.5]))
    return out


def metric_cases():
    rng = np.random.default_rng(19)
    m = random_matrix(40, 30, 500, 20)
    model = FactorModel(rng.normal(size=(40, 6)), rng.normal(size=(30, 6)))
    return dict(rows=m.users, cols=m.items, vals=m.ratings, P=model.user_factors,
                Q=model.item_factors,
                rmse=np.array([rmse(m, model).value]),
                loss=np.array([regularized_loss(m, model, 0.3, 0.7)]))


def plan_cases():
    cases = []
    m = shuffle_triples(synthetic_ratings(300, 280, rank=4, density=0.2, noise=0.1, seed=9), 9)
    for ns, nb in [(1, 0), (0, 1), (0, 2), (0, 4), (0, 8), (3, 0), (4, 2)]:
        p = uniform_plan(DeviceTopology(ns, nb), shape=(m.n_users, m.n_items))
        cases.append(dict(kind="uniform", n_stream=ns, n_batch=nb,
                          row_cuts=p.row_cuts.tolist(), col_cuts=p.col_cuts.tolist()))
    for ns, nb, alpha in [(2, 1, 0.4), (1, 1, 0.5), (4, 2, 0.3), (1, 8, 0.9), (3, 1, 0.25)]:
        p = nonuniform_plan(DeviceTopology(ns, nb), alpha, m)
        cases.append(dict(kind="nonuniform", n_stream=ns, n_batch=nb, alpha=alpha,
                          row_cuts=p.row_cuts.tolist(), col_cuts=p.col_cuts.tolist(),
                          region_of_row=p.region_of_row.tolist(),
                          sub_row_parent=p.sub_row_parent.tolist(),
                          boundary=int(p.region_boundary_row)))
    return dict(matrix=dict(n_users=m.n_users, n_items=m.n_items), cases=cases,
                users=m.users, items=m.items)


def scheduler_trace(policy, grid, classes, seed, steps, rng_seed, prefetch=True):
    sched = GridScheduler(grid, policy, max_epochs=10 ** 6, seed=seed, batch_prefetch=prefetch)
    rng = np.random.default_rng(rng_seed)
    held = {}
    events = []
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
    return dict(events=events, counts=sched.counts.tolist(), epoch=sched.epoch,
                phase=sched.phase)


def scheduler_cases():
    m = shuffle_triples(synthetic_ratings(150, 150, rank=4, density=0.2, noise=0.1, seed=31), 31)
    out = {}
    g = build_grid(m, np.linspace(0, 150, 4, dtype=int), np.linspace(0, 150, 5, dtype=int))
    out["quota_3x4"] = scheduler_trace(POLICY_QUOTA, g, {0: CLASS_BATCH, 1: CLASS_BATCH,
                                                         2: CLASS_BATCH}, 5, 400, 6)
    out["free_3x4"] = scheduler_trace(POLICY_FREE, g, {0: CLASS_STREAM, 1: CLASS_STREAM}, 7, 300, 8)
    plan = nonuniform_plan(DeviceTopology(3, 1), 0.4, m)
    g2 = build_grid(m, plan.row_cuts, plan.col_cuts, plan.region_of_row, plan.sub_row_parent)
    out["regions_3p1"] = scheduler_trace(POLICY_REGIONS, g2, {0: CLASS_STREAM, 1: CLASS_STREAM,
                                                              2: CLASS_STREAM, 3: CLASS_BATCH},
                                         32, 600, 33)
    out["regions_geometry"] = dict(row_cuts=plan.row_cuts.tolist(), col_cuts=plan.col_cuts.tolist(),
                                   region_of_row=plan.region_of_row.tolist(),
                                   sub_row_parent=plan.sub_row_parent.tolist())
    return out, m


def data_cases():
    s = synthetic_ratings(60, 50, rank=4, density=0.2, noise=0.1, seed=3)
    sh = shuffle_triples(s, 11)
    g = build_grid(sh, [0, 20, 60], [0, 10, 30, 50])
    init = init_model(7, 5, Hyperparams(n_factors=3), 4)
    return dict(syn_users=s.users, syn_items=s.items, syn_ratings=s.ratings,
                sh_users=sh.users, sh_items=sh.items, sh_ratings=sh.ratings,
                g_users=g.users, g_items=g.items, g_ratings=g.ratings, g_ptr=g.block_ptr,
                init_P=init.user_factors, init_Q=init.item_factors)


def training_cases():
    """Reference stream-only training RMSE trajectories (quality-gate anchors)."""
    out = {}
    full = synthetic_ratings(6040, 3706, rank=8, density=1.05e6 / (6040 * 3706), noise=0.1,
                             seed=0)
    rng = np.random.default_rng(1)
    perm = rng.permutation(full.nnz)
    n_test = full.nnz // 21  # 1.0 M train / 50 K test
    test_idx, train_idx = perm[:n_test], perm[n_test:]
    train = RatingMatrix(full.n_users, full.n_items, full.users[train_idx],
                         full.items[train_idx], full.ratings[train_idx])
    test = RatingMatrix(full.n_users, full.n_items, full.users[test_idx], full.items[test_idx],
                        full.ratings[test_idx])
    for epochs, label in [(1, "e1"), (5, "e5"), (20, "e20")]:
        cfg = RunConfig(schedule="stream-only", n_stream=8, n_factors=32, learning_rate=0.01,
                        reg_user=0.01, reg_item=0.01, epochs=epochs, seed=0,
                        log_train_loss=False)
        res = run_training(cfg, matrix=train)
        out[label] = dict(test_rmse=rmse(test, res.model).value,
                          train_rmse=rmse(train, res.model).value,
                          updates=int(res.scheduler.total_updates),
                          wall=res.wall_seconds)
    out["data"] = dict(nnz_full=int(full.nnz), n_test=int(n_test), split_seed=1,
                       generator="synthetic_ratings(6040, 3706, rank=8, "
                                 "density=1.05e6/(6040*3706), noise=0.1, seed=0)",
                       hyper=dict(k=32, lr=0.01, reg=0.01, seed=0, n_stream=8))
    return out


def main():
    kernels.warmup(4)
    np.savez_compressed(OUT / "sgd_range.npz",
                        **{f"{name}__{key}": val for name, case in sgd_cases().items()
                           for key, val in case.items()})
    orders = {}
    for n, seed in [(1, 5), (2, 9), (5, 1), (4095, 3), (4096, 4), (4097, 77),
                    (9753, 2 ** 62 + 1), (20000, 0)]:
        orders[f"n{n}_s{seed}"] = visit_order(n, seed)
    np.savez_compressed(OUT / "visit_order.npz", **orders)
    np.savez_compressed(OUT / "metrics.npz", **metric_cases())
    np.savez_compressed(OUT / "data.npz", **data_cases())
    plans = plan_cases()
    np.savez_compressed(OUT / "plan_matrix.npz", users=plans.pop("users"),
                        items=plans.pop("items"))
    sched, sm = scheduler_cases()
    np.savez_compressed(OUT / "sched_matrix.npz", users=sm.users, items=sm.items,
                        ratings=sm.ratings)
    meta = dict(mix64=mix64_cases(), plans=plans, scheduler=sched)
    (OUT / "golden.json").write_text(json.dumps(meta, indent=1))
    if "--no-training" not in sys.argv:
        (OUT / "training.json").write_text(json.dumps(training_cases(), indent=1))
    print("wrote fixtures to", OUT)


if __name__ == "__main__":
    main()
