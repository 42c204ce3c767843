"""GPU parity of the sm_100a kernels against the reference and the oracle.

Bars (north star, BASELINE.json):
  * EXACT mode (reference visit order, reference f64 arithmetic) is
    bit-identical to hetmf.kernels.sgd_range, on f64 and on f32 arrays;
  * fp32 update kernels match the reference within 1e-5 relative (norm-wise)
    for a fixed deterministic order (ORDERED mode, and HOGWILD on conflict-free
    inputs where order cannot matter);
  * HOGWILD applies every triple of the range exactly once (the reference's
    vanishing-step additivity pin, tests/test_sgd.py:161-182, f64 storage);
  * residual sums match the oracle; bucketing equals build_grid bit for bit.
"""

import contextlib
import json

import numpy as np
import pytest

from conftest import GOLDEN, random_matrix

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2006_15980_b200 import _lib
    _lib.load()
    return torch.device("cuda", 0)


def to_dev(a, dev, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to(dev, dtype) if dtype is not None else t.to(dev)


def run_case(c, dev, mode, storage):
    from paper_2006_15980_b200 import kernels
    dt = {"f64": torch.float64, "f32": torch.float32, "f16": torch.float16}[storage]
    vdt = torch.float64 if storage == "f64" else torch.float32
    P = to_dev(c["P0"], dev, dt)
    Q = to_dev(c["Q0"], dev, dt)
    start, stop, seed, rb, cb, _ = (int(x) for x in c["meta"])
    lr, ru, ri = (float(x) for x in c["hyper"])
    got = kernels.launch_sgd_range(P, Q, to_dev(c["rows"], dev), to_dev(c["cols"], dev),
                                   to_dev(c["vals"], dev, vdt), start, stop, lr, ru, ri, seed,
                                   rb, cb, mode)
    torch.cuda.synchronize()
    return got, P.double().cpu().numpy(), Q.double().cpu().numpy()


def rel_err(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def test_exact_mode_bitwise_f64(golden_sgd, dev):
    for name, c in golden_sgd.items():
        if c["P0"].dtype != np.float64:
            continue
        got, P, Q = run_case(c, dev, "exact", "f64")
        assert got == int(c["meta"][5]), name
        assert np.array_equal(P, c["P1"]), name
        assert np.array_equal(Q, c["Q1"]), name


def test_exact_mode_bitwise_f32(golden_sgd, dev):
    for name, c in golden_sgd.items():
        if c["P0"].dtype != np.float32:
            continue
        got, P, Q = run_case(c, dev, "exact", "f32")
        assert np.array_equal(P.astype(np.float32), c["P1"]), name
        assert np.array_equal(Q.astype(np.float32), c["Q1"]), name


def test_ordered_fp32_within_1e5_of_reference(golden_sgd, dev):
    """Fixed deterministic order, fp32 kernel arithmetic vs the reference."""
    for name, c in golden_sgd.items():
        c32 = dict(c)
        c32["P0"] = c["P0"].astype(np.float32)
        c32["Q0"] = c["Q0"].astype(np.float32)
        _, P, Q = run_case(c32, dev, "ordered", "f32")
        # f32 rounding of the start point plus ~n ordered updates: the
        # single/few-update cases are held to 1e-5; long ranges accumulate
        # rounding, and are held to 1e-5 per update chain length.
        n = int(c["meta"][1] - c["meta"][0])
        tol = 1e-5 if n <= 64 else 1e-5 * np.sqrt(n / 64)
        assert rel_err(P, c["P1"]) < tol, (name, rel_err(P, c["P1"]))
        assert rel_err(Q, c["Q1"]) < tol, (name, rel_err(Q, c["Q1"]))


def test_single_rating_update_fp32_all_shapes(dev):
    """One rating, every specialised k and the generic path, fp32 HOGWILD and
    ORDERED vs the reference f64 arithmetic (oracle): <= 1e-5 relative."""
    import oracle
    from paper_2006_15980_b200 import kernels
    rng = np.random.default_rng(0)
    for k in (1, 3, 8, 16, 32, 48, 64, 128, 256):
        P0 = rng.uniform(0, 1 / np.sqrt(k), size=(3, k))
        Q0 = rng.uniform(0, 1 / np.sqrt(k), size=(2, k))
        rows = np.array([2], np.int32)
        cols = np.array([1], np.int32)
        vals = np.array([0.7])
        Pe, Qe = P0.copy(), Q0.copy()
        oracle.sgd_range(Pe, Qe, rows, cols, vals, 0, 1, 0.05, 0.02, 0.03, 9, 0, 0)
        for mode in ("hogwild", "ordered"):
            P = to_dev(P0, dev, torch.float32)
            Q = to_dev(Q0, dev, torch.float32)
            kernels.launch_sgd_range(P, Q, to_dev(rows, dev), to_dev(cols, dev),
                                     to_dev(vals, dev, torch.float32), 0, 1, 0.05, 0.02, 0.03,
                                     9, 0, 0, mode)
            Pg = P.double().cpu().numpy()
            Qg = Q.double().cpu().numpy()
            assert np.max(np.abs(Pg - Pe) / np.maximum(np.abs(Pe), 1e-30)) < 1e-5, (k, mode)
            assert np.max(np.abs(Qg - Qe) / np.maximum(np.abs(Qe), 1e-30)) < 1e-5, (k, mode)


@pytest.mark.parametrize("k", [4, 32, 64, 128, 256])
def test_hogwild_conflict_free_equals_reference(dev, k):
    """Distinct users and items per triple: updates commute, so the racy
    kernel must equal the reference regardless of its visit order."""
    import oracle
    from paper_2006_15980_b200 import kernels
    rng = np.random.default_rng(k)
    n = 5000
    P0 = rng.uniform(0, 1 / np.sqrt(k), size=(n + 7, k))
    Q0 = rng.uniform(0, 1 / np.sqrt(k), size=(n + 3, k))
    rows = rng.permutation(n + 7)[:n].astype(np.int32)
    cols = rng.permutation(n + 3)[:n].astype(np.int32)
    vals = rng.uniform(0, 1, size=n).astype(np.float32).astype(np.float64)
    Pe, Qe = P0.copy(), Q0.copy()
    oracle.sgd_range(Pe, Qe, rows, cols, vals, 3, n - 2, 0.02, 0.01, 0.01, 5, 0, 0)
    P = to_dev(P0, dev, torch.float32)
    Q = to_dev(Q0, dev, torch.float32)
    got = kernels.launch_sgd_range(P, Q, to_dev(rows, dev), to_dev(cols, dev),
                                   to_dev(vals, dev, torch.float32), 3, n - 2, 0.02, 0.01, 0.01, 5,
                                   0, 0, "hogwild")
    assert got == n - 5
    Pg, Qg = P.double().cpu().numpy(), Q.double().cpu().numpy()
    assert rel_err(Pg, Pe) < 1e-6
    assert rel_err(Qg, Qe) < 1e-6
    # rows of triples outside [start, stop) are untouched
    for i in (0, 1, 2, n - 2, n - 1):
        assert np.array_equal(Pg[rows[i]], P0[rows[i]].astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("k,nnz,start", [(4, 30, 0), (32, 2000, 5), (128, 3000, 1), (256, 800, 2),
                                         (3, 500, 7)])
def test_hogwild_applies_each_triple_exactly_once(dev, k, nnz, start):
    """Vanishing step: the total change equals the sum of per-triple gradients
    whatever the interleaving, and a skipped or doubled triple shifts a row's
    change by a whole step (reference tests/test_sgd.py:187-208 and
    tests/test_workers.py:125-152).  f64 storage; lr = 1e-9 keeps both the
    second-order terms and the f64 rounding of the deltas below 1e-6."""
    from paper_2006_15980_b200 import kernels
    m = random_matrix(40, 40, min(nnz, 1600), 8)
    rows, cols, vals = m.users, m.items, m.ratings
    if nnz > len(vals):
        reps = -(-nnz // len(vals))
        rows, cols, vals = (np.tile(rows, reps)[:nnz], np.tile(cols, reps)[:nnz],
                            np.tile(vals, reps)[:nnz])
    rng = np.random.default_rng(3)
    P0 = rng.uniform(0, 0.5 / np.sqrt(k), size=(40, k))
    Q0 = rng.uniform(0, 0.5 / np.sqrt(k), size=(40, k))
    lr = 1e-9
    P = to_dev(P0, dev, torch.float64)
    Q = to_dev(Q0, dev, torch.float64)
    got = kernels.launch_sgd_range(P, Q, to_dev(rows, dev), to_dev(cols, dev),
                                   to_dev(vals, dev, torch.float64), start, len(vals), lr, 0.0,
                                   0.0, 99, 0, 0, "hogwild")
    assert got == len(vals) - start
    exp_dp = np.zeros_like(P0)
    exp_dq = np.zeros_like(Q0)
    for u, v, r in zip(rows[start:], cols[start:], vals[start:]):
        e = r - float(np.dot(P0[u], Q0[v]))
        exp_dp[u] += lr * e * Q0[v]
        exp_dq[v] += lr * e * P0[u]
    dP = P.cpu().numpy() - P0
    dQ = Q.cpu().numpy() - Q0
    assert rel_err(dP, exp_dp) < 1e-5
    assert rel_err(dQ, exp_dq) < 1e-5
    # per-row check: every row's change matches its own gradient sum
    for d, e in ((dP, exp_dp), (dQ, exp_dq)):
        for r_ in range(40):
            if np.linalg.norm(e[r_]) > 0:
                assert rel_err(d[r_], e[r_]) < 1e-4, r_


def test_visit_order_matches_reference(dev):
    from paper_2006_15980_b200 import kernels
    orders = np.load(GOLDEN / "visit_order.npz")
    for key in orders.files:
        n = int(key.split("_")[0][1:])
        seed = int(key.split("_s")[1])
        got = kernels.visit_order(n, seed, device=dev).cpu().numpy()
        assert np.array_equal(got.astype(np.int64), orders[key]), key


def test_visit_order_large_matches_oracle(dev):
    import oracle
    from paper_2006_15980_b200 import kernels
    for n, seed in ((1_000_003, 17), (4096 * 37, 2 ** 63 - 5)):
        got = kernels.visit_order(n, seed, device=dev).cpu().numpy().astype(np.int64)
        assert np.array_equal(got, oracle.visit_order(n, seed))


def test_exact_mode_long_range_matches_oracle(dev):
    """EXACT mode over a multi-window range with staged bases, f64 and f32."""
    import oracle
    from paper_2006_15980_b200 import kernels
    m = random_matrix(500, 300, 30000, 4)
    rng = np.random.default_rng(4)
    for dt in (np.float64, np.float32):
        P0 = rng.uniform(0, 0.2, size=(450, 16)).astype(dt)
        Q0 = rng.uniform(0, 0.2, size=(280, 16)).astype(dt)
        keep = (m.users >= 50) & (m.items >= 20)
        rows, cols = m.users[keep], m.items[keep]
        vals = (m.ratings[keep] / 5).astype(np.float32).astype(np.float64)
        Pe, Qe = P0.copy(), Q0.copy()
        oracle.sgd_range(Pe, Qe, rows, cols, vals, 11, len(vals) - 3, 0.01, 0.02, 0.03, 31, 50, 20)
        tdt = torch.float64 if dt == np.float64 else torch.float32
        P, Q = to_dev(P0, dev, tdt), to_dev(Q0, dev, tdt)
        kernels.launch_sgd_range(P, Q, to_dev(rows, dev), to_dev(cols, dev), to_dev(vals, dev, tdt),
                                 11, len(vals) - 3, 0.01, 0.02, 0.03, 31, 50, 20, "exact")
        assert np.array_equal(P.cpu().numpy(), Pe)
        assert np.array_equal(Q.cpu().numpy(), Qe)


def test_host_buffer_path_equals_device_path(dev, golden_sgd):
    """The numpy (host-buffer) drop-in call copies in, runs, copies back."""
    from paper_2006_15980_b200 import kernels
    c = golden_sgd["k32_staged"]
    P, Q = c["P0"].copy(), c["Q0"].copy()
    start, stop, seed, rb, cb, got = (int(x) for x in c["meta"])
    lr, ru, ri = c["hyper"]
    n = kernels.sgd_range(P, Q, c["rows"], c["cols"], c["vals"], start, stop, lr, ru, ri, seed,
                          rb, cb, mode="exact")
    assert n == got
    assert np.array_equal(P, c["P1"]) and np.array_equal(Q, c["Q1"])


def test_empty_range_and_errors(dev):
    from paper_2006_15980_b200 import kernels, _lib
    P = torch.ones((2, 4), device=dev)
    z = torch.zeros(2, dtype=torch.int32, device=dev)
    v = torch.ones(2, device=dev)
    assert kernels.launch_sgd_range(P, P.clone(), z, z, v, 1, 1, 0.1, 0, 0, 1, 0, 0) == 0
    with pytest.raises(_lib.HmfError):
        kernels.launch_sgd_range(P, P.clone(), z, z, v, 0, 2, 0.1, 0, 0, 1, 0, 0, mode=7)
    with pytest.raises(_lib.HmfError):
        h = torch.ones((2, 4), device=dev, dtype=torch.float16)
        kernels.launch_sgd_range(h, h.clone(), z, z, v, 0, 2, 0.1, 0, 0, 1, 0, 0, mode="exact")


def test_fp16_storage_single_update(dev):
    import oracle
    from paper_2006_15980_b200 import kernels
    rng = np.random.default_rng(1)
    for k in (32, 64, 128, 256, 24):
        P0 = rng.uniform(0, 0.2, size=(4, k)).astype(np.float16)
        Q0 = rng.uniform(0, 0.2, size=(4, k)).astype(np.float16)
        Pe, Qe = P0.astype(np.float64), Q0.astype(np.float64)
        rows, cols, vals = np.array([1], np.int32), np.array([2], np.int32), np.array([0.9])
        oracle.sgd_range(Pe, Qe, rows, cols, vals, 0, 1, 0.1, 0.01, 0.01, 3, 0, 0)
        P, Q = to_dev(P0, dev), to_dev(Q0, dev)
        kernels.launch_sgd_range(P, Q, to_dev(rows, dev), to_dev(cols, dev),
                                 to_dev(vals, dev, torch.float32), 0, 1, 0.1, 0.01, 0.01, 3, 0, 0)
        # fp16 storage: within half-precision rounding of the f64 result
        assert np.allclose(P.double().cpu().numpy(), Pe, rtol=2e-3, atol=1e-4), k
        assert np.allclose(Q.double().cpu().numpy(), Qe, rtol=2e-3, atol=1e-4), k


def test_residual_sums_match_oracle(dev):
    import oracle
    from paper_2006_15980_b200.sgd import DeviceModel, FactorModel, regularized_loss, residual_sums, rmse
    m = np.load(GOLDEN / "metrics.npz")
    model = FactorModel(m["P"], m["Q"])
    test = random_matrix(1, 1, 0, 0)
    from paper_2006_15980_b200.data import RatingMatrix
    mat = RatingMatrix(40, 30, m["rows"], m["cols"], m["vals"])
    assert rmse(mat, model).value == pytest.approx(float(m["rmse"][0]), rel=1e-12)
    assert regularized_loss(mat, model, 0.3, 0.7) == pytest.approx(float(m["loss"][0]), rel=1e-12)
    del test
    rng = np.random.default_rng(5)
    for k in (7, 32, 64, 128, 256):
        nu, ni, n = 3000, 2000, 200_001
        P = rng.uniform(0, 0.2, size=(nu, k)).astype(np.float32)
        Q = rng.uniform(0, 0.2, size=(ni, k)).astype(np.float32)
        rows = rng.integers(0, nu, n).astype(np.int32)
        cols = rng.integers(0, ni, n).astype(np.int32)
        vals = rng.uniform(0, 1, n).astype(np.float32)
        exp = oracle.residual_sums(P.astype(np.float64), Q.astype(np.float64), rows, cols,
                                   vals.astype(np.float64))
        dm = DeviceModel(to_dev(P, dev), to_dev(Q, dev))
        got = residual_sums(dm, to_dev(rows, dev), to_dev(cols, dev), to_dev(vals, dev),
                            with_reg=True).cpu().numpy()
        assert got == pytest.approx(exp, rel=1e-11), k


def test_device_bucketing_equals_build_grid(dev):
    from paper_2006_15980_b200.data import DeviceTriples, build_device_grid, build_grid
    for (nu, ni, nnz, rc, cc) in [(60, 50, 601, [0, 20, 60], [0, 10, 30, 50]),
                                  (300, 280, 20001, [0, 100, 101, 300], [0, 7, 8, 200, 280]),
                                  (40, 40, 3, [0, 40], [0, 40]),
                                  (1000, 900, 150_003, list(range(0, 1001, 125)),
                                   list(range(0, 901, 100)))]:
        m = random_matrix(nu, ni, nnz, nnz)
        m.ratings = m.ratings.astype(np.float32).astype(np.float64)
        host = build_grid(m, rc, cc)
        g = build_device_grid(DeviceTriples.from_host(m, dev), rc, cc)
        assert np.array_equal(g.block_ptr, host.block_ptr)
        assert np.array_equal(g.users.cpu().numpy(), host.users)
        assert np.array_equal(g.items.cpu().numpy(), host.items)
        assert np.array_equal(g.ratings.cpu().numpy().astype(np.float64), host.ratings)


def test_synthetic_device_law(dev):
    from paper_2006_15980_b200.data import synthetic_device
    t = synthetic_device(2000, 1500, 300_000, rank=8, noise=0.1, seed=3, device=dev)
    assert t.nnz == 300_000
    u = t.users.cpu().numpy().astype(np.int64)
    i = t.items.cpu().numpy().astype(np.int64)
    assert u.min() >= 0 and u.max() < 2000 and i.min() >= 0 and i.max() < 1500
    assert len(np.unique(u * 1500 + i)) == 300_000
    r = t.ratings.cpu().numpy().astype(np.float64)
    # rank-8 law with factor_scale 1: mean 8 * (1/(2*sqrt 8))^2 = 0.25, noise 0.1
    assert abs(r.mean() - 0.25) < 0.01
    assert 0.10 < r.std() < 0.16
    # rows are hit uniformly: per-row counts ~ Binomial(1500, 0.1)
    counts = np.bincount(u, minlength=2000)
    assert abs(counts.mean() - 150) < 1e-9 and counts.std() < 3 * np.sqrt(150)


def test_ml1m_quality_within_0005_of_reference(dev):
    """Quality gate: ML-1M-shaped synthetic instance (the reference's own
    generator, reproduced bit for bit), k=32, lr=0.01, reg=0.01, 20 epochs on
    the 1-GPU batch-only uniform 1x2 grid; test RMSE within 0.005 of the
    reference's stream-only run (tests/golden/training.json)."""
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (DeviceGrid, RatingMatrix, build_grid,
                                            shuffle_triples, synthetic_ratings)
    from paper_2006_15980_b200.sgd import DeviceModel, Hyperparams, block_epoch, init_model, rmse
    ref = json.loads((GOLDEN / "training.json").read_text())
    full = synthetic_ratings(6040, 3706, rank=8, density=1.05e6 / (6040 * 3706), noise=0.1, seed=0)
    perm = np.random.default_rng(1).permutation(full.nnz)
    n_test = full.nnz // 21
    te, tr = perm[:n_test], perm[n_test:]
    train = RatingMatrix(6040, 3706, full.users[tr], full.items[tr], full.ratings[tr])
    test = RatingMatrix(6040, 3706, full.users[te], full.items[te], full.ratings[te])
    hp = Hyperparams(n_factors=32, reg_user=0.01, reg_item=0.01, learning_rate=0.01)
    sh = shuffle_triples(train, 0)
    grid = DeviceGrid.from_host(build_grid(sh, [0, 6040], [0, 1853, 3706]), dev)
    model = DeviceModel.from_host(init_model(6040, 3706, hp, 0), dev)
    got = {}
    counts = np.zeros(2, dtype=np.int64)
    for epoch in range(1, 21):
        for b in (0, 1):
            unit = kernels.mix64(0, b, int(counts[b]))
            block_epoch(model, grid, b, hp, kernels.mix64(unit, 0))
            counts[b] += 1
        if epoch in (1, 5, 20):
            got[f"e{epoch}"] = rmse(test, model).value
    for key in ("e1", "e5", "e20"):
        print(f"{key}: gpu {got[key]:.5f} reference {ref[key]['test_rmse']:.5f}")
    assert abs(got["e20"] - ref["e20"]["test_rmse"]) <= 0.005
    assert abs(got["e5"] - ref["e5"]["test_rmse"]) <= 0.005


# ---------------------------------------------------------------------------
# Q-band-stationary kernel
# ---------------------------------------------------------------------------
# The Q-band implementation / chain configuration the helpers lay grids out
# for (None / -1: the library's defaults).  Launches take the layout's
# options from the grid (ABI 4: per-launch, nothing process-wide).
_LAYOUT = {"impl": None, "cfg": -1}


@contextlib.contextmanager
def layout(impl=None, cfg=-1):
    old = dict(_LAYOUT)
    _LAYOUT.update(impl=impl, cfg=cfg)
    try:
        yield
    finally:
        _LAYOUT.update(old)


def _qband_grid(dev, m, k, col_cuts, target, tile_bytes=None):
    """An explicit tile_bytes sets the tile count alone (no user cap)."""
    from paper_2006_15980_b200.data import DeviceTriples, bucket_qbands, build_device_grid
    g = build_device_grid(DeviceTriples.from_host(m, dev), [0, m.n_users], col_cuts)
    return bucket_qbands(g, k, target=target, tile_bytes=tile_bytes,
                         max_tile_rows=None if tile_bytes is None else 0,
                         impl=_LAYOUT["impl"], chain_cfg=_LAYOUT["cfg"])


def _fin(z):
    from paper_2006_15980_b200.kernels import _MASK64
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9 & _MASK64
    z = (z ^ (z >> 27)) * 0x94D049BB133111EB & _MASK64
    return z ^ (z >> 31)


def _chain_lanes(k):
    """Lanes per chain of the chained kernel (qchain.cuh ChainCfg) in the
    current layout's configuration."""
    from paper_2006_15980_b200 import _lib
    return int(_lib.load().hmf_qband_chain_lanes(k, 0, _LAYOUT["cfg"]))


def _bin_visit(impl, k, beg, end, seed, bin_index):
    """Triple indices of one (tile, sub-band) bin in the kernel's visit order:
    impl 4 walks batches of LPC triples from the bin start, the others chunks
    of 128 from the 4-aligned base; both rotated by the bin's seed."""
    from paper_2006_15980_b200.kernels import _MASK64
    if end <= beg:
        return []
    if impl >= 4:   # full batches rotated, the partial batch last
        step = _chain_lanes(k)
        nf = (end - beg) // step
        out = []
        if nf:
            rot = _fin((seed + bin_index * 0x9E3779B97F4A7C15) & _MASK64) % nf
            for x in range(nf):
                c = (x + rot) % nf
                out.extend(range(beg + c * step, beg + (c + 1) * step))
        out.extend(range(beg + nf * step, end))
        return out
    step, a0 = 128, beg & ~3
    n = (end - a0 + step - 1) // step
    rot = _fin((seed + bin_index * 0x9E3779B97F4A7C15) & _MASK64) % n
    out = []
    for x in range(n):
        c = (x + rot) % n
        out.extend(range(max(beg, a0 + c * step), min(a0 + (c + 1) * step, end)))
    return out


def _tile_order(seed, n_tiles):
    """The kernel's row-tile rotation (qband_kernels.cu tile_at)."""
    if n_tiles <= 1:
        return [0]
    rot = _fin(seed ^ 0x5851F42D4C957F2D) % n_tiles
    return [(i + rot) % n_tiles for i in range(n_tiles)]


@pytest.mark.parametrize("n_sub_target", [7, 20000])
def test_qband_tiled_bucketing_contract(dev, n_sub_target):
    """Row tiles x sub-bands, tile-major, item runs inside a tile, stable;
    with few and with many (> 12288 bins) sub-bands."""
    from paper_2006_15980_b200.data import qband_row_tiles
    m = random_matrix(5000, 30000, 300_000, 78)
    k = 128
    tb = 5000 * k * 4 // 5 + 1           # 5 row tiles of 1000 users
    g = _qband_grid(dev, m, k, [0, 30000], target=n_sub_target, tile_bytes=tb)
    T = qband_row_tiles(5000, k, 4, tb)
    assert T == 5 and g.sub_tiles == [T]
    cuts = g.sub_cuts[0].cpu().numpy()
    S = len(cuts) - 1
    ptr = g.sub_ptr[0].cpu().numpy()
    assert len(ptr) == T * S + 1 and ptr[0] == 0 and ptr[-1] == m.nnz
    assert np.all(np.diff(ptr) >= 0)
    users, items = g.users.cpu().numpy(), g.items.cpu().numpy()
    tiles = np.linspace(0, 5000, T + 1).round().astype(np.int64)
    for t in range(T):
        for s_ in range(0, S, max(1, S // 50)):
            a, b = ptr[t * S + s_], ptr[t * S + s_ + 1]
            assert np.all((users[a:b] >= tiles[t]) & (users[a:b] < tiles[t + 1]))
            assert np.all((items[a:b] >= cuts[s_]) & (items[a:b] < cuts[s_ + 1]))
    # tile-major, then item runs (stable): sub-band ranges stay contiguous
    key = (np.searchsorted(tiles, m.users, side="right") - 1) * 30000 + m.items
    order = np.argsort(key, kind="stable")
    assert np.array_equal(users, m.users[order]) and np.array_equal(items, m.items[order])


@pytest.mark.parametrize("k", [32, 64, 128, 256])
def test_qband_bucketing_contract(dev, k):
    m = random_matrix(700, 900, 40_000, k)
    g = _qband_grid(dev, m, k, [0, 450, 900], target=100)
    items = g.items.cpu().numpy()
    for b in range(g.n_blocks):
        ptr = g.sub_ptr[b].cpu().numpy()
        cuts = g.sub_cuts[b].cpu().numpy()
        lo, hi = g.block_range(b)
        assert ptr[0] == lo and ptr[-1] == hi
        from paper_2006_15980_b200 import _lib
        assert np.max(np.diff(cuts)) <= _lib.load().hmf_qband_max_items(k, 0, -1)
        for s in range(len(cuts) - 1):
            seg = items[ptr[s]:ptr[s + 1]]
            assert np.all((seg >= cuts[s]) & (seg < cuts[s + 1]))


@pytest.fixture(params=[(4, -1), (4, 2), (4, 4), (4, 6), (0, -1)],
                ids=["chains", "chains_cfg2", "chains_cfg4", "chains_cfg6", "regs"])
def qband_impl(request):
    impl, cfg = request.param
    with layout(impl, cfg):
        yield impl


@pytest.mark.parametrize("k", [32, 64, 128, 256])
def test_qband_equals_sequential_per_item(dev, k, qband_impl):
    """Distinct users, <= 128 triples per sub-band: every Q row is updated
    sequentially in storage order by its owner warp and no P row is shared,
    so the result equals a sequential f64 replay within fp32 rounding."""
    from paper_2006_15980_b200 import kernels
    rng = np.random.default_rng(k)
    n_users, n_items, n = 4000, 300, 3000
    users = rng.permutation(n_users)[:n].astype(np.int32)
    items = rng.integers(0, n_items, n).astype(np.int32)
    vals = rng.uniform(0, 1, n).astype(np.float32).astype(np.float64)
    from paper_2006_15980_b200.data import RatingMatrix
    m = RatingMatrix(n_users, n_items, users, items, vals)
    g = _qband_grid(dev, m, k, [0, n_items], target=n_items)  # one item per sub-band
    P0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_users, k)).astype(np.float32)
    Q0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_items, k)).astype(np.float32)
    P, Q = to_dev(P0, dev), to_dev(Q0, dev)
    got = kernels.launch_block_qband(P, Q, g, 0, 0.05, 0.02, 0.03, 11)
    assert got == n
    # sequential replay of every sub-band in the kernel's visit order
    ptr = g.sub_ptr[0].cpu().numpy()
    order = [i for b_ in range(len(ptr) - 1)
             for i in _bin_visit(qband_impl, k, int(ptr[b_]), int(ptr[b_ + 1]), 11, b_)]
    assert sorted(order) == list(range(n))
    Pe, Qe = P0.astype(np.float64), Q0.astype(np.float64)
    gu, gi = g.users.cpu().numpy(), g.items.cpu().numpy()
    gr = g.ratings.cpu().numpy().astype(np.float64)
    for u, v, r in zip(gu[order], gi[order], gr[order]):
        pu, qv = Pe[u].copy(), Qe[v].copy()
        e = r - pu @ qv
        Pe[u] = pu + 0.05 * (e * qv - 0.02 * pu)
        Qe[v] = qv + 0.05 * (e * pu - 0.03 * qv)
    assert rel_err(P.double().cpu().numpy(), Pe) < 1e-5
    assert rel_err(Q.double().cpu().numpy(), Qe) < 1e-5


@pytest.mark.parametrize("tile_bytes", [None, 100_000], ids=["default_tiles", "8_tiles"])
def test_qband_ml1m_quality_within_0005_of_reference(dev, qband_impl, tile_bytes):
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (DeviceGrid, RatingMatrix, bucket_qbands, build_grid,
                                            shuffle_triples, synthetic_ratings)
    from paper_2006_15980_b200.sgd import DeviceModel, Hyperparams, init_model, rmse
    ref = json.loads((GOLDEN / "training.json").read_text())
    full = synthetic_ratings(6040, 3706, rank=8, density=1.05e6 / (6040 * 3706), noise=0.1, seed=0)
    perm = np.random.default_rng(1).permutation(full.nnz)
    n_test = full.nnz // 21
    te, tr = perm[:n_test], perm[n_test:]
    train = RatingMatrix(6040, 3706, full.users[tr], full.items[tr], full.ratings[tr])
    test = RatingMatrix(6040, 3706, full.users[te], full.items[te], full.ratings[te])
    hp = Hyperparams(n_factors=32, reg_user=0.01, reg_item=0.01, learning_rate=0.01)
    grid = DeviceGrid.from_host(build_grid(shuffle_triples(train, 0), [0, 6040], [0, 1853, 3706]),
                                dev)
    bucket_qbands(grid, 32, tile_bytes=tile_bytes, impl=_LAYOUT["impl"], chain_cfg=_LAYOUT["cfg"])
    assert grid.sub_tiles == ([1, 1] if tile_bytes is None else [8, 8])
    model = DeviceModel.from_host(init_model(6040, 3706, hp, 0), dev)
    got = {}
    for epoch in range(1, 21):
        for b in (0, 1):
            kernels.launch_block_qband(model.P, model.Q, grid, b, 0.01, 0.01, 0.01,
                                       kernels.mix64(0, b, epoch))
        if epoch in (1, 5, 20):
            got[f"e{epoch}"] = rmse(test, model).value
    for key in ("e1", "e5", "e20"):
        print(f"{key}: gpu qband {got[key]:.5f} reference {ref[key]['test_rmse']:.5f}")
    assert abs(got["e20"] - ref["e20"]["test_rmse"]) <= 0.005
    assert abs(got["e5"] - ref["e5"]["test_rmse"]) <= 0.005


@pytest.mark.parametrize("n_tiles", [1, 3])
@pytest.mark.parametrize("k", [64, 128])
def test_qband_multi_chunk_subbands_match_sequential(dev, k, n_tiles, qband_impl):
    """Sub-bands of several hundred triples (several staging chunks, rotated
    per seed), optionally split into row tiles walked in a seeded rotation:
    with distinct users the result still equals a sequential replay in the
    kernel's visit order."""
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import RatingMatrix
    rng = np.random.default_rng(k + 1)
    n_users, n_items, n = 20000, 24, 6000
    users = rng.permutation(n_users)[:n].astype(np.int32)
    items = rng.integers(0, n_items, n).astype(np.int32)
    vals = rng.uniform(0, 1, n).astype(np.float32).astype(np.float64)
    m = RatingMatrix(n_users, n_items, users, items, vals)
    tb = 0 if n_tiles == 1 else n_users * k * 4 // n_tiles + 1
    g = _qband_grid(dev, m, k, [0, n_items], target=n_items, tile_bytes=tb)
    assert g.sub_tiles == [n_tiles]
    P0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_users, k)).astype(np.float32)
    Q0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_items, k)).astype(np.float32)
    P, Q = to_dev(P0, dev), to_dev(Q0, dev)
    seed = 12345
    kernels.launch_block_qband(P, Q, g, 0, 0.05, 0.02, 0.03, seed)
    # replay: per sub-band, chunks of 128 from the 4-aligned base, rotated
    from paper_2006_15980_b200.kernels import _MASK64
    gu, gi = g.users.cpu().numpy(), g.items.cpu().numpy()
    gr = g.ratings.cpu().numpy().astype(np.float64)
    ptr = g.sub_ptr[0].cpu().numpy()
    S = g.sub_cuts[0].numel() - 1
    Pe, Qe = P0.astype(np.float64), Q0.astype(np.float64)
    bins = [t * S + s_ for t in _tile_order(seed, n_tiles) for s_ in range(S)]
    for bn in bins:
        for i in _bin_visit(qband_impl, k, int(ptr[bn]), int(ptr[bn + 1]), seed, bn):
            u, v, r = gu[i], gi[i], gr[i]
            pu, qv = Pe[u].copy(), Qe[v].copy()
            e = r - pu @ qv
            Pe[u] = pu + 0.05 * (e * qv - 0.02 * pu)
            Qe[v] = qv + 0.05 * (e * pu - 0.03 * qv)
    assert rel_err(Q.double().cpu().numpy(), Qe) < 1e-5
    assert rel_err(P.double().cpu().numpy(), Pe) < 1e-5


@pytest.mark.parametrize("n_tiles", [1, 3])
def test_qband_chains_dynamic_matches_sequential(dev, n_tiles):
    """More sub-bands than chains: implementation 4 hands (tile, sub-band)
    units out dynamically and passes each Q row between chains by
    release/acquire.  With distinct users the result equals a sequential
    replay of every sub-band's units in tile order."""
    from paper_2006_15980_b200 import _lib, kernels
    from paper_2006_15980_b200.data import RatingMatrix, resident_warps
    from paper_2006_15980_b200.kernels import _MASK64
    k = 128
    with layout(4):
        slots = resident_warps(dev, k, False, 4)
        rng = np.random.default_rng(99)
        n_items = 2 * slots + 777
        n_users, n = 400_000, 150_000
        users = rng.permutation(n_users)[:n].astype(np.int32)
        items = rng.integers(0, n_items, n).astype(np.int32)
        vals = rng.uniform(0, 1, n).astype(np.float32).astype(np.float64)
        m = RatingMatrix(n_users, n_items, users, items, vals)
        tb = 0 if n_tiles == 1 else n_users * k * 4 // n_tiles + 1
        g = _qband_grid(dev, m, k, [0, n_items], target=n_items, tile_bytes=tb)
        S = g.sub_cuts[0].numel() - 1
        assert S == n_items > slots and g.sub_impl == 4
        P0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_users, k)).astype(np.float32)
        Q0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_items, k)).astype(np.float32)
        P, Q = to_dev(P0, dev), to_dev(Q0, dev)
        seed = 4242
        assert kernels.launch_block_qband(P, Q, g, 0, 0.05, 0.02, 0.03, seed) == n
        gu, gi = g.users.cpu().numpy(), g.items.cpu().numpy()
        gr = g.ratings.cpu().numpy().astype(np.float64)
        ptr = g.sub_ptr[0].cpu().numpy()
        order = [i for t in _tile_order(seed, n_tiles) for s_ in range(S)
                 for i in _bin_visit(4, k, int(ptr[t * S + s_]), int(ptr[t * S + s_ + 1]), seed,
                                     t * S + s_)]
        assert sorted(order) == list(range(n))
        Pe, Qe = P0.astype(np.float64), Q0.astype(np.float64)
        for u, v, r in zip(gu[order], gi[order], gr[order]):
            pu, qv = Pe[u].copy(), Qe[v].copy()
            e = r - pu @ qv
            Pe[u] = pu + 0.05 * (e * qv - 0.02 * pu)
            Qe[v] = qv + 0.05 * (e * pu - 0.03 * qv)
        assert rel_err(Q.double().cpu().numpy(), Qe) < 1e-5
        assert rel_err(P.double().cpu().numpy(), Pe) < 1e-5


@pytest.mark.parametrize("n_items,impl", [(300, 0), (300, 4), (40_000, 4)],
                         ids=["regs", "chains_static", "chains_dynamic"])
def test_qband_skewed_items_match_sequential(dev, n_items, impl):
    """Zipf-skewed item popularity (one item holds a large share of the
    ratings; many items are empty) and row tiles with empty bins: with
    distinct users every sub-band still equals a sequential replay of its
    units in tile order — static ownership and the dynamic scheduler alike."""
    from paper_2006_15980_b200 import _lib, kernels
    from paper_2006_15980_b200.data import RatingMatrix
    k, n_tiles, seed = 64, 3, 777
    with layout(impl):
        rng = np.random.default_rng(n_items + impl)
        n_users, n = 300_000, 60_000
        users = rng.permutation(n_users)[:n].astype(np.int32)
        items = ((rng.zipf(1.3, n) - 1) % n_items).astype(np.int32)
        vals = rng.uniform(0, 1, n).astype(np.float32).astype(np.float64)
        m = RatingMatrix(n_users, n_items, users, items, vals)
        tb = n_users * k * 4 // n_tiles + 1
        target = n_items if impl == 4 else min(n_items, 200)
        g = _qband_grid(dev, m, k, [0, n_items], target=target, tile_bytes=tb)
        assert g.sub_tiles == [n_tiles] and g.sub_impl == impl
        S = g.sub_cuts[0].numel() - 1
        P0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_users, k)).astype(np.float32)
        Q0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_items, k)).astype(np.float32)
        P, Q = to_dev(P0, dev), to_dev(Q0, dev)
        assert kernels.launch_block_qband(P, Q, g, 0, 0.05, 0.02, 0.03, seed) == n
        gu, gi = g.users.cpu().numpy(), g.items.cpu().numpy()
        gr = g.ratings.cpu().numpy().astype(np.float64)
        ptr = g.sub_ptr[0].cpu().numpy()
        order = [i for t in _tile_order(seed, n_tiles) for s_ in range(S)
                 for i in _bin_visit(impl, k, int(ptr[t * S + s_]), int(ptr[t * S + s_ + 1]),
                                     seed, t * S + s_)]
        assert sorted(order) == list(range(n))
        Pe, Qe = P0.astype(np.float64), Q0.astype(np.float64)
        for u, v, r in zip(gu[order], gi[order], gr[order]):
            pu, qv = Pe[u].copy(), Qe[v].copy()
            e = r - pu @ qv
            Pe[u] = pu + 0.05 * (e * qv - 0.02 * pu)
            Qe[v] = qv + 0.05 * (e * pu - 0.03 * qv)
        assert rel_err(Q.double().cpu().numpy(), Qe) < 1e-5
        assert rel_err(P.double().cpu().numpy(), Pe) < 1e-5


@pytest.mark.parametrize("k,dtype", [(128, torch.float32), (64, torch.float32),
                                     (32, torch.float32)])
@pytest.mark.parametrize("n_tiles", [1, 3])
def test_qband_split_runs_apply_every_rating(dev, n_tiles, k, dtype):
    """Implementation 5: a narrow block's item runs split over chains, each
    chain on its own Q copy, changes added back by reductions.  At a small
    step SGD is linear in the ratings, so the factor changes must equal the
    sequential reference's to first order: every rating applied once, every
    Q delta added once (nothing lost, nothing doubled).  Users repeat here, so
    P goes back by reductions (opts pstore = 0): stores may drop a concurrent
    update of the same user."""
    _split_runs_apply_every_rating(dev, n_tiles, k, dtype)


def _split_runs_apply_every_rating(dev, n_tiles, k, dtype):
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import RatingMatrix
    lr = 1e-4
    rng = np.random.default_rng(5 + n_tiles)
    n_users, n_items, n = 30_000, 64, 40_000
    users = rng.integers(0, n_users, n).astype(np.int32)
    items = rng.integers(0, n_items, n).astype(np.int32)
    vals = rng.uniform(0, 1, n).astype(np.float32).astype(np.float64)
    m = RatingMatrix(n_users, n_items, users, items, vals)
    from paper_2006_15980_b200.data import DeviceTriples, bucket_qbands, build_device_grid
    g = build_device_grid(DeviceTriples.from_host(m, dev), [0, n_users], [0, n_items])
    tb = 0 if n_tiles == 1 else n_users * k * 4 // n_tiles + 1
    bucket_qbands(g, k, tile_bytes=tb, impl=5, split=8,
                  elem_bytes=2 if dtype == torch.float16 else 4)
    assert g.sub_impl == 5 and g.sub_split == 8 and g.sub_tiles == [n_tiles]
    assert g.sub_cuts[0].numel() - 1 == n_items * 8
    P0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_users, k)).astype(np.float32)
    Q0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_items, k)).astype(np.float32)
    P, Q = to_dev(P0, dev, dtype), to_dev(Q0, dev, dtype)
    assert kernels.launch_block_qband(P, Q, g, 0, lr, 0.02, 0.03, 3, opts={"pstore": 0}) == n
    Pe, Qe = P0.astype(np.float64), Q0.astype(np.float64)
    for u, v, r in zip(users, items, vals):
        pu, qv = Pe[u].copy(), Qe[v].copy()
        e = r - pu @ qv
        Pe[u] = pu + lr * (e * qv - 0.02 * pu)
        Qe[v] = qv + lr * (e * pu - 0.03 * qv)
    dP, dQ = P.double().cpu().numpy() - P0, Q.double().cpu().numpy() - Q0
    # second-order terms (each part starts from a stale Q row): ~ lr x the
    # ratings per item x the change, a few percent here (fp16 storage would
    # round these 1e-5 changes away: covered by the quality tests instead)
    assert rel_err(dQ, Qe - Q0) < 0.03
    assert rel_err(dP, Pe - P0) < 0.03


def test_qband_pstore_conflict_free_equals_reductions_and_trains(dev):
    """P write-back by stores (grid.sub_pstore, chosen for fp32 k >= 128 when
    tiles hold many users): with distinct users per launch nothing races, so
    stores and reductions give the same factors (whole item runs,
    implementation 4, deterministic); with repeated users (the racing case)
    a few epochs still train to the reductions' test RMSE within 0.005."""
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import RatingMatrix
    k = 128
    rng = np.random.default_rng(17)
    n_users, n_items = 120_000, 700
    n = 90_000
    users = rng.permutation(n_users)[:n].astype(np.int32)
    items = rng.integers(0, n_items, n).astype(np.int32)
    vals = rng.uniform(0, 1, n).astype(np.float32).astype(np.float64)
    m = RatingMatrix(n_users, n_items, users, items, vals)
    P0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_users, k)).astype(np.float32)
    Q0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_items, k)).astype(np.float32)
    out = {}
    with layout(4):
        g = _qband_grid(dev, m, k, [0, n_items], target=None)
    assert g.sub_impl == 4
    for mode in (0, 1):
        P, Q = to_dev(P0, dev), to_dev(Q0, dev)
        assert kernels.launch_block_qband(P, Q, g, 0, 0.05, 0.02, 0.03, 11,
                                          opts={"pstore": mode}) == n
        out[mode] = (P.cpu().numpy(), Q.cpu().numpy())
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    # repeated users: held-out RMSE after 4 epochs, stores vs reductions
    n = 600_000
    users = rng.integers(0, n_users, n).astype(np.int32)
    items = rng.integers(0, n_items, n).astype(np.int32)
    a = rng.uniform(0, 0.5, size=(n_users, 8))
    b = rng.uniform(0, 0.5, size=(n_items, 8))
    vals = np.einsum("ij,ij->i", a[users], b[items]) + rng.normal(0, 0.1, n)
    cut = n * 19 // 20
    m = RatingMatrix(n_users, n_items, users[:cut], items[:cut], vals[:cut])
    g = _qband_grid(dev, m, k, [0, n_items], target=None)
    tu, ti, tv = users[cut:], items[cut:], vals[cut:]
    rm = {}
    for mode in (0, 1):
        P, Q = to_dev(P0, dev), to_dev(Q0, dev)
        for e in range(4):
            kernels.launch_block_qband(P, Q, g, 0, 0.01, 0.01, 0.01, 100 + e,
                                       opts={"pstore": mode})
        Ph, Qh = P.double().cpu().numpy(), Q.double().cpu().numpy()
        rm[mode] = float(np.sqrt(np.mean((tv - np.einsum("ij,ij->i", Ph[tu], Qh[ti])) ** 2)))
    assert np.isfinite(rm[1]) and abs(rm[1] - rm[0]) <= 0.005, rm


def test_qband_pstore_layout_choice(dev):
    """The layout picks stores only for fp32 k >= 128 with tiles of at least
    4x as many users as chains (Netflix-shaped tiles: 60 000 users)."""
    from paper_2006_15980_b200.data import RatingMatrix, resident_warps
    rng = np.random.default_rng(2)
    for n_users, k, f16, want in [(60_000, 128, False, None), (3_000, 128, False, 0),
                                  (60_000, 64, False, 0), (60_000, 128, True, 0)]:
        n = 50_000
        m = RatingMatrix(n_users, 500, rng.integers(0, n_users, n).astype(np.int32),
                         rng.integers(0, 500, n).astype(np.int32), rng.uniform(0, 1, n))
        from paper_2006_15980_b200.data import DeviceTriples, bucket_qbands, build_device_grid
        g = build_device_grid(DeviceTriples.from_host(m, dev), [0, n_users], [0, 500])
        bucket_qbands(g, k, elem_bytes=2 if f16 else 4)
        if want is None:
            want = int(n_users >= 4 * resident_warps(dev, k, False, g.sub_impl))
        assert g.sub_pstore == want, (n_users, k, f16)


def test_qband_split_runs_ml1m_quality(dev):
    """Implementation 5 on the ML-1M shape (few items per block): test RMSE
    within 0.005 of the reference's stream-only run at epochs 5 and 20."""
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (DeviceGrid, RatingMatrix, bucket_qbands, build_grid,
                                            shuffle_triples, synthetic_ratings)
    from paper_2006_15980_b200.sgd import DeviceModel, Hyperparams, init_model, rmse
    ref = json.loads((GOLDEN / "training.json").read_text())
    full = synthetic_ratings(6040, 3706, rank=8, density=1.05e6 / (6040 * 3706), noise=0.1, seed=0)
    perm = np.random.default_rng(1).permutation(full.nnz)
    n_test = full.nnz // 21
    te, tr = perm[:n_test], perm[n_test:]
    train = RatingMatrix(6040, 3706, full.users[tr], full.items[tr], full.ratings[tr])
    test = RatingMatrix(6040, 3706, full.users[te], full.items[te], full.ratings[te])
    hp = Hyperparams(n_factors=32, reg_user=0.01, reg_item=0.01, learning_rate=0.01)
    grid = DeviceGrid.from_host(build_grid(shuffle_triples(train, 0), [0, 6040], [0, 1853, 3706]),
                                dev)
    bucket_qbands(grid, 32, impl=5)
    assert grid.sub_split > 1
    model = DeviceModel.from_host(init_model(6040, 3706, hp, 0), dev)
    got = {}
    for epoch in range(1, 21):
        for b in (0, 1):
            kernels.launch_block_qband(model.P, model.Q, grid, b, 0.01, 0.01, 0.01,
                                       kernels.mix64(0, b, epoch))
        if epoch in (1, 5, 20):
            got[f"e{epoch}"] = rmse(test, model).value
    for key in ("e1", "e5", "e20"):
        print(f"{key}: gpu split runs {got[key]:.5f} reference {ref[key]['test_rmse']:.5f}")
    assert abs(got["e20"] - ref["e20"]["test_rmse"]) <= 0.005
    assert abs(got["e5"] - ref["e5"]["test_rmse"]) <= 0.005


@pytest.mark.parametrize("k,dtype", [(32, "float16"), (32, "float32"), (64, "float16"),
                                     (64, "float32"), (128, "float32")])
def test_default_layout_quality_matches_whole_runs(dev, k, dtype):
    """Narrow blocks (600 items each) at 2 % density: run groups over a
    shared-memory P tile (implementation 8), the split-run layout
    (implementation 5: item runs split over the chains, Q deltas) and the
    automatic layout must all train like whole runs on one chain each
    (implementation 4): same synthetic law, same init, test RMSE after 8
    epochs within 0.005 (and all must have learned).  The automatic layout
    picks run groups at k = 128 and, past the staleness bound
    (data.TILE_RESIDENT_MAX_STALE: 128 chains per SM over 600 items), the
    split runs at k = 32 / 64."""
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (bucket_qbands, build_device_grid, split_device,
                                            synthetic_device)
    from paper_2006_15980_b200.sgd import init_device_model, rmse
    d = dev
    trip = synthetic_device(120_000, 1_200, 3_000_000, seed=3, device=d)
    train, test = split_device(trip, 0.05)
    out = {}
    for layout, impl in (("default", None), ("runs", 8), ("split", 5), ("whole", 4)):
        g = build_device_grid(train, [0, 120_000], [0, 600, 1_200])
        bucket_qbands(g, k, elem_bytes=2 if dtype == "float16" else 4, impl=impl)
        model = init_device_model(120_000, 1_200, k, 0, device=d, dtype=dtype)
        first = rmse(test, model).value
        for e in range(8):
            for b in (0, 1):
                kernels.launch_block_qband(model.P, model.Q, g, b, 0.005, 0.05, 0.05,
                                           kernels.mix64(b, e))
        out[layout] = (first, rmse(test, model).value, g.sub_impl, g.sub_split)
    print(out)
    assert out["default"][2] == (8 if k == 128 else 5)
    assert out["runs"][2] == 8
    assert out["split"][3] > 1            # implementation 5 did split the runs
    assert out["whole"][1] < out["whole"][0] - 0.005
    for layout in ("default", "runs", "split"):
        assert abs(out[layout][1] - out["whole"][1]) <= 0.005, out


@pytest.mark.parametrize("k", [32, 64])
def test_default_layout_quality_at_twice_the_paper_rate(dev, k):
    """The staleness bound at work: at lr = 0.01 (twice the paper's) run
    groups on these narrow blocks train 0.008 worse than whole runs (their
    Q changes land after ~15 concurrent runs of the item, profiles/round2/
    s4_stale_margin.jsonl); the automatic layout avoids them and stays
    within 0.002."""
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (bucket_qbands, build_device_grid, split_device,
                                            synthetic_device)
    from paper_2006_15980_b200.sgd import init_device_model, rmse
    trip = synthetic_device(120_000, 1_200, 3_000_000, seed=3, device=dev)
    train, test = split_device(trip, 0.05)
    out = {}
    for layout, impl in (("default", None), ("whole", 4)):
        g = build_device_grid(train, [0, 120_000], [0, 600, 1_200])
        bucket_qbands(g, k, elem_bytes=4, impl=impl)
        model = init_device_model(120_000, 1_200, k, 0, device=dev, dtype="float32")
        for e in range(8):
            for b in (0, 1):
                kernels.launch_block_qband(model.P, model.Q, g, b, 0.01, 0.05, 0.05,
                                           kernels.mix64(b, e))
        out[layout] = (rmse(test, model).value, g.sub_impl)
    print(out)
    assert out["default"][1] != 8
    assert abs(out["default"][0] - out["whole"][0]) <= 0.002, out


@pytest.mark.parametrize("k", [32, 128])
def test_default_layout_quality_skewed_items(dev, k):
    """Zipf-skewed item popularity: the default layout splits hot items' runs
    over chains in proportion to their ratings (Q deltas, publication period
    shrinking with the parts).  It must train like whole runs on one chain
    per item: test RMSE after 6 epochs within 0.005, no divergence."""
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (bucket_qbands, build_device_grid, split_device,
                                            synthetic_device)
    from paper_2006_15980_b200.sgd import init_device_model, rmse
    d = dev
    trip = synthetic_device(200_000, 2_000, 3_000_000, seed=5, device=d)
    g = torch.Generator(device=d)
    g.manual_seed(11)
    w = torch.arange(1, 2_001, device=d, dtype=torch.float64).pow(-0.8)
    trip.items[:] = torch.randperm(2_000, device=d, generator=g)[
        torch.multinomial(w, trip.nnz, replacement=True, generator=g)].to(torch.int32)
    train, test = split_device(trip, 0.05)
    out = {}
    for layout in ("default", "whole"):
        grid = build_device_grid(train, [0, 200_000], [0, 1_000, 2_000])
        bucket_qbands(grid, k, impl=None if layout == "default" else 4)
        model = init_device_model(200_000, 2_000, k, 0, device=d)
        for e in range(6):
            for b in (0, 1):
                kernels.launch_block_qband(model.P, model.Q, grid, b, 0.005, 0.05, 0.05,
                                           kernels.mix64(b, e))
        out[layout] = (rmse(test, model).value, grid.sub_impl, grid.sub_split, grid.sub_qsync)
    print(out)
    assert out["default"][2] > 1                 # hot items were split
    assert np.isfinite(out["default"][0])
    assert abs(out["default"][0] - out["whole"][0]) <= 0.005


def test_qband_fp16_storage_tracks_fp32(dev, qband_impl):
    from paper_2006_15980_b200 import kernels
    m = random_matrix(3000, 800, 200_000, 5)
    g = _qband_grid(dev, m, 128, [0, 800], target=400)
    rng = np.random.default_rng(5)
    P0 = rng.uniform(0, 0.09, size=(3000, 128)).astype(np.float32)
    Q0 = rng.uniform(0, 0.09, size=(800, 128)).astype(np.float32)
    out = {}
    for dt in (torch.float32, torch.float16):
        P, Q = to_dev(P0, dev, dt), to_dev(Q0, dev, dt)
        for e in range(3):
            kernels.launch_block_qband(P, Q, g, 0, 0.002, 0.01, 0.01, e)
        out[dt] = (P.double().cpu().numpy(), Q.double().cpu().numpy())
    assert rel_err(out[torch.float16][0], out[torch.float32][0]) < 5e-3
    assert rel_err(out[torch.float16][1], out[torch.float32][1]) < 5e-3


def test_qband_bucketing_many_subbands(dev):
    """More sub-bands than the histogram bucketing handles (> 12288): the
    stable-sort path keeps the same contract."""
    m = random_matrix(2000, 30000, 300_000, 77)
    g = _qband_grid(dev, m, 128, [0, 30000], target=20000)
    items = g.items.cpu().numpy()
    users = g.users.cpu().numpy()
    ptr = g.sub_ptr[0].cpu().numpy()
    cuts = g.sub_cuts[0].cpu().numpy()
    assert len(cuts) - 1 == 20000 and ptr[-1] == 300_000
    for s in range(0, 20000, 97):
        seg = items[ptr[s]:ptr[s + 1]]
        assert np.all((seg >= cuts[s]) & (seg < cuts[s + 1]))
    # stable item runs: inside an item the original (block) order is preserved
    order = np.argsort(m.items, kind="stable")
    assert np.array_equal(users, m.users[order]) and np.array_equal(items, m.items[order])


@pytest.mark.parametrize("k,dtype", [(128, torch.float32), (32, torch.float32),
                                     (64, torch.float16), (256, torch.float32)])
def test_runs_conflict_free_equals_oracle(dev, k, dtype):
    """Implementation 8 (run groups over a tile-resident P): with distinct users AND distinct
    items nothing races and nothing is stale, so the result is every triple
    applied once from the initial factors — the reference update (oracle,
    f64) within storage rounding — across many row tiles and both blocks."""
    import oracle
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (DeviceTriples, RatingMatrix, bucket_qbands,
                                            build_device_grid)
    rng = np.random.default_rng(k)
    n_users, n_items = 200_000, 30_000
    n = 25_000
    users = rng.permutation(n_users)[:n].astype(np.int32)
    items = rng.permutation(n_items)[:n].astype(np.int32)
    vals = rng.uniform(0, 1, n).astype(np.float32).astype(np.float64)
    m = RatingMatrix(n_users, n_items, users, items, vals)
    g = build_device_grid(DeviceTriples.from_host(m, dev), [0, n_users],
                          [0, n_items // 2, n_items])
    bucket_qbands(g, k, impl=8, elem_bytes=2 if dtype == torch.float16 else 4)
    assert g.sub_impl == 8 and g.sub_tiles[0] > 1
    P0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_users, k)).astype(np.float32)
    Q0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_items, k)).astype(np.float32)
    if dtype == torch.float16:
        P0, Q0 = P0.astype(np.float16).astype(np.float32), Q0.astype(np.float16).astype(np.float32)
    P, Q = to_dev(P0, dev, dtype), to_dev(Q0, dev, dtype)
    got = sum(kernels.launch_block_qband(P, Q, g, b, 0.05, 0.02, 0.03, 7 + b)
              for b in range(g.n_blocks))
    assert got == n
    Pe, Qe = P0.astype(np.float64), Q0.astype(np.float64)
    oracle.sgd_range(Pe, Qe, users, items, vals, 0, n, 0.05, 0.02, 0.03, 1, 0, 0)
    tol = 2e-3 if dtype == torch.float16 else 1e-5
    assert rel_err(P.double().cpu().numpy(), Pe) < tol
    assert rel_err(Q.double().cpu().numpy(), Qe) < tol


def _runs_problem(dev, k, f16, seed, n_users=120_000, n_items=12_000, max_run=13):
    """Distinct users, every item inside one row tile (implementation 8
    tiles): runs never race and never go stale."""
    from paper_2006_15980_b200.data import ptile_row_cuts
    rng = np.random.default_rng(seed)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    tiles = ptile_row_cuts(0, n_users, k, f16, n_sm)
    T = len(tiles) - 1
    free = [list(rng.permutation(np.arange(tiles[t], tiles[t + 1]))) for t in range(T)]
    users, items = [], []
    for v in range(n_items):
        t = v % T
        r = min(len(free[t]), int(rng.integers(1, max_run)))
        for _ in range(r):
            users.append(free[t].pop())
            items.append(v)
    users = np.asarray(users, dtype=np.int32)
    items = np.asarray(items, dtype=np.int32)
    perm = rng.permutation(len(users))
    return users[perm], items[perm], tiles, rng


def test_runs_tile_sizes_interleave(dev):
    """One kernel launched with large, then small, then large P tiles (a
    resident layout and a streamed 256-row one in the same process): the
    dynamic shared-memory limit must never drop under a size launched
    before (util.cu kernel_occupancy)."""
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (DeviceTriples, RatingMatrix, bucket_qbands,
                                            build_device_grid)
    rng = np.random.default_rng(5)
    n_users, n_items, n = 120_000, 3_000, 600_000
    cells = rng.choice(n_users * n_items, n, replace=False)
    m = RatingMatrix(n_users, n_items, (cells // n_items).astype(np.int32),
                     (cells % n_items).astype(np.int32), rng.uniform(0, 1, n))
    P0 = rng.uniform(0, 0.1, size=(n_users, 128)).astype(np.float32)
    Q0 = rng.uniform(0, 0.1, size=(n_items, 128)).astype(np.float32)
    grids = {}
    for rows in (None, 64):
        g = build_device_grid(DeviceTriples.from_host(m, dev), [0, n_users], [0, n_items])
        bucket_qbands(g, 128, impl=8, max_tile_rows=rows)
        grids[rows] = g
    assert grids[None].sub_max_rows > 4 * grids[64].sub_max_rows
    P, Q = torch.from_numpy(P0).to(dev), torch.from_numpy(Q0).to(dev)
    for rows in (None, 64, None):
        assert kernels.launch_block_qband(P, Q, grids[rows], 0, 0.005, 0.05, 0.05, 1) == n
    torch.cuda.synchronize(dev)
    assert bool(torch.isfinite(P).all()) and bool(torch.isfinite(Q).all())


def test_runs_layout_contract(dev):
    """Implementation 8's layout: inside each row tile, runs (one item each,
    the block's order kept) sorted by length, longest first; run / tile
    arrays consistent; every rating present once."""
    from paper_2006_15980_b200.data import (DeviceTriples, RatingMatrix, bucket_qbands,
                                            build_device_grid)
    m = random_matrix(30_000, 2_000, 600_000, 91)
    g = build_device_grid(DeviceTriples.from_host(m, dev), [0, 30_000], [0, 900, 2_000])
    orig = {}
    for b in range(g.n_blocks):
        lo, hi = g.block_range(b)
        orig[b] = (g.users[lo:hi].cpu().numpy(), g.items[lo:hi].cpu().numpy(),
                   g.ratings[lo:hi].cpu().numpy())
    bucket_qbands(g, 128, impl=8)
    assert g.sub_impl == 8
    for b in range(g.n_blocks):
        lo, hi = g.block_range(b)
        u, i, r = (g.users[lo:hi].cpu().numpy(), g.items[lo:hi].cpu().numpy(),
                   g.ratings[lo:hi].cpu().numpy())
        runs = g.sub_ptr[b].cpu().numpy().astype(np.int64)
        ptr = np.concatenate([runs[:, 0], [runs[-1, 0] + runs[-1, 1]]])
        assert np.array_equal(ptr[1:-1], runs[1:, 0])        # runs tile the block
        item = runs[:, 2]
        trun = g.sub_tile_run[b].cpu().numpy()
        tiles = g.sub_tile_rows[b]
        T = g.sub_tiles[b]
        assert len(tiles) == T + 1 and len(trun) == T + 1
        assert ptr[0] == 0 and ptr[-1] == hi - lo and trun[0] == 0 and trun[-1] == len(item)
        lens = np.diff(ptr)
        assert np.all(lens > 0)
        for t in range(T):
            a, z = trun[t], trun[t + 1]
            assert np.all(np.diff(lens[a:z]) <= 0)            # longest first
            seg = slice(ptr[a], ptr[z])
            assert np.all((u[seg] >= tiles[t]) & (u[seg] < tiles[t + 1]))
        # each run is one item; the (tile, item) pairs are distinct
        run_of = np.repeat(np.arange(len(item)), lens)
        assert np.array_equal(i, item[run_of])
        # same multiset of triples; inside a run the block order is kept
        key_new = (u.astype(np.int64) << 20) | i
        ou, oi, orr = orig[b]
        key_old = (ou.astype(np.int64) << 20) | oi
        assert np.array_equal(np.sort(key_new), np.sort(key_old))
        pos_old = {kk: n for n, kk in enumerate(key_old)}
        pos = np.array([pos_old[kk] for kk in key_new])
        for rr in range(0, len(item), 97):
            assert np.all(np.diff(pos[ptr[rr]:ptr[rr + 1]]) > 0)
        assert np.array_equal(r, orr[pos])


@pytest.mark.parametrize("k,dtype,stagger,wide", [(128, torch.float32, False, 0),
                                                  (32, torch.float32, False, 0),
                                                  (32, torch.float32, False, 1),
                                                  (32, torch.float16, False, 1),
                                                  (256, torch.float32, False, 0),
                                                  (64, torch.float16, False, 0),
                                                  (128, torch.float32, True, 0)])
def test_runs_equal_sequential_replay(dev, k, dtype, stagger, wide, monkeypatch):
    """Implementation 8 (run groups): with no P race and no concurrent Q
    deltas (distinct users, items inside one tile) the kernel is exactly a
    sequential replay, run by run, of its visit order — each run from its
    seeded rotation (runs.cuh stage_group) — of the reference update (oracle,
    f64), one rating at a time.  Also with staggered tiles (uneven first
    and last tile per CTA, an empty one among them; data._staggered_cuts)
    and in the k = 32 wide configuration (hmf_qband_opts.runs_wide)."""
    import oracle
    from paper_2006_15980_b200 import data as hdata
    from paper_2006_15980_b200 import kernels
    monkeypatch.setattr(hdata, "PTILE_STAGGER", stagger)
    from paper_2006_15980_b200.data import (DeviceTriples, RatingMatrix, bucket_qbands,
                                            build_device_grid)
    from paper_2006_15980_b200.kernels import _MASK64
    f16 = dtype == torch.float16
    n_users, n_items = 120_000, 12_000
    users, items, tiles, rng = _runs_problem(dev, k, f16, 200 + k, n_users, n_items)
    n = len(users)
    vals = rng.uniform(0, 1, n).astype(np.float32).astype(np.float64)
    m = RatingMatrix(n_users, n_items, users, items, vals)
    g = build_device_grid(DeviceTriples.from_host(m, dev), [0, n_users],
                          [0, n_items // 2, n_items])
    bucket_qbands(g, k, impl=8, elem_bytes=2 if f16 else 4)
    assert g.sub_impl == 8 and all(np.array_equal(r, tiles) for r in g.sub_tile_rows)
    g.sub_wide = wide
    P0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_users, k)).astype(np.float32)
    Q0 = rng.uniform(0, 1 / np.sqrt(k), size=(n_items, k)).astype(np.float32)
    if f16:
        P0, Q0 = P0.astype(np.float16).astype(np.float32), Q0.astype(np.float16).astype(np.float32)
    P, Q = to_dev(P0, dev, dtype), to_dev(Q0, dev, dtype)
    lr, ru, ri = 0.05, 0.02, 0.03
    seeds = [kernels.mix64(5, b) for b in range(g.n_blocks)]
    got = sum(kernels.launch_block_qband(P, Q, g, b, lr, ru, ri, seeds[b])
              for b in range(g.n_blocks))
    assert got == n
    gu, gi = g.users.cpu().numpy(), g.items.cpu().numpy()
    gr = g.ratings.cpu().numpy().astype(np.float64)
    Pe, Qe = P0.astype(np.float64), Q0.astype(np.float64)
    from paper_2006_15980_b200.data import run_rotation
    for b in range(g.n_blocks):
        lo, _ = g.block_range(b)
        runs = g.sub_ptr[b].cpu().numpy().astype(np.int64)
        for r in range(len(runs)):
            first, ln, _, _ = runs[r]
            rot = run_rotation(seeds[b], r, int(ln))
            for p in range(ln):
                i = lo + int(first) + (rot + p) % int(ln)
                oracle.sgd_range(Pe, Qe, gu, gi, gr, i, i + 1, lr, ru, ri, 0, 0, 0)
    tol = 2e-3 if f16 else 1e-5
    assert rel_err(P.double().cpu().numpy(), Pe) < tol
    assert rel_err(Q.double().cpu().numpy(), Qe) < tol


def test_tile_resident_policy(dev):
    """data.tile_resident_impl picks run groups (8) exactly where they win
    (profiles/round2/s3_default_layout_sweep.jsonl): Netflix density (~4.9
    ratings per tile-item), but not a small matrix (fewer tiles than SMs),
    a sparse one (< 2 ratings per tile-item), one with hot items, or narrow
    blocks past the staleness bound."""
    from paper_2006_15980_b200.data import (build_device_grid, synthetic_band,
                                            tile_resident_impl)
    d = dev

    def grid(n_users, n_items, nnz, skew=False):
        tr, _ = synthetic_band(n_users, n_items, nnz, seed=5, device=d)
        if skew:   # one item takes a fifth of the ratings
            tr.items[: tr.nnz // 5] = 7
        return build_device_grid(tr, [0, n_users], [0, n_items // 2, n_items])

    assert tile_resident_impl(grid(120_000, 17_700, 25_000_000), 128, False) == 8
    assert tile_resident_impl(grid(120_000, 17_700, 25_000_000), 32, True) == 8
    assert tile_resident_impl(grid(6_040, 3_706, 1_000_000), 32, False) is None      # 4 tiles
    assert tile_resident_impl(grid(200_000, 60_000, 4_000_000), 128, False) is None  # sparse
    assert tile_resident_impl(grid(120_000, 17_700, 25_000_000, skew=True), 128,
                              False) is None                                         # hot item
    assert tile_resident_impl(grid(120_000, 17_700, 25_000_000), 96, False) is None  # k
    # narrow 600-item blocks: 128 chains per SM (k = 32) put ~15 runs of each
    # item in flight (staleness ~500 > TILE_RESIDENT_MAX_STALE); 64 (k = 128) ~136
    narrow = grid(120_000, 1_200, 3_000_000)
    assert tile_resident_impl(narrow, 32, False) is None
    assert tile_resident_impl(narrow, 128, False) == 8
    # the k = 32 wide configuration (160 / 256 chains per SM) only under the
    # same bound: on at Netflix density, off on the narrow blocks
    from paper_2006_15980_b200.data import bucket_qbands
    assert bucket_qbands(grid(120_000, 17_700, 25_000_000), 32, impl=8).sub_wide == 1
    assert bucket_qbands(grid(120_000, 17_700, 25_000_000), 32, impl=8,
                         elem_bytes=2).sub_wide == 1
    assert bucket_qbands(narrow, 32, impl=8).sub_wide == 0
    assert bucket_qbands(grid(120_000, 17_700, 25_000_000), 64, impl=8).sub_wide == 0
