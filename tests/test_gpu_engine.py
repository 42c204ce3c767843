"""The CUDA batch engine behind the reference's seams (workers / engine),
modelled on the reference's tests/test_workers.py and test_acceptance.py."""

import json

import ctypes

import numpy as np
import pytest

from conftest import GOLDEN, random_matrix

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return 0


def test_staging_round_trip_leaves_factors_unchanged(dev):
    """workers.py stage_rows/stage_in/stage_out/flush_rows, f64 storage."""
    from paper_2006_15980_b200.data import build_grid
    from paper_2006_15980_b200.scheduler import Unit
    from paper_2006_15980_b200.sgd import Hyperparams, init_model
    from paper_2006_15980_b200.workers import BatchEngine, BatchWorkerConfig
    m = random_matrix(20, 20, 133, 3)
    grid = build_grid(m, [0, 20], [0, 20])
    hp = Hyperparams(n_factors=4)
    model = init_model(20, 20, hp, 3)
    before = model.copy()
    eng = BatchEngine(BatchWorkerConfig(device=dev, precision="f64", kernel="range"), model, hp)
    assert eng.stage_rows(0, 20) >= 0
    assert eng.stage_in("k", grid, Unit(blocks=(0,), rows=(0,), col=0)) >= 0
    eng.stage_out("k")
    eng.flush_rows()
    eng.close()
    assert np.array_equal(model.user_factors, before.user_factors)
    assert np.array_equal(model.item_factors, before.item_factors)


def test_batch_worker_exact_equals_reference_stream_replay(dev):
    """A CUDA batch worker in EXACT mode over a real lease sequence equals the
    reference algorithm replayed serially over the same leases, bit for bit
    (reference tests/test_workers.py:43-70 and 155-183)."""
    import oracle
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import build_grid
    from paper_2006_15980_b200.scheduler import CLASS_BATCH, POLICY_QUOTA, GridScheduler
    from paper_2006_15980_b200.sgd import Hyperparams, init_model
    from paper_2006_15980_b200.workers import BatchWorker, BatchWorkerConfig, FactorStore
    m = random_matrix(48, 48, 48 * 48 // 3, 7)
    grid = build_grid(m, [0, 24, 48], [0, 16, 32, 48])
    hp = Hyperparams(n_factors=4, reg_user=0.01, reg_item=0.01, learning_rate=0.02)
    model = init_model(48, 48, hp, 7)
    start = model.copy()
    store = FactorStore(model, "f64", grid)
    sched = GridScheduler(grid, POLICY_QUOTA, max_epochs=3, seed=7, trace=True)
    cfg = BatchWorkerConfig(device=dev, precision="f64", kernel="range", mode="exact")
    w = BatchWorker(0, sched, model, grid, hp, cfg, store)
    w.start()
    w.join(timeout=120)
    assert w.error is None and sched.epoch == 3
    store.sync_host()
    P, Q = start.user_factors.copy(), start.item_factors.copy()
    counts = np.zeros(grid.n_blocks, dtype=np.int64)
    for ev in sched.trace:
        b = ev.block
        unit_seed = kernels.mix64(7, b, int(counts[b]))
        lo, hi = grid.block_range(b)
        oracle.sgd_range(P, Q, grid.users, grid.items, grid.ratings, lo, hi, 0.02, 0.01, 0.01,
                         kernels.mix64(unit_seed, 0), 0, 0)
        counts[b] += 1
    assert np.array_equal(model.user_factors, P)
    assert np.array_equal(model.item_factors, Q)


def test_run_training_ml1m_quality(dev):
    """run_training (batch-only, 1 GPU, Q-band kernel) on the ML-1M-shaped
    instance: test RMSE within 0.005 of the reference's after 20 epochs, the
    per-epoch metrics on device, and every block updated once per epoch."""
    from paper_2006_15980_b200.data import RatingMatrix, synthetic_ratings
    from paper_2006_15980_b200.engine import RunConfig, run_training
    ref = json.loads((GOLDEN / "training.json").read_text())
    full = synthetic_ratings(6040, 3706, rank=8, density=1.05e6 / (6040 * 3706), noise=0.1, seed=0)
    perm = np.random.default_rng(1).permutation(full.nnz)
    n_test = full.nnz // 21
    te, tr = perm[:n_test], perm[n_test:]
    train = RatingMatrix(6040, 3706, full.users[tr], full.items[tr], full.ratings[tr])
    test = RatingMatrix(6040, 3706, full.users[te], full.items[te], full.ratings[te])
    cfg = RunConfig(n_factors=32, learning_rate=0.01, reg_user=0.01, reg_item=0.01, epochs=20,
                    seed=0, n_batch=1, devices=(dev,))
    res = run_training(cfg, matrix=train, testset=test)
    assert res.epochs_run == 20 and len(res.metrics) == 20
    assert np.all(res.scheduler.counts == 20)
    assert res.scheduler.total_updates == 20 * train.nnz
    print("gpu", [round(r.test_rmse, 5) for r in res.metrics][:5], res.test_report.value,
          "reference", ref["e20"]["test_rmse"])
    assert abs(res.test_report.value - ref["e20"]["test_rmse"]) <= 0.005
    assert abs(res.metrics[4].test_rmse - ref["e5"]["test_rmse"]) <= 0.005
    assert res.metrics[-1].train_loss < res.metrics[0].train_loss
    assert res.model.all_finite()


def test_run_training_rejects_cpu_schedules():
    from paper_2006_15980_b200.engine import ConfigError, RunConfig
    with pytest.raises(ConfigError):
        RunConfig(schedule="stream-only", n_stream=2, synthetic=True).validate()
    with pytest.raises(ConfigError):
        RunConfig(schedule="hsgd-star", division="nonuniform", n_stream=2, n_batch=1,
                  synthetic=True).validate()


def test_gpu_calibration_fits_profile(dev, tmp_path):
    from paper_2006_15980_b200.costmodel import (DeviceTopology, calibrate_gpu, load_profile,
                                                 save_profile)
    from paper_2006_15980_b200.data import shuffle_triples, synthetic_ratings
    from paper_2006_15980_b200.sgd import Hyperparams
    from paper_2006_15980_b200.workers import BatchWorkerConfig
    m = shuffle_triples(synthetic_ratings(4000, 3000, rank=8, density=0.15, seed=1), 1)
    prof = calibrate_gpu(m, Hyperparams(n_factors=64), BatchWorkerConfig(device=dev),
                         DeviceTopology(0, 1), segments=8, repeats=3)
    # stage curves are fitted from CUDA-event timings; the kernel stage grows
    # with the workload (the transfer stages are PCIe-noise dominated here)
    assert prof.kernel.eval(m.nnz) > 0
    assert prof.kernel.eval(m.nnz) > prof.kernel.eval(m.nnz // 8)
    for stage in (prof.transfer_in, prof.transfer_out):
        assert np.isfinite(stage.eval(m.nnz))
    save_profile(tmp_path / "prof.txt", prof)
    assert load_profile(tmp_path / "prof.txt").kernel == prof.kernel


def test_throughput_sweep_reports_stages(dev):
    from paper_2006_15980_b200.sgd import Hyperparams
    from paper_2006_15980_b200.workers import BatchWorkerConfig, throughput_sweep
    out = throughput_sweep("batch", [10_000, 400_000], repeats=2, hparams=Hyperparams(n_factors=32),
                           batch_config=BatchWorkerConfig(device=dev), n_rows=2048, n_cols=2048)
    assert [r["size"] for r in out] == [10_000, 400_000]
    for r in out:
        assert r["kernel_seconds"] > 0 and r["stage_in_seconds"] > 0
        assert r["seconds"] >= r["kernel_seconds"]
    with pytest.raises(ValueError):
        throughput_sweep("batch", [2, 1], batch_config=BatchWorkerConfig(device=dev))


@pytest.mark.parametrize("k,impl,tiles,last", [(64, -1, 1, 0), (128, -1, 1, 0), (64, 0, 1, 0),
                                                (128, -1, 2, 0), (64, -1, 3, 0), (64, 0, 3, 0),
                                                (128, -1, 2, 1), (64, 0, 3, 1)])
def test_streaming_epoch_applies_every_triple_once(dev, k, impl, tiles, last):
    """StreamingEpoch (triples streamed from pinned host memory in chunks of
    `tiles` row tiles, double buffered) on conflict-free triples equals the
    reference update of each triple exactly once."""
    import oracle
    from paper_2006_15980_b200.data import DeviceTriples, build_device_grid
    from paper_2006_15980_b200.sgd import Hyperparams
    from paper_2006_15980_b200.workers import StreamingEpoch
    from paper_2006_15980_b200.data import RatingMatrix
    rng = np.random.default_rng(3)
    n = 6000
    users = rng.permutation(9000)[:n].astype(np.int32)
    items = rng.permutation(7000)[:n].astype(np.int32)
    vals = rng.uniform(0, 1, n).astype(np.float32).astype(np.float64)
    m = RatingMatrix(9000, 7000, users, items, vals)
    d = torch.device("cuda", dev)
    g = build_device_grid(DeviceTriples.from_host(m, d), [0, 9000], [0, 3500, 7000])
    se = StreamingEpoch(g, k, tile_bytes=9000 * k * 4 // 3 + 1,   # 3 row tiles per block
                        tiles_per_chunk=tiles, last_chunk_tiles=last, n_buffers=2,
                        reuse=True, impl=impl)
    se_all = StreamingEpoch(g, k, tile_bytes=9000 * k * 4 // 3 + 1, tiles_per_chunk=tiles,
                            last_chunk_tiles=last, reuse=False, impl=impl)
    assert se.n_chunks == 2 * ((1 + -(-2 // tiles)) if last else -(-3 // tiles))
    P0 = rng.uniform(0, 0.1, size=(9000, k)).astype(np.float32)
    Q0 = rng.uniform(0, 0.1, size=(7000, k)).astype(np.float32)
    P, Q = torch.from_numpy(P0).to(d), torch.from_numpy(Q0).to(d)
    hp = Hyperparams(n_factors=k, reg_user=0.02, reg_item=0.03, learning_rate=0.05)
    assert se.run(P, Q, hp, seed=1) == n
    torch.cuda.synchronize()
    Pe, Qe = P0.astype(np.float64), Q0.astype(np.float64)
    oracle.sgd_range(Pe, Qe, users, items, vals, 0, n, 0.05, 0.02, 0.03, 1, 0, 0)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    assert rel(P.double().cpu().numpy(), Pe) < 1e-6
    assert rel(Q.double().cpu().numpy(), Qe) < 1e-6
    # the chained kernel (default) with single-item sub-bands: items implicit,
    # 2-byte user ids relative to the row tile; warp-per-rating: triples
    chained = impl != 0
    assert se.implicit_items == chained and se.u16 == chained
    assert se.h2d_bytes == (6 if chained else 12) * n
    assert se.h2d_bytes_last() == se.h2d_bytes          # first epoch: every chunk uploaded
    # a second epoch starts on the two chunks still staged and does not upload them
    assert se.run(P, Q, hp, seed=2) == n
    torch.cuda.synchronize()
    assert se.h2d_bytes_last() < se.h2d_bytes
    assert se.h2d_bytes_last() > 0 or se.n_chunks <= se.n_buffers
    # without reuse every epoch uploads all of its triples
    for e in range(2):
        assert se_all.run(P, Q, hp, seed=3 + e) == n
        assert se_all.h2d_bytes_last() == se_all.h2d_bytes


def test_u16_single_tile_entry_equals_tiles_entry(dev):
    """hmf_sgd_block_qband_u16_* (one tile, row_base = -first row) and
    hmf_sgd_block_qband_u16_tiles_* (first rows per tile) update the same
    rows the same way: whole item runs (implementation 4), distinct users."""
    from paper_2006_15980_b200 import _lib
    from paper_2006_15980_b200.data import DeviceTriples, RatingMatrix, bucket_qbands, build_device_grid
    lib = _lib.load()
    rng = np.random.default_rng(8)
    n_users, n_items, k = 50_000, 300, 64
    n = 20_000
    users = (10_000 + rng.permutation(40_000)[:n]).astype(np.int32)   # one tile: rows 10000..49999
    items = rng.integers(0, n_items, n).astype(np.int32)
    vals = rng.uniform(0, 1, n).astype(np.float32).astype(np.float64)
    d = torch.device("cuda", dev) if isinstance(dev, int) else dev
    m = RatingMatrix(n_users, n_items, users, items, vals)
    g = build_device_grid(DeviceTriples.from_host(m, d), [0, n_users], [0, n_items])
    bucket_qbands(g, k, tile_bytes=0, target=n_items, impl=4)
    assert g.sub_tiles == [1] and g.sub_impl == 4
    sc, sp = g.sub_cuts[0], g.sub_ptr[0]
    assert bool(torch.all(sc[1:] - sc[:-1] == 1))      # one item per sub-band: cols = NULL
    rel16 = (g.users - 10_000).to(torch.int32).to(torch.int16)
    first = torch.tensor([10_000], dtype=torch.int32, device=d)
    P0 = rng.uniform(0, 0.1, size=(n_users, k)).astype(np.float32)
    Q0 = rng.uniform(0, 0.1, size=(n_items, k)).astype(np.float32)
    opts = _lib.QbandOpts(impl=4)
    out = []
    for tiles in (False, True):
        P, Q = torch.from_numpy(P0).to(d), torch.from_numpy(Q0).to(d)
        s = torch.cuda.current_stream(d).cuda_stream
        head = (P.data_ptr(), Q.data_ptr(), k, rel16.data_ptr(), 0, g.ratings.data_ptr(),
                sp.data_ptr(), sc.data_ptr(), int(sc.numel()) - 1, 1)
        if tiles:
            got = lib.hmf_sgd_block_qband_u16_tiles_f32(*head, first.data_ptr(),
                                                         ctypes.byref(opts), 0.05, 0.02, 0.03, 5,
                                                         0, s)
        else:
            got = lib.hmf_sgd_block_qband_u16_f32(*head, ctypes.byref(opts), 0.05, 0.02, 0.03, 5,
                                                   -10_000, 0, s)
        _lib.check(got, "u16 entry")
        torch.cuda.synchronize(d)
        out.append((P.cpu().numpy(), Q.cpu().numpy()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert not np.array_equal(out[0][0], P0)


def test_concurrent_layouts_equal_serial(dev):
    """ABI 4: launch options are per call.  Two threads launch two different
    layouts at once (implementation 4 with P by stores, configuration 5;
    implementation 0, warp per rating), each on its own stream and factors.
    With distinct users and whole item runs both kernels are deterministic, so
    the concurrent results equal the serial ones bit for bit — impossible
    when options were process-wide (one thread's settings leaked into the
    other's launches)."""
    import threading
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (DeviceTriples, RatingMatrix, bucket_qbands,
                                            build_device_grid)
    d = torch.device("cuda", dev) if isinstance(dev, int) else dev
    rng = np.random.default_rng(31)
    k, n_users, n_items, n = 128, 60_000, 400, 30_000
    cases = []
    for impl, opts in ((4, {"pstore": 1, "chain_cfg": 5}), (0, {})):
        users = rng.permutation(n_users)[:n].astype(np.int32)
        items = rng.integers(0, n_items, n).astype(np.int32)
        vals = rng.uniform(0, 1, n).astype(np.float32).astype(np.float64)
        m = RatingMatrix(n_users, n_items, users, items, vals)
        g = build_device_grid(DeviceTriples.from_host(m, d), [0, n_users], [0, n_items])
        bucket_qbands(g, k, impl=impl, target=n_items if impl else 50, tile_bytes=0)
        assert g.sub_impl == impl
        P0 = rng.uniform(0, 0.1, size=(n_users, k)).astype(np.float32)
        Q0 = rng.uniform(0, 0.1, size=(n_items, k)).astype(np.float32)
        cases.append((g, opts, P0, Q0))

    def run(case, stream, out, i, reps=20):
        g, opts, P0, Q0 = case
        with torch.cuda.stream(stream):
            P, Q = torch.from_numpy(P0).to(d), torch.from_numpy(Q0).to(d)
            for r in range(reps):
                kernels.launch_block_qband(P, Q, g, 0, 0.01, 0.02, 0.03, 50 + r,
                                           stream=stream.cuda_stream, opts=opts)
            stream.synchronize()
            out[i] = (P.cpu().numpy(), Q.cpu().numpy())

    streams = [torch.cuda.Stream(device=d) for _ in cases]
    serial = [None, None]
    for i, c in enumerate(cases):
        run(c, streams[i], serial, i)
    conc = [None, None]
    ts = [threading.Thread(target=run, args=(c, streams[i], conc, i)) for i, c in enumerate(cases)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for a, b in zip(serial, conc):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("k,chunks,max_rows", [(128, 2, None), (32, 3, None), (256, 1, None),
                                              (128, 2, 256)])
def test_streaming_epoch_runs_equals_resident_launches(dev, k, chunks, max_rows):
    """StreamingEpoch over an implementation-8 layout (run groups): 6 bytes
    per rating from pinned host memory (uint16 tile-relative users + the
    rating; items from the resident run descriptors) — 5 when the tiles hold
    at most 256 users (one-byte ids: k=256, or tiles capped at 256) — whole
    fractions of a block per launch.  On triples whose runs never race or go stale it
    equals the resident launches of the same layout under the same seeds —
    and the first upload replaced poisoned device copies."""
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (DeviceTriples, RatingMatrix, bucket_qbands,
                                            build_device_grid, ptile_row_cuts)
    from paper_2006_15980_b200.sgd import Hyperparams
    from paper_2006_15980_b200.workers import StreamingEpoch
    d = torch.device("cuda", dev)
    rng = np.random.default_rng(k)
    n_users, n_items = 90_000, 9_000
    n_sm = torch.cuda.get_device_properties(d).multi_processor_count
    tiles = ptile_row_cuts(0, n_users, k, False, n_sm, max_rows)
    T = len(tiles) - 1
    free = [list(rng.permutation(np.arange(tiles[t], tiles[t + 1]))) for t in range(T)]
    users, items = [], []
    for v in range(n_items):
        t = v % T
        for _ in range(min(len(free[t]), int(rng.integers(1, 9)))):
            users.append(free[t].pop())
            items.append(v)
    users, items = np.asarray(users, np.int32), np.asarray(items, np.int32)
    vals = rng.uniform(0, 1, len(users)).astype(np.float32).astype(np.float64)
    m = RatingMatrix(n_users, n_items, users, items, vals)
    g = build_device_grid(DeviceTriples.from_host(m, d), [0, n_users], [0, 4_000, n_items])
    bucket_qbands(g, k, impl=8, max_tile_rows=max_rows)
    se = StreamingEpoch(g, k, runs_chunks_per_block=chunks)
    one_byte = int(g.sub_max_rows) <= 256
    assert se.runs and se.u16 and se.implicit_items and se.u8 == one_byte
    assert se.h2d_bytes == (5 if one_byte else 6) * len(users)
    assert se.n_chunks == sum(len(range(0, t, -(-t // chunks))) for t in g.sub_tiles)
    P0 = rng.uniform(0, 0.1, size=(n_users, k)).astype(np.float32)
    Q0 = rng.uniform(0, 0.1, size=(n_items, k)).astype(np.float32)
    hp = Hyperparams(n_factors=k, reg_user=0.02, reg_item=0.03, learning_rate=0.05)
    P, Q = torch.from_numpy(P0).to(d), torch.from_numpy(Q0).to(d)
    # the streamed epoch reads only what it uploads: poison the device arrays
    saved = (g.users.clone(), g.ratings.clone())
    g.users.fill_(-1)
    g.ratings.fill_(float("nan"))
    assert se.run(P, Q, hp, seed=7) == len(users)
    torch.cuda.synchronize()
    g.users.copy_(saved[0])
    g.ratings.copy_(saved[1])
    # the oracle replay: block b's chunk c runs under mix64(mix64(seed, b), c);
    # with no races the order of runs does not matter, each run from its
    # seeded rotation (data.run_rotation), one rating at a time
    import oracle
    from paper_2006_15980_b200.data import run_rotation
    gu, gi = g.users.cpu().numpy(), g.items.cpu().numpy()
    gr = g.ratings.cpu().numpy().astype(np.float64)
    Pe, Qe = P0.astype(np.float64), Q0.astype(np.float64)
    for b, (chs, _) in enumerate(se.blocks):
        blo, _ = g.block_range(b)
        bseed = kernels.mix64(7, b) & 0xFFFFFFFFFFFFFFFF
        runs = g.sub_ptr[b].cpu().numpy().astype(np.int64)
        trun = g.sub_tile_run[b].cpu().numpy()
        for c, (lo, hi, nt, off, t0) in enumerate(chs):
            tseed = kernels.mix64(bseed, c) & 0xFFFFFFFFFFFFFFFF
            for r in range(trun[t0], trun[t0 + nt]):
                first, ln = int(runs[r, 0]), int(runs[r, 1])
                rot = run_rotation(tseed, r, ln)
                for p in range(ln):
                    i = blo + first + (rot + p) % ln
                    oracle.sgd_range(Pe, Qe, gu, gi, gr, i, i + 1, 0.05, 0.02, 0.03, 0, 0, 0)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    assert rel(P.double().cpu().numpy(), Pe) < 1e-5
    assert rel(Q.double().cpu().numpy(), Qe) < 1e-5
