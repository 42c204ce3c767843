"""Host-side data contract vs the reference's own outputs (tests/golden/data.npz)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN / "data.npz")


def test_synthetic_ratings_bit_identical(gold):
    from paper_2006_15980_b200.data import synthetic_ratings
    s = synthetic_ratings(60, 50, rank=4, density=0.2, noise=0.1, seed=3)
    assert np.array_equal(s.users, gold["syn_users"])
    assert np.array_equal(s.items, gold["syn_items"])
    assert np.array_equal(s.ratings, gold["syn_ratings"])


def test_shuffle_and_build_grid_bit_identical(gold):
    from paper_2006_15980_b200.data import build_grid, shuffle_triples, synthetic_ratings
    sh = shuffle_triples(synthetic_ratings(60, 50, rank=4, density=0.2, noise=0.1, seed=3), 11)
    assert np.array_equal(sh.users, gold["sh_users"])
    assert np.array_equal(sh.ratings, gold["sh_ratings"])
    g = build_grid(sh, [0, 20, 60], [0, 10, 30, 50])
    assert np.array_equal(g.block_ptr, gold["g_ptr"])
    assert np.array_equal(g.users, gold["g_users"])
    assert np.array_equal(g.items, gold["g_items"])
    assert np.array_equal(g.ratings, gold["g_ratings"])


def test_init_model_bit_identical(gold):
    from paper_2006_15980_b200.sgd import Hyperparams, init_model
    m = init_model(7, 5, Hyperparams(n_factors=3), 4)
    assert np.array_equal(m.user_factors, gold["init_P"])
    assert np.array_equal(m.item_factors, gold["init_Q"])


def test_mix64_matches_reference():
    from paper_2006_15980_b200.kernels import mix64
    meta = json.loads((GOLDEN / "golden.json").read_text())["mix64"]
    for parts, value in zip(meta["parts"], meta["values"]):
        assert mix64(*parts) == value


def test_factors_file_round_trip(tmp_path):
    from paper_2006_15980_b200.sgd import FactorModel, load_factors, save_factors
    rng = np.random.default_rng(23)
    model = FactorModel(rng.normal(size=(7, 3)), rng.normal(size=(5, 3)))
    save_factors(tmp_path / "f.bin", model)
    back = load_factors(tmp_path / "f.bin")
    assert np.array_equal(back.user_factors, model.user_factors)
    assert np.array_equal(back.item_factors, model.item_factors)
    raw = (tmp_path / "f.bin").read_bytes()
    assert raw[:5] == b"HMFP1" and len(raw) == 5 + 24 + 8 * (7 * 3 + 3 * 5)
    (tmp_path / "bad.bin").write_bytes(b"XXXXX" + b"\0" * 24)
    with pytest.raises(ValueError, match="magic"):
        load_factors(tmp_path / "bad.bin")


def test_cache_round_trip(tmp_path):
    from paper_2006_15980_b200.data import load_cache, save_cache, synthetic_ratings
    s = synthetic_ratings(30, 20, rank=2, density=0.3, seed=1)
    save_cache(tmp_path / "c.bin", s)
    back = load_cache(tmp_path / "c.bin")
    assert np.array_equal(back.users, s.users) and np.array_equal(back.ratings, s.ratings)


def test_align_ratings_skips_unseen(tmp_path):
    from paper_2006_15980_b200.data import align_ratings, load_ratings
    (tmp_path / "train.txt").write_text("1 1 2.0\n2 2 3.0\n")
    (tmp_path / "test.txt").write_text("1 1 2.0\n9 1 1.0\n1 9 1.0\n")
    u, i, r, skipped = align_ratings(load_ratings(tmp_path / "test.txt"),
                                     load_ratings(tmp_path / "train.txt"))
    assert len(r) == 1 and skipped == 2 and u[0] == 0 and i[0] == 0


def test_qband_row_tiles():
    from paper_2006_15980_b200.data import qband_row_tiles
    # Netflix k=128 fp32: 480 000 rows x 512 B = 246 MB -> 8 tiles of <= 32 MB
    assert qband_row_tiles(480_000, 128, 4) == 8
    assert qband_row_tiles(480_000, 128, 2, max_rows=0) == 4   # fp16 rows, bytes only
    assert qband_row_tiles(480_000, 128, 2) == 8           # at most 65536 users per tile
    assert qband_row_tiles(480_000, 128, 4, tile_bytes=0, max_rows=0) == 1
    assert qband_row_tiles(480_000, 32, 4, tile_bytes=0) == 8
    assert qband_row_tiles(50_000_000, 128, 4) == 763       # Hugewiki on one GPU
    assert qband_row_tiles(100, 128, 4, tile_bytes=1) == 100  # never more tiles than rows


def test_qband_split_policy():
    """data.qband_split_for on the measured configurations."""
    from paper_2006_15980_b200.data import qband_split_for
    slots = 9472
    assert qband_split_for(slots, 8850, 50e6, 8, 128) == 4           # Netflix k=128
    assert qband_split_for(slots, 8850, 50e6, 4, 128, True) == 4     # fp16
    assert qband_split_for(18944, 8850, 50e6, 2, 32) == 2            # k=32: chains > items
    assert qband_split_for(slots, 1853, 5e5, 1, 32) == 5             # ML-1M
    assert qband_split_for(slots, 20_000, 1.55e9, 763) == 1          # Hugewiki: whole runs
    assert qband_split_for(slots, 312_500, 1.25e8, 16) == 1          # Yahoo
    assert qband_split_for(slots, 2353, 22.8e6, 100) == 4            # 8-GPU Hugewiki band
    assert qband_split_for(slots, 8000, 124e6, 381) == 2             # 2-GPU Hugewiki band
    assert qband_split_for(slots, 40, 1e6, 1) == 16                  # capped
    assert qband_split_for(slots, 0, 0.0, 1) == 1


def test_bench_l2_ceiling_lookup():
    """bench.l2_ceiling reads the committed microbenchmark (a B200 measurement)."""
    import bench
    f32, f16 = bench.l2_ceiling(128, "f32"), bench.l2_ceiling(128, "f16")
    assert f32 is not None and 8e9 < f32 < 12e9          # 512-byte rows, load + reduction
    assert f16 is not None and f16 > 1.5 * f32           # 256-byte rows
    assert bench.bytes_per_update(128, "f32") == 2060
    assert bench.bytes_per_update(128, "f16") == 12 + 8 * 128
    st = bench.l2_ceiling(128, "f32", stores=True)
    assert st is not None and st > f32                   # load + store beats load + reduction


def test_stream_chunk_cuts():
    """workers.chunk_cuts: runs of tiles per chunk, an optional short last chunk."""
    from paper_2006_15980_b200.workers import chunk_cuts
    assert chunk_cuts(8, 4) == [0, 4, 8]
    assert chunk_cuts(8, 4, 1) == [0, 4, 7, 8]
    assert chunk_cuts(8, 3) == [0, 3, 6, 8]
    assert chunk_cuts(3, 1) == [0, 1, 2, 3]
    assert chunk_cuts(3, 2, 1) == [0, 2, 3]
    assert chunk_cuts(1, 4, 1) == [0, 1]                 # one tile: no separate last chunk
    assert chunk_cuts(15, 4) == [0, 4, 8, 12, 15]


def test_ptile_row_cuts():
    """Row tiles of the shared-memory P tile (implementations 7 and 8): every
    tile fits hmf_ptile_max_rows, tiles are equal to within one row, at least
    one per SM once that leaves >= PTILE_MIN_ROWS rows each, and a multiple of
    the SM count when more than half the SMs get one."""
    from paper_2006_15980_b200 import _lib
    from paper_2006_15980_b200.data import PTILE_MIN_ROWS, ptile_row_cuts
    lib = _lib.load()
    for k, f16 in ((128, False), (32, False), (256, False), (64, True)):
        cap = lib.hmf_ptile_max_rows(k, 1 if f16 else 0)
        assert cap == 208 * 1024 // (k * (2 if f16 else 4))
        for lo, hi in ((0, 480_000), (1000, 121_000), (0, 6040), (5, 9_000)):
            cuts = ptile_row_cuts(lo, hi, k, f16, 148)
            sizes = np.diff(cuts)
            T = len(sizes)
            assert cuts[0] == lo and cuts[-1] == hi and np.all(sizes > 0)
            assert sizes.max() <= cap and sizes.max() - sizes.min() <= 1
            if hi - lo >= 148 * PTILE_MIN_ROWS:
                assert T >= 148 and T % 148 == 0
    # NF at k=128 fp32: 1 184 tiles of ~405 users per block
    assert len(ptile_row_cuts(0, 480_000, 128, False, 148)) - 1 == 1184


def test_run_rotation_range_and_spread():
    """Implementation 8's per-run start rotation (csrc/runs.cuh run_rotation,
    restated in data.run_rotation): always inside the run, spread over it,
    and a function of (seed, run) only."""
    from paper_2006_15980_b200.data import run_rotation
    for length in (1, 2, 5, 17, 416):
        rots = [run_rotation(123456789, r, length) for r in range(4000)]
        assert min(rots) >= 0 and max(rots) < length
        counts = np.bincount(rots, minlength=length)
        if 1 < length <= 17:
            assert counts.min() > 0.5 * 4000 / length
        elif length > 17:
            assert (counts > 0).mean() > 0.95
    assert run_rotation(7, 3, 10) == run_rotation(7, 3, 10)
    assert [run_rotation(s, 3, 1000) for s in range(5)] != [run_rotation(0, 3, 1000)] * 5


def test_staggered_tile_cuts():
    """data._staggered_cuts: CTA i (tiles i, i + n_sm, ...) gets an uneven
    first and last tile (f_i and 1 - f_i of a full one) and full tiles in
    between, so every CTA trains the same rows and the tile switches of
    different CTAs fall at different times; cuts are monotonic and cover
    the band exactly."""
    import numpy as np
    from paper_2006_15980_b200.data import _staggered_cuts
    n_sm, waves = 148, 8
    cuts = _staggered_cuts(1000, 481_000, waves, n_sm)
    sizes = np.diff(cuts)
    assert cuts[0] == 1000 and cuts[-1] == 481_000 and np.all(sizes >= 0)
    assert len(sizes) == (waves + 1) * n_sm
    per_cta = sizes.reshape(waves + 1, n_sm).sum(axis=0)
    assert per_cta.max() - per_cta.min() <= waves + 1  # rounding only
    first = sizes[:n_sm]
    assert len(np.unique(first)) > n_sm // 2          # switches spread out
    assert np.all(sizes[n_sm:-n_sm] >= 405) and np.all(sizes <= 406)


def test_run_group_staleness_bound():
    """data.run_group_staleness against the numbers the layout policy was
    calibrated on: Netflix at N = 1 (two 8 850-item blocks,
    50 M ratings, 1 184 tiles, 128 chains per SM) ~10.5; one of 17 column
    bands at N = 8 ~89; the narrow 600-item blocks at 2 % density ~500
    (k = 32: 128 chains, 148 tiles) — over TILE_RESIDENT_MAX_STALE; and the
    k = 32 wide configuration (160 chains) stays far under it at NF."""
    from paper_2006_15980_b200.data import TILE_RESIDENT_MAX_STALE, run_group_staleness
    nf = run_group_staleness(128, 148, 50_000_000, 1184, 8_850)
    assert 9 < nf < 12
    band8 = run_group_staleness(128, 148, 100_000_000 // 17, 1184, 17_700 // 17)
    assert 80 < band8 < 100 < TILE_RESIDENT_MAX_STALE
    narrow = run_group_staleness(128, 148, 1_425_000, 148, 600)
    assert narrow > TILE_RESIDENT_MAX_STALE
    assert run_group_staleness(160, 148, 50_000_000, 296, 8_850) < 60
