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
