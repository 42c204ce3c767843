"""The bench's own configuration, quality-gated at full size (B200).

BASELINE configs[1] exactly: a Netflix-shaped 480 000 x 17 700 matrix with
100 M training ratings (the synthetic law, device generator, 5 % held out),
k = 128, fp32, lr = 0.005, reg = 0.05, the 1 x 2 plan.  The GPU side is
bench.py's path — data.bucket_qbands' automatic layout (run groups over a
shared-memory P tile, implementation 8) and one launch per block per epoch —
and the reference side is the unmodified hetmf.run_training(stream-only) on
the host cores (oracle/_ref), both from identical initial factors on the
identical triples.  North star: test RMSE within 0.005 of the reference after
the same epochs; every epoch is checked.
"""

import numpy as np
import pytest

import qgate

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N_USERS, N_ITEMS, EPOCHS, K = 480_000, 17_700, 4, 128
NNZ = int(round(100_000_000 / 0.95))      # bench.py: 100 M training ratings + 5 % test


@pytest.fixture(scope="module")
def hetmf():
    from oracle import reference
    if not reference.installed():
        pytest.skip("reference not installed under oracle/_ref (__graft_entry__.build())")
    return reference.hetmf()


@pytest.mark.parametrize("k,precision", [(K, "f32"), (32, "f32"), (32, "f16")])
def test_netflix_full_size_rmse_within_0005_of_reference(hetmf, k, precision):
    """Also at k = 32 (BASELINE configs[4]), where the layout picks the wide
    run-group configuration (160 / 256 chains per SM) under the staleness
    bound."""
    train, test, tr, te = qgate.problem(N_USERS, N_ITEMS, NNZ, seed=0,
                                        device=torch.device("cuda", 0))
    ref, init = qgate.reference_rmse(hetmf, N_USERS, N_ITEMS, k, tr, te, EPOCHS)
    ours, grid = qgate.ours_rmse(train, test, init, k, precision, EPOCHS)
    print(f"NF full size k={k} {precision}: layout impl {grid.sub_impl} wide {grid.sub_wide} "
          f"tiles {grid.sub_tiles}; "
          f"ours {np.round(ours, 5).tolist()} reference {np.round(ref, 5).tolist()}")
    assert grid.sub_impl == 8
    assert grid.sub_wide == (1 if k == 32 else 0)
    gaps = np.abs(np.asarray(ours) - np.asarray(ref))
    assert np.all(gaps <= 0.005), (ours, ref)
