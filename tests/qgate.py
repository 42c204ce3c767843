"""Quality gate helper (test infrastructure): the headline kernel path vs the
unmodified reference's CPU training on identical triples and initial factors.

GPU side: exactly the bench's path (bench.py run_ours) — the 1-GPU uniform
1 x 2 plan (partition.py:89-107), data.bucket_qbands' automatic layout (at
Netflix shape: implementation 5, item runs split 4 ways, P written back by
stores in fp32, the dynamic unit scheduler), one launch per block per epoch
with the scheduler's seed chain.  Reference side: hetmf.run_training(
RunConfig(schedule="stream-only", ...)) (engine.py:190-268) from oracle/_ref,
numba sgd_range on the host cores, its own per-epoch test RMSE.
"""

from __future__ import annotations

import os

import numpy as np

LR, REG = 0.005, 0.05        # the bench's (the paper's)


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def problem(n_users, n_items, nnz, seed, device):
    """Identical triples for both sides: the device generator's matrix
    (synthetic_band, the bench's), train/test copied to the host."""
    from paper_2006_15980_b200.data import synthetic_band
    train, test = synthetic_band(n_users, n_items, nnz, seed=seed, device=device)
    host = lambda t: (t.users.cpu().numpy(), t.items.cpu().numpy(),  # noqa: E731
                      t.ratings.cpu().numpy().astype(np.float64))
    return train, test, host(train), host(test)


def reference_rmse(hetmf, n_users, n_items, k, tr, te, epochs, seed=0, threads=None):
    """Per-epoch test RMSE of the reference's stream-only training, and its
    initial factors (init_model(seed), sgd.py:77-89)."""
    M = hetmf.RatingMatrix
    train = M(n_users, n_items, tr[0], tr[1], tr[2])
    test = M(n_users, n_items, te[0], te[1], te[2])
    cfg = hetmf.RunConfig(schedule="stream-only", n_stream=threads or host_threads(),
                          n_factors=k, learning_rate=LR, reg_user=REG, reg_item=REG,
                          epochs=epochs, seed=seed, log_train_loss=False)
    res = hetmf.run_training(cfg, matrix=train, testset=test)
    init = hetmf.init_model(n_users, n_items, cfg.hyperparams(), seed)
    return [m.test_rmse for m in res.metrics], init


def ours_rmse(train, test, init, k, precision, epochs, seed=0, opts=None, impl=None):
    """Per-epoch test RMSE of the bench's GPU path; returns (rmses, grid)."""
    import torch
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import bucket_qbands, build_device_grid
    from paper_2006_15980_b200.sgd import DeviceModel, rmse
    dev = train.users.device
    n_users, n_items = train.n_users, train.n_items
    grid = build_device_grid(train, np.array([0, n_users]),
                             np.array([0, (n_items + 1) // 2, n_items]))
    bucket_qbands(grid, k, elem_bytes=2 if precision == "f16" else 4, impl=impl)
    dt = torch.float16 if precision == "f16" else torch.float32
    model = DeviceModel(torch.from_numpy(init.user_factors).to(dev, dt).contiguous(),
                        torch.from_numpy(init.item_factors).to(dev, dt).contiguous())
    counts = np.zeros(grid.n_blocks, dtype=np.int64)
    out = []
    for _ in range(epochs):
        for b in range(grid.n_blocks):
            s = kernels.mix64(kernels.mix64(seed, b, int(counts[b])), 0)
            kernels.launch_block_qband(model.P, model.Q, grid, b, LR, REG, REG, s, opts=opts)
            counts[b] += 1
        out.append(rmse(test, model).value)
    return out, grid
