#!/usr/bin/env python
"""Netflix-scale throughput through the drop-in driver surface:
paper_2006_15980_b200.run_training (the reference's engine.py:190-268 entry
point: host shuffle, plan, grid, init, GridScheduler, BatchWorker lease loop
over BatchEngine, per-epoch device metrics) on the bench's NF-shaped
workload (480 000 x 17 700, 100 M ratings, k = 128, fp32).

The ratings are generated on the device (the reference law,
data.synthetic_device) and handed to run_training as host RatingMatrix
arrays, as a reference user would.  Per-epoch time is the spacing of the
TrainResult metrics rows (each includes the epoch-end device test RMSE);
setup (host shuffle, grid build, upload) is reported separately.

    python scripts/run_training_nf.py [--epochs 6] > out.json
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=6)
    ap.add_argument("--k", type=int, default=128)
    args = ap.parse_args()
    import torch
    from paper_2006_15980_b200 import RunConfig, run_training
    from paper_2006_15980_b200.data import split_device, synthetic_device
    dev = torch.device("cuda", 0)
    n_users, n_items, n_total = 480_000, 17_700, 105_263_158
    t0 = time.perf_counter()
    trip = synthetic_device(n_users, n_items, n_total, seed=0, device=dev)
    train_d, test_d = split_device(trip, 0.05)
    train, test = train_d.to_host(), test_d.to_host()
    del trip, train_d, test_d
    torch.cuda.empty_cache()
    gen_s = time.perf_counter() - t0
    cfg = RunConfig(n_factors=args.k, learning_rate=0.005, reg_user=0.05, reg_item=0.05,
                    epochs=args.epochs, n_batch=1, log_train_loss=False, precision="f32")
    t1 = time.perf_counter()
    res = run_training(cfg, matrix=train, testset=test)
    total_s = time.perf_counter() - t1
    walls = [m.wall_seconds for m in res.metrics]
    per_epoch = np.diff([0.0] + walls)
    steady = float(np.median(per_epoch[1:])) if len(per_epoch) > 1 else float(per_epoch[0])
    print(json.dumps({
        "path": "paper_2006_15980_b200.run_training(RunConfig(batch-only, n_batch=1, k=128, "
                "f32)) on host RatingMatrix arrays: BatchWorker lease loop over BatchEngine, "
                "device test RMSE every epoch",
        "workload": "NF-shaped 480000x17700, 100M train ratings (synthetic law), k=%d" % args.k,
        "train_ratings": int(train.nnz), "epochs": res.epochs_run,
        "epoch_seconds": [float(x) for x in per_epoch],
        "updates_per_s_steady": train.nnz / steady,
        "updates_per_s_all_epochs": train.nnz * res.epochs_run / walls[-1],
        "setup_seconds": total_s - walls[-1], "generate_seconds": gen_s,
        "test_rmse": [m.test_rmse for m in res.metrics],
        "qband_impl": None,
    }))


if __name__ == "__main__":
    main()
