#!/usr/bin/env python
"""Quality of split item runs (implementation 5) against whole runs on a
narrow synthetic block: test RMSE after E epochs per (k, dtype, split).
One JSON line per case."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_15980_b200 import kernels  # noqa: E402
from paper_2006_15980_b200.data import (bucket_qbands, build_device_grid, split_device,  # noqa: E402
                                        synthetic_device)
from paper_2006_15980_b200.sgd import init_device_model, rmse  # noqa: E402


def main():
    d = torch.device("cuda", 0)
    n_users, n_items, nnz = 120_000, 1_200, 3_000_000
    trip = synthetic_device(n_users, n_items, nnz, seed=3, device=d)
    train, test = split_device(trip, 0.05)
    from paper_2006_15980_b200 import _lib
    qs = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    _lib.check(_lib.load().hmf_qband_set_qsync(qs), "qsync")
    for k in (32, 64, 128):
        for dtype in ("float32", "float16"):
            for split in (1, 4, 15):
                g = build_device_grid(train, [0, n_users], [0, 600, 1_200])
                bucket_qbands(g, k, elem_bytes=2 if dtype == "float16" else 4,
                              impl=4 if split == 1 else 5, split=None if split == 1 else split)
                model = init_device_model(n_users, n_items, k, 0, device=d, dtype=dtype)
                for e in range(8):
                    for b in (0, 1):
                        kernels.launch_block_qband(model.P, model.Q, g, b, 0.005, 0.05, 0.05,
                                                   kernels.mix64(b, e))
                run = train.nnz / 2 / 600
                print(json.dumps({"k": k, "dtype": dtype, "split": split, "qsync": qs,
                                  "ratings_per_part": run / split,
                                  "rmse": rmse(test, model).value}), flush=True)


if __name__ == "__main__":
    main()
