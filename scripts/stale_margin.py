#!/usr/bin/env python
"""Staleness margin of the run-group kernel (implementation 8): test RMSE
after 8 epochs on narrow 2 %-density blocks (the setting of
test_default_layout_quality_matches_whole_runs) against whole runs on one
chain each (implementation 4), at rising learning rates.  One JSON line per
(k, precision, lr)."""
import json
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__))))


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("ks", nargs="?", default="32,64")
    ap.add_argument("--shape", default="120000,1200,3000000",
                    help="users,items,ratings (default: the narrow 2 %-density blocks)")
    ap.add_argument("--lrs", default="0.005,0.01,0.02")
    ap.add_argument("--dtypes", default="float32,float16")
    ap.add_argument("--epochs", type=int, default=8)
    args = ap.parse_args()
    n_users, n_items, nnz = (int(x) for x in args.shape.split(","))
    import torch
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (bucket_qbands, build_device_grid, split_device,
                                            synthetic_device)
    from paper_2006_15980_b200.sgd import init_device_model, rmse
    d = torch.device("cuda", 0)
    trip = synthetic_device(n_users, n_items, nnz, seed=3, device=d)
    train, test = split_device(trip, 0.05)
    for k in (int(x) for x in args.ks.split(",")):
        for dtype in args.dtypes.split(","):
            for lr in (float(x) for x in args.lrs.split(",")):
                out = {}
                for layout, impl in (("default", None), ("runs", 8), ("split", 5), ("whole", 4)):
                    g = build_device_grid(train, [0, n_users], [0, n_items // 2, n_items])
                    bucket_qbands(g, k, elem_bytes=2 if dtype == "float16" else 4, impl=impl)
                    model = init_device_model(n_users, n_items, k, 0, device=d, dtype=dtype)
                    for e in range(args.epochs):
                        for b in (0, 1):
                            kernels.launch_block_qband(model.P, model.Q, g, b, lr, 0.05, 0.05,
                                                       kernels.mix64(b, e))
                    out[layout] = rmse(test, model).value
                    out[layout + "_impl"] = g.sub_impl
                print(json.dumps({"shape": args.shape, "k": k, "dtype": dtype, "lr": lr, **out,
                                  "gap_default": out["default"] - out["whole"],
                                  "gap_runs": out["runs"] - out["whole"],
                                  "gap_split": out["split"] - out["whole"]}), flush=True)


if __name__ == "__main__":
    main()
