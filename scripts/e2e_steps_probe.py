#!/usr/bin/env python
"""Per-step anatomy of the streamed epoch (e2e): host time per step, split
into enqueue time (host returns from StreamingEpoch.run) and wait time (the
RMSE read), and the device time of the step's copy and compute streams.
Prints one JSON line with the slowest steps."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_15980_b200.data import (bucket_qbands, build_device_grid, split_device,  # noqa: E402
                                        synthetic_device)
from paper_2006_15980_b200.sgd import DeviceModel, Hyperparams, init_device_model, residual_sums  # noqa: E402
from paper_2006_15980_b200.workers import StreamingEpoch  # noqa: E402


def main():
    d = torch.device("cuda", 0)
    trip = synthetic_device(480_000, 17_700, int(round(1e8 / 0.95)), seed=0, device=d)
    train, test = split_device(trip, 0.05)
    grid = build_device_grid(train, [0, 480_000], [0, 8850, 17_700])
    variant = sys.argv[1] if len(sys.argv) > 1 else "default"
    bucket_qbands(grid, 128, impl=4 if variant == "whole" else None)
    se = StreamingEpoch(grid, 128)
    model = init_device_model(480_000, 17_700, 128, 0, device=d)
    dm = DeviceModel(model.P, model.Q)
    hp = Hyperparams(n_factors=128, reg_user=0.05, reg_item=0.05, learning_rate=0.005)
    rows = []
    se.trace = []
    anchor = torch.cuda.Event(enable_timing=True)
    anchor.record()
    for i in range(60):
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        se.run(model.P, model.Q, hp, seed=i)
        t1 = time.perf_counter()
        if variant == "normse":
            torch.cuda.synchronize()
        else:
            s = residual_sums(dm, test.users, test.items, test.ratings)[0].item()
        t2 = time.perf_counter()
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        torch.cuda.synchronize()
        chunks = [{"chunk": c["chunk"],
                   "copy": (round(anchor.elapsed_time(c["c0"]), 2), round(anchor.elapsed_time(c["c1"]), 2)) if c["copied"] else None,
                   "kernel": (round(anchor.elapsed_time(c["k0"]), 2), round(anchor.elapsed_time(c["k1"]), 2))}
                  for c in se.trace]
        se.trace = []
        rows.append({"step": i, "host_ms": 1e3 * (t2 - t0), "enqueue_ms": 1e3 * (t1 - t0),
                     "wait_ms": 1e3 * (t2 - t1), "device_ms": e0.elapsed_time(e1),
                     "t0": round(anchor.elapsed_time(e0), 2), "chunks": chunks})
    host = np.array([r["host_ms"] for r in rows[3:]])
    out = {"variant": variant, "impl": grid.sub_impl, "median_ms": float(np.median(host)), "p90_ms": float(np.percentile(host, 90)),
           "max_ms": float(host.max()),
           "slowest": [round(r["device_ms"], 1) for r in sorted(rows[3:], key=lambda r: -r["host_ms"])[:5]],
           "slowest_detail": sorted(rows[3:], key=lambda r: -r["host_ms"])[:2],
           "typical_detail": rows[10]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
