#!/usr/bin/env python
"""Device time of sgd.residual_sums (the e2e step's RMSE read) per k and
storage precision on the Netflix-shaped test set (5.26 M ratings)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_15980_b200.data import split_device, synthetic_device  # noqa: E402
from paper_2006_15980_b200.sgd import DeviceModel, init_device_model, residual_sums  # noqa: E402

d = torch.device("cuda", 0)
trip = synthetic_device(480_000, 17_700, int(round(1e8 / 0.95)), seed=0, device=d)
_, test = split_device(trip, 0.05)
order = torch.argsort(test.users)
tu, ti, tr = test.users[order].contiguous(), test.items[order].contiguous(), test.ratings[order].contiguous()
for k in (32, 64, 128, 256):
    for dt in ("float32", "float16"):
        m = init_device_model(480_000, 17_700, k, 0, device=d, dtype=dt)
        dm = DeviceModel(m.P, m.Q)
        for _ in range(3):
            residual_sums(dm, tu, ti, tr)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            residual_sums(dm, tu, ti, tr)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"k": k, "dtype": dt, "residual_ms": e0.elapsed_time(e1) / 10}))
