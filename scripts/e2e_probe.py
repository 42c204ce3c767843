#!/usr/bin/env python
"""Where the streamed-epoch (e2e) time goes on the GPU box: H2D bandwidth of
pinned chunks, kernel time of the streamed layout with data resident, and the
pipelined epoch.  Prints one JSON line."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2006_15980_b200 import _lib, kernels  # noqa: E402
from paper_2006_15980_b200.data import build_device_grid, split_device, synthetic_device  # noqa: E402
from paper_2006_15980_b200.sgd import Hyperparams, init_device_model  # noqa: E402
from paper_2006_15980_b200.workers import StreamingEpoch  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    _lib.load()
    out = {}
    # raw pinned H2D bandwidth
    for mb in (50, 100, 400):
        h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
        d = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        out[f"h2d_GBps_{mb}MB"] = 5 * (mb << 20) / (e0.elapsed_time(e1) / 1e3) / 1e9
    n_users, n_items, k = 480_000, 17_700, 128
    trip = synthetic_device(n_users, n_items, int(round(100_000_000 / 0.95)), seed=0, device=dev)
    train, _ = split_device(trip, 0.05)
    grid = build_device_grid(train, [0, n_users], [0, (n_items + 1) // 2, n_items])
    model = init_device_model(n_users, n_items, k, 0, device=dev)
    hp = Hyperparams(n_factors=k, reg_user=0.05, reg_item=0.05, learning_rate=0.005)
    from paper_2006_15980_b200.data import bucket_qbands
    bucket_qbands(grid, k)
    for stripes in (0,):
        se = StreamingEpoch(grid, k)
        # kernel only: the streamed layout with every chunk resident
        chunks = [(lo, hi, rel, sc) for tiles, sc in se.blocks for lo, hi, rel in tiles]
        dbufs = [(se.host[0][lo:hi].to(dev), se.host[-1][lo:hi].to(dev)) for lo, hi, _, _ in chunks]
        fn = _lib.load().hmf_sgd_block_qband_f32
        s = torch.cuda.current_stream(dev)

        def kernels_only(seed):
            for b, (lo, hi, sp, sc) in enumerate(chunks):
                u, r = dbufs[b]
                _lib.check(fn(model.P.data_ptr(), model.Q.data_ptr(), k, u.data_ptr(),
                              0 if se.implicit_items else None, r.data_ptr(), sp.data_ptr(),
                              sc.data_ptr(), int(sc.numel()) - 1, 1, se.sub_impl,
                              0.005, 0.05, 0.05, kernels.mix64(seed, b), 0, 0, s.cuda_stream),
                           "qband")
        if se.implicit_items:
            kernels_only(0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(5):
                kernels_only(1 + i)
            e1.record()
            torch.cuda.synchronize()
            out[f"kernel_ms_per_epoch_s{stripes}"] = e0.elapsed_time(e1) / 5
        del dbufs
        se.run(model.P, model.Q, hp, 0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(5):
            se.run(model.P, model.Q, hp, 1 + i)
        torch.cuda.synchronize()
        out[f"streamed_ms_per_epoch_s{stripes}"] = (time.perf_counter() - t0) / 5 * 1e3
        out[f"h2d_MB_per_epoch_s{stripes}"] = se.h2d_bytes / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
