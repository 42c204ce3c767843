#!/usr/bin/env python
"""Per-chunk copy and kernel times of the streamed epoch (StreamingEpoch.trace)
at one k / precision, next to the resident launches of the same layout.

  python scripts/stream_chunk_probe.py K f32|f16 [MAX_TILE_ROWS]
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2006_15980_b200 import kernels  # noqa: E402
from paper_2006_15980_b200.data import (bucket_qbands, build_device_grid, split_device,  # noqa: E402
                                        synthetic_device)
from paper_2006_15980_b200.sgd import Hyperparams, init_device_model  # noqa: E402
from paper_2006_15980_b200.workers import StreamingEpoch  # noqa: E402


def main():
    k, prec = int(sys.argv[1]), sys.argv[2]
    cap = int(sys.argv[3]) if len(sys.argv) > 3 else None
    d = torch.device("cuda", 0)
    trip = synthetic_device(480_000, 17_700, int(round(1e8 / 0.95)), seed=0, device=d)
    train, _ = split_device(trip, 0.05)
    grid = build_device_grid(train, [0, 480_000], [0, 8850, 17_700])
    eb = 2 if prec == "f16" else 4
    bucket_qbands(grid, k, elem_bytes=eb, max_tile_rows=cap)
    se = StreamingEpoch(grid, k, elem_bytes=eb)
    model = init_device_model(480_000, 17_700, k, 0, device=d,
                              dtype="float16" if prec == "f16" else "float32")
    hp = Hyperparams(n_factors=k, reg_user=0.05, reg_item=0.05, learning_rate=0.005)
    res = []
    for i in range(4):        # resident launches of the same layout
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for b in range(grid.n_blocks):
            kernels.launch_block_qband(model.P, model.Q, grid, b, 0.005, 0.05, 0.05, i * 7 + b)
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1))
    se.trace = []
    for i in range(4):
        se.run(model.P, model.Q, hp, seed=i)
    torch.cuda.synchronize()
    tr = se.trace[-se.n_chunks:]
    out = {"k": k, "precision": prec, "cap": cap, "u16": se.u16, "row_tiles": list(grid.sub_tiles),
           "impl": grid.sub_impl, "split": grid.sub_split, "qsync": grid.sub_qsync,
           "resident_epoch_ms": float(np.median(res)),
           "chunks": [{"chunk": c["chunk"], "copy_ms": round(c["c0"].elapsed_time(c["c1"]), 3),
                       "kernel_ms": round(c["k0"].elapsed_time(c["k1"]), 3)} for c in tr]}
    out["stream_kernel_ms"] = round(sum(c["kernel_ms"] for c in out["chunks"]), 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
