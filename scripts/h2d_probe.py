#!/usr/bin/env python
"""Pinned host->device copy stability: 60 rounds of 525 MB in 37 MB chunks
(the streamed epoch's traffic) on one stream; per-round device time."""
import json

import numpy as np
import torch


def main():
    d = torch.device("cuda", 0)
    chunk = 37 << 20
    n = 14
    host = torch.empty(chunk * n, dtype=torch.uint8).pin_memory()
    dev = [torch.empty(chunk, dtype=torch.uint8, device=d) for _ in range(2)]
    s = torch.cuda.Stream()
    times = []
    for r in range(60):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for c in range(n):
                dev[c & 1].copy_(host[c * chunk:(c + 1) * chunk], non_blocking=True)
            e1.record(s)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    t = np.array(times[3:])
    print(json.dumps({"median_ms": float(np.median(t)), "p90_ms": float(np.percentile(t, 90)),
                      "max_ms": float(t.max()), "GBps_median": chunk * n / (np.median(t) / 1e3) / 1e9,
                      "slowest": sorted(times[3:])[-5:]}))


if __name__ == "__main__":
    main()
