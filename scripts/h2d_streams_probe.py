#!/usr/bin/env python
"""Pinned host->device bandwidth with the epoch's 600 MB split over 1, 2 or 4
copy streams (concurrent copies may use more than one copy engine), and with
chunk sizes of 37 / 150 / 300 MB; device time per round, median of 20."""
import json

import numpy as np
import torch


def main():
    d = torch.device("cuda", 0)
    total = 600 << 20
    host = torch.empty(total, dtype=torch.uint8).pin_memory()
    dev = torch.empty(total, dtype=torch.uint8, device=d)
    for n_streams in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(n_streams)]
        for chunk_mb in (37, 150, 300):
            chunk = chunk_mb << 20
            n = total // chunk
            times = []
            for r in range(23):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for s in streams:
                    s.wait_event(e0)
                for c in range(n):
                    with torch.cuda.stream(streams[c % n_streams]):
                        dev[c * chunk:(c + 1) * chunk].copy_(host[c * chunk:(c + 1) * chunk],
                                                             non_blocking=True)
                for s in streams:
                    ev = torch.cuda.Event()
                    ev.record(s)
                    torch.cuda.current_stream().wait_event(ev)
                e1.record()
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            t = float(np.median(times[3:]))
            print(json.dumps({"streams": n_streams, "chunk_MB": chunk_mb, "median_ms": t,
                              "GBps": n * chunk / (t / 1e3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
