#!/usr/bin/env python
"""Lease-protocol efficiency at N GPUs, on the host (no GPU needed).

Each of N processes runs distributed.RowBandTrainer over the node-local lease
table (csrc/lease.cu) exactly as a GPU rank does, with a stand-in device: a
block's "kernel" occupies the rank's device timeline for (ratings / rate)
seconds, queued behind the block before it (compute() returns at once,
finish() waits until the block's end), Q pulls take bytes / NVLink bandwidth.
What it measures is what a one-GPU box cannot: how much of an epoch ranks
spend waiting for a free column band (the 2N+1 column rule, the staged-ahead
column) and on lease operations, against the ideal epoch (the rank's blocks
back to back).

    python scripts/lease_sim.py --gpus 8 --epochs 6 [--cols-per-gpu 2]

Per-GPU kernel rates come from the measured --sim-world runs (profiles/
round2/s3_sim_world.jsonl); block sizes from the workload's shape.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
import uuid

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class SimBand:
    """CudaRowBand's backend protocol on a simulated device timeline."""

    def __init__(self, n_cols, block_seconds, pull_seconds):
        self.n_cols = n_cols
        self.block_seconds = block_seconds      # per column band
        self.pull_seconds = pull_seconds
        self.busy_until = time.perf_counter()
        self.ends = {}
        self.pulls = 0
        self.busy = 0.0                         # device seconds of block compute

    def pull(self, c, owner):
        if owner >= 0:
            self.pulls += 1
            self.busy_until = max(self.busy_until, time.perf_counter()) + self.pull_seconds

    def compute(self, c, seed):
        start = max(self.busy_until, time.perf_counter())
        self.busy_until = start + self.block_seconds[c]
        self.busy += self.block_seconds[c]
        self.ends[c] = self.busy_until
        return 1

    def finish(self, c):
        end = self.ends.pop(c)
        while True:
            left = end - time.perf_counter()
            if left <= 0:
                return
            time.sleep(min(left, 2e-4) if left > 3e-4 else 0)


def rank_main(rank, world, run_id, n_cols, block_seconds, pull_seconds, epochs, out, policy, barrier):
    from paper_2006_15980_b200.distributed import RowBandTrainer, ShmLeaseTable
    table = ShmLeaseTable(n_cols, rank, run_id)
    while True:                     # rank 0 of the parent created the segment
        try:
            table.holder(0)
            break
        except Exception:
            time.sleep(0.01)
    band = SimBand(n_cols, block_seconds, pull_seconds)
    trainer = RowBandTrainer(band, table, rank, seed=rank, policy=policy, world=world)
    barrier.wait()                  # every rank starts together
    band.busy_until = time.perf_counter()
    t0 = time.perf_counter()
    per_epoch = []
    for _ in range(epochs):
        e0 = time.perf_counter()
        trainer.run_epoch()
        per_epoch.append(time.perf_counter() - e0)
    st = trainer.lease_stats()
    with open(f"{out}.{rank}", "w") as fh:
        json.dump({"rank": rank, "epoch_seconds": per_epoch, "total": time.perf_counter() - t0,
                   "pulls": band.pulls, "busy": band.busy, "blocks": int(trainer.counts.sum()),
                   "lease": st}, fh)
    table.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=8)
    ap.add_argument("--epochs", type=int, default=6)
    ap.add_argument("--cols-per-gpu", type=int, default=2, help="column bands = this x N + 1")
    ap.add_argument("--ratings-per-gpu", type=float, default=100e6)
    ap.add_argument("--rate", type=float, default=14.1e9, help="per-GPU updates/s (sim-world)")
    ap.add_argument("--q-band-mb", type=float, default=9.0 / 17, help="Q band size per column")
    ap.add_argument("--nvlink-gbs", type=float, default=700.0)
    ap.add_argument("--policy", choices=["quota", "free"], default="quota",
                    help="RowBandTrainer policy (the reference's batch-only quota or hsgd free)")
    ap.add_argument("--slow", type=float, default=1.0,
                    help="rank N-1 runs at rate / slow (a heterogeneous or throttled GPU)")
    ap.add_argument("--scale", type=float, default=20.0,
                    help="time dilation: block durations x scale, so host jitter is small")
    args = ap.parse_args()
    n, n_cols = args.gpus, args.cols_per_gpu * args.gpus + 1
    rng = np.random.default_rng(0)
    # blocks of a rank's row band: equal-mass column bands, +-3 % jitter
    per_block = args.ratings_per_gpu / n_cols
    block_seconds = [args.scale * per_block * (1 + 0.03 * rng.standard_normal()) / args.rate
                     for _ in range(n_cols)]
    pull_seconds = args.scale * args.q_band_mb * 1e6 / (args.nvlink_gbs * 1e9)
    run = uuid.uuid4().hex[:10]
    from paper_2006_15980_b200.distributed import ShmLeaseTable
    owner = ShmLeaseTable(n_cols, 0, run)
    owner.initialize()
    out = f"/tmp/lease_sim_{run}"
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(n)
    def blocks_of(r):
        return [b * (args.slow if r == n - 1 else 1.0) for b in block_seconds]
    procs = [ctx.Process(target=rank_main, args=(r, n, run, n_cols, blocks_of(r), pull_seconds,
                                                 args.epochs, out, args.policy, barrier))
             for r in range(n)]
    for p in procs:
        p.start()
    for p in procs:
        p.join()
    owner.close(unlink=True)
    res = [json.load(open(f"{out}.{r}")) for r in range(n)]
    ideal = sum(block_seconds)                      # one rank's blocks back to back
    # epochs end at different times per rank; the job's epoch is the slowest rank's
    epoch = [max(r["epoch_seconds"][e] for r in res) for e in range(args.epochs)]
    steady = float(np.median(epoch[1:])) if len(epoch) > 1 else epoch[0]
    # device utilisation over the whole run: block compute seconds of all
    # ranks over N x the slowest rank's wall time (the free policy's epochs
    # end at different times per rank, so per-epoch times do not compare)
    wall = max(r["total"] for r in res)
    util = sum(r["busy"] for r in res) / (n * wall)
    # block updates per second against every rank running its blocks back to back
    ideal_rate = sum(n_cols / sum(blocks_of(r)) for r in range(n))
    thru = sum(r["blocks"] for r in res) / wall / ideal_rate
    line = {"gpus": n, "column_bands": n_cols, "epochs": args.epochs, "policy": args.policy,
            "slow": args.slow, "device_utilisation": util, "throughput_efficiency": thru,
            "blocks_per_rank": [r["blocks"] for r in res],
            "ideal_epoch_s": ideal / args.scale, "median_epoch_s": steady / args.scale,
            "protocol_efficiency": ideal / steady,
            "lease_us_per_lease_max": max(r["lease"]["us_per_lease"] for r in res),
            "wait_seconds_max": max(r["lease"]["wait_seconds"] for r in res) / args.scale,
            "pulls_per_rank": float(np.mean([r["pulls"] for r in res])),
            "rate_per_gpu": args.rate, "time_dilation": args.scale}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
