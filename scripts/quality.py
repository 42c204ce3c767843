#!/usr/bin/env python
"""Quality and tuning experiments on the GPU box (results go to stdout as JSON).

  python scripts/quality.py ml1m   [--modes hogwild,hogwild_lww] [--epochs 20]
      ML-1M-shaped instance from the reference generator (bit-identical host
      restatement), k=32, lr=reg=0.01, 1x2 grid; test RMSE per epoch vs the
      reference's stream-only run (tests/golden/training.json).
  python scripts/quality.py netflix [--epochs 5] [--threads N]
      Netflix-shaped instance (device generator), k=128, lr=0.005, reg=0.05:
      the GPU engine and the CPU oracle (C port of the reference's stream-only
      path, all host threads) from identical factors on identical triples;
      test RMSE after each epoch on both.
  python scripts/quality.py sweep [--variants 0-7] [--modes ...]
      HOGWILD kernel variants x write policies on the Netflix shape: updates/s
      (CUDA events, 3 warm-up + 5 timed epochs) and test RMSE after 8 epochs.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def ml1m(args):
    import torch
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (DeviceGrid, RatingMatrix, build_grid, shuffle_triples,
                                            synthetic_ratings)
    from paper_2006_15980_b200.sgd import DeviceModel, Hyperparams, block_epoch, init_model, rmse
    dev = torch.device("cuda", 0)
    ref = json.loads((ROOT / "tests" / "golden" / "training.json").read_text())
    full = synthetic_ratings(6040, 3706, rank=8, density=1.05e6 / (6040 * 3706), noise=0.1, seed=0)
    perm = np.random.default_rng(1).permutation(full.nnz)
    n_test = full.nnz // 21
    te, tr = perm[:n_test], perm[n_test:]
    train = RatingMatrix(6040, 3706, full.users[tr], full.items[tr], full.ratings[tr])
    test = RatingMatrix(6040, 3706, full.users[te], full.items[te], full.ratings[te])
    hp = Hyperparams(n_factors=32, reg_user=0.01, reg_item=0.01, learning_rate=0.01)
    grid = DeviceGrid.from_host(build_grid(shuffle_triples(train, 0), [0, 6040], [0, 1853, 3706]),
                                dev)
    out = {"reference": {k: v["test_rmse"] for k, v in ref.items() if k.startswith("e")}}
    for mode in args.modes.split(","):
        model = DeviceModel.from_host(init_model(6040, 3706, hp, 0), dev)
        traj = []
        counts = np.zeros(2, dtype=np.int64)
        t0 = time.perf_counter()
        for epoch in range(1, args.epochs + 1):
            for b in (0, 1):
                seed = kernels.mix64(kernels.mix64(0, b, int(counts[b])), 0)
                block_epoch(model, grid, b, hp, seed, mode=mode)
                counts[b] += 1
            traj.append(rmse(test, model).value)
        torch.cuda.synchronize()
        out[mode] = {"test_rmse": traj, "seconds": time.perf_counter() - t0}
    print(json.dumps(out))


def netflix(args):
    import torch
    import oracle
    from paper_2006_15980_b200 import kernels
    from paper_2006_15980_b200.data import (build_device_grid, build_grid, split_device,
                                            synthetic_device, RatingMatrix)
    from paper_2006_15980_b200.sgd import DeviceModel, FactorModel, rmse
    dev = torch.device("cuda", 0)
    n_users, n_items, n_train, k = 480_000, 17_700, args.nnz, args.k
    lr, reg = 0.005, 0.05
    trip = synthetic_device(n_users, n_items, int(round(n_train / 0.95)), seed=0, device=dev)
    train, test = split_device(trip, 0.05)
    grid = build_device_grid(train, [0, n_users], [0, (n_items + 1) // 2, n_items])
    rng = np.random.default_rng(0)
    top = 1 / np.sqrt(k)
    P0 = rng.uniform(0, top, size=(n_users, k)).astype(np.float32)
    Q0 = rng.uniform(0, top, size=(n_items, k)).astype(np.float32)
    h_test = test.to_host()
    out = {"config": dict(n_users=n_users, n_items=n_items, train=train.nnz, test=test.nnz, k=k,
                          lr=lr, reg=reg, epochs=args.epochs)}
    # Q-band modes: qband (default implementation, fp32), qband_f16 (fp16
    # storage), qband_implN (implementation N, fp32)
    qgrids = {}
    for mode in args.modes.split(","):
        if mode.startswith("qband"):
            from paper_2006_15980_b200.data import bucket_qbands
            impl = int(mode[len("qband_impl"):]) if mode.startswith("qband_impl") else None
            g = build_device_grid(train, [0, n_users], [0, (n_items + 1) // 2, n_items])
            qgrids[mode] = bucket_qbands(g, k, impl=impl,
                                         elem_bytes=2 if mode == "qband_f16" else 4)
    for mode in args.modes.split(","):
        dt = torch.float16 if mode == "qband_f16" else torch.float32
        model = DeviceModel(torch.from_numpy(P0).to(dev, dt), torch.from_numpy(Q0).to(dev, dt))
        traj = []
        counts = np.zeros(2, dtype=np.int64)
        for epoch in range(args.epochs):
            for b in (0, 1):
                lo, hi = grid.block_range(b)
                seed = kernels.mix64(kernels.mix64(0, b, int(counts[b])), 0)
                if mode in qgrids:
                    kernels.launch_block_qband(model.P, model.Q, qgrids[mode], b, lr, reg, reg,
                                               seed)
                else:
                    kernels.launch_sgd_range(model.P, model.Q, grid.users, grid.items,
                                             grid.ratings, lo, hi, lr, reg, reg, seed, 0, 0, mode)
                counts[b] += 1
            traj.append(rmse(test, model).value)
        out[f"gpu_{mode}"] = traj
        if mode in qgrids:
            out[f"gpu_{mode}_impl"] = qgrids[mode].sub_impl
    if args.threads:
        # CPU reference path on the same triples (host copy) and same init
        h_train = train.to_host()
        threads = args.threads
        g = build_grid(h_train, np.linspace(0, n_users, threads + 1).astype(np.int64),
                       np.linspace(0, n_items, threads + 2).astype(np.int64))
        P, Q = P0.astype(np.float64), Q0.astype(np.float64)
        counts = None
        traj = []
        t0 = time.perf_counter()
        for epoch in range(args.epochs):
            _, counts = oracle.stream_train(P, Q, g.users, g.items, g.ratings, g.block_ptr,
                                            threads, threads + 1, lr, reg, reg, 0, 1, threads,
                                            counts)
            traj.append(oracle.rmse(P, Q, h_test.users, h_test.items, h_test.ratings))
        out["cpu_reference"] = traj
        out["cpu_seconds"] = time.perf_counter() - t0
        out["cpu_threads"] = threads
    print(json.dumps(out))


def sweep(args):
    import torch
    from paper_2006_15980_b200 import _lib, kernels
    from paper_2006_15980_b200.data import build_device_grid, split_device, synthetic_device
    from paper_2006_15980_b200.sgd import init_device_model, rmse
    dev = torch.device("cuda", 0)
    n_users, n_items, k = 480_000, 17_700, args.k
    trip = synthetic_device(n_users, n_items, int(round(args.nnz / 0.95)), seed=0, device=dev)
    train, test = split_device(trip, 0.05)
    grid = build_device_grid(train, [0, n_users], [0, (n_items + 1) // 2, n_items])
    lo_v, hi_v = (int(x) for x in args.variants.split("-"))
    res = []
    for mode in args.modes.split(","):
        for v in range(lo_v, hi_v + 1):
            _lib.set_variant(v)
            model = init_device_model(n_users, n_items, k, 0, device=dev,
                                      dtype="float16" if args.precision == "f16" else "float32")

            def epoch(e):
                for b in (0, 1):
                    lo, hi = grid.block_range(b)
                    kernels.launch_sgd_range(model.P, model.Q, grid.users, grid.items,
                                             grid.ratings, lo, hi, 0.005, 0.05, 0.05,
                                             kernels.mix64(b, e), 0, 0, mode)
            for e in range(3):
                epoch(e)
            torch.cuda.synchronize()
            s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for e in range(5):
                epoch(3 + e)
            t.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(t) / 5
            res.append({"mode": mode, "variant": v, "ms_per_epoch": ms,
                        "updates_per_s": train.nnz / (ms / 1e3),
                        "test_rmse_8ep": rmse(test, model).value})
            print(json.dumps(res[-1]), flush=True)
    _lib.set_variant(-1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["ml1m", "netflix", "sweep"])
    ap.add_argument("--modes", default="hogwild,hogwild_lww")
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--nnz", type=int, default=100_000_000)
    ap.add_argument("--variants", default="0-7")
    ap.add_argument("--k", type=int, default=128)
    ap.add_argument("--precision", default="f32")
    ap.add_argument("--kernel", default="hogwild")
    ap.add_argument("--pstore", type=int, default=-1,
                    help="chained Q-band kernel P write-back (hmf_qband_set_pstore)")
    args = ap.parse_args()
    if args.pstore >= 0:
        from paper_2006_15980_b200 import kernels
        kernels.PSTORE_OVERRIDE = args.pstore
    {"ml1m": ml1m, "netflix": netflix, "sweep": sweep}[args.what](args)


if __name__ == "__main__":
    main()
