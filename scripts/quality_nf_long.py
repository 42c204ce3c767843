#!/usr/bin/env python
"""Twenty-epoch test-RMSE trajectory at the bench's full configuration
(NF-shaped 480 000 x 17 700, 100 M training ratings, k = 128 fp32, the
automatic layout) against the unmodified reference's run_training
(stream-only, oracle/_ref) from identical factors on identical triples —
the full training run behind the 4-epoch gate of
tests/test_gpu_quality_netflix_full.py.  One JSON line.

    python scripts/quality_nf_long.py [--epochs 20] [--k 128] [--precision f32]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--k", type=int, default=128)
    ap.add_argument("--precision", default="f32")
    args = ap.parse_args()
    import numpy as np
    import torch

    import qgate
    from oracle import reference
    hetmf = reference.hetmf()
    n_users, n_items = 480_000, 17_700
    nnz = int(round(100_000_000 / 0.95))
    train, test, tr, te = qgate.problem(n_users, n_items, nnz, seed=0,
                                        device=torch.device("cuda", 0))
    ref, init = qgate.reference_rmse(hetmf, n_users, n_items, args.k, tr, te, args.epochs)
    ours, grid = qgate.ours_rmse(train, test, init, args.k, args.precision, args.epochs)
    gaps = np.abs(np.asarray(ours) - np.asarray(ref))
    print(json.dumps({"workload": "NF-shaped 480000x17700, 100M train ratings", "k": args.k,
                      "precision": args.precision, "epochs": args.epochs,
                      "layout_impl": grid.sub_impl, "wide": int(getattr(grid, "sub_wide", 0)),
                      "ours": [float(x) for x in ours], "reference": [float(x) for x in ref],
                      "max_gap": float(gaps.max()), "final_gap": float(gaps[-1])}))


if __name__ == "__main__":
    main()
