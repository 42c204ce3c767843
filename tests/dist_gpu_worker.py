"""torchrun worker for tests/test_gpu_distributed.py (not collected by pytest).

Each rank: one row band on a CUDA device (ranks may share a GPU), Q replicas
exchanged by CUDA IPC, columns leased through the store, EXACT-mode kernel so
the result can be compared with a serial replay bit for bit.
"""

import os
import pickle
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

N_USERS, N_ITEMS, K, NNZ = 300, 260, 32, 12_000
EPOCHS, SEED, LR, REG = 3, 9, 0.02, 0.01


def problem(conflict_free=False):
    rng = np.random.default_rng(21)
    cells = rng.permutation(N_USERS * N_ITEMS)[:NNZ]
    users = (cells // N_ITEMS).astype(np.int32)
    items = (cells % N_ITEMS).astype(np.int32)
    if conflict_free:   # every user and every item in at most one rating
        n = min(N_USERS, N_ITEMS)
        users = rng.permutation(N_USERS)[:n].astype(np.int32)
        items = rng.permutation(N_ITEMS)[:n].astype(np.int32)
    vals = rng.uniform(0, 1, len(users)).astype(np.float32).astype(np.float64)
    P0 = rng.uniform(0, 0.3, size=(N_USERS, K)).astype(np.float32)
    Q0 = rng.uniform(0, 0.3, size=(N_ITEMS, K)).astype(np.float32)
    return users, items, vals, P0, Q0


def main(out_dir, kernel="exact", stage=False, policy="quota"):
    impl = None
    if kernel == "qband8":        # the tile-resident run-group layout, forced
        kernel, impl = "qband", 8
    import torch
    import torch.distributed as dist
    from paper_2006_15980_b200.data import DeviceTriples
    from paper_2006_15980_b200.distributed import CudaRowBand, RowBandTrainer, make_lease_table
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"]) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    users, items, vals, P0, Q0 = problem(conflict_free=kernel != "exact")
    row_cuts = np.linspace(0, N_USERS, world + 1).astype(np.int64)
    col_cuts = np.linspace(0, N_ITEMS, 2 * world + 2).astype(np.int64)
    lo, hi = int(row_cuts[rank]), int(row_cuts[rank + 1])
    keep = (users >= lo) & (users < hi)
    dev = torch.device("cuda", local)
    trip = DeviceTriples(hi, N_ITEMS, torch.from_numpy(users[keep]).to(dev),
                         torch.from_numpy(items[keep]).to(dev),
                         torch.from_numpy(vals[keep].astype(np.float32)).to(dev))
    band = CudaRowBand(dist, rank, world, dev, trip, lo, hi, col_cuts, K, LR, REG, REG,
                       kernel=kernel, init=(P0[lo:hi], Q0), impl=impl)
    run_id = [f"gputest{os.getpid()}"]
    dist.broadcast_object_list(run_id, src=0)
    table = make_lease_table("shm", dist.distributed_c10d._get_default_store(), band.n_cols,
                             rank, run_id[0])
    if rank == 0:
        table.initialize()
    dist.barrier()
    if stage:      # every block's ratings uploaded from pinned host memory per lease
        band.stage_from_host(True)
        # poison the device copies: only the per-lease uploads can make the
        # result right (a broken or skipped upload trains on zeros / NaNs)
        if band.compact is not None:
            band.dev_rel.zero_()
        else:
            band.grid.users.fill_(lo)
            band.grid.items.zero_()
        band.grid.ratings.fill_(float("nan"))
        torch.cuda.synchronize()
        if rank == 0:
            with open(os.path.join(out_dir, "staged.txt"), "w") as fh:
                fh.write("compact" if band.compact is not None else "triples")
    trainer = RowBandTrainer(band, table, rank, seed=SEED, record=True, policy=policy,
                             world=world)
    for _ in range(EPOCHS):
        trainer.run_epoch()
        dist.barrier()
    band.refresh_q(table)
    torch.cuda.synchronize()
    res = [None] * world
    dist.all_gather_object(res, (trainer.log, band.P.cpu().numpy(), trainer.counts.tolist()))
    if rank == 0:
        with open(os.path.join(out_dir, "result.pkl"), "wb") as fh:
            pickle.dump((res, band.Q.cpu().numpy(), row_cuts, col_cuts), fh)
    dist.barrier()
    table.close(unlink=rank == 0)
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "exact", "stage" in sys.argv[3:],
         "free" if "free" in sys.argv[3:] else "quota")
