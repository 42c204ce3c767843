#!/usr/bin/env python
"""Benchmark: SGD updates/sec of the B200 hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload netflix|ml1m|yahoo|hugewiki] [--k K] [--precision f32|f16]

A step is one epoch of the hot path over the workload's rating matrix: every
block of the division plan once, each block one launch of the sm_100a update
kernel (HOGWILD mode) — the work one `hetmf.kernels.sgd_range` call per block
does in the reference (StreamWorker / BatchEngine.compute, workers.py:222-302).

Default (N=1): the Netflix-shaped configuration BASELINE.json's metric is
quoted on (configs[1]): 480 000 x 17 700, 100 M training ratings (plus a 5 %
held-out test set), k = 128, fp32, the 1-GPU batch-only uniform plan (1 x 2
blocks, partition.py:89-107).  Inputs are larger than L2 (P 246 MB, triples
1.2 GB), so no L2 flush is needed between steps.

Printed (rank 0, one JSON line): value = whole-job updates/s from CUDA events
over exactly K steps (barrier + synchronize both sides, max over ranks);
roofline of the dominant kernel (algorithmic bytes 12 + 16k per update over
its mean event-timed launch); e2e = the same metric through the drop-in
host-buffer call (kernels.sgd_range on numpy arrays: H2D of triples and
factors, launch, D2H of factors, per block); cpu_baseline = the CPU oracle
(a C port of the reference's stream-only path) on a bounded sample, all host
threads.  --impl reference prints the reference arm: that CPU path timed
alone on the same workload shape.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (n_users, n_items, n_train, default k, description)
    "ml1m": (6040, 3706, 1_000_000, 32, "MovieLens-1M-shaped 6040x3706, 1M ratings"),
    "netflix": (480_000, 17_700, 100_000_000, 128, "Netflix-shaped 480000x17700, 100M ratings"),
    "yahoo": (1_000_000, 625_000, 250_000_000, 128, "Yahoo!Music-R1-shaped 1Mx625K, 250M ratings"),
    "hugewiki": (50_000_000, 40_000, 3_100_000_000, 128, "Hugewiki-shaped 50Mx40K, 3.1B ratings"),
}
TEST_FRACTION = 0.05
LR, REG = 0.005, 0.05  # the paper's gamma / lambda
SEED = 0


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


def l2_ceiling(k: int, precision: str, stores: bool = False):
    """The measured ceiling of the dominant kernel's memory pattern once the
    P tile sits in L2: one random k-row load plus one vector reduction into it
    (or, with P written back by stores, one store of it) per update, no
    arithmetic (scripts/l2_rowbench.cu on a B200, 32 MB buffer;
    profiles/r02/l2_rowbench.jsonl).  Best rows/s over prefetch depths and
    lane layouts; None when that row size was not measured."""
    p = ROOT / "profiles" / "r02" / "l2_rowbench.jsonl"
    if not p.exists():
        return None
    row = k * (2 if precision == "f16" else 4)
    mode = ("load+red_f16x2" if precision == "f16"
            else "load+store" if stores else "load+red")
    best, buf = None, None
    for line in p.read_text().splitlines():
        try:
            d = json.loads(line)
        except ValueError:
            continue
        if "buffer_MB" in d:
            buf = d["buffer_MB"]
        elif buf == 32 and d.get("mode") == mode and d.get("row_bytes") == row:
            best = max(best or 0.0, float(d["rows_per_s"]))
    return best


def bytes_per_update(k: int, precision: str) -> int:
    s = 2 if precision == "f16" else 4
    return 12 + 4 * k * s  # triple + read+write of p_u and q_v


class ClockSampler:
    """nvidia-smi style clock / throttle sampling during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
            return self
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()
        return self

    def _run(self):
        nv = self._nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
            "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for n, bit in names.items():
                    if mask & bit and n != "gpu_idle":
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # NCCL init lines (nranks, transports) in the log, for the driver
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        n_dev = torch.cuda.device_count()
        local = local % n_dev            # several ranks may share a GPU (testing)
        torch.cuda.set_device(local)
        if world <= n_dev:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def _reduce_device():
    import torch.distributed as dist
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_reduce_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_reduce_device())
    dist.all_reduce(t)
    return float(t.item())


# ---------------------------------------------------------------------------
# CPU arm: the reference's own stream-only path on the host cores
# ---------------------------------------------------------------------------
def reference_module():
    """The unmodified reference package installed under oracle/_ref (test and
    baseline infrastructure, oracle/reference.py), or None."""
    try:
        from oracle import reference
        return reference.hetmf() if reference.installed() else None
    except Exception:
        return None


def workload_sample(n_users, n_items, sample_nnz, seed=SEED):
    """A bounded sample of the workload under its law (synthetic_ratings,
    data.py:311-336: rank 8, factors U[0, 1/sqrt 8], noise N(0, 0.1)) over
    the FULL user x item space: cells uniform (duplicates are ~nnz^2/cells,
    negligible at these sizes), so the timed run touches full-size P and Q."""
    rng = np.random.default_rng(seed)
    users = rng.integers(0, n_users, sample_nnz, dtype=np.int32)
    items = rng.integers(0, n_items, sample_nnz, dtype=np.int32)
    top = 1.0 / np.sqrt(8.0)
    A = rng.uniform(0.0, top, size=(n_users, 8))
    B = rng.uniform(0.0, top, size=(n_items, 8))
    vals = np.einsum("ij,ij->i", A[users], B[items]) + rng.normal(0.0, 0.1, sample_nnz)
    return users, items, vals


def cpu_reference_run(n_users, n_items, k, sample_nnz, threads, epochs, seed=SEED):
    """The reference's CPU path on a sample: hetmf.run_training(RunConfig(
    schedule="stream-only", n_stream=threads, ...)) (engine.py:190-268), its
    numba sgd_range on `threads` stream workers, log_train_loss off.  Returns
    (updates/s, updates, seconds) from the reference's own TrainResult
    (scheduler.total_updates / wall_seconds: the training loop, not setup)."""
    ref = reference_module()
    users, items, vals = workload_sample(n_users, n_items, sample_nnz, seed)
    m = ref.RatingMatrix(n_users, n_items, users, items, vals)
    cfg = ref.RunConfig(schedule="stream-only", n_stream=threads, n_factors=k, learning_rate=LR,
                        reg_user=REG, reg_item=REG, epochs=epochs, seed=seed,
                        log_train_loss=False)
    res = ref.run_training(cfg, matrix=m)
    got = int(res.scheduler.total_updates)
    return got / res.wall_seconds, got, res.wall_seconds


def cpu_port_run(n_users, n_items, k, sample_nnz, threads, epochs, seed=SEED):
    """The oracle's C port of the same stream-only path (threads x (threads+1)
    uniform grid, f64 P/Q) on the same sample: used when the reference is not
    installed, and to state the port / reference speed ratio."""
    import oracle
    from paper_2006_15980_b200.data import build_grid, RatingMatrix
    users, items, vals = workload_sample(n_users, n_items, sample_nnz, seed)
    m = RatingMatrix(n_users, n_items, users, items, vals)
    rows_cut = np.linspace(0, n_users, threads + 1).astype(np.int64)
    cols_cut = np.linspace(0, n_items, threads + 2).astype(np.int64)
    g = build_grid(m, rows_cut, cols_cut)
    rng = np.random.default_rng(seed)
    top = 1.0 / np.sqrt(k)
    P = rng.uniform(0, top, size=(n_users, k))
    Q = rng.uniform(0, top, size=(n_items, k))
    oracle.lib()
    t0 = time.perf_counter()
    got, _ = oracle.stream_train(P, Q, g.users, g.items, g.ratings, g.block_ptr, threads,
                                 threads + 1, LR, REG, REG, seed, epochs, threads)
    dt = time.perf_counter() - t0
    return got / dt, got, dt


def cpu_run(n_users, n_items, k, sample_nnz, threads, epochs, seed=SEED):
    """(kind, updates/s, updates, seconds): the reference when installed,
    else the port."""
    if reference_module() is not None:
        return ("reference",) + cpu_reference_run(n_users, n_items, k, sample_nnz, threads,
                                                  epochs, seed)
    return ("port",) + cpu_port_run(n_users, n_items, k, sample_nnz, threads, epochs, seed)


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def workload_config(args) -> dict:
    """The workload description both arms print (deterministic, no data-
    dependent counts: those are top-level keys)."""
    n_users, n_items, n_train, k0, desc = WORKLOADS[args.workload]
    k = args.k or k0
    return {"workload": f"{desc}, k={k}, {args.precision} storage", "k": k,
            "lr": LR, "reg": REG, "test_fraction": TEST_FRACTION, "seed": SEED,
            "scaling": args.scaling if args.gpus > 1 or "WORLD_SIZE" in os.environ else "weak",
            "l2": ("inputs larger than L2 (triples alone > 126 MB); no flush"
                   if n_train * 12 > (126 << 20) else
                   "inputs fit in the 126 MB L2 (not a headline configuration); no flush")}


def run_reference_arm(args, world, rank):
    n_users, n_items, n_train, k0, desc = WORKLOADS[args.workload]
    k = args.k or k0
    if rank != 0:
        return
    threads = host_threads()
    sample = int(min(n_train, 1_000_000 * threads))
    times, kind = [], None
    for step in range(args.warmup + args.steps):
        kind, rate, got, dt = cpu_run(n_users, n_items, k, sample, threads, 1, seed=SEED + step)
        if step >= args.warmup:
            times.append((got, dt))
    ups = sum(g for g, _ in times) / sum(d for _, d in times)
    ms = 1e3 * sum(d for _, d in times) / len(times)
    what = ("hetmf.run_training(stream-only, numba sgd_range), unmodified reference from "
            "oracle/_ref" if kind == "reference" else "oracle C port of the stream-only path")
    line = {
        "impl": "reference", "metric": "sgd_updates_per_sec", "value": ups, "unit": "updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (the workload's law, host sample)",
        "config": workload_config(args),
        "cpu_baseline": {"value": ups, "unit": "updates/s", "cores": threads, "kind": kind,
                         "sample": f"{sample} ratings of the workload's law over the full "
                                   f"{n_users}x{n_items} matrix, 1 epoch per step, {threads} "
                                   f"stream workers: {what}"},
        "e2e": {"value": ups, "unit": "updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def ncu_summary(key: str):
    """The committed ncu --set full summary of the dominant kernel for this
    workload (profiles/round2/ncu_summary.json, scripts/ncu_summary.py), or
    None."""
    p = ROOT / "profiles" / "round2" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(key)
    except ValueError:
        return None


def binding_unit(ncu: dict) -> str:
    """The busiest unit of an ncu capture, named for this kernel family."""
    units = {"L1TEX / shared-memory data pipe (P-row loads and stores, shuffles)":
             ncu.get("l1tex_pct", 0.0),
             "L2 (LTS)": ncu.get("lts_pct", 0.0), "DRAM": ncu.get("dram_pct", 0.0),
             "instruction issue (latency-bound: few eligible warps)": ncu.get("issue_pct", 0.0)}
    return max(units, key=units.get)


def roofline_fields(args, achieved, peak, peak_kind, bpu, mean_ms, mean_updates, compulsory,
                    l2_rows, kernel_ups, p_stores, impl=None) -> dict:
    """The dominant kernel against its bounds.

    frac (the contract's roofline): ALGORITHMIC bytes per launch (12 + 16k per
    update in fp32: the rating, p_u and q_v read and written) over
    the live CUDA-event launch time, over the measured HBM copy bandwidth —
    the north star's "% of HBM roofline".  It exceeds 1 because the row-tile
    layout keeps each tile's P rows in the 126 MB L2: the P traffic is served
    on chip.  What the kernel does to DRAM and to the on-chip units comes from
    the committed ncu capture: `dram` (measured DRAM bytes per launch over the
    live launch time, over the same peak), `compulsory` (the bytes that must
    cross HBM once per launch) and `binding_unit` (the busiest unit)."""
    k = args.k or WORKLOADS[args.workload][3]
    base = f"{args.workload}_k{k}_{args.precision}_{args.kernel}"
    ncu = ncu_summary(f"{base}_impl{impl}") if impl is not None else None
    if ncu is None and impl in (None, 5):
        ncu = ncu_summary(base)            # round-2 baseline capture (implementation 5)
    dram = None
    if ncu:
        gbs = ncu["dram_bytes"] / (mean_ms / 1e3) / 1e9
        dram = {"bytes_per_launch": ncu["dram_bytes"], "achieved_gbs": gbs, "frac": gbs / peak,
                "ncu_launch_ms": 1e3 * ncu["duration"], "source": ncu["source"]}
    out = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
           "frac": achieved / peak, "traffic": ncu["dram_bytes"] if ncu else None,
           "peak_kind": peak_kind, "bytes_per_update": bpu,
           "frac_meaning": "north-star ratio: algorithmic bytes (rating + p_u, q_v read and "
                           "written) per launch / live launch time / measured HBM copy BW; > 1 "
                           "because P rows are served on chip (L2 row tiles; shared-memory "
                           "tiles for implementation 8); see dram, compulsory, "
                           "binding_unit for the measured picture",
           "kernel": ncu["kernel"] if ncu else (
               "sgd_hogwild_kernel" if args.kernel != "qband" else
               {0: "qband_kernel", 8: "runs_kernel"}.get(impl,
                                                                             "qchain_kernel")),
           "qband_impl": impl,
           "mean_launch_ms": mean_ms, "updates_per_launch": mean_updates,
           "dram": dram,
           "compulsory": (None if compulsory is None else {
               "bytes_per_launch": compulsory,
               "what": "triples once + one read and one write of the block's P band and Q band",
               "dram_over_compulsory": (ncu["dram_bytes"] / compulsory) if ncu else None}),
           "binding_unit": (None if not ncu else {
               "unit": binding_unit(ncu),
               "l1tex_pct": ncu["l1tex_pct"], "lts_pct": ncu["lts_pct"],
               "dram_pct": ncu["dram_pct"], "sm_pct": ncu["sm_pct"],
               "issue_pct": ncu.get("issue_pct"),
               "l2_hit_pct": ncu["l2_hit_pct"],
               "instructions_per_update": (ncu["instructions"] / mean_updates
                                           if ncu.get("instructions") else None),
               "source": ncu["source"]}),
           "l2_ceiling": (None if l2_rows is None else {
               "updates_per_s": l2_rows, "kernel_updates_per_s": kernel_ups,
               "frac": kernel_ups / l2_rows,
               "source": "scripts/l2_rowbench.cu: random P-row load + "
                         + ("store" if p_stores else "vector reduction")
                         + ", L2-resident 32 MB, no arithmetic (profiles/r02/l2_rowbench.jsonl)"})}
    if ncu and ncu.get("smem_wavefronts") and impl == 8:
        # P rows live in shared memory: the bound is the SM's L1/shared data
        # pipe, one 128-byte wavefront per cycle per SM (P-row loads and
        # stores, 8 per update at fp32 k=128, plus shuffles and the global
        # loads that pass through L1)
        n_sm, mhz = sm_geometry()
        wpu = ncu["smem_wavefronts"] / mean_updates
        peak_w = n_sm * mhz * 1e6
        out["smem_pipe"] = {
            "shared_wavefronts_per_update": wpu,
            "peak_wavefronts_per_s": peak_w, "sm_count": n_sm, "sm_max_mhz": mhz,
            "ceiling_updates_per_s": peak_w / wpu, "kernel_updates_per_s": kernel_ups,
            "frac": kernel_ups / (peak_w / wpu),
            "lsu_data_pipe_pct": ncu.get("l1tex_pct"),
            "source": ncu["source"] + " (l1tex__data_pipe_lsu_wavefronts_mem_shared.sum)"}
    return out


def sm_geometry():
    """(SM count, max SM clock in MHz) of device 0 (148, 1965 on B200)."""
    try:
        import torch
        n = int(torch.cuda.get_device_properties(0).multi_processor_count)
    except Exception:
        n = 148
    try:
        import pynvml
        pynvml.nvmlInit()
        mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(pynvml.nvmlDeviceGetHandleByIndex(0),
                                                     pynvml.NVML_CLOCK_SM))
    except Exception:
        mhz = 1965.0
    return n, mhz


def cpu_baseline(n_users, n_items, k, nnz) -> dict:
    """~10-30 s of the reference's CPU path on the host cores (all threads):
    the reference itself (oracle/_ref) when installed, else the C port; plus
    the port on the same sample, so the line states the port / reference
    speed ratio measured on this host."""
    threads = host_threads()
    sample = int(min(nnz, 1_000_000 * threads))
    kind, rate, got, dt = cpu_run(n_users, n_items, k, sample, threads, 1)
    epochs = 1
    if dt < 10.0:
        more = max(1, int(round((10.0 - dt) / max(dt, 1e-3))))
        _, _, got2, dt2 = cpu_run(n_users, n_items, k, sample, threads, more, seed=SEED + 1)
        got, dt, epochs = got + got2, dt + dt2, 1 + more
        rate = got / dt
    out = {"value": rate, "unit": "updates/s", "cores": threads, "kind": kind,
           "sample": f"{sample} ratings of the workload's law over the full {n_users}x{n_items}"
                     f" matrix (f64 P/Q, k={k}), {epochs} epochs, {threads} stream workers, "
                     f"{dt:.1f} s: " + ("hetmf.run_training(stream-only), the unmodified "
                                        "reference (numba sgd_range) from oracle/_ref"
                                        if kind == "reference" else
                                        "oracle C port of the stream-only path")}
    if kind == "reference":
        prate, _, _ = cpu_port_run(n_users, n_items, k, sample, threads, 1)
        out["port_vs_reference"] = {"port_updates_per_s": prate, "ratio": prate / rate,
                                    "note": "oracle C port on the same sample, 1 epoch"}
    return out


def launch_overrides(args) -> dict:
    """Command-line overrides of the layout's per-launch Q-band options."""
    return {"impl": args.qband_impl if args.qband_impl >= 0 else None,
            "chain_cfg": args.chain_cfg if args.chain_cfg >= 0 else None,
            "pstore": args.pstore if args.pstore >= 0 else None,
            "qsync": args.qsync, "lockstep": args.chain_lockstep}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(args, world, rank, local):
    import torch
    from paper_2006_15980_b200 import _lib, kernels
    from paper_2006_15980_b200.data import bucket_qbands, build_device_grid, synthetic_band
    from paper_2006_15980_b200.sgd import init_device_model, rmse

    _lib.load()
    if args.variant is not None:
        _lib.set_variant(args.variant)
    # per-launch overrides of the layout's Q-band options (ABI 4)
    overrides = launch_overrides(args)
    dev = torch.device("cuda", local)
    n_users, n_items, n_train, k0, desc = WORKLOADS[args.workload]
    k = args.k or k0
    precision = args.precision
    n_total = int(round(n_train / (1.0 - TEST_FRACTION)))
    # the whole matrix on one GPU: synthetic_band over every row (the same
    # generator the N > 1 ranks use for their bands of one matrix)
    t0 = time.perf_counter()
    train, test = synthetic_band(n_users, n_items, n_total, 0, n_users, rank=8, noise=0.1,
                                 seed=SEED, test_fraction=TEST_FRACTION, device=dev)
    if args.item_skew > 0:
        # Zipf-like item popularity (p(item of rank r) ~ r^-alpha), for the
        # layout's handling of hot items; ratings keep the law's values
        g = torch.Generator(device=dev)
        g.manual_seed(SEED + 17)
        w = torch.arange(1, n_items + 1, device=dev, dtype=torch.float64).pow(-args.item_skew)
        perm = torch.randperm(n_items, device=dev, generator=g)
        for part in (train, test):
            for a in range(0, part.nnz, 1 << 24):
                z = min(part.nnz, a + (1 << 24))
                part.items[a:z] = perm[torch.multinomial(w, z - a, replacement=True,
                                                         generator=g)].to(torch.int32)
        del w, perm
    nnz = train.nnz
    # 1-GPU batch-only uniform plan: 1 row band x 2 column bands
    row_cuts = np.array([0, n_users], dtype=np.int64)
    col_cuts = np.array([0, (n_items + 1) // 2, n_items], dtype=np.int64)
    grid = build_device_grid(train, row_cuts, col_cuts)
    tile_bytes = None if args.tile_mb is None else int(args.tile_mb * (1 << 20))
    # free the generator's arrays (train/test are views of them): keep a
    # compact copy of the test set only — Hugewiki needs the headroom
    from paper_2006_15980_b200.data import DeviceTriples
    # the test set in user order: the residual kernel's P reads then walk
    # user ranges (L2-friendly); a sum does not depend on the order
    order = torch.argsort(test.users)
    test = DeviceTriples(test.n_users, test.n_items, test.users[order].contiguous(),
                         test.items[order].contiguous(), test.ratings[order].contiguous())
    del order
    del train
    torch.cuda.empty_cache()
    if args.kernel == "qband":
        bucket_qbands(grid, k, tile_bytes=tile_bytes, elem_bytes=2 if precision == "f16" else 4,
                      impl=(5 if args.split else (args.qband_impl if args.qband_impl >= 0
                                                  else None)),
                      split=args.split or None, max_tile_rows=args.tile_rows,
                      chain_cfg=args.chain_cfg)
    stream_epoch = None
    if not args.no_e2e and args.kernel == "qband" and world == 1:
        # e2e streams the same kind of layout from pinned host memory, tile by
        # tile; run groups over tiles of at most --stream-tile-rows users, so
        # each user id crosses PCIe as one byte (5 B per rating, not 6)
        from paper_2006_15980_b200.workers import StreamingEpoch
        sgrid = grid
        if (getattr(grid, "sub_impl", None) == 8 and args.stream_tile_rows
                and int(grid.sub_max_rows) > args.stream_tile_rows):
            from paper_2006_15980_b200.data import DeviceGrid
            sgrid = DeviceGrid(grid.n_rows, grid.n_cols, grid.row_cuts, grid.col_cuts,
                               grid.region_of_row, grid.sub_row_parent, grid.users.clone(),
                               grid.items.clone(), grid.ratings.clone(),
                               np.asarray(grid.block_ptr).copy())
            bucket_qbands(sgrid, k, elem_bytes=2 if precision == "f16" else 4, impl=8,
                          max_tile_rows=args.stream_tile_rows)
        stream_epoch = StreamingEpoch(sgrid, k, n_buffers=args.stream_buffers,
                                      tiles_per_chunk=args.stream_tiles,
                                      runs_chunks_per_block=args.stream_chunks,
                                      last_chunk_tiles=args.stream_last,
                                      reuse=args.stream_reuse, opts=overrides)
    model = init_device_model(n_users, n_items, k, SEED, device=dev,
                              dtype="float16" if precision == "f16" else "float32")
    torch.cuda.synchronize(dev)
    setup_s = time.perf_counter() - t0

    stream = torch.cuda.current_stream(dev)
    counts = np.zeros(grid.n_blocks, dtype=np.int64)
    launch_events = []

    def step(record):
        for b in range(grid.n_blocks):
            lo, hi = grid.block_range(b)
            if hi <= lo:
                continue
            seed = kernels.mix64(kernels.mix64(SEED, b, int(counts[b])), 0)
            if record:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            if args.kernel == "qband":
                kernels.launch_block_qband(model.P, model.Q, grid, b, LR, REG, REG, seed,
                                           stream=stream.cuda_stream, opts=overrides)
            else:
                kernels.launch_sgd_range(model.P, model.Q, grid.users, grid.items, grid.ratings,
                                         lo, hi, LR, REG, REG, seed, 0, 0, args.mode,
                                         stream.cuda_stream)
            if record:
                e1.record(stream)
                launch_events.append((e0, e1, hi - lo))
            counts[b] += 1

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize(dev)
    barrier(world)
    torch.cuda.synchronize(dev)
    start_ev = torch.cuda.Event(enable_timing=True)
    end_ev = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start_ev.record(stream)
        for _ in range(args.steps):
            step(True)
        end_ev.record(stream)
        torch.cuda.synchronize(dev)
    barrier(world)
    elapsed_ms = start_ev.elapsed_time(end_ev)
    elapsed_ms = max_over_ranks(elapsed_ms, world)
    updates = sum_over_ranks(float(nnz * args.steps), world)
    value = updates / (elapsed_ms / 1e3)

    # dominant kernel: the HOGWILD update launches
    durs = [(a.elapsed_time(b), n) for a, b, n in launch_events]
    mean_ms = sum(d for d, _ in durs) / len(durs)
    mean_updates = sum(n for _, n in durs) / len(durs)
    bpu = bytes_per_update(k, precision)
    achieved = mean_updates * bpu / (mean_ms / 1e3) / 1e9
    peak, peak_kind = measured_peak()
    p_stores = (precision == "f32" and args.kernel == "qband"
                and (getattr(grid, "sub_impl", None) or 0) >= 4
                and (args.pstore == 1 or (args.pstore < 0 and getattr(grid, "sub_pstore", 0))))
    impl_used = getattr(grid, "sub_impl", None)
    # the L2 row-load ceiling describes the L2 row-tile kernels; 7 and 8 keep
    # P in shared memory
    l2_rows = None if (impl_used or 0) == 8 else l2_ceiling(k, precision, bool(p_stores))
    kernel_ups = mean_updates / (mean_ms / 1e3)
    # compulsory DRAM bytes of one launch: its triples once, one read and one
    # write of every P row of its row band and of every Q row of its column
    # band (what must cross HBM if nothing stayed in L2 between launches)
    s_el = 2 if precision == "f16" else 4
    comp = []
    for b in range(grid.n_blocks):
        lo, hi = grid.block_range(b)
        if hi <= lo:
            continue
        r0, r1 = grid.row_span(b // grid.n_col_bands)
        c0, c1 = grid.col_span(b % grid.n_col_bands)
        if impl_used == 8:
            # users + ratings (items live in the run descriptors, 16 B each)
            n_runs = int(grid.sub_ptr[b].shape[0])
            comp.append((hi - lo) * 8 + 16 * n_runs + 2 * ((r1 - r0) + (c1 - c0)) * k * s_el)
        else:
            comp.append((hi - lo) * 12 + 2 * ((r1 - r0) + (c1 - c0)) * k * s_el)
    compulsory = float(np.mean(comp)) if comp else None

    # test RMSE after the epochs run (not timed)
    test_rmse = rmse(test, model).value
    epochs_run = args.warmup + args.steps

    # e2e: the drop-in host-buffer call, per block, with pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = (run_e2e_stream(args, stream_epoch, model, test, dev) if stream_epoch is not None
               else None)
        e2e_dropin = run_e2e(args, grid, model, k, precision, dev, world)
        if e2e is None:
            e2e = e2e_dropin
        else:
            e2e["sgd_range_host_buffers"] = e2e_dropin

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(n_users, n_items, k, nnz)

    if rank == 0:
        line = {
            "metric": "sgd_updates_per_sec", "value": value, "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": precision,
            "data": "synthetic (synthetic_ratings law, device generator)",
            "config": workload_config(args),
            "counts": {"train_ratings": nnz, "test_ratings": test.nnz},
            "layout": {"grid": "uniform 1x2 (1 batch worker per GPU, partition.py:89-107)",
                       "parallelism": "single GPU", "mode": args.mode, "kernel": args.kernel,
                       "variant": args.variant,
                       "qband_impl": getattr(grid, "sub_impl", None),
                       "chain_cfg": (args.chain_cfg if (getattr(grid, "sub_impl", None) or 0) >= 4
                                     else None),
                       "item_run_split": getattr(grid, "sub_split", None),
                       "p_writeback": ((["vector reductions", "stores"][
                                           args.pstore if args.pstore >= 0
                                           else int(getattr(grid, "sub_pstore", 0) or 0)]
                                        if precision == "f32" else "vector reductions")
                                       if (getattr(grid, "sub_impl", None) or 0) >= 4 else None),
                       "item_skew": args.item_skew or None,
                       "row_tiles": (list(grid.sub_tiles) if getattr(grid, "sub_tiles", None)
                                     else None)},
            "roofline": roofline_fields(args, achieved, peak, peak_kind, bpu, mean_ms,
                                        mean_updates, compulsory, l2_rows, kernel_ups, p_stores,
                                        getattr(grid, "sub_impl", None)),
            "rmse": {"epochs": epochs_run, "test": test_rmse},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": len(launch_events),
            "clocks": clocks.summary(),
            "setup_seconds": setup_s,
        }
        print(json.dumps(line), flush=True)


def run_ours_multi(args, world, rank, local):
    """N > 1: one process per GPU over ONE synthetic matrix (data.synthetic_band:
    every rank generates its own row band, keyed by global ids, so the bands
    are pieces of the same matrix with the same held-out cells).
    * weak scaling (default): the matrix is N x the workload's users (each
      rank's band Netflix-shaped: 480 000 users, 100 M training ratings),
      items shared (17 700);
    * strong scaling: the workload's matrix itself, split into N row bands.
    P bands stay resident; Q column bands (2N+1) move between GPUs through
    the lease table and CUDA IPC peer pulls.  A step is one quota epoch of
    every GPU's blocks + a barrier."""
    import torch
    import torch.distributed as dist
    from paper_2006_15980_b200 import _lib
    from paper_2006_15980_b200.data import synthetic_band
    from paper_2006_15980_b200.distributed import CudaRowBand, RowBandTrainer, make_lease_table
    from paper_2006_15980_b200.sgd import DeviceModel, residual_sums

    _lib.load()
    dev = torch.device("cuda", local)
    n_users, n_items, n_train, k0, desc = WORKLOADS[args.workload]
    k = args.k or k0
    n_total = int(round(n_train / (1.0 - TEST_FRACTION)))
    geo = args.sim_world or world      # --sim-world: rank 0's share of a larger job
    if args.scaling == "strong":
        m_users, m_total = n_users, n_total            # the workload's matrix, split
        band_rows = -(-n_users // geo)
    else:
        m_users, m_total = n_users * geo, n_total * geo  # a workload-sized band per GPU
        band_rows = n_users
    row_lo, row_hi = rank * band_rows, min(m_users, (rank + 1) * band_rows)
    t0 = time.perf_counter()
    train, test = synthetic_band(m_users, n_items, m_total, row_lo, row_hi, rank=8, noise=0.1,
                                 seed=SEED, test_fraction=TEST_FRACTION, device=dev)
    n_cols = args.cols_per_gpu * geo + 1
    col_cuts = np.linspace(0, n_items, n_cols + 1).astype(np.int64)
    band = CudaRowBand(dist, rank, world, dev, train, row_lo, row_hi, col_cuts, k, LR, REG, REG,
                       init_seed=SEED, kernel=args.multi_kernel,
                       concurrency=args.multi_concurrency, split=args.split or None)
    del train
    torch.cuda.synchronize(dev)
    setup_s = time.perf_counter() - t0
    run_id = [f"bench{os.getpid()}"]
    dist.broadcast_object_list(run_id, src=0)
    table = make_lease_table(args.lease, dist.distributed_c10d._get_default_store(), n_cols,
                             rank, run_id[0])
    if rank == 0:
        table.initialize()
    dist.barrier()
    trainer = RowBandTrainer(band, table, rank, seed=SEED, policy=args.policy, world=world)
    for _ in range(args.warmup):
        trainer.run_epoch()
        dist.barrier()
    torch.cuda.synchronize(dev)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    upd0 = trainer.total_updates
    blocks0 = int(trainer.counts.sum())
    with ClockSampler(local) as clocks:
        e0.record(band.stream)
        for _ in range(args.steps):
            trainer.run_epoch()
            dist.barrier()
        e1.record(band.stream)
        torch.cuda.synchronize(dev)
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    updates = sum_over_ranks(float(trainer.total_updates - upd0), world)
    # lease-table cost (all epochs so far), worst rank, against the timed step
    st = trainer.lease_stats()
    lease_stats = {"table": st["table"], "leases_rank0": st["leases"],
                   "ops_per_lease": st["ops_per_lease"],
                   "us_per_lease_max_rank": max_over_ranks(st["us_per_lease"], world),
                   "share_of_step_max_rank": max_over_ranks(
                       st["seconds"] / max(1, args.warmup + args.steps) / (ms / args.steps / 1e3),
                       world)}
    # one kernel launch per granted block (CudaRowBand.compute)
    launches = int(sum_over_ranks(float(int(trainer.counts.sum()) - blocks0), world))
    # test RMSE after exactly warmup + steps epochs (the N = 1 line's count)
    band.refresh_q(table)
    dist.barrier()
    sums = residual_sums(DeviceModel(band.P, band.Q), test.users, test.items, test.ratings,
                         row_base=row_lo).to(_reduce_device())
    dist.all_reduce(sums)
    n_test = sum_over_ranks(float(test.nnz), world)
    test_rmse = float(np.sqrt(sums[0].item() / n_test))
    n_train = sum_over_ranks(float(band.grid.nnz), world)
    e2e = None
    if not args.no_e2e:
        # end to end through the same lease loop: every granted block's
        # triples uploaded from pinned host memory before its launch, and
        # each rank's residual sums (its band, its Q replica) read back per
        # step; wall clock with device syncs, max over ranks
        band.stage_from_host(True)
        e2e_steps = max(3, args.steps)
        torch.cuda.synchronize(dev)
        dist.barrier()
        b0, u0 = band.staged_bytes, trainer.total_updates
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            trainer.run_epoch()
            float(residual_sums(DeviceModel(band.P, band.Q), test.users, test.items,
                                test.ratings, row_base=row_lo)[0].item())
            dist.barrier()
        torch.cuda.synchronize(dev)
        dt = max_over_ranks(time.perf_counter() - t0, world)
        band.stage_from_host(False)
        e2e = {"value": sum_over_ranks(float(trainer.total_updates - u0), world) / dt,
               "unit": "updates/s",
               "h2d_bytes_per_step": int(sum_over_ranks(float(band.staged_bytes - b0), world)
                                         / e2e_steps),
               "d2h_bytes_per_step": 24 * world, "steps": e2e_steps,
               "path": "distributed.RowBandTrainer lease loop with CudaRowBand.stage_from_host: "
                       "each granted block's ratings uploaded from pinned host memory ("
                       + ("6 B/rating: uint16 user ids relative to the row tile, item implicit"
                          if band.compact is not None else "12 B/rating triples")
                       + ") on the copy stream, the block granted ahead uploading while the "
                       "current one trains; per-rank residual sums read back every step. The "
                       "device copy of the band's ratings stays allocated (each lease "
                       "overwrites its block from the host): a data-off-device run is the N=1 "
                       "workers.StreamingEpoch path"}
    if rank == 0:
        print(json.dumps({
            "metric": "sgd_updates_per_sec", "value": updates / (ms / 1e3), "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (synthetic_ratings law, device generator)",
            "config": workload_config(args),
            "counts": {"train_ratings": int(n_train), "test_ratings": int(n_test)},
            "layout": {"matrix": (f"{desc} row band per GPU of one {m_users}x{n_items} matrix "
                                  "(weak scaling)" if args.scaling == "weak" else
                                  f"{desc} split into {geo} row bands (strong scaling)")
                                 + ": each rank generates its row band of it "
                                   "(data.synthetic_band, keyed by global ids)",
                       "grid": f"{geo} row bands x {n_cols} column bands",
                       "devices": int(torch.cuda.device_count()),
                       "simulated": (None if not args.sim_world else
                                     f"one process with rank 0's band and column geometry of "
                                     f"a {geo}-GPU job (per-GPU throughput; peer pulls of Q "
                                     f"bands not exercised)"),
                       "parallelism": f"dp{world} row bands, Q bands leased and pulled peer-to-peer",
                       "kernel": band.kernel, "qband_impl": getattr(band.grid, "sub_impl", None),
                       "item_run_split": getattr(band.grid, "sub_split", None),
                       "blocks_in_flight": band.concurrency},
            "rmse": {"epochs": args.warmup + args.steps, "test": test_rmse},
            "lease_wait_seconds_rank0": trainer.wait_seconds,
            "leases": lease_stats, "policy": args.policy,
            "setup_seconds": setup_s,
            "gpu_launches": launches, "clocks": clocks.summary(), "e2e": e2e,
        }), flush=True)
    dist.barrier()
    table.close(unlink=rank == 0)


def run_e2e_stream(args, se, model, test, dev):
    """e2e through the public engine API: every step streams that epoch's
    triples from pinned host memory (workers.StreamingEpoch: chunk c+1
    uploads while chunk c trains; every chunk is uploaded every epoch unless
    --stream-reuse) and reads the step's result —
    the test RMSE sum — back to the host.  P and Q stay resident, as in
    training.  Steps are software-pipelined: step i+1's uploads and kernels
    are queued before the host waits for step i's result, so the GPU does not
    idle while the host reads it.  h2d_bytes_per_step counts the bytes
    actually uploaded."""
    import torch
    from paper_2006_15980_b200.sgd import Hyperparams, residual_sums
    from paper_2006_15980_b200.sgd import DeviceModel
    hp = Hyperparams(n_factors=model.n_factors, reg_user=REG, reg_item=REG, learning_rate=LR)
    dm = DeviceModel(model.P, model.Q)
    steps = max(3, args.steps)
    result = torch.empty((steps + 2, 3), dtype=torch.float64).pin_memory()

    def launch(i):
        se.run(model.P, model.Q, hp, seed=1000 + i)
        h2d = se.h2d_bytes_last()
        result[i].copy_(residual_sums(dm, test.users, test.items, test.ratings),
                        non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return ev, h2d

    for i in range(2):                      # warm-up steps
        launch(steps + i)[0].synchronize()
    torch.cuda.synchronize(dev)
    import gc
    gc.collect()
    gc.disable()          # no collector pauses inside the timed host loop
    h2d, sq = 0, None
    try:
        marks = [time.perf_counter()]
        pending = None
        for i in range(steps):
            ev, b = launch(i)
            h2d += b
            if pending is not None:         # the previous step's result, read back
                pending.synchronize()
                sq = float(result[i - 1, 0])
                marks.append(time.perf_counter())
            pending = ev
        pending.synchronize()
        sq = float(result[steps - 1, 0])
        marks.append(time.perf_counter())
    finally:
        gc.enable()
    dt = marks[-1] - marks[0]
    per = sorted(1e3 * (b - a) for a, b in zip(marks, marks[1:]))
    return {"value": se.nnz * steps / dt, "unit": "updates/s",
            "h2d_bytes_per_step": int(round(h2d / steps)), "d2h_bytes_per_step": 24,
            "steps": steps,
            "ms_per_step": {"min": per[0], "median": per[len(per) // 2], "max": per[-1]},
            "test_rmse_after": float(np.sqrt(sq / test.nnz)),
            "path": "workers.StreamingEpoch (pinned host triples streamed per epoch, "
                    + (f"{se.bytes_per_rating} B/rating: "
                       + (f"{1 if se.u8 else 2}-byte user ids relative to the row tile, "
                          if se.u16 else "")
                       + ("item from its run descriptor (resident); " if se.runs else
                          "item implicit in its sub-band; " if se.implicit_items else "triples; "))
                    + (f"run groups (implementation 8), tiles of <= {se.sg.sub_max_rows} users, "
                       f"{se.n_chunks} chunks" if se.runs else
                       f"{se.n_chunks} chunks of {se.tiles_per_chunk} row tile(s)")
                    + (f" (each block's last {se.last_chunk_tiles})" if se.last_chunk_tiles
                       and not se.runs else "") + ", "
                    f"{se.n_buffers} staging buffers, H2D overlapped with the Q-band kernel; "
                    + ("chunks still staged from the previous epoch are not uploaded again"
                       if se.reuse else "every chunk uploaded every epoch")
                    + ") + device RMSE sums read back every step (steps pipelined: step i+1 "
                    "queued before step i's result is read)"}


def run_e2e(args, grid, model, k, precision, dev, world):
    """Same metric through the reference-facing host-buffer call."""
    import torch
    from paper_2006_15980_b200 import kernels
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    h_users = pin(grid.users).numpy()
    h_items = pin(grid.items).numpy()
    h_vals = pin(grid.ratings).numpy()
    h_P = pin(model.P).numpy()
    h_Q = pin(model.Q).numpy()
    steps = max(1, min(args.steps, 3))
    h2d = d2h = 0
    for b in range(grid.n_blocks):
        lo, hi = grid.block_range(b)
        lo_al = lo & ~3
        h2d += (hi - lo_al) * 12 + h_P.nbytes + h_Q.nbytes
        d2h += h_P.nbytes + h_Q.nbytes

    def step():
        for b in range(grid.n_blocks):
            lo, hi = grid.block_range(b)
            kernels.sgd_range(h_P, h_Q, h_users, h_items, h_vals, lo, hi, LR, REG, REG,
                              kernels.mix64(SEED, b, 99), 0, 0, mode=args.mode, device=dev.index)

    step()  # warm-up
    torch.cuda.synchronize(dev)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t0
    dt = max_over_ranks(dt, world)
    ups = sum_over_ranks(float(grid.nnz * steps), world) / dt
    return {"value": ups, "unit": "updates/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "path": "kernels.sgd_range(numpy pinned host arrays) per block"}


def free_port() -> int:
    import socket
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        return int(sock.getsockname()[1])


def self_launch(n: int, argv: list) -> int:
    """Re-run this script under torch.distributed.run with n ranks on this
    node (rendezvous on 127.0.0.1); rank 0 prints the JSON line.  NCCL's init
    log is on so every rank's communicator (nranks) shows in the output."""
    import subprocess
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), str(Path(__file__).resolve()), *argv]
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="netflix")
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--precision", choices=["f32", "f16"], default="f32")
    ap.add_argument("--variant", type=int, default=None)
    ap.add_argument("--mode", choices=["hogwild", "hogwild_lww"], default="hogwild")
    ap.add_argument("--kernel", choices=["qband", "hogwild"], default="qband",
                    help="qband: Q band in shared memory (engine fast path); hogwild: "
                         "global-Q kernel behind hmf_sgd_range")
    ap.add_argument("--multi-kernel", choices=["auto", "qband", "range"], default="auto")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="N>1: a workload-sized band per GPU (weak) or the workload split (strong)")
    ap.add_argument("--cols-per-gpu", type=int, default=2,
                    help="N>1: column bands = this x N + 1 (2: a primary and a staged-ahead "
                         "band per GPU plus a spare)")
    ap.add_argument("--lease", choices=["shm", "store"], default="shm",
                    help="N>1: column-lease table: node-local shared memory (csrc/lease.cu) "
                         "or the torch.distributed store")
    ap.add_argument("--policy", choices=["free", "quota"], default="free",
                    help="N>1 lease policy: free = any free column band, an epoch being "
                         "N x bands block updates claimed job-wide (the reference's POLICY_FREE, "
                         "scheduler.py:411-429); quota = each GPU trains each of its blocks once "
                         "per epoch")
    ap.add_argument("--multi-concurrency", type=int, default=1,
                    help="N>1: column blocks in flight per GPU (each on its own stream)")
    ap.add_argument("--qband-impl", type=int, choices=[-1, 0, 4, 5, 6, 8], default=-1,
                    help="Q-band kernel: 0 = warp per rating, 4-6 chained item runs, 8 run "
                         "groups over a tile-resident P (-1: the layout's choice, "
                         "data.tile_resident_impl, else 5)")
    ap.add_argument("--chain-cfg", type=int, choices=[-1, 2, 4, 5, 6], default=-1,
                    help="configuration of the chained kernel (qchain.cuh ChainCfg)")
    ap.add_argument("--chain-lockstep", type=int, choices=[0, 1, 2, 3], default=None)
    ap.add_argument("--pstore", type=int, choices=[-1, 0, 1], default=-1,
                    help="chained kernel P write-back: -1 the layout's (grid.sub_pstore), "
                         "0 reductions, 1 stores")
    ap.add_argument("--stream-buffers", type=int, default=3,
                    help="e2e: device staging buffers (ring)")
    ap.add_argument("--stream-tile-rows", type=int, default=256,
                    help="e2e with implementation 8: row tiles of at most this many users "
                         "(256: one-byte user ids, 5 B per streamed rating; 0: the resident "
                         "layout's tiles)")
    ap.add_argument("--stream-chunks", type=int, default=2,
                    help="e2e with implementation 8: chunks per block (each a whole fraction "
                         "of the block's row tiles)")
    ap.add_argument("--stream-tiles", type=int, default=4,
                    help="e2e: row tiles per streamed chunk (one launch each)")
    ap.add_argument("--stream-last", type=int, default=0,
                    help="e2e: row tiles in each block's last chunk (0 = --stream-tiles)")
    ap.add_argument("--stream-reuse", action="store_true",
                    help="e2e: do not re-upload chunks still staged from the previous epoch "
                         "(default: every epoch uploads all of its triples)")
    ap.add_argument("--qsync", type=int, default=None,
                    help="implementation 5: ratings between Q-delta publications "
                         "(default: the layout's grid.sub_qsync)")
    ap.add_argument("--item-skew", type=float, default=0.0,
                    help="Zipf exponent of item popularity (0 = the synthetic law's uniform cells)")
    ap.add_argument("--split", type=int, default=0,
                    help="implementation 5 with this many parts per item run (0 = default layout)")
    ap.add_argument("--tile-rows", type=int, default=None,
                    help="cap on users per row tile (default data.QBAND_MAX_TILE_ROWS; 0 = none)")
    ap.add_argument("--tile-mb", type=float, default=None,
                    help="P rows per Q-band row tile in MiB (default data.QBAND_TILE_BYTES; 0 = no byte bound)")
    ap.add_argument("--tile-stagger", action="store_true",
                    help="experimental: uneven first/last P tiles per CTA (data.PTILE_STAGGER)")
    ap.add_argument("--sim-world", type=int, default=0,
                    help="N=1 only: run rank 0 of an N-GPU job's geometry (projected per-GPU rate)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--spawn-probe", action="store_true",
                    help="print each rank's RANK/WORLD_SIZE and exit (tests the self-launch)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.tile_stagger:
        import paper_2006_15980_b200.data as _data
        _data.PTILE_STAGGER = True
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # `python bench.py --gpus N`: one process per GPU, launched here
        sys.exit(self_launch(args.gpus, sys.argv[1:]))
    if args.spawn_probe:
        print(json.dumps({"rank": int(os.environ.get("RANK", "0")),
                          "world": int(os.environ.get("WORLD_SIZE", "1")),
                          "local_rank": int(os.environ.get("LOCAL_RANK", "0"))}), flush=True)
        return
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
        rank = int(os.environ.get("RANK", "0"))
        run_reference_arm(args, world, rank)
        return
    world, rank, local = dist_setup()
    if world == 1 and args.sim_world:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29000 + os.getpid() % 1000))
        dist.init_process_group("gloo", rank=0, world_size=1)
        run_ours_multi(args, world, rank, local)
        dist.destroy_process_group()
        return
    if world > 1:
        run_ours_multi(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
