"""The per-rating SGD update on B200 — drop-in for hetmf.kernels.

Mirrors the reference module's surface (hetmf/kernels.py): SHUFFLE_WINDOW,
mix64, sgd_range, warmup.  `sgd_range` keeps the reference signature
(kernels.py:62-63) and in-place semantics; the arrays may be

* CUDA tensors (torch) — the device-resident fast path: one stream-ordered
  launch of the hand-written sm_100a kernel, no copies; or
* host numpy arrays — the drop-in path: the call copies the triples and both
  factor arrays to the device, runs the same kernel and copies the factors
  back in place, so callers holding numpy arrays (the reference's own layout)
  see the reference's contract.

Factor storage follows the array dtype: float32 (fp32), float16 (fp16
storage, fp32 arithmetic) or float64.  `mode` picks HOGWILD (throughput,
lock-free), ORDERED (the reference's exact visit order, fp32 arithmetic) or
EXACT (reference order and reference f64 arithmetic: bit-identical output).
There is no CPU path: without the CUDA library every call raises.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib

SHUFFLE_WINDOW = 4096  # hetmf/kernels.py:24

_MASK64 = 0xFFFFFFFFFFFFFFFF


def mix64(*parts: int) -> int:
    """splitmix64 fold of integer parts, clipped to 63 bits (kernels.py:32-48).

    Host-side integer arithmetic (it seeds launches; it is not on the device
    path); hmf_mix64 in libhmf computes the same function for C callers.
    """
    h = 0x6A09E667F3BCC909
    for p in parts:
        h = ((h ^ (int(p) & _MASK64)) + 0x9E3779B97F4A7C15) & _MASK64
        h = ((h ^ (h >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
        h = ((h ^ (h >> 27)) * 0x94D049BB133111EB) & _MASK64
        h ^= h >> 31
    return h & 0x7FFFFFFFFFFFFFFF


def _torch():
    import torch
    return torch


def current_stream_handle(device=None) -> int:
    torch = _torch()
    return int(torch.cuda.current_stream(device).cuda_stream)


_STORAGE = {"float32": "f32", "float16": "f16", "float64": "f64"}


def _storage_of(dtype) -> str:
    name = str(dtype).replace("torch.", "")
    if name not in _STORAGE:
        raise TypeError(f"factor arrays must be float32, float16 or float64, not {name}")
    return _STORAGE[name]


def _check_factor(t, name):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dim() != 2 or not t.is_contiguous():
        raise ValueError(f"{name} must be a C-contiguous 2-D array")


def launch_sgd_range(user_f, item_f, rows, cols, vals, start, stop, lr, reg_user, reg_item,
                     seed, row_base=0, col_base=0, mode="hogwild", stream=None) -> int:
    """Device fast path: all arrays are CUDA tensors; returns triples processed."""
    torch = _torch()
    _check_factor(user_f, "user_f")
    _check_factor(item_f, "item_f")
    if user_f.dtype != item_f.dtype:
        raise TypeError("user_f and item_f must share a dtype")
    k = user_f.shape[1]
    if item_f.shape[1] != k:
        raise ValueError("factor arrays disagree on the factor count")
    st = _storage_of(user_f.dtype)
    want_vals = torch.float64 if st == "f64" else torch.float32
    for t, name, dt in ((rows, "rows", torch.int32), (cols, "cols", torch.int32),
                        (vals, "vals", want_vals)):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dt:
            raise TypeError(f"{name} must be a CUDA {dt} tensor")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    start, stop = int(start), int(stop)
    if stop - start <= 0:
        return 0
    if start < 0 or stop > rows.numel() or stop > cols.numel() or stop > vals.numel():
        raise IndexError("triple range out of bounds")
    m = _lib.MODES[mode] if isinstance(mode, str) else int(mode)
    s = current_stream_handle(user_f.device) if stream is None else int(stream)
    fn = getattr(_lib.load(), f"hmf_sgd_range_{st}")
    got = fn(user_f.data_ptr(), item_f.data_ptr(), k, rows.data_ptr(), cols.data_ptr(),
             vals.data_ptr(), start, stop, float(lr), float(reg_user), float(reg_item),
             int(seed) & _MASK64, int(row_base), int(col_base), m, s)
    return _lib.check(got, f"hmf_sgd_range_{st}")


QbandOpts = _lib.QbandOpts


def qband_opts(grid=None, **overrides) -> "QbandOpts":
    """The per-launch options (hmf_qband_opts, ABI 4) of a layout: what
    data.bucket_qbands chose for `grid` (sub_impl, sub_cfg, sub_pstore,
    sub_qsync), then every override that is not None (impl, chain_cfg,
    pstore, qsync, grid_share, lockstep).  Options travel with each launch;
    nothing is process-wide, so threads launching different layouts at once
    do not interfere."""
    vals = {}
    if grid is not None:
        impl = getattr(grid, "sub_impl", None)
        vals["impl"] = -1 if impl is None else int(impl)
        cfg = getattr(grid, "sub_cfg", None)
        vals["chain_cfg"] = -1 if cfg is None else int(cfg)
        vals["pstore"] = int(getattr(grid, "sub_pstore", 0) or 0)
        q = int(getattr(grid, "sub_qsync", 0) or 0)
        vals["qsync"] = q if q > 0 else -1
        if int(getattr(grid, "sub_wide", 0) or 0):
            vals["runs_wide"] = 1
    vals.update({k: v for k, v in overrides.items() if v is not None})
    return QbandOpts(**vals)


def _as_opts(grid, opts) -> "QbandOpts":
    if opts is None:
        return qband_opts(grid)
    if isinstance(opts, QbandOpts):
        return opts
    return qband_opts(grid, **dict(opts))


def launch_block_qband(user_f, item_f, grid, block, lr, reg_user, reg_item, seed, row_base=0,
                       col_base=0, stream=None, opts=None) -> int:
    """Q-band-stationary update of one block of a DeviceGrid bucketed by
    data.bucket_qbands (the engine fast path).  `opts`: a QbandOpts, a dict
    of overrides of the layout's options, or None (the layout's).  Returns
    triples processed."""
    _check_factor(user_f, "user_f")
    _check_factor(item_f, "item_f")
    if grid.sub_ptr is None:
        raise ValueError("grid has no Q-band sub-bucketing (data.bucket_qbands)")
    st = _storage_of(user_f.dtype)
    if st == "f64":
        raise TypeError("the Q-band kernel stores f32 or f16 factors")
    lo, hi = grid.block_range(block)
    if hi <= lo:
        return 0
    s = current_stream_handle(user_f.device) if stream is None else int(stream)
    o = _as_opts(grid, opts)
    if int(grid.sub_impl) == 8:
        # run groups: per-block run descriptors, offsets relative to the block start
        fn = getattr(_lib.load(), f"hmf_sgd_block_runs_{st}")
        _lib.check(fn(user_f.data_ptr(), item_f.data_ptr(), user_f.shape[1],
                      grid.users.data_ptr() + 4 * lo, grid.ratings.data_ptr() + 4 * lo,
                      grid.sub_ptr[block].data_ptr(),
                      grid.sub_tile_run[block].data_ptr(), grid.sub_tile_cuts[block].data_ptr(),
                      grid.sub_tiles[block], int(grid.sub_max_rows), ctypes.byref(o), float(lr),
                      float(reg_user), float(reg_item), int(seed) & _MASK64, int(row_base),
                      int(col_base), s), f"hmf_sgd_block_runs_{st}")
        return hi - lo
    sp, sc = grid.sub_ptr[block], grid.sub_cuts[block]
    n_tiles = grid.sub_tiles[block] if grid.sub_tiles is not None else 1
    n_sub = int(sc.numel()) - 1
    if int(sp.numel()) != n_tiles * n_sub + 1:
        raise ValueError("sub_ptr does not match sub_cuts x sub_tiles")
    fn = getattr(_lib.load(), f"hmf_sgd_block_qband_{st}")
    _lib.check(fn(user_f.data_ptr(), item_f.data_ptr(), user_f.shape[1], grid.users.data_ptr(),
                  grid.items.data_ptr(), grid.ratings.data_ptr(), sp.data_ptr(), sc.data_ptr(),
                  n_sub, n_tiles, ctypes.byref(o), float(lr), float(reg_user),
                  float(reg_item), int(seed) & _MASK64, int(row_base), int(col_base), s),
               f"hmf_sgd_block_qband_{st}")
    return hi - lo


def sgd_range(user_f, item_f, rows, cols, vals, start, stop, lr, reg_user, reg_item, seed,
              row_base, col_base, *, mode="hogwild", stream=None, device=None) -> int:
    """Apply one SGD pass over triples[start:stop] (hetmf/kernels.py:61-133).

    user_f is indexed by rows[i] - row_base, item_f by cols[i] - col_base.
    Returns the number of triples processed (stop - start, 0 when empty).
    """
    torch = _torch()
    if isinstance(user_f, torch.Tensor):
        return launch_sgd_range(user_f, item_f, rows, cols, vals, start, stop, lr, reg_user,
                                reg_item, seed, row_base, col_base, mode, stream)
    # Host arrays: stage [start, stop) and both factor arrays on the device,
    # run, write the factors back in place.
    if not (isinstance(user_f, np.ndarray) and isinstance(item_f, np.ndarray)):
        raise TypeError("factor arrays must be numpy arrays or CUDA tensors")
    if not (user_f.flags.c_contiguous and item_f.flags.c_contiguous):
        raise ValueError("factor arrays must be C-contiguous")
    start, stop = int(start), int(stop)
    if stop - start <= 0:
        return 0
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    # One call at a time per pair of host factor arrays: each call uploads
    # both arrays whole and writes them back whole, so two concurrent calls
    # on the same arrays (the reference's BatchEngine lanes, workers.py:
    # 244-255) would otherwise overwrite each other's updates.  Serialised,
    # every call sees all updates of the calls before it.
    with _host_lock(user_f, item_f):
        return _sgd_range_host(user_f, item_f, rows, cols, vals, start, stop, lr, reg_user,
                               reg_item, seed, row_base, col_base, mode, stream, dev)


_host_locks: dict = {}
_host_locks_guard = threading.Lock()


def _host_lock(user_f, item_f):
    key = (user_f.__array_interface__["data"][0], item_f.__array_interface__["data"][0])
    with _host_locks_guard:
        lock = _host_locks.get(key)
        if lock is None:
            lock = _host_locks[key] = threading.Lock()
        return lock


def _sgd_range_host(user_f, item_f, rows, cols, vals, start, stop, lr, reg_user, reg_item, seed,
                    row_base, col_base, mode, stream, dev) -> int:
    torch = _torch()
    st = _storage_of(user_f.dtype)
    vdt = np.float64 if st == "f64" else np.float32
    lo = start & ~3  # keep the device triple arrays 16-byte aligned at `lo`
    d_rows = torch.from_numpy(np.ascontiguousarray(rows[lo:stop], dtype=np.int32)).to(dev, non_blocking=True)
    d_cols = torch.from_numpy(np.ascontiguousarray(cols[lo:stop], dtype=np.int32)).to(dev, non_blocking=True)
    d_vals = torch.from_numpy(np.ascontiguousarray(vals[lo:stop], dtype=vdt)).to(dev, non_blocking=True)
    d_p = torch.from_numpy(user_f).to(dev, non_blocking=True)
    d_q = torch.from_numpy(item_f).to(dev, non_blocking=True)
    got = launch_sgd_range(d_p, d_q, d_rows, d_cols, d_vals, start - lo, stop - lo, lr, reg_user,
                           reg_item, seed, row_base, col_base, mode, stream)
    if stream is not None:
        torch.cuda.synchronize(dev)
    torch.from_numpy(user_f).copy_(d_p, non_blocking=False)
    torch.from_numpy(item_f).copy_(d_q, non_blocking=False)
    return got


def visit_order(n: int, seed: int, device=None):
    """The reference visit order of n triples (offsets), computed on device."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    out = torch.empty(max(int(n), 0), dtype=torch.int32, device=dev)
    if n > 0:
        _lib.check(_lib.load().hmf_visit_order(int(n), int(seed) & _MASK64, out.data_ptr(),
                                               current_stream_handle(dev)), "hmf_visit_order")
    return out


def warmup(k: int = 8) -> None:
    """Load the library and initialise the CUDA context (kernels.py:136-143)."""
    torch = _torch()
    _lib.load()
    if not torch.cuda.is_available():
        raise _lib.HmfError("no CUDA device: the B200 engine has no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device())
    P = torch.zeros((2, k), dtype=torch.float32, device=dev)
    Q = torch.zeros((2, k), dtype=torch.float32, device=dev)
    r = torch.zeros(2, dtype=torch.int32, device=dev)
    v = torch.zeros(2, dtype=torch.float32, device=dev)
    launch_sgd_range(P, Q, r, r, v, 0, 2, 0.0, 0.0, 0.0, 1, 0, 0)
    torch.cuda.synchronize(dev)
