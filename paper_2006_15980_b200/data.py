"""Rating triples, block grids and synthetic instances (host and device).

Host side keeps the reference's data contract (hetmf/data.py): RatingMatrix
(int32 users/items, f64 ratings, id remap tables), shuffle_triples,
BlockGrid/build_grid (block-major, CSR block_ptr, stable within a block) and
synthetic_ratings with the reference's law *and* its numpy RNG call sequence,
so small instances are bit-identical to the reference's.

Device side is the B200 layout the hot path reads:
  DeviceTriples  SoA int32 users, int32 items, f32 (or f64) ratings in HBM;
  DeviceGrid     the same, bucketed block-major by hmf_bucket_triples (a
                 stable partition, data.py:238-280), plus block_ptr;
  synthetic_device  the synthetic_ratings law generated on the GPU for shapes
                 the reference generator cannot reach (Netflix, Yahoo R1,
                 Hugewiki), with hmf_synthetic_{count,cells,fill}.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib

CACHE_MAGIC = b"HMF1"
REGION_STREAM = 0
REGION_BATCH = 1


class DataError(ValueError):
    """Malformed input or inconsistent rating data (data.py:23-24)."""


class GridError(ValueError):
    """Invalid block-grid geometry (data.py:27-28)."""


@dataclass
class RatingMatrix:
    """Coordinate-form ratings with dense 0-based indices (data.py:31-73).

    user_ids / item_ids map dense index -> original id; the inverse maps
    user_index / item_index are built lazily (a dict over 50 M Hugewiki users
    is not free).
    """

    n_users: int
    n_items: int
    users: np.ndarray
    items: np.ndarray
    ratings: np.ndarray
    user_ids: np.ndarray = field(default=None)
    item_ids: np.ndarray = field(default=None)
    _user_index: dict = field(default=None, repr=False)
    _item_index: dict = field(default=None, repr=False)

    def __post_init__(self):
        if self.user_ids is None:
            self.user_ids = np.arange(self.n_users, dtype=np.int64)
        if self.item_ids is None:
            self.item_ids = np.arange(self.n_items, dtype=np.int64)

    @property
    def user_index(self) -> dict:
        if self._user_index is None:
            self._user_index = {int(x): i for i, x in enumerate(self.user_ids)}
        return self._user_index

    @property
    def item_index(self) -> dict:
        if self._item_index is None:
            self._item_index = {int(x): i for i, x in enumerate(self.item_ids)}
        return self._item_index

    @property
    def nnz(self) -> int:
        return len(self.ratings)

    def validate(self) -> None:
        if not (len(self.users) == len(self.items) == len(self.ratings)):
            raise DataError("triple arrays have mismatched lengths")
        if self.nnz:
            if self.users.min() < 0 or self.users.max() >= self.n_users:
                raise DataError("user index out of range")
            if self.items.min() < 0 or self.items.max() >= self.n_items:
                raise DataError("item index out of range")
        if not np.all(np.isfinite(self.ratings)):
            raise DataError("non-finite rating value")


def _with_order(matrix: RatingMatrix, order) -> RatingMatrix:
    return RatingMatrix(matrix.n_users, matrix.n_items, matrix.users[order],
                        matrix.items[order], matrix.ratings[order], matrix.user_ids,
                        matrix.item_ids, matrix._user_index, matrix._item_index)


def shuffle_triples(matrix: RatingMatrix, seed: int) -> RatingMatrix:
    """Seed-deterministic permutation of the triples (data.py:153-166)."""
    return _with_order(matrix, np.random.default_rng(seed).permutation(matrix.nnz))


def align_ratings(testset: RatingMatrix, train: RatingMatrix):
    """Map held-out triples into the training index space (data.py:135-150).

    Vectorised: original ids are looked up by binary search in the training
    id tables.  Returns (users, items, ratings, n_skipped)."""
    def lookup(dense, ids_test, ids_train):
        orig = np.asarray(ids_test, dtype=np.int64)[dense]
        order = np.argsort(ids_train, kind="stable")
        sorted_ids = np.asarray(ids_train, dtype=np.int64)[order]
        pos = np.searchsorted(sorted_ids, orig)
        pos_c = np.minimum(pos, max(len(sorted_ids) - 1, 0))
        hit = (len(sorted_ids) > 0) & (sorted_ids[pos_c] == orig) if len(sorted_ids) else \
            np.zeros(len(orig), dtype=bool)
        return np.where(hit, order[pos_c], -1)

    users = lookup(testset.users, testset.user_ids, train.user_ids)
    items = lookup(testset.items, testset.item_ids, train.item_ids)
    ok = (users >= 0) & (items >= 0)
    return (users[ok].astype(np.int32), items[ok].astype(np.int32), testset.ratings[ok],
            int((~ok).sum()))


def load_ratings(path) -> RatingMatrix:
    """Text "user item rating" file, keep-last dedup, dense remap (data.py:76-132)."""
    try:
        raw = np.loadtxt(path, comments="#", ndmin=2)
    except (OSError, ValueError) as exc:
        raise DataError(f"cannot read {path}: {exc}") from exc
    if raw.size == 0:
        raw = np.zeros((0, 3))
    if raw.shape[1] != 3:
        raise DataError(f"{path}: expected 'user item rating' lines")
    u, v, r = raw[:, 0].astype(np.int64), raw[:, 1].astype(np.int64), raw[:, 2]
    if not np.all(np.isfinite(r)):
        raise DataError(f"{path}: non-finite rating")
    if len(u):
        _, last = np.unique(np.stack([u, v], 1)[::-1], axis=0, return_index=True)
        keep = np.sort(len(u) - 1 - last)
        u, v, r = u[keep], v[keep], r[keep]
    user_ids, users = np.unique(u, return_inverse=True)
    item_ids, items = np.unique(v, return_inverse=True)
    return RatingMatrix(len(user_ids), len(item_ids), users.astype(np.int32),
                        items.astype(np.int32), r, user_ids, item_ids)


# ---------------------------------------------------------------------------
# Host block grid (the reference contract)
# ---------------------------------------------------------------------------
@dataclass
class BlockGrid:
    """Block-major triples + CSR block_ptr (data.py:169-224)."""

    n_rows: int
    n_cols: int
    row_cuts: np.ndarray
    col_cuts: np.ndarray
    region_of_row: np.ndarray
    sub_row_parent: np.ndarray | None
    users: np.ndarray
    items: np.ndarray
    ratings: np.ndarray
    block_ptr: np.ndarray

    @property
    def n_row_bands(self) -> int:
        return len(self.row_cuts) - 1

    @property
    def n_col_bands(self) -> int:
        return len(self.col_cuts) - 1

    @property
    def n_blocks(self) -> int:
        return self.n_row_bands * self.n_col_bands

    @property
    def nnz(self) -> int:
        return len(self.ratings)

    def block_id(self, row_band: int, col_band: int) -> int:
        return row_band * self.n_col_bands + col_band

    def block_range(self, block: int):
        return int(self.block_ptr[block]), int(self.block_ptr[block + 1])

    def block_nnz(self, block: int) -> int:
        lo, hi = self.block_range(block)
        return hi - lo

    def block_counts(self) -> np.ndarray:
        return np.diff(self.block_ptr)

    def row_span(self, row_band: int):
        return int(self.row_cuts[row_band]), int(self.row_cuts[row_band + 1])

    def col_span(self, col_band: int):
        return int(self.col_cuts[col_band]), int(self.col_cuts[col_band + 1])


def check_cuts(cuts, extent, axis) -> np.ndarray:
    cuts = np.asarray(cuts, dtype=np.int64)
    if len(cuts) < 2:
        raise GridError(f"{axis} cuts need at least two boundaries")
    if cuts[0] != 0 or cuts[-1] != extent:
        raise GridError(f"{axis} cuts must start at 0 and end at {extent}")
    if np.any(np.diff(cuts) <= 0):
        raise GridError(f"{axis} cuts must be strictly ascending")
    return cuts


def _grid_tags(n_row_bands, region_of_row, sub_row_parent):
    if region_of_row is None:
        region = np.full(n_row_bands, REGION_STREAM, dtype=np.int8)
    else:
        region = np.asarray(region_of_row, dtype=np.int8)
        if len(region) != n_row_bands:
            raise GridError("region_of_row length must match row band count")
    if sub_row_parent is not None:
        sub_row_parent = np.asarray(sub_row_parent, dtype=np.int64)
        if len(sub_row_parent) != n_row_bands:
            raise GridError("sub_row_parent length must match row band count")
    return region, sub_row_parent


def build_grid(matrix: RatingMatrix, row_cuts, col_cuts, region_of_row=None,
               sub_row_parent=None) -> BlockGrid:
    """Host bucketing with the reference semantics (data.py:238-280)."""
    row_cuts = check_cuts(row_cuts, matrix.n_users, "row")
    col_cuts = check_cuts(col_cuts, matrix.n_items, "column")
    nrb, ncb = len(row_cuts) - 1, len(col_cuts) - 1
    region, sub_row_parent = _grid_tags(nrb, region_of_row, sub_row_parent)
    bid = ((np.searchsorted(row_cuts, matrix.users, side="right") - 1) * ncb
           + np.searchsorted(col_cuts, matrix.items, side="right") - 1)
    order = np.argsort(bid, kind="stable")
    ptr = np.zeros(nrb * ncb + 1, dtype=np.int64)
    np.cumsum(np.bincount(bid, minlength=nrb * ncb), out=ptr[1:])
    return BlockGrid(matrix.n_users, matrix.n_items, row_cuts, col_cuts, region, sub_row_parent,
                     np.ascontiguousarray(matrix.users[order]),
                     np.ascontiguousarray(matrix.items[order]),
                     np.ascontiguousarray(matrix.ratings[order]), ptr)


def save_cache(path, matrix: RatingMatrix) -> None:
    """HMF1 binary cache (data.py:283-294)."""
    with open(path, "wb") as fh:
        fh.write(CACHE_MAGIC)
        fh.write(struct.pack("<QQQ", matrix.n_users, matrix.n_items, matrix.nnz))
        fh.write(np.asarray(matrix.users).astype("<u8").tobytes())
        fh.write(np.asarray(matrix.items).astype("<u8").tobytes())
        fh.write(np.asarray(matrix.ratings).astype("<f8").tobytes())


def load_cache(path) -> RatingMatrix:
    """HMF1 reader (data.py:297-308)."""
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != CACHE_MAGIC:
            raise DataError(f"{path}: not a rating cache (bad magic {magic!r})")
        n_users, n_items, nnz = struct.unpack("<QQQ", fh.read(24))
        users = np.frombuffer(fh.read(8 * nnz), dtype="<u8").astype(np.int32)
        items = np.frombuffer(fh.read(8 * nnz), dtype="<u8").astype(np.int32)
        ratings = np.frombuffer(fh.read(8 * nnz), dtype="<f8").astype(np.float64)
    m = RatingMatrix(int(n_users), int(n_items), users, items, ratings)
    m.validate()
    return m


def synthetic_ratings(n_users=500, n_items=500, rank=8, density=0.05, noise=0.1, seed=0,
                      factor_scale=1.0) -> RatingMatrix:
    """Low-rank synthetic instance, the reference law and RNG stream (data.py:311-336).

    Cells: unique uniform draws topped up until `target` distinct cells exist,
    then a random `target`-subset in random order; values: sum over `rank` of
    U[0, factor_scale/sqrt(rank)] factors plus N(0, noise).  Uses the same
    numpy Generator calls in the same order as the reference, so the output is
    bit-identical for the same arguments (pinned by tests/golden/data.npz).
    Host-only; use synthetic_device() for Netflix-scale shapes.
    """
    gen = np.random.default_rng(seed)
    cells_total = n_users * n_items
    target = min(int(round(density * cells_total)), cells_total)
    picked = np.empty(0, dtype=np.int64)
    while picked.size < target:
        extra = gen.integers(0, cells_total, size=int((target - picked.size) * 1.3) + 16)
        picked = np.unique(np.concatenate([picked, extra]))
    picked = gen.permutation(picked)[:target]
    users = (picked // n_items).astype(np.int32)
    items = (picked % n_items).astype(np.int32)
    top = factor_scale / np.sqrt(rank)
    a = gen.uniform(0.0, top, size=(n_users, rank))
    b = gen.uniform(0.0, top, size=(n_items, rank))
    values = np.einsum("ij,ij->i", a[users], b[items])
    if noise > 0:
        values = values + gen.normal(0.0, noise, size=target)
    return RatingMatrix(n_users, n_items, users, items, values)


# ---------------------------------------------------------------------------
# Device-resident triples and grids
# ---------------------------------------------------------------------------
def _torch():
    import torch
    return torch


def _stream(dev) -> int:
    return int(_torch().cuda.current_stream(dev).cuda_stream)


@dataclass
class DeviceTriples:
    """SoA triples in HBM: int32 users, int32 items, f32/f64 ratings."""

    n_users: int
    n_items: int
    users: object
    items: object
    ratings: object

    @property
    def nnz(self) -> int:
        return int(self.ratings.numel())

    @property
    def device(self):
        return self.ratings.device

    @classmethod
    def from_host(cls, m: RatingMatrix, device, rating_dtype="float32") -> "DeviceTriples":
        torch = _torch()
        rdt = getattr(torch, rating_dtype)
        return cls(m.n_users, m.n_items,
                   torch.from_numpy(np.ascontiguousarray(m.users, dtype=np.int32)).to(device),
                   torch.from_numpy(np.ascontiguousarray(m.items, dtype=np.int32)).to(device),
                   torch.from_numpy(np.ascontiguousarray(m.ratings)).to(device=device, dtype=rdt))

    def to_host(self) -> RatingMatrix:
        return RatingMatrix(self.n_users, self.n_items, self.users.cpu().numpy(),
                            self.items.cpu().numpy(),
                            self.ratings.cpu().numpy().astype(np.float64))

    def take(self, index) -> "DeviceTriples":
        return DeviceTriples(self.n_users, self.n_items, self.users[index].contiguous(),
                             self.items[index].contiguous(), self.ratings[index].contiguous())


@dataclass
class DeviceGrid:
    """A BlockGrid whose triples live in HBM (block-major, 16-byte aligned).

    block_ptr and the cuts stay on the host (the scheduler reads them); the
    triple arrays are single contiguous device allocations, so a block is a
    [block_ptr[b], block_ptr[b+1]) range of one launch.
    """

    n_rows: int
    n_cols: int
    row_cuts: np.ndarray
    col_cuts: np.ndarray
    region_of_row: np.ndarray
    sub_row_parent: np.ndarray | None
    users: object
    items: object
    ratings: object
    block_ptr: np.ndarray

    # Q-band sub-bucketing (optional): per block, device int64 sub_ptr[S+1]
    # (absolute triple offsets) and int32 sub_cuts[S+1] (absolute item ids);
    # see hmf_sgd_block_qband_* and bucket_qbands().
    sub_ptr: list | None = None
    sub_cuts: list | None = None
    # row tiles per block (L2 residency of P): sub_ptr[b] then holds
    # sub_tiles[b] * S + 1 offsets, tile-major
    sub_tiles: list | None = None
    sub_impl: int = -1          # Q-band implementation the layout is for
    sub_cfg: int = -1           # chain configuration it is for (-1: by k and storage)
    sub_tile_rows: list | None = None   # per block: row cuts of its tiles (host int64)
    sub_split: int = 1                  # parts per item run (implementation 5)
    sub_qsync: int = 0                  # Q publication period for implementation 5
    sub_pstore: int = 0                 # chained kernel P write-back: 1 stores, 0 reductions
    sub_tile_cuts: list | None = None   # implementation 8: per block, device int32 tile cuts
    sub_max_rows: int = 0               # implementation 8: rows of the largest tile
    sub_tile_run: list | None = None    # implementation 8: per block, first run of each tile
    sub_wide: int = 0                   # implementation 8 at k = 32: the wide configuration

    n_row_bands = BlockGrid.n_row_bands
    n_col_bands = BlockGrid.n_col_bands
    n_blocks = BlockGrid.n_blocks
    block_id = BlockGrid.block_id
    block_range = BlockGrid.block_range
    block_nnz = BlockGrid.block_nnz
    block_counts = BlockGrid.block_counts
    row_span = BlockGrid.row_span
    col_span = BlockGrid.col_span

    @property
    def nnz(self) -> int:
        return int(self.ratings.numel())

    @property
    def device(self):
        return self.ratings.device

    @classmethod
    def from_host(cls, grid: BlockGrid, device, rating_dtype="float32") -> "DeviceGrid":
        torch = _torch()
        rdt = getattr(torch, rating_dtype)
        return cls(grid.n_rows, grid.n_cols, grid.row_cuts, grid.col_cuts, grid.region_of_row,
                   grid.sub_row_parent,
                   torch.from_numpy(np.ascontiguousarray(grid.users, dtype=np.int32)).to(device),
                   torch.from_numpy(np.ascontiguousarray(grid.items, dtype=np.int32)).to(device),
                   torch.from_numpy(np.ascontiguousarray(grid.ratings)).to(device=device, dtype=rdt),
                   np.asarray(grid.block_ptr, dtype=np.int64))

    def to_host(self) -> BlockGrid:
        return BlockGrid(self.n_rows, self.n_cols, self.row_cuts, self.col_cuts,
                         self.region_of_row, self.sub_row_parent, self.users.cpu().numpy(),
                         self.items.cpu().numpy(), self.ratings.cpu().numpy().astype(np.float64),
                         self.block_ptr.copy())


def build_device_grid(triples: DeviceTriples, row_cuts, col_cuts, region_of_row=None,
                      sub_row_parent=None) -> DeviceGrid:
    """Bucket device triples block-major on the GPU (stable; data.py:238-280)."""
    torch = _torch()
    row_cuts = check_cuts(row_cuts, triples.n_users, "row")
    col_cuts = check_cuts(col_cuts, triples.n_items, "column")
    nrb, ncb = len(row_cuts) - 1, len(col_cuts) - 1
    region, sub_row_parent = _grid_tags(nrb, region_of_row, sub_row_parent)
    dev = triples.device
    if triples.ratings.dtype != torch.float32:
        raise TypeError("device bucketing takes f32 ratings")
    n = triples.nnz
    out_u = torch.empty(n, dtype=torch.int32, device=dev)
    out_i = torch.empty(n, dtype=torch.int32, device=dev)
    out_r = torch.empty(n, dtype=torch.float32, device=dev)
    d_rc = torch.from_numpy(row_cuts).to(dev)
    d_cc = torch.from_numpy(col_cuts).to(dev)
    d_ptr = torch.empty(nrb * ncb + 1, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().hmf_bucket_triples(
        triples.users.data_ptr(), triples.items.data_ptr(), triples.ratings.data_ptr(), n,
        d_rc.data_ptr(), nrb, d_cc.data_ptr(), ncb, out_u.data_ptr(), out_i.data_ptr(),
        out_r.data_ptr(), d_ptr.data_ptr(), _stream(dev)), "hmf_bucket_triples")
    ptr = d_ptr.cpu().numpy()
    return DeviceGrid(triples.n_users, triples.n_items, row_cuts, col_cuts, region,
                      sub_row_parent, out_u, out_i, out_r, ptr)


def resident_warps(device, k: int = 128, f16: bool = False, impl: int = -1,
                   chain_cfg: int = -1) -> int:
    """Sub-band slots the Q-band kernel keeps resident on `device` (warps for
    implementation 0, lane-group chains for 4-6): SMs x slots per SM of that
    launch shape (hmf_qband_slots_per_sm, per-device occupancy)."""
    torch = _torch()
    opts = _lib.QbandOpts(impl=int(impl), chain_cfg=int(chain_cfg))
    with torch.cuda.device(device):
        per_sm = int(_lib.load().hmf_qband_slots_per_sm(int(k), 1 if f16 else 0,
                                                         ctypes.byref(opts)))
    return int(torch.cuda.get_device_properties(device).multi_processor_count) * max(per_sm, 1)


def qband_impl_for(device, k: int, f16: bool, n_items: int) -> int:
    """The Q-band implementation a grid is laid out and launched for when the
    caller names none: the library's default (hmf_qband_resolve_impl), the
    chained kernel with Q deltas (5), whose layout splits item runs only when
    a block has fewer items than chains (bucket_qbands)."""
    return int(_lib.load().hmf_qband_resolve_impl(int(k), 1 if f16 else 0))


# mean ratings per (row tile, item) pair from which a tile-resident-P layout
# (implementations 7, 8) beats the L2 row-tile kernels (5, 6): one B200,
# profiles/round2/s3_layout_by_workload.jsonl — Netflix (4.8 at k = 128, 19
# at k = 32) wins 1.3-1.8x; Hugewiki (0.65) and Yahoo-R1 (0.16) lose 10-35 %
TILE_RESIDENT_MIN_RUN = 2.0
# Staleness bound of implementation 8.  A run adds its Q change at its end,
# so an item's runs training at the same time in different tiles all start
# from the same Q row: on average chains_in_flight / items runs of L ratings,
# S = chains_per_sm x CTAs x L / items ratings trained against one stale row.
# Measured on narrow 2 %-density blocks (scripts/stale_margin.py, profiles/
# round2/s4_stale_margin.jsonl): lr x S <= 2.5 trains within 0.0005 of whole
# runs, lr x S ~ 5 loses 0.008-0.023 and 10 diverges.  Capped at 250: twice
# the paper's learning rate (0.005) stays inside the measured-good range.
# Netflix: S = 10.5 at N = 1, 89 per band at N = 8 (17 column bands).
TILE_RESIDENT_MAX_STALE = 250.0


def run_group_staleness(chains_per_sm: int, n_sm: int, ratings: int, tiles: int,
                        items: int) -> float:
    """S of TILE_RESIDENT_MAX_STALE for one block: the ratings of an item
    training at once against one stale Q row — chains in flight (chains per
    SM x the CTAs, one per SM up to the tiles) spread over the block's items,
    times the mean run length (ratings per tile and item)."""
    items = max(1, int(items))
    tiles = max(1, int(tiles))
    run_len = ratings / (tiles * items)
    return chains_per_sm * min(tiles, n_sm) * run_len / items


def runs_chains_per_sm(k: int, f16: bool, wide: bool = False) -> int:
    """Run-group chains resident per SM (implementation 8's configuration
    for k and the element size, hmf_qband_slots_per_sm; `wide`: the k = 32
    wide one)."""
    opts = _lib.QbandOpts(impl=8, runs_wide=1 if wide else 0)
    return int(_lib.check(_lib.load().hmf_qband_slots_per_sm(int(k), 1 if f16 else 0,
                                                              ctypes.byref(opts)),
                          "hmf_qband_slots_per_sm"))


def tile_resident_impl(grid, k: int, f16: bool, max_rows: int | None = None) -> int | None:
    """Implementation 8 (run groups over a shared-memory P tile) when every
    non-empty block of `grid` suits it, else None (the L2 row-tile kernels):
    * k in {32, 64, 128, 256};
    * at least one tile per SM (a CTA trains one tile at a time: ML-1M's
      6 040 users make 4 tiles at k = 32 — 1.4 vs 16 G upd/s);
    * item runs long enough: on average >= TILE_RESIDENT_MIN_RUN ratings per
      (tile, item) — each run costs a Q-row load and a Q-delta reduction;
    * no hot items (an item's ratings > 4x the block mean): one run per tile
      would then be long and train concurrently in every tile from the same
      Q row; the item-split kernel (5) handles that case;
    * Q staleness S <= TILE_RESIDENT_MAX_STALE (few items for the runs in
      flight: narrow column blocks).
    Returns 8 (Netflix fp32 k = 32 / 64 / 128 / 256: 74.7 / 40.0 / 19.4 / 7.6
    G upd/s against 30.6 / 19.7 / 11.8 / 5.9 for implementation 5; fp16 83 /
    49 / 22.6 / 9.4 against 42 / 27 / 16.4 / 8.5; profiles/round2/
    s4_ksweep.jsonl)."""
    torch = _torch()
    if k not in (32, 64, 128, 256) or grid.nnz == 0:
        return None
    dev = grid.device
    n_sm = int(torch.cuda.get_device_properties(dev).multi_processor_count)
    chains = runs_chains_per_sm(k, f16)
    for b in range(grid.n_blocks):
        lo, hi = grid.block_range(b)
        if hi <= lo:
            continue
        if hi - lo >= (1 << 31):
            return None
        c_lo, c_hi = grid.col_span(b % grid.n_col_bands)
        r_lo, r_hi = grid.row_span(b // grid.n_col_bands)
        T = len(ptile_row_cuts(r_lo, r_hi, k, f16, n_sm, max_rows)) - 1
        W = max(1, c_hi - c_lo)
        run_len = (hi - lo) / (T * W)
        if T < n_sm or run_len < TILE_RESIDENT_MIN_RUN:
            return None
        if run_group_staleness(chains, n_sm, hi - lo, T, W) > TILE_RESIDENT_MAX_STALE:
            return None
        cnt = torch.bincount(grid.items[lo:hi] - c_lo, minlength=W)
        if float(cnt.max()) > 4 * (hi - lo) / W:
            return None
    return 8


def qband_sub_cuts(c_lo: int, c_hi: int, k: int, target: int, cap: int | None = None) -> np.ndarray:
    """Equal-width item sub-bands of [c_lo, c_hi): about `target` of them
    (one per resident warp or chain), never more than the items, and at most
    `cap` items wide (the kernel's Q-slice bound; default hmf_qband_max_items)."""
    items = c_hi - c_lo
    cap = int(_lib.load().hmf_qband_max_items(int(k), 0, -1)) if cap is None else int(cap)
    if cap <= 0:
        raise ValueError(f"Q-band kernel does not support k={k}")
    n_sub = min(items, max(target, -(-items // cap)))
    base, rem = divmod(items, n_sub)
    widths = np.full(n_sub, base, dtype=np.int64)
    widths[:rem] += 1
    return np.concatenate([[c_lo], c_lo + np.cumsum(widths)]).astype(np.int64)


# P rows per row tile of the Q-band kernel: one tile's P rows, the Q band and
# the triple stream share the 126 MB L2 (sweep: profiles/r02_tile_sweep*).
QBAND_TILE_BYTES = 32 << 20
# users per row tile at most: tile-relative user ids then fit 16 bits, so a
# streamed epoch (workers.StreamingEpoch) sends 6 bytes per rating at every k
# and precision (NF k = 32..64, fp16 k = 128: 8.9-9.0 G upd/s end to end vs
# 6.7-6.8 with 4-byte ids; resident throughput within -4.5..+1.5 %,
# profiles/r02/tile_rows_cap.jsonl)
QBAND_MAX_TILE_ROWS: int | None = 65536


def qband_row_tiles(n_rows: int, k: int, elem_bytes: int = 4,
                    tile_bytes: int | None = None, max_rows: int | None = None) -> int:
    """Row tiles for a block spanning n_rows users: the fewest equal tiles
    whose P rows (n_rows/T x k x elem_bytes) fit tile_bytes and, when
    max_rows is set (default QBAND_MAX_TILE_ROWS), hold at most max_rows
    rows.  tile_bytes <= 0 disables the byte bound."""
    tb = QBAND_TILE_BYTES if tile_bytes is None else int(tile_bytes)
    mr = QBAND_MAX_TILE_ROWS if max_rows is None else int(max_rows)
    if n_rows <= 0:
        return 1
    t = 1 if tb <= 0 else -(-(n_rows * k * elem_bytes) // tb)
    if mr and mr > 0:
        t = max(t, -(-n_rows // mr))
    return max(1, min(n_rows, t))


def qband_split_for(slots: int, items: int, block_nnz: float, n_tiles: int, k: int = 128,
                    f16: bool = False) -> int:
    """Parts per item run for implementation 5 (measured on one B200,
    profiles/r02/split_*.jsonl).

    The parts of one run go to different chains at the same time, each on
    its own copy of the item's Q row.  Without bounds, R concurrent parts
    pile up an item's steps before the deltas meet (test RMSE 0.42 vs 0.12 at
    k = 32); every chain therefore publishes its change and re-reads the row
    every few ratings (grid.sub_qsync: 512 // parts, or 128 // parts when hot
    items are split, clamped to 4..32; hmf_qband_set_qsync), which keeps every
    split within 0.0001 of whole runs at k = 32..128, fp32 and fp16.  Then:
    * at least twice as many items as chains: whole runs (Yahoo, Hugewiki);
    * fewer items than chains: slots // items parts, so every chain has a
      unit per tile (ML-1M: 5; an 8-GPU column band: 4-9); when that is 1
      and runs are short (< 192 ratings), 2 parts, scheduled dynamically
      (Hugewiki split over 2 GPUs, 8 000 items against 9 472 chains and
      40-rating runs: 9.05 vs 7.29 G upd/s);
    * k >= 64 and long runs (>= 192 ratings): 4 parts, scheduled
      dynamically (Netflix k = 128: 9.9 vs 9.1 fp32, 16.6 vs 15.9 fp16;
      k = 64: 17.3 vs 16.8; k = 256: 4.8 vs 4.5 G upd/s); at k = 32 whole runs
      were faster."""
    if items <= 0 or items >= 2 * slots:
        return 1
    avg_run = block_nnz / (max(1, n_tiles) * items)
    dyn = 4 if (k >= 64 and avg_run >= 192) else 1
    static = slots // items if items < slots else 1
    if items < slots and static == 1 and avg_run < 192:
        static = 2
    return max(1, min(16, max(static, dyn)))


def bucket_qbands(grid: DeviceGrid, k: int, target: int | None = None,
                  tile_bytes: int | None = None, elem_bytes: int = 4,
                  impl: int | None = None, split: int | None = None,
                  max_tile_rows: int | None = None, chain_cfg: int = -1) -> DeviceGrid:
    """Re-bucket every block of a device grid for the Q-band kernel, in place:
    row tile major, then item (both stable), and attach sub_ptr / sub_cuts /
    sub_tiles.  Row tiles are equal user ranges of the block's row band, sized
    by qband_row_tiles (tile_bytes <= 0 and no row cap: one tile).  Sorting by item inside a
    tile makes every (tile, sub-band) range contiguous and lays each item's
    ratings out as one run, so the kernel keeps the current item's Q row in
    registers.  The order of ratings within an item is the block order
    (stable), i.e. the reference's shuffled order (data.py:242-244, 264).
    The grid records the implementation it is laid out for (sub_impl;
    qband_impl_for unless `impl` is given) and launches use it.

    Implementation 5 (Q deltas) splits every (tile, item) run into `split`
    consecutive parts, each its own sub-band (default: enough parts for
    every chain to have one), so a block with few items still feeds every
    chain; sub-band s then holds part s % split of item sub_cuts[s]."""
    torch = _torch()
    dev = grid.device
    lib = _lib.load()
    s = _stream(dev)
    f16 = elem_bytes == 2
    # an implementation asked for keeps its layout rules; the automatic
    # choice (None or -1) also splits hot items' runs
    if impl is not None and int(impl) < 0:
        impl = None
    auto = impl is None
    chain_cfg = int(chain_cfg)
    split_given = split is not None
    if impl is None and tile_bytes is None:
        impl = tile_resident_impl(grid, k, f16, max_tile_rows)
    if impl is None:
        impl = qband_impl_for(dev, k, f16, max((grid.col_span(c)[1] - grid.col_span(c)[0]
                                                for c in range(grid.n_col_bands)), default=0))
    impl = int(impl)
    if impl == 7:
        raise ValueError("implementation 7 (item bins over a P tile) was removed: run groups (8) "
                         "beat it at every k")
    if impl == 8:
        return _bucket_runs(grid, k, f16, max_tile_rows)
    widest = max((grid.col_span(c)[1] - grid.col_span(c)[0]
                  for c in range(grid.n_col_bands)), default=0)
    if impl == 5 and split is None:
        sizes = np.diff(np.asarray(grid.block_ptr))
        full = [b for b in range(grid.n_blocks) if sizes[b] > 0]
        rows = max((grid.row_span(b // grid.n_col_bands)[1] - grid.row_span(b // grid.n_col_bands)[0]
                    for b in full), default=1)
        split = 1 if target is not None else qband_split_for(
            resident_warps(dev, k, f16, 5, chain_cfg), widest,
            float(np.mean(sizes[full])) if full else 0.0,
            qband_row_tiles(rows, k, elem_bytes, tile_bytes, max_tile_rows), k, f16)
    split = 1 if impl != 5 or not split else int(split)
    if split > 1:
        target = widest          # one item per sub-band, then its parts
    elif target is None:
        # one sub-band per resident slot; for the chained kernel with at least
        # twice as many items as chains, narrower sub-bands (up to 4 per
        # chain) that its dynamic scheduler balances (qchain.cuh)
        target = resident_warps(dev, k, f16, impl, chain_cfg)
        if impl >= 4 and widest >= 2 * target:
            target = min(widest, 4 * target)
    target = int(target)
    cap = int(lib.hmf_qband_max_items(int(k), 1 if f16 else 0, impl))
    out_u = torch.empty_like(grid.users)
    out_i = torch.empty_like(grid.items)
    out_r = torch.empty_like(grid.ratings)
    sub_ptrs, sub_cuts, sub_tiles, tile_rows = [], [], [], []
    max_parts = 1
    any_skewed = False
    for b in range(grid.n_blocks):
        lo, hi = grid.block_range(b)
        c_lo, c_hi = grid.col_span(b % grid.n_col_bands)
        r_lo, r_hi = grid.row_span(b // grid.n_col_bands)
        n_tiles = qband_row_tiles(r_hi - r_lo, k, elem_bytes, tile_bytes, max_tile_rows)
        tiles = np.linspace(r_lo, r_hi, n_tiles + 1).round().astype(np.int64)
        cuts = qband_sub_cuts(c_lo, c_hi, k, target, cap)
        parts = None             # parts per item (single-item sub-bands), device int64
        if hi > lo and not split_given and (impl == 5 or (auto and impl >= 4)) and c_hi > c_lo:
            cnt = torch.bincount(grid.items[lo:hi] - c_lo, minlength=c_hi - c_lo)
            mean = (hi - lo) / (c_hi - c_lo)
            skewed = float(cnt.max()) > 4 * mean
            any_skewed = any_skewed or skewed
            if split > 1 or skewed:
                # parts in proportion to the item's ratings: a hot item gets
                # several chains (Q deltas), cold ones keep one
                # (at most 16 parts; with sub_qsync below, parts x period
                # stays at ~128 stale item steps for skewed layouts)
                parts = torch.clamp(torch.round(cnt.double() * (max(split, 1) / mean)),
                                    1, 16).to(torch.int64)
        elif split > 1:
            parts = torch.full((c_hi - c_lo,), split, dtype=torch.int64, device=dev)
        if parts is not None:
            cuts = np.arange(c_lo, c_hi + 1, dtype=np.int64)   # single items, then parts
            part_base = torch.cumsum(parts, 0) - parts              # first sub-band of item i
            n_sub = int(parts.sum())
            item_of = torch.repeat_interleave(torch.arange(c_hi - c_lo, device=dev), parts)
            part_no = torch.arange(n_sub, device=dev) - part_base[item_of]
            split_used = int(parts.max())
        else:
            n_sub = len(cuts) - 1
        rel = torch.from_numpy(cuts[:-1] - c_lo).to(dev)
        ptr = torch.full((n_tiles * n_sub + 1,), hi, dtype=torch.int64, device=dev)
        if hi > lo:
            # 1. row-tile major (stable), grid arrays -> out_*
            if n_tiles == 1:
                out_u[lo:hi], out_i[lo:hi], out_r[lo:hi] = (grid.users[lo:hi],
                                                            grid.items[lo:hi],
                                                            grid.ratings[lo:hi])
                tp = np.array([lo, hi], dtype=np.int64)
            else:
                d_tiles = torch.from_numpy(tiles).to(dev)
                tptr = torch.zeros(n_tiles + 1, dtype=torch.int64, device=dev)
                if n_tiles <= 12288:
                    d_cc = torch.tensor([c_lo, c_hi], dtype=torch.int64, device=dev)
                    _lib.check(lib.hmf_bucket_triples(
                        grid.users.data_ptr() + 4 * lo, grid.items.data_ptr() + 4 * lo,
                        grid.ratings.data_ptr() + 4 * lo, hi - lo, d_tiles.data_ptr(), n_tiles,
                        d_cc.data_ptr(), 1, out_u.data_ptr() + 4 * lo,
                        out_i.data_ptr() + 4 * lo, out_r.data_ptr() + 4 * lo, tptr.data_ptr(),
                        s), "hmf_bucket_triples")
                else:
                    key = torch.bucketize(grid.users[lo:hi], d_tiles[1:-1].to(torch.int32),
                                          right=True)
                    order = torch.sort(key, stable=True).indices
                    out_u[lo:hi] = grid.users[lo:hi][order]
                    out_i[lo:hi] = grid.items[lo:hi][order]
                    out_r[lo:hi] = grid.ratings[lo:hi][order]
                    tptr[1:] = torch.cumsum(torch.bincount(key, minlength=n_tiles), 0)
                    del key, order
                tp = tptr.cpu().numpy() + lo
            # 2. by item inside each tile (stable), out_* -> grid arrays
            n_items = c_hi - c_lo
            for t in range(n_tiles):
                a, z = int(tp[t]), int(tp[t + 1])
                if z <= a:
                    ptr[t * n_sub:(t + 1) * n_sub] = a
                    continue
                key = out_i[a:z] - c_lo
                order = torch.sort(key, stable=True).indices
                grid.users[a:z] = out_u[a:z][order]
                grid.items[a:z] = out_i[a:z][order]
                grid.ratings[a:z] = out_r[a:z][order]
                iptr = torch.zeros(n_items + 1, dtype=torch.int64, device=dev)
                iptr[1:] = torch.cumsum(torch.bincount(key, minlength=n_items), 0)
                if parts is not None:
                    # part r of item i starts at iptr[i] + len_i * r // parts_i
                    ln = (iptr[1:] - iptr[:-1])[item_of]
                    ptr[t * n_sub:(t + 1) * n_sub] = (iptr[:-1][item_of]
                                                      + ln * part_no // parts[item_of] + a)
                else:
                    ptr[t * n_sub:(t + 1) * n_sub] = iptr[rel] + a
                del key, order, iptr
        sub_ptrs.append(ptr)
        if parts is not None:
            cuts = np.concatenate([np.repeat(cuts[:-1], parts.cpu().numpy()), cuts[-1:]])
            max_parts = max(max_parts, split_used)
        sub_cuts.append(torch.from_numpy(cuts).to(device=dev, dtype=torch.int32))
        sub_tiles.append(n_tiles)
        tile_rows.append(tiles)
    del out_u, out_i, out_r
    grid.sub_ptr, grid.sub_cuts, grid.sub_tiles = sub_ptrs, sub_cuts, sub_tiles
    if max_parts > 1 and auto and impl in (4, 6):
        impl = 5                 # a hot item's runs are split: Q deltas
    split = max(split, max_parts)
    if impl == 5 and split == 1:
        # whole item runs.  No more sub-bands than chains (static owners): Q
        # rows are never shared, plain stores (implementation 4).  More: the
        # dynamic scheduler runs units of one sub-band in consecutive tiles
        # side by side on Q deltas without hand-off waits, published at item
        # changes only (implementation 6; Yahoo 9.7 vs 9.1 G upd/s with the
        # 16-rating publication, RMSE equal)
        slots = resident_warps(dev, k, f16, 4, chain_cfg)
        impl = 4 if all(len(c) - 1 <= slots for c in sub_cuts) else 6
    grid.sub_impl = impl
    grid.sub_cfg = chain_cfg
    grid.sub_split = split
    # Q publication period for split runs, bounding an item's steps in
    # flight across its parts (parts x period): ~128 when hot items are split
    # (16 parts publishing every 16 ratings diverged on skewed items, every 8
    # trained like whole runs, profiles/r02/skew_item_popularity.jsonl), ~512
    # for uniform popularity (15 parts x 32 matched whole runs,
    # profiles/r02/split_quality_bounded_staleness.jsonl)
    bound = 128 if any_skewed else 512
    grid.sub_qsync = max(4, min(32, bound // max(split, 1))) if impl == 5 else 0
    grid.sub_tile_rows = tile_rows
    # P rows written back by plain stores (the reference's racing lanes)
    # instead of reductions where that is measured faster (fp32, k >= 128:
    # +19 %) and where a tile holds at least 4x as many users as there are
    # chains, so concurrent updates of one user stay rare (Netflix-shaped
    # k = 128: test RMSE within 0.0015 of reductions at every epoch, equal
    # after 10, profiles/r02/pstore.jsonl; a 3 000-user tile lost ~10 % of
    # its P change)
    min_rows = min((int(np.min(np.diff(r))) for r in tile_rows if len(r) > 1), default=0)
    grid.sub_pstore = int(impl >= 4 and not f16 and k >= 128
                          and min_rows >= 4 * resident_warps(dev, k, f16, impl, chain_cfg))
    return grid


PTILE_MIN_ROWS = 64


def ptile_row_cuts(r_lo: int, r_hi: int, k: int, f16: bool, n_sm: int,
                   max_rows: int | None = None, stagger: bool = False) -> np.ndarray:
    """Row tiles of implementation 8 (tile-resident P): the fewest
    equal tiles whose P rows fit one CTA's shared memory (hmf_ptile_max_rows),
    at least one per SM when that leaves PTILE_MIN_ROWS rows per tile (a CTA
    trains one tile at a time) — rounded up to a multiple of the SM count,
    so the persistent CTAs finish their last tiles together.  With
    `stagger` (or PTILE_STAGGER) and at least two waves, the first and last
    tile of each CTA are uneven (_staggered_cuts)."""
    n = r_hi - r_lo
    cap = int(_lib.load().hmf_ptile_max_rows(int(k), 1 if f16 else 0))
    if max_rows:
        cap = min(cap, int(max_rows))
    t = max(1, -(-n // cap))
    if t < n_sm and n >= n_sm * PTILE_MIN_ROWS:
        t = n_sm
    if t > n_sm // 2:
        t = -(-t // n_sm) * n_sm
    t = max(1, min(n, t))
    if (stagger or PTILE_STAGGER) and t % n_sm == 0 and t // n_sm >= 2:
        return _staggered_cuts(r_lo, r_hi, t // n_sm, n_sm)
    return np.linspace(r_lo, r_hi, t + 1).round().astype(np.int64)


# Staggered tile switches: every CTA moves its P tile at the same moments
# when tiles are equal, and those switches are L2-throughput bound (~60 MB
# at once, ~5 us).  Staggered, the first and last tile of CTA i are f_i and
# 1 - f_i of a tile (f_i spread over [0, 1)), so the switches of different
# CTAs fall at different times.  Worth it only where a tile trains briefly:
# at the 8-GPU geometry (5 k ratings per tile) +2.9 %, at N = 1 (42 k) -4 to
# -9 % (the partial tiles' shorter runs; profiles/round2/s4_stagger.jsonl).
# _bucket_runs staggers resident layouts below PTILE_STAGGER_BELOW ratings
# per tile; PTILE_STAGGER forces it everywhere (experiments, tests).
PTILE_STAGGER = False
PTILE_STAGGER_BELOW = 10_000
PTILE_STAGGER_MIN_BLOCK = 1_000_000


def _staggered_cuts(r_lo: int, r_hi: int, waves: int, n_sm: int) -> np.ndarray:
    R = (r_hi - r_lo) / (waves * n_sm)
    f = ((np.arange(n_sm) * 53) % n_sm) / n_sm
    sizes = np.concatenate([f * R, np.full((waves - 1) * n_sm, R), (1 - f) * R])
    cuts = r_lo + np.concatenate([[0.0], np.cumsum(sizes)])
    cuts = cuts.round().astype(np.int64)
    cuts[-1] = r_hi
    return cuts


def _coprime_multiplier(w: int) -> int:
    """An odd multiplier near 0.618 w that is coprime with w (item
    scrambling inside a tile is then a bijection)."""
    import math
    m = max(1, int(w * 0.6180339887)) | 1
    while math.gcd(m, w) != 1:
        m += 2
    return m


def run_rotation(seed: int, r: int, length: int) -> int:
    """Where implementation 8 starts run r's visit (csrc/runs.cuh
    run_rotation): a 32-bit hash of (seed, r) scaled to [0, length)."""
    s32 = (int(seed) ^ (int(seed) >> 32)) & 0xFFFFFFFF
    h = ((r * 0x9E3779B1) & 0xFFFFFFFF) ^ s32
    h ^= h >> 15
    h = (h * 0x2C1B3C6D) & 0xFFFFFFFF
    h ^= h >> 12
    h = (h * 0x297A2D39) & 0xFFFFFFFF
    h ^= h >> 15
    return (h * length) >> 32


def _bucket_runs(grid: DeviceGrid, k: int, f16: bool, max_rows: int | None) -> DeviceGrid:
    """The layout of implementation 8 (csrc/runs.cuh): per block, row tiles
    whose P rows fit shared memory (ptile_row_cuts); inside a tile the runs — all
    ratings of one item, in the block's (shuffled) order, data.py:242-244,
    264 — sorted by length, longest first, then in a per-tile scrambled item
    order.  Two stable device sorts per block: by (tile, item) to measure the
    runs, then by (tile, -length, scrambled item).  Attaches per block:
    sub_ptr = the run descriptors (int32 [n_runs, 4]: first rating relative
    to the block's first, length, item, run index), sub_cuts = their items (a view),
    sub_tile_run (int32, first run of each tile), sub_tile_cuts (int32 row
    cuts of the tiles)."""
    torch = _torch()
    dev = grid.device
    n_sm = int(torch.cuda.get_device_properties(dev).multi_processor_count)
    run_descs, tile_runs, tile_rows, tile_cuts, n_tiles = [], [], [], [], []
    for b in range(grid.n_blocks):
        lo, hi = grid.block_range(b)
        c_lo, c_hi = grid.col_span(b % grid.n_col_bands)
        r_lo, r_hi = grid.row_span(b // grid.n_col_bands)
        tiles = ptile_row_cuts(r_lo, r_hi, k, f16, n_sm, max_rows)
        if (max_rows is None and hi - lo >= PTILE_STAGGER_MIN_BLOCK
                and hi - lo < PTILE_STAGGER_BELOW * (len(tiles) - 1)):
            tiles = ptile_row_cuts(r_lo, r_hi, k, f16, n_sm, max_rows, stagger=True)
        T = len(tiles) - 1
        W = max(1, c_hi - c_lo)
        if hi - lo >= (1 << 31):
            raise ValueError("implementation 8 takes blocks of < 2^31 ratings")
        if hi > lo:
            d_tiles = torch.from_numpy(tiles[1:-1]).to(dev, torch.int32)
            tile_of = torch.bucketize(grid.users[lo:hi], d_tiles, right=True).to(torch.int64)
            item_rel = (grid.items[lo:hi] - c_lo).to(torch.int64)
            key = tile_of * W + item_rel
            v1, i1 = torch.sort(key, stable=True)
            _, inv, counts = torch.unique_consecutive(v1, return_inverse=True,
                                                      return_counts=True)
            run_len = torch.empty_like(key)
            run_len[i1] = counts[inv]
            lmax = int(counts.max())
            del v1, i1, inv, counts
            # equal-length runs in a per-tile pseudo-random item order (a
            # bijection of [0, W)), so the CTAs working on different tiles do
            # not walk the same items at the same time (fewer concurrent Q
            # deltas on one item)
            mult = _coprime_multiplier(W)
            scram = (item_rel * mult + tile_of * 0x9E3779B1) % W
            key = tile_of * ((lmax + 1) * W) + (lmax - run_len) * W + scram
            del run_len, item_rel, tile_of, scram
            v2, order = torch.sort(key, stable=True)
            grid.users[lo:hi] = grid.users[lo:hi][order]
            grid.items[lo:hi] = grid.items[lo:hi][order]
            grid.ratings[lo:hi] = grid.ratings[lo:hi][order]
            del order
            uniq, counts = torch.unique_consecutive(v2, return_counts=True)
            del v2, key
            runs = torch.zeros((uniq.numel(), 4), dtype=torch.int32, device=dev)
            runs[1:, 0] = torch.cumsum(counts, 0)[:-1].to(torch.int32)
            runs[:, 1] = counts.to(torch.int32)
            runs[:, 2] = grid.items[lo:hi][runs[:, 0].to(torch.int64)]
            runs[:, 3] = torch.arange(uniq.numel(), dtype=torch.int32, device=dev)
            run_tile = uniq // ((lmax + 1) * W)
            trun = torch.searchsorted(run_tile, torch.arange(T + 1, device=dev))
            run_descs.append(runs)
            tile_runs.append(trun.to(torch.int32))
            del uniq, counts, run_tile
        else:
            run_descs.append(torch.zeros((0, 4), dtype=torch.int32, device=dev))
            tile_runs.append(torch.zeros(T + 1, dtype=torch.int32, device=dev))
        tile_rows.append(tiles)
        tile_cuts.append(torch.from_numpy(tiles).to(device=dev, dtype=torch.int32))
        n_tiles.append(T)
    # sub_ptr: the run descriptors; sub_cuts: their items (a view)
    grid.sub_ptr, grid.sub_tiles = run_descs, n_tiles
    grid.sub_cuts = [r[:, 2] for r in run_descs]
    grid.sub_tile_run = tile_runs
    grid.sub_impl, grid.sub_cfg, grid.sub_split, grid.sub_qsync, grid.sub_pstore = 8, -1, 1, 0, 0
    grid.sub_tile_rows = tile_rows
    grid.sub_tile_cuts = tile_cuts
    grid.sub_max_rows = max((int(np.max(np.diff(t))) for t in tile_rows if len(t) > 1),
                            default=1)
    # k = 32: the wide configuration (more chains per SM, faster) wherever
    # its staleness stays under the bound in every block
    grid.sub_wide = 0
    if k == 32:
        wide = runs_chains_per_sm(k, f16, wide=True)
        ok = True
        for b in range(grid.n_blocks):
            lo, hi = grid.block_range(b)
            if hi <= lo:
                continue
            c_lo, c_hi = grid.col_span(b % grid.n_col_bands)
            W, T = max(1, c_hi - c_lo), max(1, n_tiles[b])
            if run_group_staleness(wide, n_sm, hi - lo, T, W) > TILE_RESIDENT_MAX_STALE:
                ok = False
        grid.sub_wide = int(ok)
    return grid


def synthetic_device(n_users: int, n_items: int, nnz: int, rank: int = 8, noise: float = 0.1,
                     seed: int = 0, factor_scale: float = 1.0, device=None) -> DeviceTriples:
    """The synthetic_ratings law at any scale, generated in HBM.

    Exactly `nnz` distinct cells, uniform over the matrix, in random order;
    values sum_r A[u,r] B[v,r] + N(0, noise) with A, B ~ U[0, fs/sqrt(rank)].
    Cells are Bernoulli-selected with probability slightly above nnz/cells
    (hmf_synthetic_count/cells), randomly permuted, and the first nnz kept —
    the reference's permutation(chosen)[:target] — so the kept set is a
    uniform nnz-subset.  Values come from hmf_synthetic_fill.
    """
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    total = n_users * n_items
    if nnz > total:
        raise DataError("more ratings than cells")
    lib = _lib.load()
    s = _stream(dev)
    p = min(1.0, nnz / total * (1.0 + 6.0 / np.sqrt(max(nnz, 1))) + 16.0 / total)
    for attempt in range(8):
        gseed = (seed * 0x9E3779B1 + attempt * 0x85EBCA77 + 1) & 0xFFFFFFFFFFFFFFFF
        row_ptr = torch.empty(n_users + 1, dtype=torch.int64, device=dev)
        got = _lib.check(lib.hmf_synthetic_count(n_users, n_items, p, gseed, 0, row_ptr.data_ptr(),
                                                 s), "hmf_synthetic_count")
        if got >= nnz:
            break
        p = min(1.0, p * 1.01 + 1.0 / total)
    else:
        raise DataError("generator could not reach the requested count")
    users = torch.empty(got, dtype=torch.int32, device=dev)
    items = torch.empty(got, dtype=torch.int32, device=dev)
    _lib.check(lib.hmf_synthetic_cells(n_users, n_items, p, gseed, 0, row_ptr.data_ptr(),
                                       users.data_ptr(), items.data_ptr(), s), "hmf_synthetic_cells")
    del row_ptr
    # random order, first nnz kept (a keyed permutation: no sort, no index array)
    out_u = torch.empty(nnz, dtype=torch.int32, device=dev)
    out_i = torch.empty(nnz, dtype=torch.int32, device=dev)
    _lib.check(lib.hmf_permute_cells(users.data_ptr(), items.data_ptr(), got, out_u.data_ptr(),
                                     out_i.data_ptr(), nnz, (seed * 0x2545F491 + 7) & 0xFFFFFFFFFFFFFFFF,
                                     s), "hmf_permute_cells")
    users, items = out_u, out_i
    vals = torch.empty(nnz, dtype=torch.float32, device=dev)
    _lib.check(lib.hmf_synthetic_fill(users.data_ptr(), items.data_ptr(), nnz, rank, noise,
                                      factor_scale, (seed + 0x5EED) & 0xFFFFFFFFFFFFFFFF,
                                      vals.data_ptr(), s), "hmf_synthetic_fill")
    return DeviceTriples(n_users, n_items, users, items, vals)


def synthetic_band(n_users: int, n_items: int, nnz: float, row_lo: int = 0,
                   row_hi: int | None = None, rank: int = 8, noise: float = 0.1, seed: int = 0,
                   test_fraction: float = 0.05, factor_scale: float = 1.0, device=None):
    """Rows [row_lo, row_hi) of ONE synthetic matrix (the synthetic_ratings
    law, data.py:311-336), generated in HBM, split into (train, test).

    Every decision is keyed by the global cell, so the bands of any row
    partition are exactly the pieces of the whole matrix — N ranks each
    generating their own band train on the same matrix as one GPU, with the
    same held-out cells and the same ground truth (latent factors hashed from
    the global user and item ids, noise from the cell):
    * a cell is present with probability nnz / cells (geometric skipping per
      global row), so the matrix holds nnz ratings in expectation (not
      exactly: there is no global truncation step);
    * a cell is a test cell iff a hash of it falls below test_fraction
      (hmf_cell_mask);
    * each band's cells are then put in a keyed random order (the
      reference's shuffle_triples, data.py:99-102), train and test kept in it.
    User ids are global.  Returns (train, test) DeviceTriples with n_users
    the whole matrix's."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    row_hi = n_users if row_hi is None else int(row_hi)
    row_lo = int(row_lo)
    if not 0 <= row_lo <= row_hi <= n_users:
        raise DataError("bad row band")
    total = float(n_users) * float(n_items)
    if nnz > total:
        raise DataError("more ratings than cells")
    p = min(1.0, float(nnz) / total)
    lib = _lib.load()
    s = _stream(dev)
    gseed = (seed * 0x9E3779B1 + 1) & 0xFFFFFFFFFFFFFFFF
    n_rows = row_hi - row_lo
    row_ptr = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
    got = _lib.check(lib.hmf_synthetic_count(n_rows, n_items, p, gseed, row_lo,
                                             row_ptr.data_ptr(), s), "hmf_synthetic_count")
    users = torch.empty(got, dtype=torch.int32, device=dev)
    items = torch.empty(got, dtype=torch.int32, device=dev)
    _lib.check(lib.hmf_synthetic_cells(n_rows, n_items, p, gseed, row_lo, row_ptr.data_ptr(),
                                       users.data_ptr(), items.data_ptr(), s), "hmf_synthetic_cells")
    del row_ptr
    # keyed random order of the band's cells (a permutation of all of them)
    out_u = torch.empty_like(users)
    out_i = torch.empty_like(items)
    _lib.check(lib.hmf_permute_cells(users.data_ptr(), items.data_ptr(), got, out_u.data_ptr(),
                                     out_i.data_ptr(), got,
                                     (seed * 0x2545F491 + 7 + row_lo * 0x9E3779B97F4A7C15)
                                     & 0xFFFFFFFFFFFFFFFF, s), "hmf_permute_cells")
    users, items = out_u, out_i
    del out_u, out_i
    vals = torch.empty(got, dtype=torch.float32, device=dev)
    _lib.check(lib.hmf_synthetic_fill(users.data_ptr(), items.data_ptr(), got, rank, noise,
                                      factor_scale, (seed + 0x5EED) & 0xFFFFFFFFFFFFFFFF,
                                      vals.data_ptr(), s), "hmf_synthetic_fill")
    mask = torch.empty(got, dtype=torch.uint8, device=dev)
    _lib.check(lib.hmf_cell_mask(users.data_ptr(), items.data_ptr(), got, float(test_fraction),
                                 (seed * 0x632BE59BD9B4E019 + 0x7E57) & 0xFFFFFFFFFFFFFFFF,
                                 mask.data_ptr(), s), "hmf_cell_mask")
    # stable split, chunk by chunk (no nnz-long index array at Hugewiki scale)
    n_test = int(mask.sum(dtype=torch.int64))
    out = [(torch.empty(got - n_test, dtype=torch.int32, device=dev),
            torch.empty(got - n_test, dtype=torch.int32, device=dev),
            torch.empty(got - n_test, dtype=torch.float32, device=dev)),
           (torch.empty(n_test, dtype=torch.int32, device=dev),
            torch.empty(n_test, dtype=torch.int32, device=dev),
            torch.empty(n_test, dtype=torch.float32, device=dev))]
    at = [0, 0]
    chunk = 1 << 27
    for a in range(0, got, chunk):
        z = min(got, a + chunk)
        sel = mask[a:z].bool()
        for which, m in ((1, sel), (0, ~sel)):
            idx = torch.nonzero(m).squeeze(1)
            n = int(idx.numel())
            for dst, src in zip(out[which], (users, items, vals)):
                dst[at[which]:at[which] + n] = src[a:z][idx]
            at[which] += n
        del sel
    del mask, users, items, vals
    train = DeviceTriples(n_users, n_items, *out[0])
    test = DeviceTriples(n_users, n_items, *out[1])
    return train, test


def split_device(triples: DeviceTriples, test_fraction: float, seed: int = 1):
    """Seeded train/test split of device triples (the test set is a random
    `test_fraction` of them).  Triples from synthetic_device are already in
    random order, so the split takes a prefix as the test set."""
    n = triples.nnz
    # a multiple of 4 keeps the train view 16-byte aligned for the bulk copies
    n_test = int(round(n * test_fraction)) & ~3
    test = DeviceTriples(triples.n_users, triples.n_items, triples.users[:n_test],
                         triples.items[:n_test], triples.ratings[:n_test])
    train = DeviceTriples(triples.n_users, triples.n_items, triples.users[n_test:],
                          triples.items[n_test:], triples.ratings[n_test:])
    return train, test
