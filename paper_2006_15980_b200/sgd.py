"""SGD numerics on B200: factor models, the update, block epochs, loss, RMSE.

Drop-in for hetmf.sgd (hetmf/sgd.py).  The host FactorModel keeps the
reference's P/Q output layout — user_factors (n_users, k) and item_factors
(n_items, k), row-major f64 (sgd.py:41-65) — and the HMFP1 file format
(sgd.py:191-209).  DeviceModel holds the same layout in HBM in the storage
precision the engine computes in (f32, f16 or f64).

Every numeric entry point here runs on the GPU through libhmf:
  block_epoch        -> hmf_sgd_range_*        (sgd.py:118-131)
  sgd_update         -> hmf_sgd_range_* on one triple, EXACT mode (sgd.py:99-115)
  rmse, regularized_loss -> hmf_residual_sums_* (sgd.py:134-188), f64 sums
There is no numpy fallback for them.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from . import _lib, kernels
from .data import (BlockGrid, DeviceGrid, DeviceTriples, RatingMatrix, align_ratings)

FACTORS_MAGIC = b"HMFP1"


@dataclass
class Hyperparams:
    """sgd.py:22-38."""

    n_factors: int = 8
    reg_user: float = 0.05
    reg_item: float = 0.05
    learning_rate: float = 0.005
    epochs: int = 10

    def validate(self) -> None:
        if self.n_factors < 1:
            raise ValueError("n_factors must be >= 1")
        if self.reg_user < 0 or self.reg_item < 0:
            raise ValueError("regularization must be >= 0")
        if self.learning_rate <= 0:
            raise ValueError("learning_rate must be > 0")
        if self.epochs < 1:
            raise ValueError("epochs must be >= 1")


@dataclass
class FactorModel:
    """Host factors: user_factors (n_users, k), item_factors (n_items, k)."""

    user_factors: np.ndarray
    item_factors: np.ndarray

    @property
    def n_factors(self) -> int:
        return self.user_factors.shape[1]

    @property
    def n_users(self) -> int:
        return self.user_factors.shape[0]

    @property
    def n_items(self) -> int:
        return self.item_factors.shape[0]

    def copy(self) -> "FactorModel":
        return FactorModel(self.user_factors.copy(), self.item_factors.copy())

    def all_finite(self) -> bool:
        return bool(np.all(np.isfinite(self.user_factors))
                    and np.all(np.isfinite(self.item_factors)))


@dataclass
class UpdateTrace:
    residual: float
    delta_user_norm: float
    delta_item_norm: float


def _torch():
    import torch
    return torch


def _device(device=None):
    torch = _torch()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


@dataclass
class DeviceModel:
    """P (n_users x k) and Q (n_items x k), row-major, resident in HBM."""

    P: object
    Q: object

    @property
    def n_factors(self) -> int:
        return int(self.P.shape[1])

    @property
    def n_users(self) -> int:
        return int(self.P.shape[0])

    @property
    def n_items(self) -> int:
        return int(self.Q.shape[0])

    @property
    def dtype(self):
        return self.P.dtype

    @property
    def device(self):
        return self.P.device

    @classmethod
    def from_host(cls, model: FactorModel, device=None, dtype="float32") -> "DeviceModel":
        torch = _torch()
        dev = _device(device)
        dt = getattr(torch, dtype) if isinstance(dtype, str) else dtype
        return cls(torch.from_numpy(np.ascontiguousarray(model.user_factors)).to(dev, dt),
                   torch.from_numpy(np.ascontiguousarray(model.item_factors)).to(dev, dt))

    def to_host(self) -> FactorModel:
        torch = _torch()
        return FactorModel(self.P.to(torch.float64).cpu().numpy(),
                           self.Q.to(torch.float64).cpu().numpy())

    def copy(self) -> "DeviceModel":
        return DeviceModel(self.P.clone(), self.Q.clone())

    def all_finite(self) -> bool:
        torch = _torch()
        return bool(torch.isfinite(self.P).all().item() and torch.isfinite(self.Q).all().item())


def init_model(n_users: int, n_items: int, hparams: Hyperparams, seed: int) -> FactorModel:
    """U[0, 1/sqrt(k)] i.i.d., users then items, numpy default_rng(seed)
    (sgd.py:77-89) — the reference's exact stream, so both engines start from
    bit-identical factors."""
    k = hparams.n_factors
    if k < 1:
        raise ValueError("n_factors must be >= 1")
    gen = np.random.default_rng(seed)
    top = 1.0 / np.sqrt(k)
    return FactorModel(gen.uniform(0.0, top, size=(n_users, k)),
                       gen.uniform(0.0, top, size=(n_items, k)))


def init_device_model(n_users: int, n_items: int, k: int, seed: int, device=None,
                      dtype="float32") -> DeviceModel:
    """The init law drawn on the device (shapes where a host f64 draw is too
    large: Hugewiki P is 50 M x 128).  Same distribution, different stream."""
    torch = _torch()
    dev = _device(device)
    dt = getattr(torch, dtype) if isinstance(dtype, str) else dtype
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    top = 1.0 / float(np.sqrt(k))
    P = (torch.rand((n_users, k), generator=gen, device=dev, dtype=torch.float32) * top).to(dt)
    Q = (torch.rand((n_items, k), generator=gen, device=dev, dtype=torch.float32) * top).to(dt)
    return DeviceModel(P.contiguous(), Q.contiguous())


def predict_one(user_vec, item_vec) -> float:
    if len(user_vec) != len(item_vec):
        raise ValueError("factor vectors must have equal length")
    return float(np.dot(np.asarray(user_vec, dtype=np.float64),
                        np.asarray(item_vec, dtype=np.float64)))


def sgd_update(model: FactorModel, user: int, item: int, rating: float,
               hparams: Hyperparams) -> UpdateTrace:
    """One update of one rating, in place (sgd.py:99-115), run by the device
    kernel in EXACT mode (f64, both sides from pre-update vectors)."""
    pu0 = model.user_factors[user].copy()
    qv0 = model.item_factors[item].copy()
    # fresh arrays: the kernel updates them in place, pu0 / qv0 stay the
    # pre-update vectors the trace is computed from
    P = pu0[None, :].copy()
    Q = qv0[None, :].copy()
    kernels.sgd_range(P, Q, np.zeros(1, np.int32), np.zeros(1, np.int32),
                      np.array([rating], dtype=np.float64), 0, 1, hparams.learning_rate,
                      hparams.reg_user, hparams.reg_item, 0, 0, 0, mode="exact")
    model.user_factors[user] = P[0]
    model.item_factors[item] = Q[0]
    return UpdateTrace(residual=float(rating - np.dot(pu0, qv0)),
                       delta_user_norm=float(np.linalg.norm(P[0] - pu0)),
                       delta_item_norm=float(np.linalg.norm(Q[0] - qv0)))


def block_epoch(model, grid, block: int, hparams: Hyperparams, order_seed: int,
                mode: str = "hogwild") -> int:
    """Apply every triple of one block once (sgd.py:118-131).

    model/grid are a DeviceModel/DeviceGrid (device fast path) or a host
    FactorModel/BlockGrid (staged through the device, in place)."""
    lo, hi = grid.block_range(block)
    if isinstance(model, DeviceModel):
        return kernels.launch_sgd_range(model.P, model.Q, grid.users, grid.items, grid.ratings,
                                        lo, hi, hparams.learning_rate, hparams.reg_user,
                                        hparams.reg_item, order_seed, 0, 0, mode)
    return kernels.sgd_range(model.user_factors, model.item_factors, grid.users, grid.items,
                             grid.ratings, lo, hi, hparams.learning_rate, hparams.reg_user,
                             hparams.reg_item, order_seed, 0, 0, mode=mode)


# ---------------------------------------------------------------------------
# Residual sums on device
# ---------------------------------------------------------------------------
_RES = {"torch.float32": "f32", "torch.float16": "f16", "torch.float64": "f64"}


def residual_sums(model: DeviceModel, users, items, ratings, with_reg: bool = False,
                  row_base: int = 0, col_base: int = 0):
    """(sum err^2, sum |p_u|^2, sum |q_v|^2) over device triples, f64 (device
    tensor of 3 doubles; call .tolist() to read)."""
    torch = _torch()
    st = _RES[str(model.P.dtype)]
    want = torch.float64 if st == "f64" else torch.float32
    if ratings.dtype != want:
        ratings = ratings.to(want)
    out = torch.empty(3, dtype=torch.float64, device=model.P.device)
    fn = getattr(_lib.load(), f"hmf_residual_sums_{st}")
    _lib.check(fn(model.P.data_ptr(), model.Q.data_ptr(), model.n_factors, users.data_ptr(),
                  items.data_ptr(), ratings.data_ptr(), int(ratings.numel()), int(row_base),
                  int(col_base), 1 if with_reg else 0, out.data_ptr(),
                  kernels.current_stream_handle(model.P.device)), f"hmf_residual_sums_{st}")
    return out


def _as_device_model(model):
    if isinstance(model, DeviceModel):
        return model
    return DeviceModel.from_host(model, dtype="float64")


def _device_triples(matrix, dev, dtype):
    torch = _torch()
    if isinstance(matrix, (DeviceTriples, DeviceGrid)):
        return matrix.users, matrix.items, matrix.ratings
    return (torch.from_numpy(np.ascontiguousarray(matrix.users, dtype=np.int32)).to(dev),
            torch.from_numpy(np.ascontiguousarray(matrix.items, dtype=np.int32)).to(dev),
            torch.from_numpy(np.ascontiguousarray(matrix.ratings, dtype=np.float64)).to(dev, dtype))


def regularized_loss(matrix, model, reg_user: float, reg_item: float) -> float:
    """Eq. (2): sum over entries of err^2 + reg_user|p_u|^2 + reg_item|q_v|^2
    (sgd.py:134-154), evaluated on the device in f64."""
    torch = _torch()
    dm = _as_device_model(model)
    dt = torch.float64 if dm.P.dtype == torch.float64 else torch.float32
    u, i, r = _device_triples(matrix, dm.P.device, dt)
    if int(r.numel()) == 0:
        return 0.0
    sq, pp, qq = residual_sums(dm, u, i, r, with_reg=True).tolist()
    total = sq
    if reg_user:
        total += reg_user * pp
    if reg_item:
        total += reg_item * qq
    return float(total)


@dataclass
class RmseReport:
    value: float
    n_evaluated: int
    n_skipped: int


def rmse(testset, model, train: RatingMatrix | None = None) -> RmseReport:
    """Root mean square error over a rating set (sgd.py:157-188), on device.

    With `train`, the test set's original ids are resolved through the
    training remap tables and unseen ids are skipped and counted."""
    torch = _torch()
    dm = _as_device_model(model)
    dt = torch.float64 if dm.P.dtype == torch.float64 else torch.float32
    skipped = 0
    if train is not None and isinstance(testset, RatingMatrix):
        users, items, ratings, skipped = align_ratings(testset, train)
        testset = RatingMatrix(dm.n_users, dm.n_items, users, items, ratings)
    u, i, r = _device_triples(testset, dm.P.device, dt)
    n = int(r.numel())
    if n == 0:
        raise ValueError("no evaluable entries in test set")
    sq = residual_sums(dm, u, i, r)[0].item()
    return RmseReport(value=float(np.sqrt(sq / n)), n_evaluated=n, n_skipped=skipped)


def save_factors(path, model) -> None:
    """HMFP1: magic, <QQQ dims, P row-major f8, then Q^T (k x n_items) f8."""
    if isinstance(model, DeviceModel):
        model = model.to_host()
    with open(path, "wb") as fh:
        fh.write(FACTORS_MAGIC)
        fh.write(struct.pack("<QQQ", model.n_users, model.n_items, model.n_factors))
        fh.write(np.ascontiguousarray(model.user_factors, dtype="<f8").tobytes())
        fh.write(np.ascontiguousarray(model.item_factors.T, dtype="<f8").tobytes())


def load_factors(path) -> FactorModel:
    with open(path, "rb") as fh:
        magic = fh.read(5)
        if magic != FACTORS_MAGIC:
            raise ValueError(f"{path}: not a factors file (bad magic {magic!r})")
        n_users, n_items, k = struct.unpack("<QQQ", fh.read(24))
        P = np.frombuffer(fh.read(8 * n_users * k), dtype="<f8").reshape(n_users, k)
        Qt = np.frombuffer(fh.read(8 * k * n_items), dtype="<f8").reshape(k, n_items)
    return FactorModel(P.astype(np.float64), np.ascontiguousarray(Qt.T))
