"""ctypes binding of libhmf.so (the C ABI declared in include/hmf.h).

The library is loaded from the in-tree build (paper_2006_15980_b200/lib/).
There is no fallback: if the library is missing or fails to load, every
product entry point raises.  ctypes releases the GIL around foreign calls, so
worker threads driving different devices or streams run concurrently, as the
reference's numba kernel does with nogil=True (hetmf/kernels.py:61).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libhmf.so"

HMF_OK = 0
HMF_ERR_ARG = -1
HMF_ERR_CUDA = -2
HMF_ERR_UNSUPPORTED = -3
HMF_ERR_ABORTED = -4

MODE_HOGWILD = 0
MODE_ORDERED = 1
MODE_EXACT = 2
MODE_HOGWILD_LWW = 3
MODES = {"hogwild": MODE_HOGWILD, "ordered": MODE_ORDERED, "exact": MODE_EXACT,
         "hogwild_lww": MODE_HOGWILD_LWW}

TUNE_VARIANT = 1
ABI_VERSION = 5

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_u64 = C.c_uint64
_f64 = C.c_double

# name -> (restype, argtypes).  Mirrors include/hmf.h one to one; the
# not-gpu test suite checks every symbol the header declares is bound here.
SIGNATURES = {
    "hmf_abi_version": (C.c_int, []),
    "hmf_last_error": (C.c_char_p, []),
    "hmf_set_tuning": (C.c_int, [_i32, _i32]),
    "hmf_sgd_range_f32": (_i64, [_p, _p, _i64, _p, _p, _p, _i64, _i64, _f64, _f64, _f64, _u64,
                                 _i64, _i64, _i32, _p]),
    "hmf_sgd_range_f16": (_i64, [_p, _p, _i64, _p, _p, _p, _i64, _i64, _f64, _f64, _f64, _u64,
                                 _i64, _i64, _i32, _p]),
    "hmf_sgd_range_f64": (_i64, [_p, _p, _i64, _p, _p, _p, _i64, _i64, _f64, _f64, _f64, _u64,
                                 _i64, _i64, _i32, _p]),
    "hmf_qband_resolve_impl": (_i32, [_i64, _i32]),
    "hmf_qband_resolve_chain_cfg": (_i32, [_i64, _i32]),
    "hmf_qband_slots_per_sm": (_i32, [_i64, _i32, _p]),
    "hmf_qband_chain_lanes": (_i32, [_i64, _i32, _i32]),
    "hmf_qband_max_items": (_i32, [_i64, _i32, _i32]),
    "hmf_sgd_block_qband_f32": (_i64, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64, _p, _f64,
                                       _f64, _f64, _u64, _i64, _i64, _p]),
    "hmf_sgd_block_qband_f16": (_i64, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64, _p, _f64,
                                       _f64, _f64, _u64, _i64, _i64, _p]),
    "hmf_sgd_block_qband_u16_f32": (_i64, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64, _p,
                                           _f64, _f64, _f64, _u64, _i64, _i64, _p]),
    "hmf_sgd_block_qband_u16_f16": (_i64, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64, _p,
                                           _f64, _f64, _f64, _u64, _i64, _i64, _p]),
    "hmf_sgd_block_qband_u16_tiles_f32": (_i64, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64,
                                                 _p, _p, _f64, _f64, _f64, _u64, _i64, _p]),
    "hmf_sgd_block_qband_u16_tiles_f16": (_i64, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64,
                                                 _p, _p, _f64, _f64, _f64, _u64, _i64, _p]),
    "hmf_ptile_max_rows": (_i32, [_i64, _i32]),
    "hmf_runs_chains_per_warp": (_i32, [_i64, _i32]),
    "hmf_sgd_block_runs_f32": (_i64, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i32, _p, _f64,
                                      _f64, _f64, _u64, _i64, _i64, _p]),
    "hmf_sgd_block_runs_f16": (_i64, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i32, _p, _f64,
                                      _f64, _f64, _u64, _i64, _i64, _p]),
    "hmf_sgd_block_runs_u16_f32": (_i64, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i32, _p,
                                          _f64, _f64, _f64, _u64, _i64, _i64, _p]),
    "hmf_sgd_block_runs_u16_f16": (_i64, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i32, _p,
                                          _f64, _f64, _f64, _u64, _i64, _i64, _p]),
    "hmf_sgd_block_runs_u8_f32": (_i64, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i32, _p,
                                         _f64, _f64, _f64, _u64, _i64, _i64, _p]),
    "hmf_sgd_block_runs_u8_f16": (_i64, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i32, _p,
                                         _f64, _f64, _f64, _u64, _i64, _i64, _p]),
    "hmf_visit_order": (C.c_int, [_i64, _u64, _p, _p]),
    "hmf_mix64": (_u64, [C.POINTER(_u64), _i32]),
    "hmf_residual_sums_f32": (C.c_int, [_p, _p, _i64, _p, _p, _p, _i64, _i64, _i64, _i32, _p, _p]),
    "hmf_residual_sums_f16": (C.c_int, [_p, _p, _i64, _p, _p, _p, _i64, _i64, _i64, _i32, _p, _p]),
    "hmf_residual_sums_f64": (C.c_int, [_p, _p, _i64, _p, _p, _p, _i64, _i64, _i64, _i32, _p, _p]),
    "hmf_bucket_triples": (C.c_int, [_p, _p, _p, _i64, _p, _i32, _p, _i32, _p, _p, _p, _p, _p]),
    "hmf_synthetic_count": (_i64, [_i64, _i64, _f64, _u64, _i64, _p, _p]),
    "hmf_synthetic_cells": (C.c_int, [_i64, _i64, _f64, _u64, _i64, _p, _p, _p, _p]),
    "hmf_cell_mask": (C.c_int, [_p, _p, _i64, _f64, _u64, _p, _p]),
    "hmf_synthetic_fill": (C.c_int, [_p, _p, _i64, _i32, _f64, _f64, _u64, _p, _p]),
    "hmf_permute_cells": (C.c_int, [_p, _p, _i64, _p, _p, _i64, _u64, _p]),
    "hmf_device_count": (C.c_int, [C.POINTER(_i32)]),
    "hmf_set_device": (C.c_int, [_i32]),
    "hmf_enable_peer_access": (C.c_int, [_i32, _i32]),
    "hmf_memcpy_peer_async": (C.c_int, [_p, _i32, _p, _i32, _i64, _p]),
    "hmf_stream_synchronize": (C.c_int, [_p]),
    "hmf_ipc_get_handle": (C.c_int, [_p, C.POINTER(C.c_uint8), C.POINTER(_i64)]),
    "hmf_ipc_open_handle": (C.c_int, [C.POINTER(C.c_uint8), C.POINTER(_p)]),
    "hmf_ipc_close_handle": (C.c_int, [_p]),
    "hmf_lease_open": (C.c_int, [C.c_char_p, _i32, _i32, C.POINTER(_p)]),
    "hmf_lease_close": (C.c_int, [_p, _i32]),
    "hmf_lease_try_acquire": (_i32, [_p, _i32, _i32]),
    "hmf_lease_acquire_first": (C.c_int, [_p, C.POINTER(_i32), _i32, _i32, C.POINTER(_i32)]),
    "hmf_lease_release": (_i32, [_p, _i32, _i32]),
    "hmf_lease_owner": (C.c_int, [_p, _i32, C.POINTER(_i32)]),
    "hmf_lease_holder": (C.c_int, [_p, _i32, C.POINTER(_i32)]),
    "hmf_lease_ticket": (_i64, [_p]),
    "hmf_lease_ops": (_i64, [_p]),
    "hmf_lease_claim": (_i64, [_p, _i64]),
    "hmf_lease_abort": (C.c_int, [_p, _i32]),
    "hmf_lease_aborted": (_i32, [_p]),
}


class HmfError(RuntimeError):
    """A libhmf call failed (bad arguments or a CUDA error)."""


_lock = threading.Lock()
_lib = None


def load() -> C.CDLL:
    """Load libhmf.so, building it first only when explicitly allowed.

    Set HMF_AUTOBUILD=1 to compile on first use (developer convenience); the
    GPU box uses the prebuilt library that travels with the repository.
    """
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if os.environ.get("HMF_AUTOBUILD") == "1":
            from . import _build
            _build.build()
        if not LIB_PATH.exists():
            raise HmfError(f"{LIB_PATH} is missing: run `python -m paper_2006_15980_b200._build` "
                           "(or __graft_entry__.build()) first; there is no CPU fallback")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.hmf_abi_version() != ABI_VERSION:
            raise HmfError("libhmf ABI version mismatch")
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().hmf_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> int:
    """Raise HmfError for a negative return code; pass counts through."""
    if rc < 0:
        raise HmfError(f"{what} failed ({rc}): {last_error()}")
    return rc


def mix64_native(*parts: int) -> int:
    arr = (_u64 * len(parts))(*[int(p) & 0xFFFFFFFFFFFFFFFF for p in parts])
    return int(load().hmf_mix64(arr, len(parts)))


class QbandOpts(C.Structure):
    """hmf_qband_opts (include/hmf.h): per-launch options of the Q-band
    kernels; -1 in a field means the library default."""
    _fields_ = [("impl", _i32), ("chain_cfg", _i32), ("pstore", _i32), ("qsync", _i32),
                ("grid_share", _i32), ("lockstep", _i32), ("runs_wide", _i32)]

    def __init__(self, **kw):
        vals = {name: -1 for name, _ in self._fields_}
        vals.update({k: int(v) for k, v in kw.items() if v is not None})
        super().__init__(**vals)

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}

    def __repr__(self):
        return f"QbandOpts({self.as_dict()})"


def set_variant(variant: int) -> None:
    check(load().hmf_set_tuning(TUNE_VARIANT, int(variant)), "hmf_set_tuning")
