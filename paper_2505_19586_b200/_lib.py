"""ctypes binding of ``libtailorkv.so`` (the C ABI in include/tailorkv.h).

This is the reference-side binding a maintainer of ``hybridkv`` would add: it
maps the C status codes onto the reference's exception classes
(hybridkv/errors.py:9-38) and marshals torch tensors into raw pointers.
There is no fallback: if the library cannot be loaded every operation raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import torch

from .errors import (
    EmptyCacheError,
    EncodingError,
    NumericError,
    ParameterError,
    SchedulingError,
    ShapeError,
)

_LIB_PATH = Path(__file__).resolve().parent / "libtailorkv.so"


class CudaError(RuntimeError):
    """A CUDA runtime failure inside the extension (no reference counterpart)."""


_STATUS = {
    1: ShapeError,
    2: ParameterError,
    3: EmptyCacheError,
    4: NumericError,
    5: EncodingError,
    6: SchedulingError,
    7: CudaError,
}


class QCache(C.Structure):
    _fields_ = [
        ("units", C.c_int32), ("d", C.c_int32), ("bits", C.c_int32), ("g", C.c_int32),
        ("capacity", C.c_int64),
        ("key_codes", C.c_void_p), ("key_lohi", C.c_void_p), ("key_resid", C.c_void_p),
        ("val_codes", C.c_void_p), ("val_lohi", C.c_void_p), ("val_smax", C.c_void_p),
        ("len", C.c_void_p), ("ticket", C.c_void_p),
    ]


class SparseLayer(C.Structure):
    _fields_ = [
        ("units", C.c_int32), ("d", C.c_int32),
        ("capacity", C.c_int64), ("local_offset", C.c_int64), ("local_capacity", C.c_int64),
        ("kt", C.c_void_p), ("chmax", C.c_void_p), ("loc_k", C.c_void_p), ("loc_v", C.c_void_p),
        ("kdev", C.c_void_p), ("host_kv", C.c_void_p), ("len", C.c_void_p), ("ticket", C.c_void_p),
        ("cache_slots", C.c_int32), ("cache_window", C.c_int32), ("slot_tok", C.c_void_p), ("slot_stamp", C.c_void_p),
        ("slot_v", C.c_void_p), ("tok_slot", C.c_void_p), ("cache_stats", C.c_void_p), ("thresh", C.c_void_p),
        ("slot_hand", C.c_void_p), ("n_sink", C.c_int32), ("part_hint", C.c_void_p),
        ("s1_ready", C.c_void_p), ("s1_flags", C.c_int32),
    ]


MAX_PARTS = 256  # TKV_MAX_PARTS (tailorkv.h)


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_SIGS = {
    "tkv_last_error": (C.c_char_p, []),
    "tkv_abi_version": (C.c_int, []),
    "tkv_event_record": (C.c_int, [_P, _P, _I32]),
    "tkv_graph_instantiate": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "tkv_graph_launch": (C.c_int, [_P, _P]),
    "tkv_graph_destroy": (C.c_int, [_P]),
    "tkv_qcache_sizes": (C.c_int, [_I32, _I32, _I32, _I32, _I64, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "tkv_qcache_pack": (C.c_int, [C.POINTER(QCache), _P, _P, _I64, _I32, _P]),
    "tkv_qcache_append": (C.c_int, [C.POINTER(QCache), _P, _P, _P]),
    "tkv_qcache_export_size": (C.c_int64, [C.POINTER(QCache), _I32, _I64]),
    "tkv_qcache_export": (C.c_int, [C.POINTER(QCache), _I32, _I32, _I64, _P, _P]),
    "tkv_qcache_dequant": (C.c_int, [C.POINTER(QCache), _I32, _I32, _I64, _P, _P]),
    "tkv_quant_decode_workspace": (C.c_int64, [C.POINTER(QCache), _I32]),
    "tkv_quant_decode": (C.c_int, [C.POINTER(QCache), _P, _I32, _P, _P, _I32, _P]),
    "tkv_qgemv_scores": (C.c_int, [C.POINTER(QCache), _I32, _I64, _P, _P, _P]),
    "tkv_qgemv_output_workspace": (C.c_int64, [C.POINTER(QCache), _I64]),
    "tkv_qgemv_output": (C.c_int, [C.POINTER(QCache), _I32, _I64, _P, _P, _P, _P]),
    "tkv_qcache_import": (C.c_int, [C.POINTER(QCache), _I32, _I32, C.c_char_p, _I64, _P, _P]),
    "tkv_attention_f64": (C.c_int, [_P, _I32, _P, _P, _I64, _I32, _P, _I64, _P, _P, _P, _P]),
    "tkv_approx_scores_f64": (C.c_int, [_P, _I32, _P, _I64, _I32, _P, _P]),
    "tkv_channel_select_f64": (C.c_int, [_P, _I32, _P, _I32, _I32, _P, _P, _P]),
    "tkv_host_gather": (C.c_int, [C.POINTER(SparseLayer), _I32, _P, _I64, _P, _P, _P]),
    "tkv_sparse_decode_plan": (C.c_int, [C.POINTER(SparseLayer), _I32, _I32, _I32, _I32]),
    "tkv_sum_at": (C.c_int, [_P, _P, _P, _P, _P]),
    "tkv_sparse_prefill": (C.c_int, [C.POINTER(SparseLayer), _P, _P, _I64, _P]),
    "tkv_sparse_append": (C.c_int, [C.POINTER(SparseLayer), _P, _P, _P]),
    "tkv_stage1_workspace": (C.c_int64, [_I32, _I32, _I32, _I32]),
    "tkv_stage1": (C.c_int, [_P, _P, _I32, _I32, _I32, _I32, _I32, _P, _I32, _P, _P, _P, _P]),
    "tkv_stage1_prefetch": (C.c_int, [_P, _P, _I32, _I32, _I32, _I32, _I32, _P, _I32, _P, _P, _P,
                                      C.POINTER(SparseLayer), _P]),
    "tkv_select_workspace": (C.c_int64, [_I32, _I64]),
    "tkv_select_tokens": (C.c_int, [C.POINTER(SparseLayer), _P, _I32, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P]),
    "tkv_topk_from_scores": (C.c_int, [_P, _I32, _I64, _I32, _I32, _P, _P, _P, _P]),
    "tkv_sparse_attn_workspace": (C.c_int64, [_I32, _I32, _I32, _I32]),
    "tkv_sparse_attention": (C.c_int, [C.POINTER(SparseLayer), _P, _I32, _P, _P, _I32, _I32, _I32, _P, _P, _P]),
    "tkv_sparse_decode_workspace": (C.c_int64, [_I32, _I64, _I32, _I32, _I32]),
    "tkv_sparse_decode": (C.c_int, [C.POINTER(SparseLayer), _P, _I32, _P, _I32, _I32, _I32, _P, _P, _P, _I32, _P, _P,
                                    _P, _P, _P]),
    "tkv_sparse_fidelity_workspace": (C.c_int64, [_I32, _I32, _I64, _I32]),
    "tkv_sparse_fidelity": (C.c_int, [C.POINTER(SparseLayer), _P, _I32, _I64, _P, _P, _I32, _I32, _P, _P, _P, _P]),
    "tkv_host_store_create": (C.c_void_p, [C.c_size_t, _I32]),
    "tkv_host_store_destroy": (C.c_int, [_P, C.c_size_t]),
    "tkv_uva_read_probe": (C.c_int, [_P, C.c_size_t, _I32, _P, _I32, _P, _P]),
    "tkv_calibrate_workspace": (C.c_int64, [_I32, _I32, _I64]),
    "tkv_dense_preference": (C.c_int, [_P, _P, _I32, _I32, _I32, _I64, _I32, _I64, _P, _P, _P]),
}

_lib = None


def exported_symbols() -> list[str]:
    return list(_SIGS)


def load():
    """Load the CUDA library (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if os.environ.get("TAILORKV_NO_BUILD") != "1":
        from . import build as _build

        try:
            if _build.needs_build():
                _build.build()
        except Exception as exc:  # a stale or missing toolkit is reported below
            if not _LIB_PATH.exists():
                raise RuntimeError(f"libtailorkv.so is missing and could not be built: {exc}") from exc
    if not _LIB_PATH.exists():
        raise RuntimeError(f"libtailorkv.so not found at {_LIB_PATH}; run paper_2505_19586_b200/build.py")
    lib = C.CDLL(str(_LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def set_sparse_kernel(mode: int) -> None:
    """Which kernel runs a fused sparse decode: -1 auto (one thread-block
    cluster per unit; the wide decode only for shapes the cluster kernel
    cannot take), 0 never the wide decode, 1 the wide decode whenever the
    shape allows (tests, experiments)."""
    load().tkv_debug_sparse_wide(int(mode))


def wide_parts(units: int) -> int:
    """Token partitions (CTAs) per unit of the wide sparse decode on this GPU."""
    return int(load().tkv_wide_parts(int(units)))


def check(status: int) -> None:
    if status != 0:
        msg = load().tkv_last_error().decode()
        raise _STATUS.get(status, CudaError)(msg)


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("the TailorKV engine needs a CUDA device (no CPU fallback)")
