"""The reference's public API, same names and signatures, on the CUDA path.

A caller of the reference package (``hybridkv``, /root/reference/pkg/src)
switches with::

    import paper_2505_19586_b200.hybridkv as hybridkv

Covered: the hot-path names of hybridkv/__init__.py:12-18 and of the modules
the decode path goes through --

* kv_model.py: ``ModelConfig``, ``LayerKV`` (:76-157), ``append_kv``,
  ``attention_weights`` / ``exact_attention`` / ``layer_attention`` (:169-242);
* quantizer.py: ``GroupAxis``, ``QuantParams``, ``GroupQuantizedTensor``
  (:187-422, with ``to_bytes`` / ``from_bytes``), ``QuantizedLayerKV``
  (:430-451), ``quantize_layer_kv`` (:479), ``qgemv_scores`` /
  ``qgemv_output`` (:505-558);
* retriever.py: ``RetrievalConfig``, ``CriticalChannelSet``,
  ``QueryEstimate``, ``estimate_query``, ``channel_scores_from_max``,
  ``group_channel_scores``, ``select_critical_channels``, ``approx_scores``,
  ``select_topk_tokens``, ``sparse_attention``, ``top_weight_tokens``,
  ``recall_at_k`` (:45-252);
* memsim.py: ``HostPool`` (:76-135), ``DeviceBuffers`` (:143-187),
  ``TransferRequest``, ``prefetch_critical_keys``, ``fetch_topk`` (:196-252);
* identifier.py: ``LayerKind``, ``SparsityProbe``, ``LayerProfile``,
  ``default_probe_k``, ``sparse_error``, ``dense_preference_score``,
  ``classify_layer``, ``calibrate(trace, probe)`` (:29-187);
* trace.py: ``read_trace`` returning a reference-shaped ``Trace``.

Arguments and results are numpy float64 like the reference's; the work runs
in this package's kernels (csrc/refops.cu, qcache.cu, sparse.cu,
calibrate.cu).  Cache contents are fp16 storage, the reference's element
semantics (kv_model.py:8-10): inputs that are not fp16-exact are rounded
when they enter a cache.  Shapes the CUDA cache does not support (head_dim
not a multiple of 32 in [32, 256]; group sizes other than 16/32/64, or 128
at 1 bit) raise ParameterError -- there is no CPU path.  Errors are the
reference's exception classes (errors.py).
"""

from __future__ import annotations

import ctypes as C
import enum
import struct
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr, stream_ptr
from .errors import (ConfigError, EmptyCacheError, EncodingError, NumericError, ParameterError, SchedulingError,
                     ShapeError, TraceFormatError)
from .hoststore import OffloadedLayerKV
from .identifier import (LayerKind, LayerProfile, SparsityProbe, classify_layer, default_probe_k,
                         dense_preference_score, head_scores)
from .kv_model import ModelConfig
from .quantizer import QuantizedLayerKV as _QCache
from .quantizer import qgemv_output as _qgemv_output
from .quantizer import qgemv_scores as _qgemv_scores
from .retriever import RetrievalConfig, stage1_select
from .retriever import select_topk_tokens as _select_topk

__all__ = [
    "ConfigError", "EmptyCacheError", "EncodingError", "NumericError", "ParameterError", "SchedulingError",
    "ShapeError", "TraceFormatError", "ModelConfig", "LayerKV", "append_kv", "attention_weights",
    "exact_attention", "layer_attention", "GroupAxis", "QuantParams", "GroupQuantizedTensor", "QuantizedLayerKV",
    "quantize_layer_kv", "qgemv_scores", "qgemv_output", "RetrievalConfig", "CriticalChannelSet", "QueryEstimate",
    "estimate_query", "channel_scores_from_max", "group_channel_scores", "select_critical_channels",
    "approx_scores", "select_topk_tokens", "sparse_attention", "top_weight_tokens", "recall_at_k", "HostPool",
    "DeviceBuffers", "TransferRequest", "prefetch_critical_keys", "fetch_topk", "LayerKind", "SparsityProbe",
    "LayerProfile", "default_probe_k", "sparse_error", "dense_preference_score", "classify_layer", "calibrate",
    "Trace", "TraceStep", "read_trace",
]

SUPPORTED_BITS = (1, 2)


def _dev(x) -> torch.Tensor:
    """float64 contiguous device copy of an array-like."""
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to("cuda")


def _host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().astype(np.float64, copy=False)


# ---------------------------------------------------------------------------
# kv_model.py
# ---------------------------------------------------------------------------
class LayerKV:
    """Append-only per-layer key/value rows [num_heads, n, head_dim] (the
    caller-side container the reference's compress and offload calls take;
    kv_model.py:76-157).  Host float64 storage with geometric growth."""

    def __init__(self, num_heads: int, head_dim: int) -> None:
        if num_heads < 1 or head_dim < 1:
            raise ConfigError("num_heads and head_dim must be >= 1")
        self.num_heads, self.head_dim = num_heads, head_dim
        self._n = 0
        self._k = np.empty((num_heads, 0, head_dim))
        self._v = np.empty((num_heads, 0, head_dim))

    @classmethod
    def from_arrays(cls, keys, values) -> "LayerKV":
        keys = np.asarray(keys, dtype=np.float64)
        values = np.asarray(values, dtype=np.float64)
        if keys.ndim != 3 or keys.shape != values.shape:
            raise ShapeError(f"keys/values must share shape [heads, n, head_dim], got {keys.shape} and "
                             f"{values.shape}")
        if not (np.isfinite(keys).all() and np.isfinite(values).all()):
            raise NumericError("cache contents must be finite")
        out = cls(keys.shape[0], keys.shape[2])
        out._k, out._v, out._n = keys.copy(), values.copy(), keys.shape[1]
        return out

    @property
    def seq_len(self) -> int:
        return self._n

    @property
    def keys(self) -> np.ndarray:
        return self._k[:, :self._n]

    @property
    def values(self) -> np.ndarray:
        return self._v[:, :self._n]

    def append(self, new_key, new_value) -> None:
        new_key = np.asarray(new_key, dtype=np.float64)
        new_value = np.asarray(new_value, dtype=np.float64)
        shape = (self.num_heads, self.head_dim)
        if new_key.shape != shape or new_value.shape != shape:
            raise ShapeError(f"appended rows must have shape {shape}, got {new_key.shape} and {new_value.shape}")
        if not (np.isfinite(new_key).all() and np.isfinite(new_value).all()):
            raise NumericError("appended rows must be finite")
        if self._n == self._k.shape[1]:
            cap = max(16, 2 * self._k.shape[1])
            for name in ("_k", "_v"):
                old = getattr(self, name)
                grown = np.empty((self.num_heads, cap, self.head_dim))
                grown[:, :self._n] = old[:, :self._n]
                setattr(self, name, grown)
        self._k[:, self._n] = new_key
        self._v[:, self._n] = new_value
        self._n += 1


def append_kv(cache: LayerKV, new_key, new_value) -> LayerKV:
    cache.append(new_key, new_value)
    return cache


def _attention(queries: np.ndarray, keys: np.ndarray, values, sel=None, want_weights=False):
    """softmax(q K^T / sqrt(d)) per query row (kv_model.py:169-194) and
    optionally @ V, over all rows or the index list ``sel`` (csrc/refops.cu)."""
    q = _dev(queries)
    k = _dev(keys)
    rows, d = q.shape
    n = k.shape[0]
    s = None if sel is None else torch.as_tensor(np.ascontiguousarray(sel, dtype=np.int64)).to("cuda")
    m = n if s is None else s.numel()
    v = _dev(values) if values is not None else None
    ws = torch.empty((rows, m), dtype=torch.float64, device="cuda")
    w = torch.empty((rows, m), dtype=torch.float64, device="cuda") if want_weights else None
    out = torch.empty((rows, d), dtype=torch.float64, device="cuda") if v is not None else None
    check(_lib.load().tkv_attention_f64(ptr(q), rows, ptr(k), ptr(v), n, d, ptr(s), m, ptr(ws), ptr(w), ptr(out),
                                        stream_ptr()))
    return (None if w is None else _host(w)), (None if out is None else _host(out))


def _check_attention_inputs(query, keys):
    query = np.asarray(query, dtype=np.float64).reshape(-1)
    keys = np.asarray(keys, dtype=np.float64)
    if keys.ndim != 2 or keys.shape[1] != query.shape[0]:
        raise ShapeError(f"keys shape {keys.shape} incompatible with query dim {query.shape[0]}")
    if keys.shape[0] == 0:
        raise EmptyCacheError("attention over an empty cache")
    if not (np.isfinite(query).all() and np.isfinite(keys).all()):
        raise NumericError("attention inputs must be finite")
    return query, keys


def attention_weights(query, keys) -> np.ndarray:
    """[n] softmax weights of one head's query (kv_model.py:169-194)."""
    query, keys = _check_attention_inputs(query, keys)
    w, _ = _attention(query[None], keys, None, want_weights=True)
    return w[0]


def exact_attention(query, keys, values) -> np.ndarray:
    """softmax(q K^T / sqrt(d)) V (kv_model.py:197-213)."""
    values = np.asarray(values, dtype=np.float64)
    if values.shape != np.asarray(keys).shape:
        raise ShapeError(f"values shape {values.shape} must match keys shape {np.asarray(keys).shape}")
    query, keys = _check_attention_inputs(query, keys)
    _, out = _attention(query[None], keys, values)
    return out[0]


def layer_attention(queries, cache: LayerKV) -> np.ndarray:
    """All query heads against their KV head's rows (kv_model.py:216-242)."""
    queries = np.asarray(queries, dtype=np.float64)
    if queries.ndim != 2 or queries.shape[1] != cache.head_dim:
        raise ShapeError(f"queries shape {queries.shape} incompatible with head_dim {cache.head_dim}")
    if queries.shape[0] % cache.num_heads:
        raise ShapeError(f"{queries.shape[0]} query heads not divisible by {cache.num_heads} KV heads")
    if cache.seq_len == 0:
        raise EmptyCacheError("attention over an empty cache")
    G = queries.shape[0] // cache.num_heads
    out = np.empty_like(queries)
    for kv in range(cache.num_heads):
        _, o = _attention(queries[kv * G:(kv + 1) * G], cache.keys[kv], cache.values[kv])
        out[kv * G:(kv + 1) * G] = o
    return out


# ---------------------------------------------------------------------------
# quantizer.py
# ---------------------------------------------------------------------------
class GroupAxis(enum.Enum):
    PER_CHANNEL = "per_channel"  # keys: g consecutive tokens of one channel
    PER_TOKEN = "per_token"      # values: g consecutive channels of one token


@dataclass(frozen=True)
class QuantParams:
    zero_point: float
    scale: float
    bits: int
    group_size: int

    def __post_init__(self) -> None:
        if self.bits not in SUPPORTED_BITS:
            raise ParameterError(f"bits must be one of {SUPPORTED_BITS}, got {self.bits}")
        if self.group_size < 1:
            raise ParameterError(f"group_size must be >= 1, got {self.group_size}")
        if self.scale < 0:
            raise ParameterError(f"scale must be non-negative, got {self.scale}")


def _cuda_shape_ok(head_dim: int, bits: int, group_size: int) -> None:
    if bits not in SUPPORTED_BITS:
        raise ParameterError(f"bits must be one of {SUPPORTED_BITS}, got {bits}")
    if group_size < 1:
        raise ParameterError("group_size must be >= 1")
    if not (32 <= head_dim <= 256 and head_dim % 32 == 0):
        raise ParameterError(f"head_dim {head_dim}: the CUDA cache needs a multiple of 32 in [32, 256]")
    if group_size not in (16, 32, 64) and not (group_size == 128 and bits == 1):
        raise ParameterError(f"group_size {group_size}: the CUDA cache supports 16, 32, 64 (128 at 1 bit)")


class GroupQuantizedTensor:
    """One head's quantized [n, head_dim] matrix, resident in HBM: a view of
    unit ``unit`` of a CUDA cache (``which`` = keys for PER_CHANNEL, values
    for PER_TOKEN).  Standalone tensors (``from_matrix`` / ``from_bytes``) own
    a one-unit cache whose other side is unused; per-head views of a layer
    cache share it (append through ``QuantizedLayerKV.append_token``)."""

    _MAGIC = b"GQT1"

    def __init__(self, cache: _QCache, unit: int, axis: GroupAxis, standalone: bool = False) -> None:
        self._cache, self._unit, self.axis, self._standalone = cache, unit, axis, standalone
        self.head_dim, self.bits, self.group_size = cache.head_dim, cache.bits, cache.group_size

    @property
    def _which(self) -> str:
        return "keys" if self.axis is GroupAxis.PER_CHANNEL else "values"

    @classmethod
    def from_matrix(cls, matrix, axis: GroupAxis, bits: int, group_size: int) -> "GroupQuantizedTensor":
        matrix = np.asarray(matrix, dtype=np.float64)
        if matrix.ndim != 2:
            raise ShapeError(f"expected a 2-D matrix, got shape {matrix.shape}")
        if not np.isfinite(matrix).all():
            raise NumericError("matrix contains non-finite values")
        n, d = matrix.shape
        _cuda_shape_ok(d, bits, group_size)
        cache = _QCache(1, d, bits, group_size, max(n, 1) + 256)
        t = cls(cache, 0, axis, standalone=True)
        if n:
            t.append_rows(matrix)
        return t

    @classmethod
    def from_bytes(cls, blob: bytes) -> "GroupQuantizedTensor":
        """GQT1 blob -> HBM cache (quantizer.py:383-422)."""
        blob = bytes(blob)
        hs = struct.calcsize("<4sBBHIIII")
        if len(blob) < hs:
            raise EncodingError("quantized tensor blob truncated")
        magic, bits, axis_code, g, rows, d, res_rows, _ = struct.unpack("<4sBBHIIII", blob[:hs])
        if magic != cls._MAGIC:
            raise EncodingError("bad quantized tensor magic")
        axis = GroupAxis.PER_CHANNEL if axis_code == 1 else GroupAxis.PER_TOKEN
        _cuda_shape_ok(d, bits, g)
        cache = _QCache(1, d, bits, g, rows + res_rows + 256)
        cache.import_bytes(0, "keys" if axis is GroupAxis.PER_CHANNEL else "values", blob)
        return cls(cache, 0, axis, standalone=True)

    def append_rows(self, rows) -> None:
        """Append token rows (quantizer.py:238-293): keys finalize a group every
        group_size rows (the rest stays in the fp16 residual), values pack
        immediately.  Standalone tensors only."""
        if not self._standalone:
            raise SchedulingError("append to a layer cache through QuantizedLayerKV.append_token")
        rows = np.asarray(rows, dtype=np.float64)
        if rows.ndim == 1:
            rows = rows[None, :]
        if rows.shape[1] != self.head_dim:
            raise ShapeError(f"rows have {rows.shape[1]} channels, expected {self.head_dim}")
        if not np.isfinite(rows).all():
            raise NumericError("rows contain non-finite values")
        c = self._cache
        if c.n + rows.shape[0] > c.capacity:
            c.grow(2 * (c.n + rows.shape[0]))
        r16 = torch.tensor(rows, dtype=torch.float16, device=c.device)
        zero = torch.zeros_like(r16[0])[None]
        if c.n == 0 and rows.shape[0] > 0:
            k, v = (r16, torch.zeros_like(r16)) if self._which == "keys" else (torch.zeros_like(r16), r16)
            fresh = _QCache.from_kv(k[None], v[None], c.bits, c.group_size, capacity=c.capacity)
            self._cache = fresh
            return
        for i in range(rows.shape[0]):
            row = r16[i][None]
            c.append_token(row if self._which == "keys" else zero, row if self._which == "values" else zero)

    # -- inspection -----------------------------------------------------------
    @property
    def logical_shape(self) -> tuple[int, int]:
        return (self._cache.n, self.head_dim)

    @property
    def num_complete_rows(self) -> int:
        n = self._cache.n
        return (n // self.group_size) * self.group_size if self.axis is GroupAxis.PER_CHANNEL else n

    @property
    def num_groups(self) -> int:
        if self.axis is GroupAxis.PER_CHANNEL:
            return (self._cache.n // self.group_size) * self.head_dim
        return self._cache.n * ((self.head_dim + self.group_size - 1) // self.group_size)

    def _params(self) -> tuple[np.ndarray, np.ndarray]:
        """Runtime (zero_point, scale) grids in float64 from the cache's fp16
        (lo, hi) pairs: scale = (hi - lo) / (2^b - 1), 1 when degenerate."""
        c, u, d, g = self._cache, self._unit, self.head_dim, self.group_size
        if self.axis is GroupAxis.PER_CHANNEL:
            words = c._bufs[1].view(torch.int32).view(c.units, c.capacity // g, d)[u, :c.n // g]
        else:
            nb = (d + g - 1) // g
            words = c._bufs[4].view(torch.int32).view(c.units, c.capacity, nb)[u, :c.n]
        w = words.cpu().numpy().view(np.uint32)
        lo = (w & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float64)
        hi = (w >> 16).astype(np.uint16).view(np.float16).astype(np.float64)
        scale = (hi - lo) / (2 ** self.bits - 1)
        scale[scale == 0.0] = 1.0
        return lo, scale

    def group_params(self, index: int) -> QuantParams:
        z, s = self._params()
        if not 0 <= index < z.size:
            raise ParameterError(f"group index {index} out of range ({z.size} groups)")
        if self.axis is GroupAxis.PER_CHANNEL:
            size = self.group_size
        else:
            start = (index % s.shape[1]) * self.group_size
            size = min(self.group_size, self.head_dim - start)
        return QuantParams(float(z.reshape(-1)[index]), float(s.reshape(-1)[index]), self.bits, size)

    @property
    def residual(self) -> np.ndarray:
        if self.axis is GroupAxis.PER_TOKEN:
            return np.empty((0, self.head_dim))
        c, g = self._cache, self.group_size
        r = c.n - (c.n // g) * g
        res = c._bufs[2].view(torch.float16).view(c.units, g, self.head_dim)[self._unit, :r]
        return res.cpu().numpy().astype(np.float64)

    def to_bytes(self) -> bytes:
        """Bit-exact GQT1 serialization (quantizer.py:358-380)."""
        return self._cache.to_bytes(self._unit, self._which)

    def packed_codes(self) -> np.ndarray:
        blob = self.to_bytes()
        plen = struct.unpack("<I", blob[20:24])[0]
        return np.frombuffer(blob[24:24 + plen], dtype=np.uint8).copy()

    def dequantize(self) -> np.ndarray:
        """[n, head_dim] reconstruction code * scale + zero (+ residual rows)."""
        if self._cache.n == 0:
            return np.empty((0, self.head_dim))
        return _host(self._cache.dequantize(self._unit, self._which).double())


class QuantizedLayerKV:
    """One layer's quantized cache, every KV head in one HBM cache
    (quantizer.py:430-451); ``keys[h]`` / ``values[h]`` are per-head views."""

    def __init__(self, cache: _QCache) -> None:
        self._cache = cache
        self.keys = [GroupQuantizedTensor(cache, h, GroupAxis.PER_CHANNEL) for h in range(cache.units)]
        self.values = [GroupQuantizedTensor(cache, h, GroupAxis.PER_TOKEN) for h in range(cache.units)]

    @property
    def num_heads(self) -> int:
        return self._cache.units

    @property
    def seq_len(self) -> int:
        return self._cache.n

    def append_token(self, new_key, new_value) -> None:
        new_key = np.asarray(new_key, dtype=np.float64)
        new_value = np.asarray(new_value, dtype=np.float64)
        shape = (self.num_heads, self._cache.head_dim)
        if new_key.shape != shape or new_value.shape != shape:
            raise ShapeError(f"appended rows must have shape {shape}")
        if not (np.isfinite(new_key).all() and np.isfinite(new_value).all()):
            raise NumericError("appended rows must be finite")
        c = self._cache
        if c.n + 1 > c.capacity:
            c.grow(2 * c.capacity)
            for t in self.keys + self.values:
                t._cache = c
        c.append_token(torch.tensor(new_key, dtype=torch.float16, device=c.device),
                       torch.tensor(new_value, dtype=torch.float16, device=c.device))

    def decode(self, queries) -> np.ndarray:
        """Quantized decode attention of every query head (pipeline.py:331-337):
        the fused tensor-core kernel, fp32 out as float64 [hq, d]."""
        q = torch.tensor(np.asarray(queries, dtype=np.float64), dtype=torch.float16, device=self._cache.device)
        return _host(self._cache.decode(q).double())


def quantize_layer_kv(cache: LayerKV, bits: int, group_size: int) -> QuantizedLayerKV:
    """Keys per channel, values per token, every head in one launch
    (quantizer.py:479-497)."""
    if cache.seq_len == 0:
        raise EmptyCacheError("cannot quantize an empty cache")
    _cuda_shape_ok(cache.head_dim, bits, group_size)
    q = _QCache.from_kv(cache.keys, cache.values, bits, group_size, capacity=cache.seq_len + 1024)
    return QuantizedLayerKV(q)


def qgemv_scores(query, qkeys: GroupQuantizedTensor) -> np.ndarray:
    """Unscaled logits [n] over quantized keys (quantizer.py:505-533)."""
    if qkeys.axis is not GroupAxis.PER_CHANNEL:
        raise ShapeError("qgemv_scores needs a per-channel (key) tensor")
    query = np.asarray(query, dtype=np.float64).reshape(-1)
    if query.shape[0] != qkeys.head_dim:
        raise ShapeError(f"query dim {query.shape[0]} != head_dim {qkeys.head_dim}")
    if qkeys._cache.n == 0:
        return np.empty(0)
    return _host(_qgemv_scores(query, qkeys._cache, qkeys._unit))


def qgemv_output(weights, qvalues: GroupQuantizedTensor) -> np.ndarray:
    """weights [n] @ dequantized values -> [head_dim] (quantizer.py:536-558)."""
    if qvalues.axis is not GroupAxis.PER_TOKEN:
        raise ShapeError("qgemv_output needs a per-token (value) tensor")
    weights = np.asarray(weights, dtype=np.float64).reshape(-1)
    if weights.shape[0] != qvalues._cache.n:
        raise ShapeError(f"weights length {weights.shape[0]} != token count {qvalues._cache.n}")
    return _host(_qgemv_output(weights, qvalues._cache, qvalues._unit))


# ---------------------------------------------------------------------------
# retriever.py
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class CriticalChannelSet:
    channel_scores: np.ndarray  # [head_dim]
    selected: np.ndarray        # ascending, d_s entries


@dataclass(frozen=True)
class QueryEstimate:
    q_hat: np.ndarray  # [num_query_heads, head_dim]
    source_layer: int


def estimate_query(w_q, hidden_state, source_layer: int) -> QueryEstimate:
    """q_hat = h . W_q (retriever.py:84-108) on the stage-1 kernel (fp16
    operands as stored, float64 result)."""
    w = np.asarray(w_q, dtype=np.float64)
    h = np.asarray(hidden_state, dtype=np.float64).reshape(-1)
    if w.ndim != 3 or w.shape[1] != h.shape[0]:
        raise ShapeError(f"w_q shape {w.shape} incompatible with hidden dim {h.shape[0]}")
    hq, _, d = w.shape
    q_hat = torch.empty((1, hq, d), dtype=torch.float64, device="cuda")
    stage1_select(torch.tensor(h[None], dtype=torch.float16, device="cuda"),
                  torch.tensor(w, dtype=torch.float16, device="cuda"),
                  torch.ones((hq, d), dtype=torch.float32, device="cuda"), 1, 1, q_hat=q_hat)
    return QueryEstimate(q_hat=_host(q_hat[0]), source_layer=source_layer)


def _channel_select(q, chmax, d_s: int):
    q = _dev(np.atleast_2d(q))
    G, d = q.shape
    cm = None if chmax is None else _dev(chmax)
    scores = torch.empty(d, dtype=torch.float64, device="cuda")
    sel = torch.empty(max(d_s, 1), dtype=torch.int32, device="cuda")
    check(_lib.load().tkv_channel_select_f64(ptr(q), G, ptr(cm), d, max(d_s, 1), ptr(scores), ptr(sel),
                                             stream_ptr()))
    return _host(scores), sel.cpu().numpy().astype(np.int64)


def channel_scores_from_max(q_hat, channel_abs_max) -> np.ndarray:
    """|q_hat_i| * max_j |K[j, i]| (retriever.py:111-119)."""
    q = np.asarray(q_hat, dtype=np.float64).reshape(-1)
    cm = np.asarray(channel_abs_max, dtype=np.float64).reshape(-1)
    if q.shape != cm.shape:
        raise ShapeError(f"query dim {q.shape[0]} != channel max dim {cm.shape[0]}")
    return _channel_select(q, cm, 1)[0]


def group_channel_scores(q_hat_group, channel_abs_max) -> np.ndarray:
    """(sum over the group of |q_hat|) * channel max (retriever.py:138-148)."""
    q = np.atleast_2d(np.asarray(q_hat_group, dtype=np.float64))
    cm = np.asarray(channel_abs_max, dtype=np.float64).reshape(-1)
    if q.shape[1] != cm.shape[0]:
        raise ShapeError(f"query dim {q.shape[1]} != channel max dim {cm.shape[0]}")
    return _channel_select(q, cm, 1)[0]


def select_critical_channels(scores, d_s: int) -> CriticalChannelSet:
    """Top d_s channels, ties to the lower index, ascending (retriever.py:151-163)."""
    s = np.asarray(scores, dtype=np.float64).reshape(-1)
    if not 1 <= d_s <= s.shape[0]:
        raise ParameterError(f"d_s must lie in [1, {s.shape[0]}], got {d_s}")
    _, sel = _channel_select(s, None, d_s)
    return CriticalChannelSet(channel_scores=s, selected=sel)


def approx_scores(query_critical, critical_keys) -> np.ndarray:
    """critical_keys [n, d_s] @ (sum over the group of the query slice)
    (retriever.py:166-189), float64."""
    qc = np.atleast_2d(np.asarray(query_critical, dtype=np.float64))
    ck = np.asarray(critical_keys, dtype=np.float64)
    if ck.ndim != 2 or ck.shape[1] != qc.shape[1]:
        raise ShapeError(f"critical keys shape {ck.shape} incompatible with query slice {qc.shape}")
    n = ck.shape[0]
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    if n:
        q, k = _dev(qc), _dev(ck)
        check(_lib.load().tkv_approx_scores_f64(ptr(q), qc.shape[0], ptr(k), n, qc.shape[1], ptr(out),
                                                stream_ptr()))
    return _host(out)


def select_topk_tokens(scores, config: RetrievalConfig) -> np.ndarray:
    """Local window + top n_topk by (score desc, index desc), ascending
    (retriever.py:192-211)."""
    return _select_topk(scores, config)


def sparse_attention(query, keys, values, selected) -> np.ndarray:
    """Exact attention over the selected rows only (retriever.py:214-226)."""
    sel = np.asarray(selected, dtype=np.int64).reshape(-1)
    if sel.size == 0:
        raise EmptyCacheError("sparse attention needs a non-empty selection")
    keys = np.asarray(keys, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    if sel.min() < 0 or sel.max() >= keys.shape[0]:
        raise ParameterError("selected indices out of range")
    query, _ = _check_attention_inputs(query, keys[sel[:1]])
    _, out = _attention(query[None], keys, values, sel=sel)
    return out[0]


def top_weight_tokens(weights, k: int) -> np.ndarray:
    """The k largest weights, ties to the more recent index, ascending
    (retriever.py:229-242) -- the top-k kernel with an empty local window."""
    w = np.asarray(weights, dtype=np.float64).reshape(-1)
    if not 1 <= k <= w.shape[0]:
        raise ParameterError(f"k must lie in [1, {w.shape[0]}], got {k}")
    return _select_topk(w, RetrievalConfig(0, k, 1))


def recall_at_k(selected, exact_topk) -> float:
    """|selected ∩ exact| / |exact| (retriever.py:245-252); index bookkeeping."""
    selected = np.asarray(selected).reshape(-1)
    exact_topk = np.asarray(exact_topk).reshape(-1)
    if selected.size == 0 or exact_topk.size == 0:
        raise ParameterError("recall needs non-empty index sets")
    return np.intersect1d(selected, exact_topk).size / exact_topk.size


# ---------------------------------------------------------------------------
# memsim.py: host pool on pinned NUMA-local memory, GPU gathers
# ---------------------------------------------------------------------------
class HostPool:
    """Offloaded per-layer K/V (memsim.py:76-135) in this package's pinned
    host stores; the running channel maxima live on the device and are
    updated by the append kernel; gathers are UVA reads by the GPU."""

    def __init__(self) -> None:
        self._layers: dict[int, OffloadedLayerKV] = {}

    def offload_layer(self, layer: int, cache: LayerKV) -> None:
        if layer in self._layers:
            raise SchedulingError(f"layer {layer} already offloaded")
        if cache.seq_len == 0:
            raise EmptyCacheError("cannot offload an empty cache")
        if cache.head_dim % 32 or not 32 <= cache.head_dim <= 256:
            raise ParameterError(f"head_dim {cache.head_dim}: the CUDA host store needs a multiple of 32 in [32, 256]")
        lay = OffloadedLayerKV(cache.num_heads, cache.head_dim, cache.seq_len + 1024, cache.seq_len, 0)
        lay.offload(cache.keys, cache.values)
        self._layers[layer] = lay

    def has_layer(self, layer: int) -> bool:
        return layer in self._layers

    def _require(self, layer: int) -> OffloadedLayerKV:
        if layer not in self._layers:
            raise ParameterError(f"layer {layer} is not offloaded")
        return self._layers[layer]

    def seq_len(self, layer: int) -> int:
        return self._require(layer).n

    def append(self, layer: int, new_key, new_value) -> None:
        lay = self._require(layer)
        k = np.asarray(new_key, dtype=np.float64)
        v = np.asarray(new_value, dtype=np.float64)
        if k.shape != (lay.units, lay.head_dim) or v.shape != k.shape:
            raise ShapeError(f"appended rows must have shape {(lay.units, lay.head_dim)}")
        lay.append(k, v)

    def channel_abs_max(self, layer: int) -> np.ndarray:
        """Running max|K| per (head, channel), all tokens incl. appended."""
        return _host(self._require(layer).chmax.double())

    def gather(self, layer: int, head: int, indices) -> tuple[np.ndarray, np.ndarray]:
        lay = self._require(layer)
        idx = np.asarray(indices, dtype=np.int64).reshape(-1)
        if idx.size == 0:
            return np.empty((0, lay.head_dim)), np.empty((0, lay.head_dim))
        if idx.min() < 0 or idx.max() >= lay.n:
            raise ParameterError("gather index out of range")
        if not 0 <= head < lay.units:
            raise ParameterError("head out of range")
        torch.cuda.synchronize()  # appends of earlier steps have landed in the store
        di = torch.as_tensor(idx).to("cuda")
        k = torch.empty((idx.size, lay.head_dim), dtype=torch.float16, device="cuda")
        v = torch.empty_like(k)
        check(_lib.load().tkv_host_gather(C.byref(lay.struct), head, ptr(di), idx.size, ptr(k), ptr(v),
                                          stream_ptr()))
        return _host(k.double()), _host(v.double())

    def gather_key_columns(self, layer: int, head: int, channels) -> np.ndarray:
        """[n, len(channels)] key columns from the device's channel-major copy."""
        lay = self._require(layer)
        ch = np.asarray(channels, dtype=np.int64).reshape(-1)
        if ch.size and (ch.min() < 0 or ch.max() >= lay.head_dim):
            raise ParameterError("channel index out of range")
        cols = lay.kt[head, torch.as_tensor(ch).to(lay.kt.device), :lay.n]
        return _host(cols.double()).T.copy()


class DeviceBuffers:
    """Double-buffered critical-key slots + staging (memsim.py:143-187): the
    reference's scheduling contract (a slot being written is never read)."""

    def __init__(self, num_heads: int, head_dim: int) -> None:
        self.num_heads, self.head_dim = num_heads, head_dim
        self._slots: list = [None, None]
        self._writing = [False, False]
        self.local = LayerKV(num_heads, head_dim)
        self.staged_topk = None

    @staticmethod
    def slot_for_step(step: int) -> int:
        return step % 2

    def begin_prefetch(self, step: int) -> int:
        s = self.slot_for_step(step)
        if self._writing[s]:
            raise SchedulingError(f"critical-key slot {s} already has a prefetch in flight")
        self._writing[s] = True
        return s

    def complete_prefetch(self, slot: int, per_head, step: int) -> None:
        if not self._writing[slot]:
            raise SchedulingError(f"slot {slot} has no prefetch in flight")
        self._slots[slot] = (step, per_head)
        self._writing[slot] = False

    def read_slot(self, step: int):
        s = self.slot_for_step(step)
        if self._writing[s]:
            raise SchedulingError(f"slot {s} is being written")
        if self._slots[s] is None or self._slots[s][0] != step:
            raise SchedulingError(f"slot {s} does not hold step {step}")
        return self._slots[s][1]


@dataclass(frozen=True)
class TransferRequest:
    label: str
    layer: int
    step: int
    nbytes: int


def prefetch_critical_keys(pool: HostPool, layer: int, channel_sets: Sequence, buffers: DeviceBuffers, step: int,
                           element_bytes: int = 2) -> TransferRequest:
    """Stage each head's selected key columns into the step's slot
    (memsim.py:205-225); n * d_s elements per head."""
    slot = buffers.begin_prefetch(step)
    per_head, nbytes = [], 0
    for head, ch in enumerate(channel_sets):
        cols = pool.gather_key_columns(layer, head, ch)
        per_head.append((np.asarray(ch, dtype=np.intp).copy(), cols))
        nbytes += cols.size * element_bytes
    buffers.complete_prefetch(slot, per_head, step)
    return TransferRequest("prefetch", layer, step, nbytes)


def fetch_topk(pool: HostPool, layer: int, indices_per_head: Sequence, buffers: DeviceBuffers | None, step: int,
               element_bytes: int = 2):
    """Selected tokens' K and V rows from the host store (memsim.py:228-252);
    2 * rows * head_dim elements."""
    rows, total, d = [], 0, None
    for head, idx in enumerate(indices_per_head):
        k, v = pool.gather(layer, head, idx)
        rows.append((k, v))
        total += k.shape[0]
        d = k.shape[1]
    if buffers is not None:
        buffers.staged_topk = {"step": step, "rows": rows}
    return rows, TransferRequest("topk_fetch", layer, step, 2 * total * (d or 0) * element_bytes)


# ---------------------------------------------------------------------------
# identifier.py
# ---------------------------------------------------------------------------
def sparse_error(weights, k: int) -> float:
    """1 - (sum of the k largest weights) (identifier.py:89-107): the top-k
    selection kernel, then a fixed-order float64 sum of the kept weights."""
    w = np.asarray(weights, dtype=np.float64).reshape(-1)
    n = w.shape[0]
    if not 1 <= k <= n:
        raise ParameterError(f"k must lie in [1, {n}], got {k}")
    lib = _lib.load()
    dw = _dev(w)[None]
    from .retriever import WORKSPACES
    ws = WORKSPACES.get("topk", lib.tkv_select_workspace(1, n), dw.device)
    ws.zero_()
    idx = torch.empty((1, k), dtype=torch.int32, device="cuda")
    cnt = torch.empty(1, dtype=torch.int32, device="cuda")
    check(lib.tkv_topk_from_scores(ptr(dw), 1, n, 0, k, ptr(idx), ptr(cnt), ptr(ws), stream_ptr()))
    kept = torch.empty(1, dtype=torch.float64, device="cuda")
    check(lib.tkv_sum_at(ptr(dw), ptr(idx), ptr(cnt), ptr(kept), stream_ptr()))
    return float(1.0 - kept.item())


def calibrate(trace, probe: SparsityProbe) -> list[LayerProfile]:
    """Classify every layer of a trace from its prefill (identifier.py:153-187):
    each query head's last n_q prefill queries against its KV head's prefill
    keys, on the calibration kernel.  ``trace``: this module's ``Trace``, the
    reference's, or a ``DeviceTrace`` (trace.load_trace)."""
    if hasattr(trace, "prefill"):
        keys = [np.asarray(c.keys) for c in trace.prefill]
        queries = [np.asarray(q) for q in trace.prefill_queries]
    else:
        keys, queries = trace.prefill_keys, trace.prefill_queries
    n = keys[0].shape[1]
    if n < probe.n_q:
        raise ParameterError(f"trace prefill length {n} is shorter than probe n_q {probe.n_q}")
    if probe.k > n:
        raise ParameterError(f"probe k {probe.k} exceeds prefill length {n}")
    out = []
    for layer, (Q, K) in enumerate(zip(queries, keys)):
        recent = Q[:, Q.shape[1] - probe.n_q:, :]
        out.append(classify_layer(layer, head_scores(recent, K, probe.k), probe.tau))
    return out


# ---------------------------------------------------------------------------
# trace.py
# ---------------------------------------------------------------------------
@dataclass
class TraceStep:
    hidden: np.ndarray      # [L, hidden]
    queries: np.ndarray     # [L, hq, d]
    new_keys: np.ndarray    # [L, h, d]
    new_values: np.ndarray


@dataclass
class Trace:
    """Reference-shaped trace (trace.py:57-76), float64 fp16-exact arrays."""

    config: ModelConfig
    prefill: list
    prefill_queries: list
    w_q: list
    steps: list
    labels: list | None = None

    @property
    def prefill_len(self) -> int:
        return self.prefill[0].seq_len

    @property
    def num_steps(self) -> int:
        return len(self.steps)


def read_trace(path) -> Trace:
    """HKVTRACE file -> Trace (trace.py:105-228 format), read through
    trace.load_trace (one device upload, fp16 sections) and returned as
    float64 host arrays like the reference reader."""
    from .trace import load_trace

    dt = load_trace(path)
    m = dt.header["model"]
    config = ModelConfig(m["num_layers"], m["num_query_heads"], m["num_kv_heads"], m["head_dim"], m["hidden_dim"])

    def f64(t):
        return t.cpu().double().numpy()

    prefill = [LayerKV.from_arrays(f64(k), f64(v)) for k, v in zip(dt.prefill_keys, dt.prefill_values)]
    steps = [TraceStep(f64(dt.hidden[t]), f64(dt.queries[t]), f64(dt.new_keys[t]), f64(dt.new_values[t]))
             for t in range(dt.num_steps)]
    return Trace(config, prefill, [f64(q) for q in dt.prefill_queries], [f64(w) for w in dt.w_q], steps,
                 list(dt.labels) or None)
