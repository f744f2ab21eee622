"""Quantized KV cache of quantization-friendly layers, resident in HBM.

Mirrors hybridkv/quantizer.py (GroupQuantizedTensor :187-422,
QuantizedLayerKV :430-451, quantize_layer_kv :479-497, qgemv_scores/_output
:505-558) on top of the sm_100a kernels in csrc/qcache.cu and csrc/decode.cu.
One object holds every KV head ("unit") of one layer (batch x kv heads);
codes are kept in the MMA-native bit-plane layout and exported to the
reference GQT1 byte stream on demand (``to_bytes``).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import QCache, check, ptr, stream_ptr
from .errors import EmptyCacheError, ParameterError, ShapeError

SUPPORTED_BITS = (1, 2)


def as_f16(x, device=None) -> torch.Tensor:
    """fp16 contiguous CUDA tensor from numpy / torch input (values are taken
    as fp16 storage, the reference's element semantics, kv_model.py:8-10)."""
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float16))
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(np.asarray(x, dtype=np.float16))
    return x.to(device=device or "cuda", dtype=torch.float16).contiguous()


class QuantizedLayerKV:
    """Bit-packed 1/2-bit cache of one layer for ``units`` KV heads.

    Keys: per-channel groups of ``group_size`` tokens, trailing rows kept in an
    fp16 residual (quantizer.py:277-293).  Values: per-token groups of
    ``group_size`` channels (quantizer.py:252-275).  The token count lives on
    the device (``len``) so decode steps can be replayed from a CUDA graph.
    """

    def __init__(self, units: int, head_dim: int, bits: int, group_size: int, capacity: int, device=None):
        _lib.require_cuda()
        lib = _lib.load()
        if bits not in SUPPORTED_BITS:
            raise ParameterError(f"bits must be one of {SUPPORTED_BITS}, got {bits}")
        sizes = (C.c_int64 * 6)()
        tile = C.c_int32()
        tile_probe = lib.tkv_qcache_sizes(units, head_dim, bits, group_size, 1 << 30, sizes, C.byref(tile))
        check(tile_probe)
        t = max(int(tile.value), group_size)
        capacity = ((int(capacity) + t - 1) // t) * t
        check(lib.tkv_qcache_sizes(units, head_dim, bits, group_size, capacity, sizes, C.byref(tile)))
        dev = torch.device(device or "cuda")
        self.device = dev
        self.units, self.head_dim, self.bits, self.group_size, self.capacity = units, head_dim, bits, group_size, capacity
        self._bufs = [torch.zeros(int(s), dtype=torch.uint8, device=dev) for s in sizes]
        self._len = torch.zeros(2, dtype=torch.int32, device=dev)  # [len, ticket]
        self.n = 0  # host mirror of the device length
        self._ws = {}
        self.struct = QCache(
            units, head_dim, bits, group_size, capacity,
            *[b.data_ptr() for b in self._bufs],
            self._len.data_ptr(), self._len.data_ptr() + 4,
        )

    # -- construction -------------------------------------------------------
    @classmethod
    def from_kv(cls, keys, values, bits: int, group_size: int, capacity: int | None = None,
                check_finite: bool = True, stream=None) -> "QuantizedLayerKV":
        """Quantize ``[units, n, d]`` keys/values (quantize_layer_kv,
        quantizer.py:479-497)."""
        k = as_f16(keys)
        v = as_f16(values)
        if k.dim() != 3 or k.shape != v.shape:
            raise ShapeError(f"keys/values must share shape [heads, n, head_dim], got {tuple(k.shape)} and {tuple(v.shape)}")
        units, n, d = k.shape
        if n == 0:
            raise EmptyCacheError("cannot quantize an empty cache")
        obj = cls(units, d, bits, group_size, capacity or n, device=k.device)
        check(_lib.load().tkv_qcache_pack(C.byref(obj.struct), ptr(k), ptr(v), n, int(check_finite), stream_ptr(stream)))
        obj.n = n
        return obj

    def grow(self, capacity: int) -> None:
        """Re-home the cache into buffers for ``capacity`` tokens (device
        copies of every unit's token prefix; the layouts are per-unit blocks
        whose token order does not depend on the capacity)."""
        if capacity <= self.capacity:
            return
        bigger = QuantizedLayerKV(self.units, self.head_dim, self.bits, self.group_size, capacity, device=self.device)
        for old, new in zip(self._bufs, bigger._bufs):
            o, nw = old.view(self.units, -1), new.view(self.units, -1)
            nw[:, :o.shape[1]].copy_(o)
        bigger._len.copy_(self._len)
        self._bufs, self._len, self.capacity, self.struct = bigger._bufs, bigger._len, bigger.capacity, bigger.struct
        self._ws = {}

    # -- properties ---------------------------------------------------------
    @property
    def num_heads(self) -> int:
        return self.units

    @property
    def seq_len(self) -> int:
        return self.n

    @property
    def len_tensor(self) -> torch.Tensor:
        return self._len[:1]

    # -- decode-time ops ----------------------------------------------------
    def append_token(self, new_keys, new_values, stream=None) -> None:
        """Append one token per unit (QuantizedLayerKV.append_token,
        quantizer.py:445-451).  ``new_keys``/``new_values``: [units, d] fp16."""
        k = new_keys if isinstance(new_keys, torch.Tensor) and new_keys.dtype == torch.float16 else as_f16(new_keys)
        v = new_values if isinstance(new_values, torch.Tensor) and new_values.dtype == torch.float16 else as_f16(new_values)
        if tuple(k.shape[-2:]) != (self.units, self.head_dim) or k.shape != v.shape:
            raise ShapeError(f"appended rows must have shape {(self.units, self.head_dim)}")
        if self.n + 1 > self.capacity:
            raise ParameterError("cache capacity exhausted")
        check(_lib.load().tkv_qcache_append(C.byref(self.struct), ptr(k), ptr(v), stream_ptr(stream)))
        self.n += 1

    def workspace(self, G: int) -> torch.Tensor:
        if G not in self._ws:
            size = _lib.load().tkv_quant_decode_workspace(C.byref(self.struct), G)
            self._ws[G] = torch.zeros(int(size), dtype=torch.uint8, device=self.device)  # arrival counters start at 0
        return self._ws[G]

    def decode(self, queries, out: torch.Tensor | None = None, impl: int = 0, stream=None) -> torch.Tensor:
        """Quantized decode attention of one layer (pipeline.py:331-337):
        ``queries`` [units*G, d] fp16 -> fp32 [units*G, d]."""
        q = queries if isinstance(queries, torch.Tensor) and queries.dtype == torch.float16 and queries.is_cuda else as_f16(queries)
        q = q.reshape(-1, self.head_dim)
        if q.shape[0] % self.units:
            raise ShapeError(f"{q.shape[0]} query heads not divisible by {self.units} KV heads")
        G = q.shape[0] // self.units
        if out is None:
            out = torch.empty((q.shape[0], self.head_dim), dtype=torch.float32, device=self.device)
        if self.n == 0:
            raise EmptyCacheError("attention over an empty cache")
        check(_lib.load().tkv_quant_decode(C.byref(self.struct), ptr(q), G, ptr(out), ptr(self.workspace(G)), impl,
                                           stream_ptr(stream)))
        return out

    # -- inspection / export ------------------------------------------------
    def to_bytes(self, unit: int, which: str = "keys") -> bytes:
        """GQT1 blob of one head, byte-identical to
        GroupQuantizedTensor.to_bytes (quantizer.py:358-380)."""
        w = 0 if which == "keys" else 1
        lib = _lib.load()
        size = lib.tkv_qcache_export_size(C.byref(self.struct), w, self.n)
        out = torch.empty(int(size), dtype=torch.uint8, device=self.device)
        check(lib.tkv_qcache_export(C.byref(self.struct), unit, w, self.n, ptr(out), stream_ptr()))
        return out.cpu().numpy().tobytes()

    def import_bytes(self, unit: int, which: str, blob: bytes) -> None:
        """Load a GQT1 blob (GroupQuantizedTensor.to_bytes, quantizer.py:358-422)
        into one unit's keys or values; the device token count becomes the
        blob's row count (all units share it)."""
        w = 0 if which == "keys" else 1
        blob = bytes(blob)
        ws = torch.empty(max(len(blob), 1), dtype=torch.uint8, device=self.device)
        check(_lib.load().tkv_qcache_import(C.byref(self.struct), unit, w, blob, len(blob), ptr(ws), stream_ptr()))
        self.n = int(self._len[0].item())

    def dequantize(self, unit: int, which: str = "keys") -> torch.Tensor:
        """[n, d] fp32 reconstruction (quantizer.py:335-352)."""
        out = torch.empty((self.n, self.head_dim), dtype=torch.float32, device=self.device)
        check(_lib.load().tkv_qcache_dequant(C.byref(self.struct), unit, 0 if which == "keys" else 1, self.n,
                                             ptr(out), stream_ptr()))
        return out


def quantize_layer_kv(keys, values, bits: int, group_size: int, capacity: int | None = None) -> QuantizedLayerKV:
    """Keys per channel, values per token (quantizer.py:479-497)."""
    return QuantizedLayerKV.from_kv(keys, values, bits, group_size, capacity)


def _f64_vector(x, device, name: str, size: int) -> torch.Tensor:
    t = torch.as_tensor(np.asarray(x, np.float64) if not isinstance(x, torch.Tensor) else x)
    t = t.to(device=device, dtype=torch.float64).reshape(-1).contiguous()
    if t.numel() != size:
        raise ShapeError(f"{name} has {t.numel()} entries, expected {size}")
    return t


def qgemv_scores(query, qkv: QuantizedLayerKV, unit: int = 0, n: int | None = None) -> torch.Tensor:
    """Unscaled float64 logits [n] of one head over its quantized keys
    (quantizer.py:505-533): complete groups from the codes, the trailing
    rows from the fp16 residual."""
    n = qkv.n if n is None else n
    if n < 1:
        raise EmptyCacheError("scores over an empty cache")
    q = _f64_vector(query, qkv.device, "query", qkv.head_dim)
    out = torch.empty(n, dtype=torch.float64, device=qkv.device)
    check(_lib.load().tkv_qgemv_scores(C.byref(qkv.struct), unit, n, ptr(q), ptr(out), stream_ptr()))
    return out


def qgemv_output(weights, qkv: QuantizedLayerKV, unit: int = 0, n: int | None = None) -> torch.Tensor:
    """float64 ``w V`` [d] of one head over its quantized values
    (quantizer.py:536-558)."""
    n = qkv.n if n is None else n
    if n < 1:
        raise EmptyCacheError("output over an empty cache")
    w = _f64_vector(weights, qkv.device, "weights", n)
    lib = _lib.load()
    ws = torch.empty(int(lib.tkv_qgemv_output_workspace(C.byref(qkv.struct), n)), dtype=torch.uint8,
                     device=qkv.device)
    out = torch.empty(qkv.head_dim, dtype=torch.float64, device=qkv.device)
    check(lib.tkv_qgemv_output(C.byref(qkv.struct), unit, n, ptr(w), ptr(out), ptr(ws), stream_ptr()))
    return out
