"""Offloaded (sparsity-friendly) layer: pinned NUMA-local host KV store plus
the device-resident state the Top-K path needs.

Mirrors hybridkv/memsim.py HostPool (:76-135: offload_layer, append,
channel_abs_max, gather) and DeviceBuffers/_SparseLayerState
(memsim.py:143-187, pipeline.py:183-200).  B200 design:

* host store: token-major rows ``[units][capacity][K|V][d]`` fp16 in a pinned,
  NUMA-local arena read by the GPU over PCIe (UVA zero-copy);
* device: channel-major keys ``[units][d][capacity]`` for the proxy scorer
  (channels change every step, so the reference's per-step PCIe prefetch of
  n*d_s columns, memsim.py:205-225, is replaced by a resident copy), the
  running channel max, and the append-only local window mirror.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib
from ._lib import SparseLayer, check, ptr, stream_ptr
from .errors import EmptyCacheError, ParameterError, ShapeError
from .quantizer import as_f16
from .retriever import RetrievalConfig


def gpu_numa_node(device_index: int = 0) -> int:
    """NUMA node of the GPU's PCIe root (sysfs), -1 when unknown."""
    try:
        props = torch.cuda.get_device_properties(device_index)
        bus = f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as fh:
            return int(fh.read().strip())
    except Exception:
        return -1


class PinnedArena:
    """Pinned (cudaHostRegister'ed), NUMA-bound host allocation."""

    def __init__(self, nbytes: int, numa_node: int = -1):
        lib = _lib.load()
        self.nbytes = int(nbytes)
        self.addr = lib.tkv_host_store_create(self.nbytes, numa_node)
        if not self.addr:
            raise MemoryError(lib.tkv_last_error().decode())
        self.numa_node = numa_node

    def as_tensor(self, count: int, dtype=torch.float16) -> torch.Tensor:
        ctype = {torch.float16: C.c_uint16}[dtype]
        arr = np.ctypeslib.as_array((ctype * count).from_address(self.addr))
        return torch.from_numpy(arr).view(dtype)

    def close(self):
        if self.addr:
            _lib.load().tkv_host_store_destroy(self.addr, self.nbytes)
            self.addr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class OffloadedLayerKV:
    """One sparsity-friendly layer for ``units`` KV heads (batch x heads)."""

    def __init__(self, units: int, head_dim: int, capacity: int, prefill_len: int, n_local: int,
                 keys_on_device: bool = False, numa_node: int | None = None, device=None, cache_rows: int = 0,
                 cache_window: int = 1, n_sink: int = 0):
        _lib.require_cuda()
        dev = torch.device(device or "cuda")
        self.device = dev
        capacity = (int(capacity) + 63) // 64 * 64  # 16-byte aligned channel rows for the scorer
        self.units, self.head_dim, self.capacity = units, head_dim, capacity
        self.local_offset = max(0, prefill_len - n_local)
        self.local_capacity = self.capacity - self.local_offset
        d = head_dim
        self.kt = torch.zeros((units, d, self.capacity), dtype=torch.float16, device=dev)
        self.chmax = torch.zeros((units, d), dtype=torch.float32, device=dev)
        self.loc_k = torch.zeros((units, self.local_capacity, d), dtype=torch.float16, device=dev)
        self.loc_v = torch.zeros_like(self.loc_k)
        self.kdev = torch.zeros((units, self.capacity, d), dtype=torch.float16, device=dev) if keys_on_device else None
        if numa_node is None:
            numa_node = gpu_numa_node(dev.index or 0)
        self.arena = PinnedArena(units * self.capacity * 2 * d * 2, numa_node)
        self.host_kv = self.arena.as_tensor(units * self.capacity * 2 * d).view(units, self.capacity, 2, d)
        self._len = torch.zeros(2, dtype=torch.int32, device=dev)
        self.n = 0
        # HBM row cache: (key|value) rows selected within the last `cache_window` steps stay resident
        self.cache_window = int(cache_window) if cache_rows else 0
        self.cache_slots = int(cache_rows) * max(1, self.cache_window) if cache_rows else 0
        if self.cache_slots:
            self.slot_tok = torch.full((units, self.cache_slots), -1, dtype=torch.int32, device=dev)
            self.slot_stamp = torch.full((units, self.cache_slots), -(1 << 30), dtype=torch.int32, device=dev)
            self.slot_v = torch.zeros((units, self.cache_slots, 2, d), dtype=torch.float16, device=dev)  # K|V
            self.tok_slot = torch.full((units, self.capacity), -1, dtype=torch.int32, device=dev)
            self.cache_stats = torch.zeros(2, dtype=torch.int64, device=dev)
            self.slot_hand = torch.zeros((units, _lib.MAX_PARTS), dtype=torch.int32, device=dev)
        else:
            self.slot_tok = self.slot_stamp = self.slot_v = self.tok_slot = self.cache_stats = None
            self.slot_hand = None
        self.thresh = torch.full((units, 4), float("nan"), dtype=torch.float32, device=dev)  # top-k threshold hint
        self.part_hint = torch.full((units, _lib.MAX_PARTS, 2), float("nan"), dtype=torch.float32, device=dev)
        self.s1_ready = None
        self.struct = SparseLayer(units, d, self.capacity, self.local_offset, self.local_capacity,
                                  self.kt.data_ptr(), self.chmax.data_ptr(), self.loc_k.data_ptr(),
                                  self.loc_v.data_ptr(), ptr(self.kdev), self.arena.addr,
                                  self._len.data_ptr(), self._len.data_ptr() + 4,
                                  self.cache_slots, self.cache_window, ptr(self.slot_tok), ptr(self.slot_stamp),
                                  ptr(self.slot_v), ptr(self.tok_slot), ptr(self.cache_stats), ptr(self.thresh),
                                  ptr(self.slot_hand), int(n_sink), self.part_hint.data_ptr())
        self.n_sink = int(n_sink)

    @property
    def keys_on_device(self) -> bool:
        return self.kdev is not None

    @property
    def seq_len(self) -> int:
        return self.n

    def offload(self, keys, values, stream=None) -> None:
        """HostPool.offload_layer + device mirror (memsim.py:88-93,
        pipeline.py:183-193); keys/values [units, n, d]."""
        k, v = as_f16(keys, self.device), as_f16(values, self.device)
        if k.dim() != 3 or k.shape != v.shape or k.shape[0] != self.units or k.shape[2] != self.head_dim:
            raise ShapeError(f"keys/values must be [{self.units}, n, {self.head_dim}]")
        n = k.shape[1]
        if n == 0:
            raise EmptyCacheError("cannot offload an empty cache")
        check(_lib.load().tkv_sparse_prefill(C.byref(self.struct), ptr(k), ptr(v), n, stream_ptr(stream)))
        self.n = n

    def append(self, new_keys, new_values, stream=None) -> None:
        """HostPool.append + local mirror append (memsim.py:106-111,
        pipeline.py:412-413); rows [units, d]."""
        k = new_keys if isinstance(new_keys, torch.Tensor) and new_keys.dtype == torch.float16 else as_f16(new_keys)
        v = new_values if isinstance(new_values, torch.Tensor) and new_values.dtype == torch.float16 else as_f16(new_values)
        if self.n + 1 > self.capacity:
            raise ParameterError("layer capacity exhausted")
        check(_lib.load().tkv_sparse_append(C.byref(self.struct), ptr(k), ptr(v), stream_ptr(stream)))
        self.n += 1

    def _check_sinks(self, cfg: RetrievalConfig) -> None:
        if cfg.n_sink != self.n_sink:
            raise ParameterError(f"RetrievalConfig.n_sink={cfg.n_sink} but the layer was built with n_sink={self.n_sink}")

    def set_stage1_handshake(self, enabled: bool, l2_prefetch: bool = True) -> None:
        """Device-side stage-1 handshake (tkv_sparse_layer.s1_ready): stage 1, given this layer as its
        prefetch layer, flags each unit's channels as written, and the fused cluster decode waits for the
        flag instead of a stream dependency on stage 1 (which costs a programmatic-launch overlap per
        layer).  Only for decodes that leave SMs free for stage 1.  ``l2_prefetch`` False keeps stage 1's
        scorer-column L2 prefetch off while the layer is passed for the handshake."""
        if enabled and self.s1_ready is None:
            self.s1_ready = torch.zeros(self.units, dtype=torch.int32, device=self.kt.device)
        self.struct.s1_ready = self.s1_ready.data_ptr() if enabled else None
        self.struct.s1_flags = 0 if l2_prefetch else 1

    def set_row_cache(self, enabled: bool) -> None:
        """Switch the HBM row cache on or off for later launches (a captured
        graph keeps the setting it was captured with).  Results are identical
        either way: cached rows are exact copies, and rows appended while the
        cache is off are simply not cached."""
        self.struct.cache_slots = self.cache_slots if enabled else 0

    def cache_counters(self) -> tuple[int, int]:
        """(rows served from the HBM row cache, rows fetched over PCIe) so far."""
        if self.cache_stats is None:
            return 0, 0
        a, b = self.cache_stats.tolist()
        return int(a), int(b)

    def channel_abs_max(self) -> torch.Tensor:
        """Running max|K| per (unit, channel) (memsim.py:113-116)."""
        return self.chmax

    def gather(self, unit: int, indices) -> tuple[np.ndarray, np.ndarray]:
        """Host rows of one head, in index order (memsim.py:118-127)."""
        torch.cuda.synchronize()
        idx = np.asarray(indices, dtype=np.int64).reshape(-1)
        if idx.size and (idx.min() < 0 or idx.max() >= self.n):
            raise ParameterError("gather index out of range")
        rows = self.host_kv[unit].numpy()[idx]
        return rows[:, 0].astype(np.float64), rows[:, 1].astype(np.float64)

    # -- decode-step pieces --------------------------------------------------
    def select(self, queries: torch.Tensor, channels: torch.Tensor, G: int, cfg: RetrievalConfig,
               sel_idx: torch.Tensor, sel_count: torch.Tensor, fetch_count: torch.Tensor, workspace: torch.Tensor,
               scores_out: torch.Tensor | None = None, stream=None) -> None:
        """Proxy scores with the true query + exact top-k (retriever.py:166-211)."""
        self._check_sinks(cfg)
        check(_lib.load().tkv_select_tokens(C.byref(self.struct), ptr(queries), G, ptr(channels), channels.shape[1],
                                            cfg.n_local, cfg.n_topk, ptr(sel_idx), ptr(sel_count), ptr(fetch_count),
                                            ptr(scores_out), ptr(workspace), stream_ptr(stream)))

    def decode(self, queries: torch.Tensor, channels: torch.Tensor, G: int, cfg: RetrievalConfig,
               sel_idx: torch.Tensor, sel_count: torch.Tensor, fetch_count: torch.Tensor, out: torch.Tensor,
               workspace: torch.Tensor, keys_from_device: bool = False, new_keys=None, new_values=None,
               stream=None) -> None:
        """One fused launch: proxy scores + exact top-k + gather + attention
        (pipeline.py:351-376); same results as ``select`` then ``attend``.
        With new_keys/new_values [units, d] the step's ``append`` runs in the
        same launch, after the attention."""
        self._check_sinks(cfg)
        if (new_keys is None) != (new_values is None):
            raise ParameterError("new_keys and new_values must both be given")
        if new_keys is not None and self.n + 1 > self.capacity:
            raise ParameterError("layer capacity exhausted")
        check(_lib.load().tkv_sparse_decode(C.byref(self.struct), ptr(queries), G, ptr(channels), channels.shape[1],
                                            cfg.n_local, cfg.n_topk, ptr(sel_idx), ptr(sel_count), ptr(fetch_count),
                                            int(keys_from_device), ptr(new_keys), ptr(new_values), ptr(out),
                                            ptr(workspace), stream_ptr(stream)))
        if new_keys is not None:
            self.n += 1

    def attend(self, queries: torch.Tensor, G: int, cfg: RetrievalConfig, sel_idx: torch.Tensor,
               sel_count: torch.Tensor, out: torch.Tensor, workspace: torch.Tensor, keys_from_device: bool = False,
               stream=None) -> None:
        """Gather + exact softmax attention over the selected rows
        (memsim.py:228-252, pipeline.py:364-376)."""
        check(_lib.load().tkv_sparse_attention(C.byref(self.struct), ptr(queries), G, ptr(sel_idx), ptr(sel_count),
                                               cfg.n_local, sel_idx.shape[1], int(keys_from_device), ptr(out),
                                               ptr(workspace), stream_ptr(stream)))
