"""Hybrid decode engine: the per-layer decode-attention calls of
hybridkv/pipeline.py:303-413 run as one stream-ordered (optionally CUDA-graph
captured) decode step on one GPU, with KV heads sharded across ranks.

Per step and layer l (pipeline.py order, attend-before-append):

* quantization-friendly: ``QuantizedLayerKV.decode`` then ``append_token``;
* sparsity-friendly: stage 1 (query estimate from hidden[l-1] + critical
  channels) runs on a side stream as soon as layer l-1 starts, like the
  reference's 1-worker prefetch executor (pipeline.py:288-313); then proxy
  scores + exact top-k, PCIe gather + sparse attention, append;
* with ``world_size > 1`` the head outputs of the layer are all-gathered
  (one NCCL all-gather per layer over NVLink).
"""

from __future__ import annotations

import os

from dataclasses import dataclass, field

import ctypes as C

import numpy as np
import torch

from .errors import ConfigError, ShapeError
from .hoststore import OffloadedLayerKV
from .identifier import LayerKind
from .kv_model import ModelConfig
from .quantizer import QuantizedLayerKV, as_f16
from .retriever import WORKSPACES, RetrievalConfig, stage1_select
from . import _lib
from ._lib import check


# timing experiments only: skip stage 1 inside the step (channels keep their last values; results are
# then not the reference's) to see what the rest of the step costs
_SKIP_STAGE1 = os.environ.get("TKV_SKIP_STAGE1") == "1"


@dataclass(frozen=True)
class EngineConfig:
    """Decode-path knobs (the subset of PipelineConfig, pipeline.py:66-111,
    that acts on the hot path) plus B200 placement options."""

    bits: int = 1
    group_size: int = 64
    n_local: int = 64
    n_topk: int = 128
    critical_channels: int = 8
    n_sink: int = 0                # extension: attention-sink tokens always selected (0 = the reference)
    keys_from_hbm: bool = True     # gather key rows from HBM; only V rows cross PCIe
    token_major_keys: bool = True  # keep a token-major HBM key copy for that gather (else read the scorer's
                                   # channel-major copy: no extra memory, 32x more DRAM sectors)
    row_cache: bool = True         # keep fetched value rows in HBM (exact; rows are immutable)
    row_cache_steps: int = 4       # a row stays cached until it has not been selected for this many steps
    fused_sparse: bool = True      # one launch per sparse layer (select + gather + attention); else two
    scorer_l2_prefetch: bool = True  # stage 1 starts moving the chosen scorer columns into L2
    overlap_stage1: bool = True    # stage 1 of layer l+1 runs on a side stream during layer l (else in line)
    stage1_handshake: bool | None = None  # decode waits for stage 1 on a device flag, not a stream edge
                                          # (None: when the fused decode leaves half the SMs free)
    quant_impl: int = 0            # 0 auto, 1 SIMT, 2 tensor-core

    def validate(self) -> None:
        if self.bits not in (1, 2):
            raise ConfigError(f"bits must be 1 or 2 on the engine path, got {self.bits}")
        if self.n_local < 0 or self.n_topk < 1 or self.critical_channels < 1 or self.n_sink < 0:
            raise ConfigError("token/channel budgets out of range")


@dataclass(frozen=True)
class ShardSlice:
    """The (sequence, KV head) block one rank owns."""

    b0: int
    batch: int
    k0: int
    kv_heads: int


def shard_plan(batch: int, num_kv_heads: int, world_size: int) -> list[ShardSlice]:
    """Split the batch x kv-head units evenly over ranks:
    heads are split inside a sequence when a rank owns fewer units than a
    sequence has heads, otherwise whole sequences are assigned."""
    units = batch * num_kv_heads
    if units % world_size:
        raise ConfigError(f"{units} (batch x kv heads) units do not split over {world_size} ranks")
    per = units // world_size
    plan = []
    for r in range(world_size):
        if per <= num_kv_heads:
            if num_kv_heads % per:
                raise ConfigError(f"{per} units per rank do not tile {num_kv_heads} kv heads")
            plan.append(ShardSlice(b0=(r * per) // num_kv_heads, batch=1, k0=(r * per) % num_kv_heads, kv_heads=per))
        else:
            if per % num_kv_heads:
                raise ConfigError(f"{per} units per rank are not whole sequences of {num_kv_heads} heads")
            nb = per // num_kv_heads
            plan.append(ShardSlice(b0=r * nb, batch=nb, k0=0, kv_heads=num_kv_heads))
    return plan


def assemble(gathered: list[torch.Tensor], plan: list[ShardSlice], batch: int, num_kv_heads: int) -> torch.Tensor:
    """Per-rank outputs [B_r, h_r*G, d] -> full [batch, hq, d]."""
    G = gathered[0].shape[1] // plan[0].kv_heads
    d = gathered[0].shape[2]
    out = gathered[0].new_empty((batch, num_kv_heads * G, d))
    for s, t in zip(plan, gathered):
        out[s.b0:s.b0 + s.batch, s.k0 * G:(s.k0 + s.kv_heads) * G] = t.reshape(s.batch, s.kv_heads * G, d)
    return out


def slice_step_input(x, shard: ShardSlice, batch: int, num_kv_heads: int, heads_per_unit: int, world: int):
    """A rank's part of one step input [L, B, ...].  Full inputs are
    recognised per dimension: the batch slice applies when dim 1 holds the
    whole batch, the head slice when dim 2 holds every head
    (``heads_per_unit`` heads per KV head; 0 = no head dimension), so an
    already-sharded [L, 1, h_r, d] input of a head-split batch-1 rank is
    left alone."""
    if world > 1:
        if x.shape[1] == batch:
            x = x[:, shard.b0:shard.b0 + shard.batch]
        if heads_per_unit and x.dim() > 2 and x.shape[2] == num_kv_heads * heads_per_unit:
            x = x[:, :, shard.k0 * heads_per_unit:(shard.k0 + shard.kv_heads) * heads_per_unit]
    return x


def _label(x) -> str:
    v = x.value if isinstance(x, LayerKind) else str(x)
    if v in ("q", LayerKind.QUANTIZATION_FRIENDLY.value):
        return "q"
    if v in ("s", LayerKind.SPARSITY_FRIENDLY.value):
        return "s"
    raise ConfigError(f"unknown layer label {x!r}")


class _PriorityGraph:
    """A captured decode step instantiated by the library with per-node launch
    priorities (cudaGraphInstantiateFlagUseNodePriority): the attention chain
    is dispatched ahead of the next layer's stage 1 when both are ready.  The
    torch graph object is kept alive: it owns the captured graph and the
    memory pool of its allocations."""

    def __init__(self, torch_graph: torch.cuda.CUDAGraph):
        self.torch_graph = torch_graph
        exe = C.c_void_p()
        check(_lib.load().tkv_graph_instantiate(C.c_void_p(torch_graph.raw_cuda_graph()), C.byref(exe)))
        self.exec = exe

    def replay(self) -> None:
        check(_lib.load().tkv_graph_launch(self.exec, C.c_void_p(torch.cuda.current_stream().cuda_stream)))

    def __del__(self):
        try:
            if self.exec:
                _lib.load().tkv_graph_destroy(self.exec)
        except Exception:
            pass


@dataclass
class _SparseState:
    layer: OffloadedLayerKV
    w_q: torch.Tensor          # [hq_r, hidden, d] fp16
    channels: torch.Tensor     # [units, d_s] int32
    s1_ws: torch.Tensor
    s1_done: torch.cuda.Event = field(default_factory=lambda: torch.cuda.Event())


class DecodeEngine:
    """All layers of one model replica shard on one GPU."""

    def __init__(self, model: ModelConfig, labels, config: EngineConfig, batch: int = 1, max_steps: int = 64,
                 rank: int = 0, world_size: int = 1, process_group=None, device=None):
        _lib.require_cuda()
        config.validate()
        self.model, self.cfg = model, config
        self.labels = [_label(x) for x in labels]
        if len(self.labels) != model.num_layers:
            raise ConfigError("one label per layer is required")
        self.batch, self.max_steps = batch, max_steps
        self.rank, self.world = rank, world_size
        self.group = process_group
        self.plan = shard_plan(batch, model.num_kv_heads, world_size)
        self._host_collective = False
        # process_group == "none": rank `rank`'s share of a world_size-GPU run without the collective
        # (bench.py --shard-of: per-GPU work of a multi-GPU configuration measured on one GPU)
        self._no_collective = process_group == "none"
        if self._no_collective:
            self.group = None
        elif world_size > 1:
            import torch.distributed as dist

            self._host_collective = dist.get_backend(process_group) != "nccl"
        self.shard = self.plan[rank]
        self.G = model.queries_per_kv_head
        self.units = self.shard.batch * self.shard.kv_heads
        self.hq_r = self.shard.kv_heads * self.G
        self.d = model.head_dim
        self.device = torch.device(device or "cuda")
        self.retrieval = RetrievalConfig(config.n_local, config.n_topk, min(config.critical_channels, self.d),
                                         config.n_sink)
        self.layers: list = [None] * model.num_layers
        self.sparse: dict[int, _SparseState] = {}
        self.prefill_len = None
        self.side = torch.cuda.Stream(device=self.device)
        L, U, d = model.num_layers, self.units, self.d
        kmax = self.retrieval.max_selected
        dev = self.device
        # static per-step buffers (graph inputs/outputs)
        self.hidden = torch.zeros((L, self.shard.batch, model.hidden_dim), dtype=torch.float16, device=dev)
        self.queries = torch.zeros((L, U * self.G, d), dtype=torch.float16, device=dev)
        self.new_keys = torch.zeros((L, U, d), dtype=torch.float16, device=dev)
        self.new_values = torch.zeros((L, U, d), dtype=torch.float16, device=dev)
        self.out = torch.zeros((L, U * self.G, d), dtype=torch.float32, device=dev)
        self.gathered = (torch.zeros((L, world_size, U * self.G, d), dtype=torch.float32, device=dev)
                         if world_size > 1 else None)
        self.sel_idx = torch.zeros((U, kmax), dtype=torch.int32, device=dev)
        self.sel_count = torch.zeros(U, dtype=torch.int32, device=dev)
        self.fetch_count = torch.zeros(U, dtype=torch.int32, device=dev)
        lib = _lib.load()
        self.attn_ws = torch.zeros(int(lib.tkv_sparse_attn_workspace(U, self.G, d, kmax)), dtype=torch.uint8, device=dev)
        self.sel_ws = self.dec_ws = None
        self.graph = None
        self.steps_done = 0
        self.record_selection = False
        self.profile = None  # list of (name, layer, start_event, end_event) when profiling
        self._event_pool = None
        self.prof_graph = None
        self.keys_from_hbm = config.keys_from_hbm
        self._s1_sync = None  # decided at the first sparse prefill (stage-1 handshake on/off)
        self.last_channels: dict[int, torch.Tensor] = {}
        self.last_selection: dict[int, tuple] = {}
        # host I/O inside the captured step (capture(host_io=True)): pinned staging for the step inputs and
        # outputs, copied by the graph on its own stream, overlapped with the layers
        self._host_io = False
        self._io_capture = None  # capture-time state while capturing with host I/O
        self.io = None
        # two staging sets, each with its own captured graph, used alternately: the host fills set k % 2
        # while the graph of the previous step (the other set) runs
        self._hio_sets = None    # [(inputs (hidden, queries, new_keys, new_values) pinned, outputs pinned)] x 2
        self._hio_graphs = None
        self._hio_done = None    # per set: host-recorded event after its last replay
        self._hio_next = 0
        self.host_inputs = None  # the staging set being captured / filled
        self.host_out = None     # the pinned output of the last step_host

    # -- prefill ---------------------------------------------------------------
    def _slice_kv(self, x):
        """[B, h, n, d] (full) or [B_r, h_r, n, d] (already sharded) -> units."""
        x = as_f16(x, self.device)
        s = self.shard
        if x.dim() == 3:
            x = x[None]
        if x.shape[0] == self.batch and x.shape[1] == self.model.num_kv_heads and (self.world > 1):
            x = x[s.b0:s.b0 + s.batch, s.k0:s.k0 + s.kv_heads]
        if x.shape[0] != s.batch or x.shape[1] != s.kv_heads:
            raise ShapeError(f"prefill K/V must be [{self.batch}, {self.model.num_kv_heads}, n, d]")
        return x.reshape(self.units, x.shape[2], x.shape[3]).contiguous()

    def prefill(self, layer: int, keys, values, w_q=None) -> None:
        """Compress (Q layer, quantize_layer_kv) or offload (S layer,
        HostPool.offload_layer) one layer's prefill cache."""
        k, v = self._slice_kv(keys), self._slice_kv(values)
        n = k.shape[1]
        if self.prefill_len is None:
            self.prefill_len = n
        cap = n + self.max_steps
        if self.labels[layer] == "q":
            self.layers[layer] = QuantizedLayerKV.from_kv(k, v, self.cfg.bits, self.cfg.group_size, capacity=cap)
            self.layers[layer].workspace(self.G)  # allocate before any graph capture
        else:
            if w_q is None:
                raise ConfigError(f"sparsity-friendly layer {layer} needs its W_q for stage 1")
            lay = OffloadedLayerKV(self.units, self.d, cap, n, self.retrieval.n_local,
                                   keys_on_device=self.cfg.keys_from_hbm and self.cfg.token_major_keys,
                                   device=self.device,
                                   cache_rows=self.retrieval.max_selected if self.cfg.row_cache else 0,
                                   cache_window=self.cfg.row_cache_steps, n_sink=self.retrieval.n_sink)
            lay.offload(k, v)
            w = as_f16(w_q, self.device)
            if w.shape[0] == self.model.num_query_heads:
                w = w[self.shard.k0 * self.G:(self.shard.k0 + self.shard.kv_heads) * self.G]
            w = w.contiguous()
            lib = _lib.load()
            ws = torch.zeros(int(lib.tkv_stage1_workspace(self.shard.batch, self.hq_r, w.shape[1], self.d)),
                             dtype=torch.uint8, device=self.device)
            chans = torch.zeros((self.units, self.retrieval.d_s), dtype=torch.int32, device=self.device)
            self.sparse[layer] = _SparseState(lay, w, chans, ws)
            self.layers[layer] = lay
            if self._s1_sync is None:
                self._s1_sync = self._stage1_handshake_ok(lay)
            lay.set_stage1_handshake(self._s1_sync, l2_prefetch=self.cfg.scorer_l2_prefetch)
            # workspaces follow the largest layer capacity seen so far (prefill lengths may differ per layer)
            kmax = self.retrieval.max_selected
            need_sel = int(lib.tkv_select_workspace(self.units, lay.capacity))
            need_dec = int(lib.tkv_sparse_decode_workspace(self.units, lay.capacity, self.G, self.d, kmax))
            if self.sel_ws is None or self.sel_ws.numel() < need_sel:
                self.sel_ws = torch.zeros(need_sel, dtype=torch.uint8, device=self.device)
            if self.dec_ws is None or self.dec_ws.numel() < need_dec:
                self.dec_ws = torch.zeros(need_dec, dtype=torch.uint8, device=self.device)
        self.graph = self.prof_graph = None  # a captured step holds the old buffers: capture again
        self._hio_graphs = None

    def _stage1_handshake_ok(self, lay) -> bool:
        """The decode may wait for stage 1 on a device flag when stage 1 is overlapped and the fused
        cluster decode leaves at least half of the SMs free (stage 1 then always finds room to run)."""
        c = self.cfg
        if c.stage1_handshake is not None:
            return bool(c.stage1_handshake) and c.fused_sparse and c.overlap_stage1
        if not (c.fused_sparse and c.overlap_stage1):
            return False
        plan = int(_lib.load().tkv_sparse_decode_plan(C.byref(lay.struct), self.G, self.retrieval.d_s,
                                                      self.retrieval.n_local, int(self.keys_from_hbm)))
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        return plan > 0 and self.units * plan <= sms // 2

    # -- one step --------------------------------------------------------------
    def load_step(self, hidden, queries, new_keys, new_values, non_blocking: bool = True) -> None:
        """Copy one step's inputs into the static buffers.  Shapes (full or
        rank slice): hidden [L, B, hidden], queries [L, B, hq, d],
        new_keys/new_values [L, B, h, d]."""
        def sl(x, heads_per_unit):
            if not isinstance(x, torch.Tensor):  # numpy / array-like step inputs (fp16 storage)
                x = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float16)))
            return slice_step_input(x, self.shard, self.batch, self.model.num_kv_heads, heads_per_unit, self.world)

        self.hidden.copy_(sl(hidden, 0).reshape(self.hidden.shape), non_blocking=non_blocking)
        self.queries.copy_(sl(queries, self.G).reshape(self.queries.shape), non_blocking=non_blocking)
        self.new_keys.copy_(sl(new_keys, 1).reshape(self.new_keys.shape), non_blocking=non_blocking)
        self.new_values.copy_(sl(new_values, 1).reshape(self.new_values.shape), non_blocking=non_blocking)

    def _stage1(self, l: int) -> None:
        st = self.sparse[l]
        src = l - 1 if l >= 1 else 0  # pipeline.py:273
        t0 = self._mark(self.side)
        if not _SKIP_STAGE1:
            # the layer goes to stage 1 for its L2 prefetch and/or the handshake flags (s1_flags says which)
            stage1_select(self.hidden[src], st.w_q, st.layer.chmax, self.G, self.retrieval.d_s,
                          channels=st.channels, workspace=st.s1_ws, stream=self.side,
                          prefetch_layer=st.layer if (self.cfg.scorer_l2_prefetch or self._s1_sync) else None)
        self._span("stage1", l, t0, self.side)
        st.s1_done.record(self.side)

    def _mark(self, stream):
        if self.profile is None:
            return None
        if self._event_pool is not None:  # inside a profiled capture: an event-record node of the graph
            ev = self._event_pool.pop()
            check(_lib.load().tkv_event_record(C.c_void_p(ev.cuda_event), C.c_void_p(stream.cuda_stream), 1))
            return ev
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        return ev

    def _span(self, name, layer, start, stream):
        if self.profile is not None:
            self.profile.append((name, layer, start, self._mark(stream)))

    def kernels_per_step(self) -> int:
        """Launches of this library per decode step."""
        q = sum(1 for x in self.labels if x == "q")
        s = len(self.labels) - q
        per_s = 2 if self.cfg.fused_sparse else 4  # stage 1 + (fused decode+append | select + gather/attend + append)
        # q: decode + append; the SIMT and per-chunk tensor-core kernels add a combine launch (the pipelined
        # tensor-core kernel merges its splits in its last CTA)
        pipe = (self.cfg.quant_impl in (0, 2) and self.model.head_dim == 128 and self.cfg.group_size == 64
                and self.cfg.bits in (1, 2) and self.G <= 16)
        return q * (2 if pipe else 3) + s * per_s

    def _io_inputs(self, main) -> None:
        """Host I/O capture: copy the staged inputs on the io stream in two phases -- the first two layers'
        slices (needed at once), then the rest, which lands while those two run -- each ending in an event
        the consumers wait on."""
        L = self.model.num_layers
        A = min(L, 2)
        fork = torch.cuda.Event()
        fork.record(main)
        self.io.wait_event(fork)
        evs = []
        with torch.cuda.stream(self.io):
            for lo, hi in ((0, A), (A, L)):
                if lo >= hi:
                    continue
                for dst, src in zip((self.hidden, self.queries, self.new_keys, self.new_values), self.host_inputs):
                    dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.io)
                evs.append((hi, ev))
        self._io_capture = {"evs": evs, "waited": set()}

    def _io_wait(self, stream, layer: int) -> None:
        """Make `stream` wait until layer `layer`'s inputs are on the device (host I/O capture only)."""
        st = self._io_capture
        if st is None:
            return
        for i, (hi, ev) in enumerate(st["evs"]):
            if layer < hi:
                if (id(stream), i) not in st["waited"]:
                    stream.wait_event(ev)
                    st["waited"].add((id(stream), i))
                return

    def _io_output(self, main, l: int) -> None:
        """Host I/O capture: copy the outputs back on the io stream in two pieces -- every layer but the last
        L/8 once those are done (overlapped with the rest of the step), then the tail at the end.  (One copy
        per layer costs more than it hides: each extra dependency on a layer's kernel breaks the programmatic
        launch overlap with the next one.)"""
        if self._io_capture is None:
            return
        L = self.model.num_layers
        tail = max(1, L // 8)
        if l == L - 1:
            lo = L - tail if L > tail else 0
        elif l == L - tail - 1:
            lo = 0
        else:
            return
        done = torch.cuda.Event()
        done.record(main)
        self.io.wait_event(done)
        with torch.cuda.stream(self.io):
            self.host_out[lo:l + 1].copy_(self.out[lo:l + 1], non_blocking=True)

    def _recheck_handshake(self) -> None:
        """The dispatch can change after prefill (set_sparse_kernel / TKV_WIDE): keep the stage-1 handshake
        only while the fused cluster decode still runs (the wide decode neither waits nor re-arms)."""
        if self._s1_sync and self.sparse:
            lay = next(iter(self.sparse.values())).layer
            if not self._stage1_handshake_ok(lay) and self.cfg.stage1_handshake is None:
                self._s1_sync = False
                for st in self.sparse.values():
                    st.layer.set_stage1_handshake(False, l2_prefetch=self.cfg.scorer_l2_prefetch)

    def _run_step(self) -> None:
        self._recheck_handshake()
        main = torch.cuda.current_stream(self.device)
        L = self.model.num_layers
        if self._io_capture is not None:
            self._io_inputs(main)
        begin = [torch.cuda.Event() for _ in range(L)]
        for l in range(L):
            self._io_wait(main, l)
            begin[l].record(main)
            nxt = [j for j in ((0, 1) if l == 0 else (l + 1,)) if j < L and self.labels[j] == "s"]
            if not self.cfg.overlap_stage1:
                nxt = [l] if self.labels[l] == "s" else []
            for j in nxt:
                self.side.wait_event(begin[l])
                self._io_wait(self.side, max(j - 1, 0))  # stage 1 of layer j reads hidden[j - 1]
                with torch.cuda.stream(self.side):
                    self._stage1(j)
            lay = self.layers[l]
            if self.labels[l] == "q":
                t0 = self._mark(main)
                lay.decode(self.queries[l], out=self.out[l], impl=self.cfg.quant_impl)
                self._span("quant_decode", l, t0, main)
                # attend, then append (pipeline.py:405-413): the append only has to land before
                # this layer's next decode, so it runs on the side stream, off the layer chain
                done = torch.cuda.Event()
                done.record(main)
                self.side.wait_event(done)
                with torch.cuda.stream(self.side):
                    t0 = self._mark(self.side)
                    lay.append_token(self.new_keys[l], self.new_values[l])
                    self._span("quant_append", l, t0, self.side)
            else:
                st = self.sparse[l]
                if not self._s1_sync:  # (with the handshake the decode waits on the device flag)
                    main.wait_event(st.s1_done)
                if self.cfg.fused_sparse:
                    t0 = self._mark(main)
                    lay.decode(self.queries[l], st.channels, self.G, self.retrieval, self.sel_idx, self.sel_count,
                               self.fetch_count, self.out[l], self.dec_ws, keys_from_device=self.keys_from_hbm,
                               new_keys=self.new_keys[l], new_values=self.new_values[l])
                    self._span("sparse_decode", l, t0, main)
                else:
                    t0 = self._mark(main)
                    lay.select(self.queries[l], st.channels, self.G, self.retrieval, self.sel_idx, self.sel_count,
                               self.fetch_count, self.sel_ws)
                    self._span("select", l, t0, main)
                    t0 = self._mark(main)
                    lay.attend(self.queries[l], self.G, self.retrieval, self.sel_idx, self.sel_count, self.out[l],
                               self.attn_ws, keys_from_device=self.keys_from_hbm)
                    self._span("gather_attend", l, t0, main)
                if self.record_selection:
                    self.last_channels[l] = st.channels.clone()
                    self.last_selection[l] = (self.sel_idx.clone(), self.sel_count.clone(), self.fetch_count.clone())
                if not self.cfg.fused_sparse:
                    t0 = self._mark(main)
                    lay.append(self.new_keys[l], self.new_values[l])
                    self._span("sparse_append", l, t0, main)
            if self.world > 1 and not self._no_collective:
                self._all_gather(l)
            self._io_output(main, l)
        main.wait_stream(self.side)
        if self._io_capture is not None:
            main.wait_stream(self.io)

    def _all_gather(self, l: int) -> None:
        """The layer's one exchange: head outputs of every rank.
        NCCL gathers device buffers in stream order (capturable); a host
        backend (gloo: the multi-process tests that share one GPU) stages
        through host memory and cannot be captured."""
        import torch.distributed as dist

        if not self._host_collective:
            dist.all_gather_into_tensor(self.gathered[l], self.out[l], group=self.group)
            return
        if torch.cuda.is_current_stream_capturing():
            raise ConfigError("a host-staged (gloo) all-gather cannot be captured in a CUDA graph")
        parts = [torch.empty(self.out[l].shape, dtype=self.out[l].dtype) for _ in range(self.world)]
        dist.all_gather(parts, self.out[l].cpu(), group=self.group)
        self.gathered[l].copy_(torch.stack(parts))

    def step(self, hidden=None, queries=None, new_keys=None, new_values=None) -> torch.Tensor:
        """Run one decode step; returns this rank's outputs [L, units*G, d]
        (fp32, device).  With inputs None the static buffers are used."""
        if hidden is not None:
            if self._host_io and self._hio_graphs is not None:
                self._stage_inputs(hidden, queries, new_keys, new_values)
            else:
                self.load_step(hidden, queries, new_keys, new_values)
        elif self._host_io and self._hio_graphs is not None:
            raise ConfigError("the host-I/O graph takes its inputs from the host: pass them (step_host)")
        if self.steps_done >= self.max_steps:
            raise ConfigError("engine max_steps exhausted")
        if self._host_io and self._hio_graphs is not None and hidden is not None:
            i = self._hio_next
            self._hio_graphs[i].replay()
            self._hio_done[i].record(torch.cuda.current_stream(self.device))
            self.host_out = self._hio_sets[i][1]
            self._hio_next = 1 - i
            for lay in self.layers:
                lay.n += 1
            self.steps_done += 1
        elif self.graph is not None:
            self.graph.replay()
            for lay in self.layers:
                lay.n += 1
            self.steps_done += 1
        else:
            self._run_step()
            self.steps_done += 1
        return self.out

    def _stage_inputs(self, hidden, queries, new_keys, new_values) -> None:
        """Write one step's host inputs (full or rank slice, as load_step) into the next staging set, once
        that set's previous replay (two steps back) has finished."""
        i = self._hio_next
        self._hio_done[i].synchronize()

        def sl(x, heads_per_unit):
            if not isinstance(x, torch.Tensor):
                x = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float16)))
            return slice_step_input(x, self.shard, self.batch, self.model.num_kv_heads, heads_per_unit, self.world)

        for dst, x, hpu in zip(self._hio_sets[i][0], (hidden, queries, new_keys, new_values), (0, self.G, 1, 1)):
            dst.copy_(sl(x, hpu).reshape(dst.shape))

    def step_host(self, hidden, queries, new_keys, new_values) -> torch.Tensor:
        """One decode step with host inputs and host outputs through the host-I/O graph
        (``capture(host_io=True)``): the inputs are staged in pinned memory, the graph copies them in
        (the first two layers' slices first) and the outputs back (all but the last L/8 layers as soon as
        those are done), on a copy stream beside the layers.  Two staging sets alternate, so the host fills
        the next step's inputs while this one runs.  Returns this step's pinned host output
        [L, units*G, d] (fp32), complete once the stream has reached the end of the step and valid until
        the step after next."""
        if not (self._host_io and self._hio_graphs is not None):
            raise ConfigError("step_host needs capture(host_io=True)")
        self.step(hidden, queries, new_keys, new_values)
        return self.host_out

    def step_profiled(self, hidden=None, queries=None, new_keys=None, new_values=None) -> dict:
        """One eager step with CUDA events around every kernel group; returns
        {name: [ms per launch]} (used by bench.py for the roofline)."""
        if hidden is not None:
            self.load_step(hidden, queries, new_keys, new_values)
        self.profile = []
        self._run_step()
        self.steps_done += 1
        torch.cuda.synchronize()
        res: dict = {}
        for name, layer, a, b in self.profile:
            res.setdefault(name, []).append(a.elapsed_time(b))
        self.profile = None
        return res

    def capture(self, host_io: bool = False) -> None:
        """Capture one decode step in a CUDA graph; ``step`` then replays it.
        Capturing executes nothing, so the caches do not advance; the host
        mirrors of the token counts are restored afterwards.  With
        ``host_io`` the graph also copies the step's inputs in from pinned
        host staging and its outputs back to pinned host memory
        (``step_host``)."""
        if self._host_collective:
            raise ConfigError("capture needs the nccl backend (the gloo all-gather is host-staged)")
        saved = [lay.n for lay in self.layers]
        torch.cuda.synchronize()

        def one(io_set):
            g = torch.cuda.CUDAGraph(keep_graph=True)
            self._io_capture = {} if io_set is not None else None
            if io_set is not None:
                self.host_inputs, self.host_out = io_set
            try:
                with torch.cuda.graph(g):
                    self._run_step()
            finally:
                self._io_capture = None
            for lay, n in zip(self.layers, saved):
                lay.n = n
            return _PriorityGraph(g)

        if host_io:
            if self._hio_sets is None:
                self._hio_sets = [(tuple(torch.empty(x.shape, dtype=x.dtype).pin_memory()
                                         for x in (self.hidden, self.queries, self.new_keys, self.new_values)),
                                   torch.empty(self.out.shape, dtype=self.out.dtype).pin_memory()) for _ in range(2)]
                self.io = torch.cuda.Stream(device=self.device)
                self._hio_done = [torch.cuda.Event(), torch.cuda.Event()]
            self._hio_graphs = [one(st) for st in self._hio_sets]
            self._hio_next = 0
            self.graph = self._hio_graphs[0]
        else:
            self._hio_graphs = None
            self.graph = one(None)
        self._host_io = host_io

    def capture_profiled(self) -> None:
        """Capture the decode step with an event-record node around every
        kernel group (cudaEventRecordExternal); ``replay_profiled`` then times
        the kernels inside a real graph replay, without host launch gaps."""
        L = self.model.num_layers
        pool = [torch.cuda.Event(enable_timing=True) for _ in range(8 * L + 8)]
        for ev in pool:
            ev.record()  # materialise the CUDA events outside the capture
        torch.cuda.synchronize()
        saved = [lay.n for lay in self.layers]
        self._event_pool, self.profile = pool, []
        g = torch.cuda.CUDAGraph(keep_graph=True)
        try:
            with torch.cuda.graph(g):
                self._run_step()
        finally:
            self._event_pool = None
        self._prof_spans, self.profile = self.profile, None
        for lay, n in zip(self.layers, saved):
            lay.n = n
        self.prof_graph = _PriorityGraph(g)

    def replay_profiled(self) -> dict:
        """One step through the profiled graph; returns {name: [ms per launch]}."""
        if self.steps_done >= self.max_steps:
            raise ConfigError("engine max_steps exhausted")
        self.prof_graph.replay()
        for lay in self.layers:
            lay.n += 1
        self.steps_done += 1
        torch.cuda.synchronize()
        res: dict = {}
        for name, layer, a, b in self._prof_spans:
            res.setdefault(name, []).append(a.elapsed_time(b))
        return res

    def layer_fidelity(self, l: int) -> dict:
        """Recall, selected mass, cosine and max-abs error of sparse layer l's
        last eager step against exact attention (pipeline.py:316-325,
        377-403), computed on the GPU.  Needs ``record_selection``."""
        from .fidelity import sparse_layer_fidelity

        if self.labels[l] != "s":
            raise ConfigError("fidelity metrics are defined for sparsity-friendly layers")
        if l not in self.last_selection:
            raise ConfigError("run an eager step with record_selection = True first")
        idx, cnt, _ = self.last_selection[l]
        lay = self.layers[l]
        return sparse_layer_fidelity(lay, self.queries[l], self.G, lay.n - 1, idx, cnt, self.retrieval.n_topk,
                                     self.out[l])

    def set_row_cache(self, enabled: bool) -> None:
        """Row cache on/off for every sparse layer; the step must be captured
        again (``capture``) for a graph to pick it up."""
        for st in self.sparse.values():
            st.layer.set_row_cache(enabled)
        self.graph = self.prof_graph = None

    def resident_bytes(self) -> dict:
        """Bytes this rank keeps resident, by structure: HBM (quantized caches,
        scorer keys, token-major key copy, row cache, local windows, W_q,
        workspaces) and pinned host memory (the offloaded K/V store)."""
        def nb(t):
            return 0 if t is None else t.numel() * t.element_size()

        q = sum(sum(nb(b) for b in self.layers[l]._bufs) for l in range(len(self.labels)) if self.labels[l] == "q")
        kt = kdev = cache = loc = wq = host = other = 0
        for st in self.sparse.values():
            lay = st.layer
            kt += nb(lay.kt)
            kdev += nb(lay.kdev)
            cache += sum(nb(x) for x in (lay.slot_tok, lay.slot_stamp, lay.slot_v, lay.tok_slot, lay.slot_hand))
            loc += nb(lay.loc_k) + nb(lay.loc_v)
            wq += nb(st.w_q)
            other += nb(lay.chmax) + nb(st.s1_ws) + nb(lay.thresh)
            host += lay.arena.nbytes
        ws = nb(self.sel_ws) + nb(self.dec_ws) + nb(self.attn_ws)
        ws += sum(sum(nb(w) for w in self.layers[l]._ws.values()) for l in range(len(self.labels)) if self.labels[l] == "q")
        hbm = {"quantized_caches": q, "scorer_keys_channel_major": kt, "token_major_key_copy": kdev,
               "row_cache": cache, "local_windows": loc, "w_q": wq, "workspaces_and_small": ws + other}
        return {"hbm": hbm, "hbm_total": sum(hbm.values()), "pinned_host_kv": host}

    def cache_counters(self) -> tuple[int, int]:
        """Summed (HBM-cache hits, PCIe-fetched rows) over the sparse layers."""
        h = m = 0
        for st in self.sparse.values():
            a, b = st.layer.cache_counters()
            h += a
            m += b
        return h, m

    def full_output(self, l: int) -> torch.Tensor:
        """Layer output [batch, hq, d] (all ranks' heads)."""
        if self.world == 1:
            return self.out[l].reshape(self.batch, self.model.num_query_heads, self.d)
        parts = [self.gathered[l][r].reshape(s.batch, s.kv_heads * self.G, self.d) for r, s in enumerate(self.plan)]
        return assemble(parts, self.plan, self.batch, self.model.num_kv_heads)
