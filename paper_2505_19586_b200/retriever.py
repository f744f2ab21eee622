"""Two-stage Top-K retrieval for sparsity-friendly layers, on the GPU.

Mirrors hybridkv/retriever.py: RetrievalConfig (:45-65), estimate_query +
group_channel_scores + select_critical_channels (:84-163, fused as
``select_critical_channels_gpu``), approx_scores + select_topk_tokens
(:166-211, fused as ``select_tokens_gpu``) and ``select_topk_tokens`` over
caller scores.  Semantics kept: channel ties to the lower index, token ties
to the more recent index, the local window always kept, everything selected
when ``n <= n_local + n_topk``.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr, stream_ptr
from .errors import EmptyCacheError, ParameterError, ShapeError


@dataclass(frozen=True)
class RetrievalConfig:
    """Token and channel budgets of one sparsity-friendly layer
    (retriever.py:45-65)."""

    n_local: int = 64
    n_topk: int = 128
    d_s: int = 8
    n_sink: int = 0  # extension: tokens [0, n_sink) always selected (attention sinks); 0 = the reference

    @property
    def max_selected(self) -> int:
        """Selected rows per head at most: sinks + Top-K + local window."""
        return self.n_local + self.n_topk + self.n_sink

    def __post_init__(self) -> None:
        if self.n_sink < 0:
            raise ParameterError(f"n_sink must be >= 0, got {self.n_sink}")
        if self.n_local < 0:
            raise ParameterError(f"n_local must be >= 0, got {self.n_local}")
        if self.n_topk < 1:
            raise ParameterError(f"n_topk must be >= 1, got {self.n_topk}")
        if self.d_s < 1:
            raise ParameterError(f"d_s must be >= 1, got {self.d_s}")


class _WS:
    """Grow-only device workspaces keyed by purpose (zero-initialised, as the
    selection kernels require)."""

    def __init__(self):
        self.bufs: dict[str, torch.Tensor] = {}

    def get(self, key: str, nbytes: int, device) -> torch.Tensor:
        b = self.bufs.get(key)
        if b is None or b.numel() < nbytes:
            b = torch.zeros(int(nbytes), dtype=torch.uint8, device=device)
            self.bufs[key] = b
        return b


WORKSPACES = _WS()


def stage1_select(hidden: torch.Tensor, w_q: torch.Tensor, chmax: torch.Tensor, G: int, d_s: int,
                  channels: torch.Tensor | None = None, q_hat: torch.Tensor | None = None, workspace=None,
                  stream=None, prefetch_layer=None) -> torch.Tensor:
    """q_hat = hidden . W_q then the top-d_s critical channels per unit.

    hidden fp16 [B, hidden]; w_q fp16 [hq, hidden, d]; chmax fp32 [B*hq/G, d].
    Returns int32 [units, d_s] sorted ascending (retriever.py:84-163).
    """
    B, H = hidden.shape
    hq, H2, d = w_q.shape
    if H2 != H:
        raise ShapeError(f"w_q shape {tuple(w_q.shape)} incompatible with hidden dim {H}")
    d_s = min(d_s, d)
    units = B * hq // G
    lib = _lib.load()
    if channels is None:
        channels = torch.empty((units, d_s), dtype=torch.int32, device=hidden.device)
    if workspace is None:
        # one zero-initialised workspace per shape: its arrival counters re-arm themselves, but a buffer shared
        # across shapes would put one shape's partials where another keeps its counters
        workspace = WORKSPACES.get(f"stage1:{B}:{hq}:{H}:{d}", lib.tkv_stage1_workspace(B, hq, H, d), hidden.device)
    if prefetch_layer is None:
        check(lib.tkv_stage1(ptr(hidden), ptr(w_q), B, hq, H, d, G, ptr(chmax), d_s, ptr(q_hat), ptr(channels),
                             ptr(workspace), stream_ptr(stream)))
    else:  # also start moving the chosen scorer columns of that layer into L2
        check(lib.tkv_stage1_prefetch(ptr(hidden), ptr(w_q), B, hq, H, d, G, ptr(chmax), d_s, ptr(q_hat),
                                      ptr(channels), ptr(workspace), C.byref(prefetch_layer.struct),
                                      stream_ptr(stream)))
    return channels


def select_topk_tokens(scores, config: RetrievalConfig) -> np.ndarray:
    """GPU exact top-k over caller scores [n] or [units, n]
    (retriever.py:192-211).  Returns the ascending index set (list per unit
    for 2-D input)."""
    s = torch.as_tensor(np.asarray(scores, np.float64) if not isinstance(scores, torch.Tensor) else scores)
    s = s.to(device="cuda", dtype=torch.float64).contiguous()
    one = s.dim() == 1
    if one:
        s = s[None]
    units, n = s.shape
    if n == 0:
        raise EmptyCacheError("token selection over an empty cache")
    k = config.n_local + config.n_topk
    lib = _lib.load()
    ws = WORKSPACES.get("topk", lib.tkv_select_workspace(units, n), s.device)
    ws.zero_()  # the carve-up depends on (units, n); start from a clean slate
    idx = torch.empty((units, k), dtype=torch.int32, device=s.device)
    cnt = torch.empty(units, dtype=torch.int32, device=s.device)
    check(lib.tkv_topk_from_scores(ptr(s), units, n, config.n_local, config.n_topk, ptr(idx), ptr(cnt), ptr(ws),
                                   stream_ptr()))
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    res = [idx[u, : cnt[u]].astype(np.int64) for u in range(units)]
    return res[0] if one else res
