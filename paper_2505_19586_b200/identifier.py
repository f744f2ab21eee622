"""Offline layer classification (hybridkv/identifier.py:29-187) on the GPU.

``dense_preference_score`` / ``calibrate`` run csrc/calibrate.cu: probe-query
logits against every prefill key, the exact top-k softmax mass per probe
(radix select of the k-th largest logit, ties counted exactly k times), and
the per-head mean.  ``classify_layer`` is the same host-side threshold rule.
"""

from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr, stream_ptr
from .errors import ParameterError, ShapeError
from .quantizer import as_f16


class LayerKind(str, enum.Enum):
    QUANTIZATION_FRIENDLY = "quantization_friendly"
    SPARSITY_FRIENDLY = "sparsity_friendly"


@dataclass(frozen=True)
class SparsityProbe:
    """Probe settings (identifier.py:34-55)."""

    k: int
    n_q: int = 32
    tau: float = 0.2

    def __post_init__(self) -> None:
        if self.k < 1:
            raise ParameterError(f"k must be >= 1, got {self.k}")
        if self.n_q < 1:
            raise ParameterError(f"n_q must be >= 1, got {self.n_q}")
        if not 0.0 <= self.tau <= 1.0:
            raise ParameterError(f"tau must lie in [0, 1], got {self.tau}")


@dataclass(frozen=True)
class LayerProfile:
    layer_index: int
    per_head_scores: tuple
    score: float
    label: LayerKind


def default_probe_k(seq_len: int) -> int:
    """5 % of the sequence, at least one token (identifier.py:58-60)."""
    return max(1, int(math.ceil(0.05 * seq_len)))


def head_scores(queries, keys, k: int) -> np.ndarray:
    """Dense preference of every query head: queries [hq, n_q, d] (the probe
    rows), keys [h, n, d] -> float64 [hq] (identifier.py:110-132)."""
    q, kk = as_f16(queries), as_f16(keys)
    if q.dim() != 3 or kk.dim() != 3 or q.shape[2] != kk.shape[2]:
        raise ShapeError(f"query/key shapes incompatible: {tuple(q.shape)} vs {tuple(kk.shape)}")
    hq, n_q, d = q.shape
    h, n, _ = kk.shape
    if not 1 <= k <= n:
        raise ParameterError(f"k must lie in [1, {n}], got {k}")
    lib = _lib.load()
    ws = torch.empty(int(lib.tkv_calibrate_workspace(hq, n_q, n)), dtype=torch.uint8, device=q.device)
    out = torch.empty(hq, dtype=torch.float64, device=q.device)
    check(lib.tkv_dense_preference(ptr(q), ptr(kk), hq, h, n_q, n, d, k, ptr(out), ptr(ws), stream_ptr()))
    return out.cpu().numpy()


def dense_preference_score(recent_queries, keys, k: int) -> float:
    """Mean residual mass outside each probe query's top-k (one head)."""
    rq = np.asarray(recent_queries) if not isinstance(recent_queries, torch.Tensor) else recent_queries
    kk = np.asarray(keys) if not isinstance(keys, torch.Tensor) else keys
    return float(head_scores(rq[None], kk[None], k)[0])


def classify_layer(layer_index: int, head_scores_: Sequence[float], tau: float) -> LayerProfile:
    """Mean over heads, quantization-friendly iff strictly above tau
    (identifier.py:135-150)."""
    scores = tuple(float(s) for s in head_scores_)
    if not scores:
        raise ParameterError("classify_layer needs at least one head score")
    mean = float(np.mean(scores))
    label = LayerKind.QUANTIZATION_FRIENDLY if mean > tau else LayerKind.SPARSITY_FRIENDLY
    return LayerProfile(layer_index, scores, mean, label)


def calibrate(prefill_queries, prefill_keys, probe: SparsityProbe) -> list[LayerProfile]:
    """Classify every layer from its prefill (identifier.py:153-187).

    prefill_queries: per layer [hq, n, d] (only the last n_q rows are read);
    prefill_keys: per layer [h, n, d].  No causal mask, as in the reference.
    """
    profiles = []
    for layer, (Q, K) in enumerate(zip(prefill_queries, prefill_keys)):
        n = K.shape[1]
        if n < probe.n_q:
            raise ParameterError(f"prefill length {n} is shorter than probe n_q {probe.n_q}")
        if probe.k > n:
            raise ParameterError(f"probe k {probe.k} exceeds prefill length {n}")
        recent = Q[:, Q.shape[1] - probe.n_q:, :]
        profiles.append(classify_layer(layer, head_scores(recent, K, probe.k), probe.tau))
    return profiles
