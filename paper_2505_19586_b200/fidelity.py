"""Per-step fidelity metrics of a sparsity-friendly layer on the GPU: the
comparison ``run_pipeline`` makes against its float64 exact oracle
(hybridkv/pipeline.py:316-325, 377-403), without the oracle.

* ``recall``: recall@k of the engine's selection against the exact top-k
  tokens of the group-summed attention weights (retriever.py:229-252);
* ``selected_mass``: attention mass of the selection (pipeline.py:385);
* ``cosine`` and ``max_abs_err`` of the engine's layer output against exact
  attention over every token (pipeline.py:143-150, 400-401).
Per-KV-head values are averaged like the reference (pipeline.py:392-393).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import check, ptr, stream_ptr
from .hoststore import OffloadedLayerKV


def sparse_layer_fidelity(layer: OffloadedLayerKV, queries: torch.Tensor, G: int, n: int, sel_idx: torch.Tensor,
                          sel_count: torch.Tensor, n_topk: int, out: torch.Tensor, stream=None) -> dict:
    """Metrics of one step whose cache held ``n`` tokens (before its append).
    queries fp16 [units*G, d]; sel_idx/sel_count as written by the decode;
    out fp32 [units*G, d], the engine's output for the step."""
    lib = _lib.load()
    units = layer.units
    ws = torch.empty(int(lib.tkv_sparse_fidelity_workspace(units, G, n, n_topk)), dtype=torch.uint8,
                     device=layer.device)
    exact = torch.empty((units * G, layer.head_dim), dtype=torch.float32, device=layer.device)
    metrics = torch.empty((units, 2), dtype=torch.float64, device=layer.device)
    check(lib.tkv_sparse_fidelity(C.byref(layer.struct), ptr(queries), G, n, ptr(sel_idx), ptr(sel_count),
                                  sel_idx.shape[1], n_topk, ptr(exact), ptr(metrics), ptr(ws), stream_ptr(stream)))
    o = out.reshape(units * G, -1).double()
    e = exact.double()
    na, nb = o.norm(), e.norm()
    cos = 1.0 if (na == 0 and nb == 0) else (0.0 if (na == 0 or nb == 0) else float((o * e).sum() / (na * nb)))
    m = metrics.cpu()
    return {
        "recall": float(m[:, 0].mean()),
        "selected_mass": float(m[:, 1].mean()),
        "cosine": cos,
        "max_abs_err": float((o - e).abs().max()),
        "per_head_recall": m[:, 0].tolist(),
        "exact_out": exact,
    }
