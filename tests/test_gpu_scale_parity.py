"""GPU parity at the BASELINE configs' full scale (not reduced contexts).

* config 2 sparse layers: 131,072 tokens, several decode steps with the HBM row
  cache (W = 4) and the previous-step threshold hint both active, checked
  against the oracle replay (``pipeline.py:303-413``) at EVERY step: stage-1
  channel sets, Top-K selections (exact, reference tie rule,
  ``retriever.py:192-211``), fetch counts (``pipeline.py:357``) and outputs;
* config 2 quantized layers: exactly 131,072 tokens x 8 KV heads, b = 1 and 2,
  against the float64 oracle of ``quantizer.py:505-558`` / ``pipeline.py:327-337``;
* config 3: 32k context, batch 16, 2-bit quantized layer + Top-K 3 %, every
  sequence against its own oracle replay.

Tolerances: index sets exact, outputs rel-err <= 2e-3 (north_star).
"""

import numpy as np
import pytest
import torch

import cases
from oracle import tailorkv_oracle as O

pytestmark = pytest.mark.gpu
REL_TOL = 2e-3


def rel_err(out, ref):
    out = np.asarray(out, np.float64).reshape(ref.shape[0], -1)
    ref = np.asarray(ref, np.float64).reshape(ref.shape[0], -1)
    return float(max(np.linalg.norm(o - r) / max(np.linalg.norm(r), 1e-30) for o, r in zip(out, ref)))


@pytest.fixture(scope="module")
def tkv():
    import paper_2505_19586_b200 as P

    return P


def _run_and_check(tkv, w, hq, h, d, bits, B, n_topk, T, graph_from=None):
    """Run the engine over T steps -- eagerly with the selections recorded,
    then (from step ``graph_from``) by replaying the captured CUDA graph, where
    the static selection buffers hold the last layer's selection -- and
    compare every sequence with the oracle replay."""
    L = len(w.labels)
    cfg = tkv.EngineConfig(bits=bits, n_local=64, n_topk=n_topk, critical_channels=8)
    eng = tkv.DecodeEngine(tkv.ModelConfig(L, hq, h, d, hq * d), w.labels, cfg, batch=B, max_steps=T)
    for l in range(L):
        eng.prefill(l, w.prefill_keys[l], w.prefill_values[l], w.w_q[l])
    eng.record_selection = True
    outs, sels, chans = [], [], []
    for t in range(T):
        if t == graph_from:
            eng.capture()
        outs.append(eng.step(w.hidden[t], w.queries[t], w.new_keys[t], w.new_values[t]).cpu().numpy().copy())
        if graph_from is not None and t >= graph_from:
            sels.append({L - 1: tuple(x.cpu().numpy() for x in (eng.sel_idx, eng.sel_count, eng.fetch_count))})
            chans.append({l: st.channels.cpu().numpy() for l, st in eng.sparse.items()})
        else:
            sels.append({l: tuple(x.cpu().numpy() for x in eng.last_selection[l]) for l in eng.last_selection})
            chans.append({l: c.cpu().numpy() for l, c in eng.last_channels.items()})
    hits = misses = 0
    for l, lay in enumerate(eng.layers):
        if w.labels[l] == "s":
            hh, mm = lay.cache_counters()
            hits, misses = hits + hh, misses + mm
    for b in range(B):
        steps = [{"hidden": w.hidden[t, :, b].double().cpu().numpy(),
                  "queries": w.queries[t, :, b].double().cpu().numpy(),
                  "new_keys": w.new_keys[t, :, b].double().cpu().numpy(),
                  "new_values": w.new_values[t, :, b].double().cpu().numpy()} for t in range(T)]
        orc = O.replay([k[b].double().cpu().numpy() for k in w.prefill_keys],
                       [v[b].double().cpu().numpy() for v in w.prefill_values],
                       [wq.double().cpu().numpy() if wq is not None else None for wq in w.w_q], steps, w.labels,
                       bits=bits, n_local=64, n_topk=n_topk, d_s=8, compute_exact=False)
        for t in range(T):
            for l in range(L):
                o = outs[t][l].reshape(B, hq, d)[b]
                assert rel_err(o, orc.outputs[t][l]) <= REL_TOL, (b, t, l)
                if w.labels[l] != "s":
                    continue
                for kvh in range(h):
                    u = b * h + kvh
                    assert np.array_equal(chans[t][l][u], orc.channels[(l, t)][kvh]), ("channels", b, t, l, kvh)
                    if l not in sels[t]:
                        continue
                    idx, cnt, fc = sels[t][l]
                    assert np.array_equal(idx[u, :cnt[u]], orc.selected[(l, t)][kvh]), ("selection", b, t, l, kvh)
                    assert int(fc[u]) == orc.fetched[(l, t)][kvh], ("fetch count", b, t, l, kvh)
    return hits, misses


def test_config2_sparse_layers_128k_multistep_row_cache_and_hint(tkv, sparse_kernel):
    """131,072-token sparse layers, 4 KV heads, 6 steps with the per-step
    outlier drift (trace.py:268-275), row cache W=4 and the threshold hint on:
    selections, channels, fetch counts and outputs equal the oracle's at every
    step (3 eager steps, then 3 replays of the captured graph), and the row
    cache both hits and misses."""
    from paper_2505_19586_b200.synth import make_workload

    hq, h, d, n, T = 16, 4, 128, 131072, 6
    w = make_workload(2, (), hq, h, d, n, T, seed=23, drift=True)
    hits, misses = _run_and_check(tkv, w, hq, h, d, 1, 1, 2621, T, graph_from=3)
    assert hits > 0 and misses > 0


@pytest.mark.parametrize("bits", [1, 2])
def test_config2_quant_decode_128k_8_heads(tkv, bits):
    """Quantized decode at exactly the config-2 layer shape: 131,072 tokens x
    8 KV heads x 32 query heads, against the float64 oracle."""
    rng = np.random.default_rng(131 + bits)
    h, G, d, n = 8, 4, 128, 131072
    keys = cases.f16(rng.normal(0, 0.05, size=(h, n, d)))
    keys[:, ::211] += cases.f16(rng.normal(0, 0.4, size=(h, 1, d)))  # a few louder tokens
    keys = cases.f16(keys)
    values = cases.f16(rng.normal(size=(h, n, d)))
    queries = cases.f16(rng.normal(size=(h * G, d)))
    q = tkv.quantize_layer_kv(keys, values, bits, 64)
    kq, vq = O.quantize_layer(keys, values, bits, 64)
    ref = O.quant_layer_decode(queries, kq, vq)
    out = q.decode(queries).cpu().numpy()
    assert rel_err(out, ref) <= REL_TOL
    assert rel_err(out, ref) <= 5e-4


def test_config3_shape_32k_batch16_2bit(tkv):
    """BASELINE config 3 on one GPU: Llama-3.1-8B heads, 32k context, batch 16
    (128 units: the 4-CTA cluster build), layer 0 2-bit quantized, two Top-K
    3 % layers; every sequence against its oracle replay for 2 steps."""
    from paper_2505_19586_b200.synth import make_workload

    hq, h, d, n, B, T = 32, 8, 128, 32768, 16, 2
    w = make_workload(3, (0,), hq, h, d, n, T, batch=B, seed=29)
    _run_and_check(tkv, w, hq, h, d, 2, B, round(0.03 * n), T)
