"""Attention-sink tokens, an opt-in extension (north_star: "sparse attention
over the gathered tokens plus sink/local-window tokens"; the reference has
none, SURVEY 8(a')9).  n_sink = 0 is the reference's selection (covered by
every other sparse test); n_sink > 0 is checked against the oracle
extension ``select_tokens_sinks``: index sets identical (ties included),
outputs within 1e-5 of the float64 oracle, on the fused decode and inside
the engine."""

import numpy as np
import pytest
import torch

import cases
from oracle import tailorkv_oracle as O

from test_gpu_parity import _keys_for, _sparse_layer, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tkv():
    import paper_2505_19586_b200 as P

    return P


def _decode(tkv, lay, queries, chans, G, cfg, kod=True):
    import paper_2505_19586_b200._lib as L
    units, d = chans.shape[0], lay.head_dim
    kmax = cfg.max_selected
    idx = torch.zeros((units, kmax), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(units, dtype=torch.int32, device="cuda")
    fc = torch.zeros(units, dtype=torch.int32, device="cuda")
    out = torch.zeros((units * G, d), dtype=torch.float32, device="cuda")
    ws = torch.zeros(int(L.load().tkv_sparse_decode_workspace(units, lay.capacity, G, d, kmax)), dtype=torch.uint8,
                     device="cuda")
    lay.decode(torch.tensor(queries, dtype=torch.float16, device="cuda"), torch.tensor(chans, device="cuda"), G, cfg,
               idx, cnt, fc, out, ws, keys_from_device=kod)
    return idx.cpu().numpy(), cnt.cpu().numpy(), fc.cpu().numpy(), out.cpu().numpy()


@pytest.mark.parametrize("n_sink", [1, 4, 37])
@pytest.mark.parametrize("dist", ["normal", "ties", "near_ties"])
@pytest.mark.parametrize("n", [20000, 700, 150])
def test_fused_decode_with_sinks_matches_oracle(tkv, n_sink, dist, n, sparse_kernel):
    rng = np.random.default_rng(n_sink * 7 + n)
    units, d, G, d_s = 3, 128, 4, 8
    keys = cases.f16(_keys_for(dist, rng, (units, n, d)))
    values = cases.f16(rng.normal(size=(units, n, d)))
    queries = cases.f16(rng.normal(size=(units * G, d)))
    cfg = tkv.RetrievalConfig(64, 100 if n < 1000 else 613, d_s, n_sink)
    lay = tkv.OffloadedLayerKV(units, d, n + 4, n, cfg.n_local, keys_on_device=True, n_sink=n_sink,
                               cache_rows=cfg.max_selected, cache_window=2)
    lay.offload(keys, values)
    chans = np.stack([np.sort(rng.choice(d, d_s, replace=False)) for _ in range(units)]).astype(np.int32)
    idx, cnt, fc, out = _decode(tkv, lay, queries, chans, G, cfg)
    ref = np.empty_like(out, dtype=np.float64)
    for u in range(units):
        qg = queries[u * G:(u + 1) * G]
        sel = O.select_tokens_sinks(O.approx_scores(qg[:, chans[u]], keys[u][:, chans[u]]), cfg.n_local, cfg.n_topk,
                                    n_sink)
        assert np.array_equal(idx[u, :cnt[u]], sel), u
        assert np.all(np.isin(np.arange(min(n_sink, n)), idx[u, :cnt[u]]))
        assert fc[u] == int((sel < max(0, n - cfg.n_local)).sum())
        for j in range(G):
            ref[u * G + j] = O.sparse_attention(qg[j], keys[u], values[u], sel)
    assert rel_err(out, ref) <= 1e-5


def test_sink_config_must_match_layer(tkv):
    rng = np.random.default_rng(0)
    keys = cases.f16(rng.normal(size=(1, 500, 128)))
    lay = _sparse_layer(tkv, keys, keys, 16)
    with pytest.raises(tkv.ParameterError):
        _decode(tkv, lay, cases.f16(rng.normal(size=(4, 128))), np.arange(8, dtype=np.int32)[None], 4,
                tkv.RetrievalConfig(16, 50, 8, 3))
    with pytest.raises(tkv.ParameterError):
        tkv.RetrievalConfig(16, 50, 8, -1)


def test_engine_with_sinks_matches_oracle_over_steps(tkv):
    """Two sparse layers, 6 graph-replayed steps with appends: every step's
    selection is sinks + Top-K + local window and the outputs follow the
    oracle (channels from the engine's own stage 1, checked separately)."""
    rng = np.random.default_rng(5)
    L, hq, h, d, n, T, n_sink = 2, 8, 2, 128, 3000, 6, 4
    model = tkv.ModelConfig(L, hq, h, d, hq * d)
    cfg = tkv.EngineConfig(bits=1, group_size=64, n_local=32, n_topk=150, critical_channels=8, n_sink=n_sink)
    eng = tkv.DecodeEngine(model, ["s", "s"], cfg, max_steps=T)
    K = [cases.f16(rng.normal(size=(h, n, d))) for _ in range(L)]
    V = [cases.f16(rng.normal(size=(h, n, d))) for _ in range(L)]
    W = [cases.f16(rng.normal(size=(hq, hq * d, d)) / np.sqrt(hq * d)) for _ in range(L)]
    for l in range(L):
        eng.prefill(l, K[l][None], V[l][None], W[l])
    G = hq // h
    eng.record_selection = True
    for t in range(T):
        hid = cases.f16(rng.normal(size=(L, 1, hq * d)))
        q = cases.f16(rng.normal(size=(L, 1, hq, d)))
        nk = cases.f16(rng.normal(size=(L, 1, h, d)))
        nv = cases.f16(rng.normal(size=(L, 1, h, d)))
        out = eng.step(hid, q, nk, nv).cpu().numpy()
        for l in range(L):
            chans = eng.last_channels[l].cpu().numpy()
            idx, cnt, _ = (x.cpu().numpy() for x in eng.last_selection[l])
            ref = np.empty((hq, d))
            for u in range(h):
                qg = q[l, 0, u * G:(u + 1) * G]
                sc = O.approx_scores(qg[:, chans[u]], K[l][u][:, chans[u]])
                sel = O.select_tokens_sinks(sc, 32, 150, n_sink)
                assert np.array_equal(idx[u, :cnt[u]], sel), (t, l, u)
                for j in range(G):
                    ref[u * G + j] = O.sparse_attention(qg[j], K[l][u], V[l][u], sel)
            assert rel_err(out[l], ref) <= 1e-4, (t, l)
            K[l] = np.concatenate([K[l], nk[l, 0][:, None]], axis=1)
            V[l] = np.concatenate([V[l], nv[l, 0][:, None]], axis=1)
