"""GPU parity: every CUDA path against the reference golden vectors and the
CPU oracle on identical fp16 inputs.

Tolerances (BASELINE.json north_star): packed bit-planes / GQT1 blobs
bit-exact; top-k and channel index sets exact (no exact score ties are
resolved differently: ties use the reference's index rule); attention
outputs within relative error 2e-3, where
    rel_err = max over query heads of ||out - ref||_2 / ||ref||_2.
"""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest
import torch

import cases
from oracle import tailorkv_oracle as O

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLD / "golden.json").read_text())
KER = np.load(GOLD / "kernels.npz")
REL_TOL = 2e-3


def rel_err(out, ref):
    out = np.asarray(out, np.float64).reshape(ref.shape[0], -1)
    ref = np.asarray(ref, np.float64).reshape(ref.shape[0], -1)
    return float(max(np.linalg.norm(o - r) / max(np.linalg.norm(r), 1e-30) for o, r in zip(out, ref)))


def sha(b):
    return hashlib.sha256(b).hexdigest()


@pytest.fixture(scope="module")
def tkv():
    import paper_2505_19586_b200 as P

    return P


# ---------------------------------------------------------------------------
# K1/K2 pack + GQT1 export: bit-exact against the reference
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case", [c for c in cases.PACK_CASES if c["gpu"]], ids=lambda c: c["name"])
def test_pack_gqt1_bit_exact(tkv, case):
    k, v = cases.pack_inputs(case)
    q = tkv.quantize_layer_kv(k[None], v[None], case["bits"], case["g"])
    gold = META["pack"][case["name"]]
    kb, vb = q.to_bytes(0, "keys"), q.to_bytes(0, "values")
    assert len(kb) == gold["keys_len"] and sha(kb) == gold["keys_sha256"]
    assert len(vb) == gold["values_len"] and sha(vb) == gold["values_sha256"]


def test_pack_multi_unit_each_head_exact(tkv):
    rng = np.random.default_rng(3)
    keys = cases.f16(rng.normal(size=(5, 700, 128)))
    values = cases.f16(rng.normal(size=(5, 700, 128)))
    for bits in (1, 2):
        q = tkv.quantize_layer_kv(keys, values, bits, 64)
        for u in range(5):
            with np.errstate(over="ignore"):
                assert q.to_bytes(u, "keys") == O.quantize_keys(keys[u], bits, 64).to_bytes()
                assert q.to_bytes(u, "values") == O.quantize_values(values[u], bits, 64).to_bytes()


def _boundary_groups(rng, ngroups, glen, bits):
    """Groups whose members sit on and next to the codec's rounding boundaries
    lo + (k - 1/2) (hi - lo) / (2^b - 1): the fp16 values nearest each boundary
    and 1-2 ulps either side, plus lo and hi; spans include mixed signs,
    subnormals, +-0 and wide magnitude ranges."""
    out = np.zeros((ngroups, glen), np.float16)
    for i in range(ngroups):
        kind = i % 5
        if kind == 0:
            lo, hi = sorted(rng.normal(size=2) * 3)
        elif kind == 1:
            lo, hi = sorted(rng.normal(size=2) * 1e-5)  # subnormal fp16
        elif kind == 2:
            lo, hi = -abs(rng.normal()) * 1e4, abs(rng.normal()) * 1e-3
        elif kind == 3:
            lo, hi = 0.0, abs(rng.normal()) + 0.1
        else:
            lo, hi = -abs(rng.normal()) - 0.1, -0.0
        lo16, hi16 = np.float16(lo), np.float16(hi)
        if lo16 == hi16:
            hi16 = np.nextafter(hi16, np.float16(np.inf))
        cand = [lo16, hi16]
        nl = (1 << bits) - 1
        for k in range(1, nl + 1):
            b = np.float16(float(lo16) + (k - 0.5) * (float(hi16) - float(lo16)) / nl)
            x = b
            for _ in range(3):
                cand.append(x)
                x = np.nextafter(x, np.float16(np.inf))
            x = b
            for _ in range(2):
                x = np.nextafter(x, np.float16(-np.inf))
                cand.append(x)
        cand = np.clip(np.array(cand, np.float16), lo16, hi16)
        row = rng.choice(cand, size=glen)
        row[rng.integers(glen)], row[rng.integers(glen)] = lo16, hi16
        if lo16 == 0:  # one zero sign per group (with both, numpy's min picks by reduction order)
            row[row == 0] = lo16
        out[i] = row
    return out


@pytest.mark.parametrize("d", [32, 64, 96, 128, 256])
@pytest.mark.parametrize("bits,g", [(1, 16), (1, 32), (1, 64), (1, 128), (2, 16), (2, 32), (2, 64)])
def test_pack_every_instantiation_exact(tkv, d, bits, g):
    # every (bits, group, head_dim) pack kernel instance -- the d = 64 / 128 specialisations and the
    # generic one -- against the oracle, with a partial key tile, a residual and a partial value chunk
    rng = np.random.default_rng(1000 + d + 10 * g + bits)
    Tk = 16 * (8 // bits)
    n = 2 * Tk + g + 7 if g < Tk else Tk + g + 7
    keys = cases.f16(rng.normal(size=(2, n, d)))
    values = cases.f16(rng.normal(size=(2, n, d)) * 3.0)
    q = tkv.quantize_layer_kv(keys, values, bits, g)
    for u in range(2):
        assert q.to_bytes(u, "keys") == O.quantize_keys(keys[u], bits, g).to_bytes(), (u, "keys")
        assert q.to_bytes(u, "values") == O.quantize_values(values[u], bits, g).to_bytes(), (u, "values")


@pytest.mark.parametrize("bits", [1, 2])
def test_pack_negative_zero_minimum(tkv, bits):
    # a group whose minimum is -0.0 stores the zero-point as -0.0 (0x8000), as
    # the reference's float64 min does; prefill and append agree
    g, d, n = 16, 32, 64
    rng = np.random.default_rng(9)
    keys = np.abs(cases.f16(rng.normal(size=(n, d))))
    values = np.abs(cases.f16(rng.normal(size=(n, d))))
    keys[::5, ::3] = np.float16(-0.0)
    values[::3, ::5] = np.float16(-0.0)
    q = tkv.quantize_layer_kv(keys[None], values[None], bits, g)
    assert q.to_bytes(0, "keys") == O.quantize_keys(keys, bits, g).to_bytes()
    assert q.to_bytes(0, "values") == O.quantize_values(values, bits, g).to_bytes()
    qa = tkv.QuantizedLayerKV.from_kv(keys[None, :20], values[None, :20], bits, g, capacity=n)
    for t in range(20, n):
        qa.append_token(keys[None, t], values[None, t])
    assert qa.to_bytes(0, "keys") == O.quantize_keys(keys, bits, g).to_bytes()
    assert qa.to_bytes(0, "values") == O.quantize_values(values, bits, g).to_bytes()


@pytest.mark.parametrize("bits", [1, 2])
@pytest.mark.parametrize("g", [16, 64])
def test_pack_rounding_boundaries_exact(tkv, bits, g):
    # the pack encodes by per-group fp16 thresholds; every value on or next to
    # a rounding boundary must still get the reference's float64 code
    rng = np.random.default_rng(40 + bits + g)
    d, n = 128, 4 * 128 + g + 5  # complete tiles, a partial key tile, a residual
    kg = _boundary_groups(rng, (n // g) * d, g, bits)  # [(group, ch)][token in group]
    keys = np.zeros((n, d), np.float16)
    keys[: (n // g) * g] = kg.reshape(n // g, d, g).transpose(0, 2, 1).reshape(-1, d)
    keys[(n // g) * g:] = cases.f16(rng.normal(size=(n - (n // g) * g, d)))
    values = _boundary_groups(rng, n * (d // g), g, bits).reshape(n, d)
    q = tkv.quantize_layer_kv(keys[None], values[None], bits, g)
    assert q.to_bytes(0, "keys") == O.quantize_keys(keys, bits, g).to_bytes()
    assert q.to_bytes(0, "values") == O.quantize_values(values, bits, g).to_bytes()


@pytest.mark.parametrize("bits", [1, 2])
def test_append_matches_batch_quantization(tkv, bits):
    # quantizer.py:445-451 + test_quantizer.py:204-222: incremental == batch
    rng = np.random.default_rng(4 + bits)
    n0, T = 250, 80  # crosses two key-group boundaries (256, 320)
    keys = cases.f16(rng.normal(size=(3, n0 + T, 128)))
    values = cases.f16(rng.normal(size=(3, n0 + T, 128)))
    q = tkv.QuantizedLayerKV.from_kv(keys[:, :n0], values[:, :n0], bits, 64, capacity=n0 + T)
    for t in range(T):
        q.append_token(keys[:, n0 + t], values[:, n0 + t])
    for u in range(3):
        assert q.to_bytes(u, "keys") == O.quantize_keys(keys[u], bits, 64).to_bytes()
        assert q.to_bytes(u, "values") == O.quantize_values(values[u], bits, 64).to_bytes()


def test_dequantize_bound(tkv):
    rng = np.random.default_rng(8)
    keys = cases.f16(rng.normal(size=(1, 513, 128)))
    values = cases.f16(rng.normal(size=(1, 513, 128)))
    q = tkv.quantize_layer_kv(keys, values, 2, 64)
    kt = O.quantize_keys(keys[0], 2, 64)
    np.testing.assert_allclose(q.dequantize(0, "keys").cpu().numpy(), kt.dequantize(), rtol=1e-6, atol=1e-6)


def test_error_mapping(tkv):
    with pytest.raises(tkv.EmptyCacheError):
        tkv.quantize_layer_kv(np.zeros((1, 0, 128)), np.zeros((1, 0, 128)), 1, 64)
    with pytest.raises(tkv.ParameterError):
        tkv.quantize_layer_kv(np.zeros((1, 64, 128)), np.zeros((1, 64, 128)), 3, 64)
    with pytest.raises(tkv.ShapeError):
        tkv.quantize_layer_kv(np.zeros((1, 64, 128)), np.zeros((1, 65, 128)), 1, 64)
    bad = np.zeros((1, 64, 128))
    bad[0, 3, 4] = np.inf
    with pytest.raises(tkv.NumericError):
        tkv.quantize_layer_kv(bad, np.zeros((1, 64, 128)), 1, 64)


# ---------------------------------------------------------------------------
# K4 quantized decode attention
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("impl", [1, 0])
@pytest.mark.parametrize("case", cases.DECODE_CASES, ids=lambda c: c["name"])
def test_quant_decode_matches_reference(tkv, case, impl):
    keys, values, queries = cases.decode_inputs(case)
    q = tkv.quantize_layer_kv(keys, values, case["bits"], case["g"])
    out = q.decode(queries, impl=impl).cpu().numpy()
    ref = KER[case["name"] + "/out"]
    assert rel_err(out, ref) <= REL_TOL


@pytest.mark.parametrize("impl", [2, 3])
@pytest.mark.parametrize("bits", [1, 2])
@pytest.mark.parametrize("n,kscale", [(32768 + 17, 0.05), (5000, 0.5), (64 * 17, 0.2)])
def test_quant_decode_tensor_core_vs_oracle(tkv, bits, n, kscale, impl):
    """The IMMA kernels (impl=2 pipelined, 3 per-chunk) at long context, dense
    (near-uniform) and peaky attention, against the float64 oracle."""
    rng = np.random.default_rng(n + bits)
    h, G, d = 2, 4, 128
    keys = cases.f16(rng.normal(0, kscale, size=(h, n, d)))
    keys[:, ::97] += cases.f16(rng.normal(0, 3 * kscale, size=(h, 1, d)))  # a few louder tokens
    keys = cases.f16(keys)
    values = cases.f16(rng.normal(size=(h, n, d)))
    queries = cases.f16(rng.normal(size=(h * G, d)))
    q = tkv.quantize_layer_kv(keys, values, bits, 64)
    kq, vq = O.quantize_layer(keys, values, bits, 64)
    ref = O.quant_layer_decode(queries, kq, vq)
    out2 = q.decode(queries, impl=impl).cpu().numpy()
    assert rel_err(out2, ref) <= REL_TOL
    assert rel_err(out2, ref) <= 5e-4  # typical margin of the exact-integer design


@pytest.mark.parametrize("G", [1, 3, 5, 7, 8])
@pytest.mark.parametrize("bits", [1, 2])
def test_quant_decode_tensor_core_head_blocks(tkv, bits, G):
    """GQA groups of any size on the pipelined IMMA kernel (Qwen2.5-7B G=7,
    Llama-3.1-70B G=8): query heads run in blocks of 4, the last block ragged."""
    rng = np.random.default_rng(300 + 10 * G + bits)
    h, d, n = 2, 128, 9000 + 21
    keys = cases.f16(rng.normal(0, 0.2, size=(h, n, d)))
    keys[:, ::131] += cases.f16(rng.normal(0, 0.6, size=(h, 1, d)))
    keys = cases.f16(keys)
    values = cases.f16(rng.normal(size=(h, n, d)))
    queries = cases.f16(rng.normal(size=(h * G, d)))
    q = tkv.quantize_layer_kv(keys, values, bits, 64)
    kq, vq = O.quantize_layer(keys, values, bits, 64)
    ref = O.quant_layer_decode(queries, kq, vq)
    out = q.decode(queries, impl=2).cpu().numpy()
    assert rel_err(out, ref) <= 5e-4
    assert np.array_equal(q.decode(queries).cpu().numpy(), out)  # impl 0 picks the tensor-core kernel
    if G > 4:
        with pytest.raises(tkv.ParameterError):
            q.decode(queries, impl=3)


@pytest.mark.parametrize("bits", [1, 2])
def test_quant_decode_pipelined_ring_wraps(tkv, bits):
    """8 heads at 60k tokens: every CTA of the pipelined kernel streams more
    chunks than its TMA ring has stages, so stages are refilled while other
    warps still compute; against the oracle and the per-chunk kernel."""
    rng = np.random.default_rng(90 + bits)
    h, G, d, n = 8, 4, 128, 60000 + 33
    keys = cases.f16(rng.normal(0, 0.2, size=(h, n, d)))
    values = cases.f16(rng.normal(size=(h, n, d)))
    queries = cases.f16(rng.normal(size=(h * G, d)))
    q = tkv.quantize_layer_kv(keys, values, bits, 64)
    kq, vq = O.quantize_layer(keys, values, bits, 64)
    ref = O.quant_layer_decode(queries, kq, vq)
    out = q.decode(queries, impl=2).cpu().numpy()
    assert rel_err(out, ref) <= 5e-4
    out3 = q.decode(queries, impl=3).cpu().numpy()
    assert rel_err(out, out3) <= 5e-4


@pytest.mark.parametrize("bits", [1, 2])
def test_quant_decode_after_appends(tkv, bits):
    rng = np.random.default_rng(77 + bits)
    h, G, d, n0, T = 2, 4, 128, 1000, 90
    keys = cases.f16(rng.normal(0, 0.3, size=(h, n0 + T, d)))
    values = cases.f16(rng.normal(size=(h, n0 + T, d)))
    queries = cases.f16(rng.normal(size=(h * G, d)))
    q = tkv.QuantizedLayerKV.from_kv(keys[:, :n0], values[:, :n0], bits, 64, capacity=n0 + T)
    for t in range(T):
        q.append_token(keys[:, n0 + t], values[:, n0 + t])
        if t % 29 == 0 or t == T - 1:
            kq, vq = O.quantize_layer(keys[:, :n0 + t + 1], values[:, :n0 + t + 1], bits, 64)
            ref = O.quant_layer_decode(queries, kq, vq)
            for impl in (1, 2, 3):
                assert rel_err(q.decode(queries, impl=impl).cpu().numpy(), ref) <= REL_TOL


def test_qgemv_raw_ops(tkv):
    keys, values, queries = cases.decode_inputs(cases.DECODE_CASES[0])
    q = tkv.quantize_layer_kv(keys, values, 1, 64)
    logits = tkv.qgemv_scores(queries[0], q, 0).cpu().numpy()
    np.testing.assert_allclose(logits, KER["dec_b1_ragged/logits0"], rtol=1e-5, atol=1e-4)
    kq, vq = O.quantize_layer(keys, values, 1, 64)
    w = O.stable_softmax(logits.astype(np.float64) / np.sqrt(128))
    ref = O.qgemv_output(w, vq[0])
    np.testing.assert_allclose(tkv.qgemv_output(w, q, 0).cpu().numpy(), ref, rtol=1e-5, atol=1e-6)


# ---------------------------------------------------------------------------
# K5-K7 retrieval
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case", cases.TOPK_CASES, ids=lambda c: c["name"])
def test_topk_exact(tkv, case):
    scores = cases.topk_scores(case)
    sel = tkv.select_topk_tokens(scores, tkv.RetrievalConfig(case["n_local"], case["n_topk"]))
    assert np.array_equal(sel, KER[case["name"]])


def test_topk_batched_units(tkv):
    rng = np.random.default_rng(9)
    s = rng.normal(size=(6, 9000))
    s[3] = np.round(s[3])  # heavy ties in one unit
    sel = tkv.select_topk_tokens(s, tkv.RetrievalConfig(32, 300))
    for u in range(6):
        assert np.array_equal(sel[u], O.select_tokens(s[u], 32, 300))


@pytest.mark.parametrize("case", cases.CHANNEL_CASES, ids=lambda c: c["name"])
def test_stage1_channels_exact(tkv, case):
    qhat, chmax = cases.channel_inputs(case)
    G, d = qhat.shape
    # hidden = concat(q_hat heads), W_q[h] selects its slice -> q_hat exactly
    hidden = torch.tensor(qhat.reshape(1, -1), dtype=torch.float16, device="cuda")
    W = torch.zeros((G, G * d, d), dtype=torch.float16, device="cuda")
    for h in range(G):
        W[h, h * d:(h + 1) * d] = torch.eye(d)
    cm = torch.tensor(chmax[None], dtype=torch.float32, device="cuda")
    ch = tkv.stage1_select(hidden, W, cm, G, case["d_s"]).cpu().numpy()[0]
    ref = O.select_channels(O.group_channel_scores(cases.f16(qhat), chmax.astype(np.float32)), case["d_s"])
    assert np.array_equal(ch, ref)


def test_stage1_estimate_matches_oracle(tkv):
    rng = np.random.default_rng(10)
    hq, H, d, G = 8, 1024, 128, 4
    w_q = cases.f16(rng.normal(size=(hq, H, d)) / np.sqrt(H))
    hid = cases.f16(rng.normal(size=(2, H)))
    chmax = cases.f16(np.abs(rng.normal(size=(2 * hq // G, d))) + 0.1)
    qhat = torch.empty((2, hq, d), dtype=torch.float64, device="cuda")
    ch = tkv.stage1_select(torch.tensor(hid, dtype=torch.float16, device="cuda"),
                           torch.tensor(w_q, dtype=torch.float16, device="cuda"),
                           torch.tensor(chmax, dtype=torch.float32, device="cuda"), G, 8, q_hat=qhat).cpu().numpy()
    for b in range(2):
        ref_q = O.estimate_query(w_q, hid[b])
        np.testing.assert_allclose(qhat[b].cpu().numpy(), ref_q, rtol=2e-5, atol=1e-6)
        for kvh in range(hq // G):
            ref = O.select_channels(O.group_channel_scores(ref_q[kvh * G:(kvh + 1) * G], chmax[b * 2 + kvh]), 8)
            assert np.array_equal(ch[b * 2 + kvh], ref)


def _sparse_layer(tkv, keys, values, n_local, steps=4, keys_on_device=False, cache_rows=0, cache_window=1):
    units, n, d = keys.shape
    lay = tkv.OffloadedLayerKV(units, d, n + steps, n, n_local, keys_on_device=keys_on_device, cache_rows=cache_rows,
                               cache_window=cache_window)
    lay.offload(keys, values)
    return lay


@pytest.mark.parametrize("path", ["cluster", "multikernel"])
@pytest.mark.parametrize("kod", [False, True])
def test_select_and_sparse_attention_match_oracle(tkv, kod, path, monkeypatch):
    if path == "multikernel":
        monkeypatch.setenv("TKV_SELECT_MULTIKERNEL", "1")
    rng = np.random.default_rng(11)
    units, n, d, G, d_s = 3, 5000, 128, 4, 8
    keys = cases.f16(rng.normal(size=(units, n, d)))
    values = cases.f16(rng.normal(size=(units, n, d)))
    queries = cases.f16(rng.normal(size=(units * G, d)))
    cfg = tkv.RetrievalConfig(64, 200, d_s)
    lay = _sparse_layer(tkv, keys, values, cfg.n_local, keys_on_device=kod)
    chans = np.stack([np.sort(rng.choice(d, d_s, replace=False)) for _ in range(units)]).astype(np.int32)
    qdev = torch.tensor(queries, dtype=torch.float16, device="cuda")
    cdev = torch.tensor(chans, device="cuda")
    import paper_2505_19586_b200._lib as L
    ws = torch.zeros(int(L.load().tkv_select_workspace(units, lay.capacity)), dtype=torch.uint8, device="cuda")
    kmax = cfg.n_local + cfg.n_topk
    idx = torch.zeros((units, kmax), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(units, dtype=torch.int32, device="cuda")
    fc = torch.zeros(units, dtype=torch.int32, device="cuda")
    scores = torch.zeros((units, lay.capacity), dtype=torch.float64, device="cuda")
    lay.select(qdev, cdev, G, cfg, idx, cnt, fc, ws, scores_out=scores)
    out = torch.zeros((units * G, d), dtype=torch.float32, device="cuda")
    aws = torch.zeros(int(L.load().tkv_sparse_attn_workspace(units, G, d, kmax)), dtype=torch.uint8, device="cuda")
    lay.attend(qdev, G, cfg, idx, cnt, out, aws, keys_from_device=kod)
    idx, cnt, fc = idx.cpu().numpy(), cnt.cpu().numpy(), fc.cpu().numpy()
    ref_out = np.empty((units * G, d))
    for u in range(units):
        qg = queries[u * G:(u + 1) * G]
        sc = O.approx_scores(qg[:, chans[u]], keys[u][:, chans[u]])
        np.testing.assert_allclose(scores[u, :n - cfg.n_local].cpu().numpy(), sc[:n - cfg.n_local], rtol=1e-12)
        sel = O.select_tokens(sc, cfg.n_local, cfg.n_topk)
        assert np.array_equal(idx[u, :cnt[u]], sel)
        assert fc[u] == int((sel < n - cfg.n_local).sum())
        for j in range(G):
            ref_out[u * G + j] = O.sparse_attention(qg[j], keys[u], values[u], sel)
    assert rel_err(out.cpu().numpy(), ref_out) <= 1e-5


@pytest.mark.parametrize("cluster", [8, 4, 2])
@pytest.mark.parametrize("dist", ["normal", "ties", "outliers"])
def test_fused_decode_every_cluster_size(tkv, cluster, dist):
    """The fused decode built with 8-, 4- and 2-CTA clusters (the dispatch picks by units): selections,
    fetch counts and outputs against the oracle, with the row cache, over two steps."""
    import paper_2505_19586_b200._lib as L
    rng = np.random.default_rng(300 + cluster)
    units, n, d, G = 3, 9000, 128, 4
    keys = cases.f16(_keys_for(dist, rng, (units, n, d)))
    values = cases.f16(rng.normal(size=(units, n, d)))
    cfg = tkv.RetrievalConfig(64, 300, 8)
    lay = _sparse_layer(tkv, keys, values, cfg.n_local, keys_on_device=True, cache_rows=cfg.n_local + cfg.n_topk,
                        cache_window=2)
    L.load().tkv_debug_sparse_cluster(cluster)
    try:
        for step in range(2):
            queries = cases.f16(rng.normal(size=(units * G, d)))
            chans = np.stack([np.sort(rng.choice(d, 8, replace=False)) for _ in range(units)]).astype(np.int32)
            res = _decode_once(tkv, lay, queries, chans, G, cfg, True)
            assert L.load().tkv_debug_sparse_path() == cluster
            assert _check_decode(keys, values, queries, chans, G, cfg, res, n) <= 1e-5
    finally:
        L.load().tkv_debug_sparse_cluster(-1)


@pytest.mark.parametrize("dist", ["ties", "zeros", "normal"])
def test_cluster_select_ties_and_sizes(tkv, dist):
    """Scorer + top-k on inputs with massive exact score ties (the cluster
    radix select resolves them toward larger indices like lexsort)."""
    rng = np.random.default_rng(21)
    units, n, d, G = 2, 20000, 64, 2
    if dist == "ties":
        keys = np.round(rng.normal(size=(units, n, d)))
    elif dist == "zeros":
        keys = np.zeros((units, n, d))
    else:
        keys = rng.normal(size=(units, n, d))
    keys = cases.f16(keys)
    values = cases.f16(rng.normal(size=(units, n, d)))
    cfg = tkv.RetrievalConfig(17, 777, 4)
    lay = _sparse_layer(tkv, keys, values, cfg.n_local)
    queries = cases.f16(np.round(rng.normal(size=(units * G, d))))
    chans = np.stack([np.sort(rng.choice(d, 4, replace=False)) for _ in range(units)]).astype(np.int32)
    import paper_2505_19586_b200._lib as L
    ws = torch.zeros(int(L.load().tkv_select_workspace(units, lay.capacity)), dtype=torch.uint8, device="cuda")
    kmax = cfg.n_local + cfg.n_topk
    idx = torch.zeros((units, kmax), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(units, dtype=torch.int32, device="cuda")
    fc = torch.zeros(units, dtype=torch.int32, device="cuda")
    lay.select(torch.tensor(queries, dtype=torch.float16, device="cuda"), torch.tensor(chans, device="cuda"), G, cfg,
               idx, cnt, fc, ws)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for u in range(units):
        sc = O.approx_scores(queries[u * G:(u + 1) * G][:, chans[u]], keys[u][:, chans[u]])
        assert np.array_equal(idx[u, :cnt[u]], O.select_tokens(sc, cfg.n_local, cfg.n_topk))


def _keys_for(dist, rng, shape):
    if dist == "ties":
        return np.round(rng.normal(size=shape))
    if dist == "zeros":
        return np.zeros(shape)
    if dist == "outliers":  # a few huge keys stretch the score range: the threshold bin is crowded -> refinement
        k = rng.normal(0, 1e-3, size=shape)
        k[:, rng.choice(shape[1], 5, replace=False)] *= 1e5
        return k
    if dist == "near_ties":  # scores equal in fp32 but not in float64 -> the exact band decides
        k = np.round(rng.normal(size=shape) * 4) / 4
        k += rng.choice([0, 2.0 ** -10], size=shape)
        return k
    return rng.normal(size=shape)


def _decode_once(tkv, lay, queries, chans, G, cfg, kod):
    import paper_2505_19586_b200._lib as L
    units, d = chans.shape[0], lay.head_dim
    kmax = cfg.n_local + cfg.n_topk
    idx = torch.zeros((units, kmax), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(units, dtype=torch.int32, device="cuda")
    fc = torch.zeros(units, dtype=torch.int32, device="cuda")
    out = torch.zeros((units * G, d), dtype=torch.float32, device="cuda")
    ws = torch.zeros(int(L.load().tkv_sparse_decode_workspace(units, lay.capacity, G, d, kmax)), dtype=torch.uint8,
                     device="cuda")
    lay.decode(torch.tensor(queries, dtype=torch.float16, device="cuda"), torch.tensor(chans, device="cuda"), G, cfg,
               idx, cnt, fc, out, ws, keys_from_device=kod)
    return idx.cpu().numpy(), cnt.cpu().numpy(), fc.cpu().numpy(), out.cpu().numpy()


def _check_decode(keys, values, queries, chans, G, cfg, res, n):
    idx, cnt, fc, out = res
    units = chans.shape[0]
    ref_out = np.empty((units * G, keys.shape[2]))
    for u in range(units):
        qg = queries[u * G:(u + 1) * G]
        sc = O.approx_scores(qg[:, chans[u]], keys[u][:n, chans[u]])
        sel = O.select_tokens(sc, cfg.n_local, cfg.n_topk)
        assert np.array_equal(idx[u, :cnt[u]], sel), u
        assert fc[u] == int((sel < max(0, n - cfg.n_local)).sum())
        for j in range(G):
            ref_out[u * G + j] = O.sparse_attention(qg[j], keys[u][:n], values[u][:n], sel)
    return rel_err(out, ref_out)


@pytest.mark.parametrize("dist", ["normal", "ties", "zeros", "outliers", "near_ties"])
@pytest.mark.parametrize("kod", [True, False], ids=["keys_hbm", "keys_pcie"])
def test_fused_sparse_decode_matches_oracle(tkv, dist, kod, sparse_kernel):
    """One launch (scores + exact top-k + gather + attention) against the
    oracle: identical index sets (ties by the reference's index rule) and
    outputs within 1e-5."""
    rng = np.random.default_rng(31)
    units, n, d, G, d_s = 3, 20000, 128, 4, 8
    keys = cases.f16(_keys_for(dist, rng, (units, n, d)))
    values = cases.f16(rng.normal(size=(units, n, d)))
    queries = cases.f16(np.round(rng.normal(size=(units * G, d))) if dist != "normal" else rng.normal(size=(units * G, d)))
    cfg = tkv.RetrievalConfig(64, 613, d_s)
    lay = _sparse_layer(tkv, keys, values, cfg.n_local, keys_on_device=kod)
    chans = np.stack([np.sort(rng.choice(d, d_s, replace=False)) for _ in range(units)]).astype(np.int32)
    res = _decode_once(tkv, lay, queries, chans, G, cfg, kod)
    assert _check_decode(keys, values, queries, chans, G, cfg, res, n) <= 1e-5


@pytest.mark.parametrize("d,G", [(64, 8), (128, 8), (32, 2), (256, 4)])
def test_fused_sparse_decode_shapes(tkv, d, G):
    rng = np.random.default_rng(32)
    units, n = 2, 3000
    keys = cases.f16(rng.normal(size=(units, n, d)))
    values = cases.f16(rng.normal(size=(units, n, d)))
    queries = cases.f16(rng.normal(size=(units * G, d)))
    cfg = tkv.RetrievalConfig(16, 100, min(8, d))
    lay = _sparse_layer(tkv, keys, values, cfg.n_local, keys_on_device=True)
    chans = np.stack([np.sort(rng.choice(d, cfg.d_s, replace=False)) for _ in range(units)]).astype(np.int32)
    res = _decode_once(tkv, lay, queries, chans, G, cfg, True)
    assert _check_decode(keys, values, queries, chans, G, cfg, res, n) <= 1e-5


@pytest.mark.parametrize("n", [300, 130, 70, 40])
def test_fused_sparse_decode_select_all(tkv, n, sparse_kernel):
    """n <= n_local + n_topk: every token is attended (retriever.py:204-205),
    including contexts shorter than the cluster's slices."""
    rng = np.random.default_rng(33)
    units, d, G = 2, 128, 4
    keys = cases.f16(rng.normal(size=(units, n, d)))
    values = cases.f16(rng.normal(size=(units, n, d)))
    queries = cases.f16(rng.normal(size=(units * G, d)))
    cfg = tkv.RetrievalConfig(64, 400, 8)
    lay = _sparse_layer(tkv, keys, values, cfg.n_local, keys_on_device=True)
    chans = np.stack([np.arange(8) for _ in range(units)]).astype(np.int32)
    res = _decode_once(tkv, lay, queries, chans, G, cfg, True)
    assert res[1].tolist() == [n, n]
    assert _check_decode(keys, values, queries, chans, G, cfg, res, n) <= 1e-5


@pytest.mark.parametrize("window,rows", [(1, None), (3, None), (100, None), (2, 60)])
def test_fused_sparse_decode_row_cache_across_steps(tkv, window, rows, sparse_kernel):
    """Decode -> append -> decode ... with the HBM row cache (rows selected in
    the last `window` steps stay resident): rows served from the cache give
    the oracle's results at every step, and slots are recycled."""
    rng = np.random.default_rng(34)
    units, n0, d, G, T = 2, 8000, 128, 4, 10
    keys = cases.f16(rng.normal(size=(units, n0 + T, d)))
    values = cases.f16(rng.normal(size=(units, n0 + T, d)))
    cfg = tkv.RetrievalConfig(32, 400, 8)
    lay = _sparse_layer(tkv, keys[:, :n0], values[:, :n0], cfg.n_local, steps=T, keys_on_device=True,
                        cache_rows=rows or cfg.n_local + cfg.n_topk, cache_window=window)  # rows: undersized cache
    chans = np.stack([np.sort(rng.choice(d, 8, replace=False)) for _ in range(units)]).astype(np.int32)
    base_q = rng.normal(size=(units * G, d))
    for t in range(T):
        n = n0 + t
        queries = cases.f16(base_q + 0.3 * rng.normal(size=base_q.shape))  # correlated steps -> cache hits
        res = _decode_once(tkv, lay, queries, chans, G, cfg, True)
        assert _check_decode(keys, values, queries, chans, G, cfg, res, n) <= 1e-5, t
        lay.append(torch.tensor(keys[:, n], dtype=torch.float16, device="cuda"),
                   torch.tensor(values[:, n], dtype=torch.float16, device="cuda"))
    hits, misses = lay.cache_counters()
    assert hits > 0 and misses > 0
    # every cached slot holds the (key | value) row of the token it claims
    tok = lay.slot_tok.cpu().numpy()
    sv = lay.slot_v.cpu().numpy().astype(np.float64)
    for u in range(units):
        for p in np.nonzero(tok[u] >= 0)[0]:
            assert np.array_equal(sv[u, p, 0], keys[u, tok[u, p]])
            assert np.array_equal(sv[u, p, 1], values[u, tok[u, p]])


@pytest.mark.parametrize("G", [4, 7])
def test_fused_sparse_decode_row_cache_staging_rounds(tkv, G):
    """(K|V) row cache with more selected rows per CTA than one staging round
    holds (n_topk 6000 over an 8-CTA cluster: ~750 rows per CTA), so hits,
    misses and local-window rows are gathered over several rounds on both
    mbarriers, across decode steps; G=7 takes the 8-head kernel."""
    rng = np.random.default_rng(36 + G)
    units, n0, d, T = 2, 40000, 128, 4
    keys = cases.f16(rng.normal(size=(units, n0 + T, d)))
    values = cases.f16(rng.normal(size=(units, n0 + T, d)))
    cfg = tkv.RetrievalConfig(40, 6000, 8)
    lay = _sparse_layer(tkv, keys[:, :n0], values[:, :n0], cfg.n_local, steps=T, keys_on_device=True,
                        cache_rows=cfg.n_local + cfg.n_topk, cache_window=2)
    chans = np.stack([np.sort(rng.choice(d, 8, replace=False)) for _ in range(units)]).astype(np.int32)
    base_q = rng.normal(size=(units * G, d))
    for t in range(T):
        n = n0 + t
        queries = cases.f16(base_q + 0.2 * rng.normal(size=base_q.shape))
        res = _decode_once(tkv, lay, queries, chans, G, cfg, True)
        assert _check_decode(keys, values, queries, chans, G, cfg, res, n) <= 1e-5, t
        lay.append(torch.tensor(keys[:, n], dtype=torch.float16, device="cuda"),
                   torch.tensor(values[:, n], dtype=torch.float16, device="cuda"))
    hits, misses = lay.cache_counters()
    assert hits > 0 and misses > 0


def test_fused_sparse_decode_many_units_4cta_clusters(tkv):
    """More units than 8-CTA clusters fit at once (16 > 15) at a context 4 CTAs cover: the
    decode takes the 4-CTA cluster build of the kernel (sparse_fused.cu, TKV_FZ_CTAS=4) and
    matches the oracle across steps with the row cache on."""
    rng = np.random.default_rng(37)
    units, n0, d, G, T = 16, 6000, 128, 4, 3
    keys = cases.f16(rng.normal(size=(units, n0 + T, d)))
    values = cases.f16(rng.normal(size=(units, n0 + T, d)))
    cfg = tkv.RetrievalConfig(24, 300, 8)
    lay = _sparse_layer(tkv, keys[:, :n0], values[:, :n0], cfg.n_local, steps=T, keys_on_device=True,
                        cache_rows=cfg.n_local + cfg.n_topk, cache_window=2)
    chans = np.stack([np.sort(rng.choice(d, 8, replace=False)) for _ in range(units)]).astype(np.int32)
    base_q = rng.normal(size=(units * G, d))
    for t in range(T):
        n = n0 + t
        queries = cases.f16(base_q + 0.2 * rng.normal(size=base_q.shape))
        res = _decode_once(tkv, lay, queries, chans, G, cfg, True)
        assert _check_decode(keys, values, queries, chans, G, cfg, res, n) <= 1e-5, t
        lay.append(torch.tensor(keys[:, n], dtype=torch.float16, device="cuda"),
                   torch.tensor(values[:, n], dtype=torch.float16, device="cuda"))
    hits, misses = lay.cache_counters()
    assert hits > 0 and misses > 0


def test_fused_sparse_decode_128k(tkv, sparse_kernel):
    """Config-2 head shape (131072 tokens, n_topk 2621, d_s 8) against the
    oracle for two heads."""
    rng = np.random.default_rng(35)
    units, n, d, G = 2, 131072, 128, 4
    keys = cases.f16(rng.normal(0, 1 / np.sqrt(d), size=(units, n, d)))
    values = cases.f16(rng.normal(size=(units, n, d)))
    queries = cases.f16(rng.normal(size=(units * G, d)))
    cfg = tkv.RetrievalConfig(64, 2621, 8)
    lay = _sparse_layer(tkv, keys, values, cfg.n_local, keys_on_device=True)
    chans = np.stack([np.sort(rng.choice(d, 8, replace=False)) for _ in range(units)]).astype(np.int32)
    res = _decode_once(tkv, lay, queries, chans, G, cfg, True)
    assert _check_decode(keys, values, queries, chans, G, cfg, res, n) <= 1e-5


def test_host_store_gather_roundtrip(tkv):
    rng = np.random.default_rng(12)
    keys = cases.f16(rng.normal(size=(2, 300, 64)))
    values = cases.f16(rng.normal(size=(2, 300, 64)))
    lay = _sparse_layer(tkv, keys, values, 16)
    idx = np.array([5, 0, 299, 17])
    k, v = lay.gather(1, idx)
    assert np.array_equal(k, keys[1][idx]) and np.array_equal(v, values[1][idx])
    np.testing.assert_array_equal(lay.channel_abs_max().cpu().numpy(), np.abs(keys).max(axis=1))


# ---------------------------------------------------------------------------
# Layer classification (identifier.py) against the reference
# ---------------------------------------------------------------------------
def test_calibrate_matches_reference(tkv):
    for c in cases.CALIB_CASES:
        pq, pk = cases.calib_inputs(c)
        g = META["calibrate"][c["name"]]
        probe = tkv.SparsityProbe(k=g["k"], n_q=c["n_q"], tau=c["tau"])
        prof = tkv.calibrate(list(pq), list(pk), probe)
        for p, ref in zip(prof, g["layers"]):
            np.testing.assert_allclose(p.per_head_scores, ref["scores"], rtol=1e-5, atol=1e-6)
            assert p.label.value == ref["label"]


# ---------------------------------------------------------------------------
# Whole decode replay vs the reference pipeline (selections) and the oracle
# (outputs), eager and CUDA-graph
# ---------------------------------------------------------------------------
def _golden_trace():
    z = np.load(GOLD / "pipeline_trace.npz")
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("graph,kfh", [(False, True), (False, False), (True, True)],
                         ids=["eager-keys_hbm", "eager-keys_pcie", "graph-keys_hbm"])
@pytest.mark.parametrize("run", list(cases.PIPELINE_CONFIGS), ids=str)
def test_engine_replays_reference_pipeline(tkv, run, graph, kfh, sparse_kernel):
    z = _golden_trace()
    ref = META["pipeline"]["runs"][run]
    rc = ref["config"]
    L, h, n0, d = z["prefill_keys"].shape
    hq = z["w_q"].shape[1]
    T = z["queries"].shape[0]
    labels = ["q" if lab == "quantization_friendly" else "s" for lab in ref["labels"]]
    cfg = tkv.EngineConfig(bits=rc.get("bits", 1), n_local=rc.get("n_local", 64), n_topk=rc.get("n_topk", 128),
                           critical_channels=rc.get("critical_channels", 8), keys_from_hbm=kfh)
    model = tkv.ModelConfig(L, hq, h, d, hq * d)
    eng = tkv.DecodeEngine(model, labels, cfg, batch=1, max_steps=T)
    for l in range(L):
        eng.prefill(l, z["prefill_keys"][l][None], z["prefill_values"][l][None], z["w_q"][l])
    eng.record_selection = not graph
    if graph:
        eng.capture()
    steps = [{"hidden": z["hidden"][t].astype(np.float64), "queries": z["queries"][t].astype(np.float64),
              "new_keys": z["new_keys"][t].astype(np.float64), "new_values": z["new_values"][t].astype(np.float64)}
             for t in range(T)]
    orc = O.replay(list(z["prefill_keys"].astype(np.float64)), list(z["prefill_values"].astype(np.float64)),
                   list(z["w_q"].astype(np.float64)), steps, labels, bits=cfg.bits, n_local=cfg.n_local,
                   n_topk=cfg.n_topk, d_s=cfg.critical_channels, compute_exact=False)
    recs = {(r["layer"], r["step"]): r for r in ref["retrieval"]}
    worst = 0.0
    for t in range(T):
        dev = lambda a: torch.tensor(a[:, None], dtype=torch.float16, device="cuda")  # noqa: E731
        out = eng.step(dev(z["hidden"][t]), dev(z["queries"][t]), dev(z["new_keys"][t]), dev(z["new_values"][t]))
        out = out.cpu().numpy()
        for l in range(L):
            worst = max(worst, rel_err(out[l], orc.outputs[t][l]))
            if not graph and labels[l] == "s":
                idx, cnt, fc = (x.cpu().numpy() for x in eng.last_selection[l])
                chans = eng.last_channels[l].cpu().numpy()
                for kvh, ph in enumerate(recs[(l, t)]["per_head"]):
                    assert chans[kvh].tolist() == ph["channels"], (l, t, kvh)
                    assert np.array_equal(idx[kvh, :cnt[kvh]], cases.hex_to_indices(ph["selected_hex"])), (l, t, kvh)
                    assert fc[kvh] == ph["fetched"]
    assert worst <= REL_TOL, worst
    if kfh and not graph and labels.count("s"):
        hits, misses = eng.cache_counters()
        assert misses > 0 and hits + misses > 0  # the HBM row cache was exercised


def test_gpu_fidelity_metrics_match_reference_records(tkv):
    """Recall@k, selected mass, cosine and max-abs error of every sparse layer
    and step, computed on the GPU against exact attention, equal the values
    run_pipeline recorded with its float64 oracle (pipeline.py:316-403)."""
    z = _golden_trace()
    ref = META["pipeline"]["runs"]["default"]
    rc = ref["config"]
    L, h, n0, d = z["prefill_keys"].shape
    hq = z["w_q"].shape[1]
    T = 24
    labels = ["q" if lab == "quantization_friendly" else "s" for lab in ref["labels"]]
    cfg = tkv.EngineConfig(bits=rc.get("bits", 1), n_local=rc.get("n_local", 64), n_topk=rc.get("n_topk", 128),
                           critical_channels=rc.get("critical_channels", 8))
    eng = tkv.DecodeEngine(tkv.ModelConfig(L, hq, h, d, hq * d), labels, cfg, batch=1, max_steps=T)
    for l in range(L):
        eng.prefill(l, z["prefill_keys"][l][None], z["prefill_values"][l][None], z["w_q"][l])
    eng.record_selection = True
    dev = lambda a: torch.tensor(a[:, None], dtype=torch.float16, device="cuda")  # noqa: E731
    checked = 0
    for t in range(T):
        eng.step(dev(z["hidden"][t]), dev(z["queries"][t]), dev(z["new_keys"][t]), dev(z["new_values"][t]))
        for l in range(L):
            if labels[l] != "s":
                continue
            f = eng.layer_fidelity(l)
            assert abs(f["recall"] - ref["recall"][l][t]) <= 1.0 / cfg.n_topk + 1e-12, (l, t)
            assert abs(f["selected_mass"] - ref["selected_mass"][l][t]) <= 1e-4, (l, t)
            assert abs(f["cosine"] - ref["cosine"][l][t]) <= 1e-4, (l, t)
            assert f["max_abs_err"] == pytest.approx(ref["max_abs_err"][l][t], rel=2e-2, abs=1e-4), (l, t)
            checked += 1
    assert checked > 0


def test_engine_runs_reference_trace_file_on_device(tkv):
    """A reference HKVTRACE file loaded straight to the device (trace.py
    container, fp16 sections) drives the engine; every output matches the
    oracle replay of the same file."""
    from paper_2505_19586_b200.trace import load_trace

    tr = load_trace(GOLD / "tiny_trace.hkv", device="cuda")
    ref = O.read_trace_file(GOLD / "tiny_trace.hkv")
    m = tr.header["model"]
    labels = ["q", "s"]
    cfg = tkv.EngineConfig(bits=1, group_size=16, n_local=4, n_topk=8, critical_channels=4)
    eng = tkv.DecodeEngine(tkv.ModelConfig(m["num_layers"], m["num_query_heads"], m["num_kv_heads"], m["head_dim"],
                                           m["hidden_dim"]), labels, cfg, max_steps=tr.num_steps)
    for l in range(m["num_layers"]):
        eng.prefill(l, tr.prefill_keys[l][None], tr.prefill_values[l][None], tr.w_q[l])
    orc = O.replay(ref["prefill_keys"], ref["prefill_values"], ref["w_q"], ref["steps"], labels, bits=1, g=16,
                   n_local=4, n_topk=8, d_s=4, compute_exact=False)
    for t in range(tr.num_steps):
        out = eng.step(*tr.step_inputs(t)).cpu().numpy()
        for l in range(m["num_layers"]):
            assert rel_err(out[l], orc.outputs[t][l]) <= REL_TOL, (t, l)


# BASELINE.json configs 3-5 as parity cases at reduced context (the bench runs config 2):
# (name, hq, h, hidden, q_layers, bits, batch, n, n_topk)
_CONFIG_CASES = [
    ("cfg3_llama8b_b2_2bit_3pct", 32, 8, 4096, (0,), 2, 2, 2048, 61),
    ("cfg4_qwen7b_g7_1pct", 28, 4, 3584, (0,), 1, 2, 4096, 41),
    ("cfg5_llama70b_g8_2pct", 64, 8, 8192, (0,), 1, 1, 2048, 41),
]


@pytest.mark.parametrize("case", _CONFIG_CASES, ids=lambda c: c[0])
def test_engine_baseline_config_shapes(tkv, case):
    """Engine outputs for the BASELINE config families (batch > 1, 2-bit,
    G = 7 and G = 8 grouped-query shapes) against the oracle replay of every
    sequence, and the Top-K selections against the oracle's."""
    from paper_2505_19586_b200.synth import make_workload

    name, hq, h, hidden, q_layers, bits, B, n, n_topk = case
    L, T, d = 3, 3, 128
    w = make_workload(L, q_layers, hq, h, d, n, T, batch=B, seed=17, keep_wq_for_q_layers=True)
    cfg = tkv.EngineConfig(bits=bits, n_local=64, n_topk=n_topk, critical_channels=8)
    eng = tkv.DecodeEngine(tkv.ModelConfig(L, hq, h, d, hidden), w.labels, cfg, batch=B, max_steps=T)
    for l in range(L):
        eng.prefill(l, w.prefill_keys[l], w.prefill_values[l], w.w_q[l])
    eng.record_selection = True
    outs, sels = [], []
    for t in range(T):
        outs.append(eng.step(w.hidden[t], w.queries[t], w.new_keys[t], w.new_values[t]).cpu().numpy().copy())
        sels.append({l: tuple(x.cpu().numpy() for x in eng.last_selection[l]) for l in eng.last_selection})
    G = hq // h
    for b in range(B):
        steps = [{"hidden": w.hidden[t, :, b].double().cpu().numpy(), "queries": w.queries[t, :, b].double().cpu().numpy(),
                  "new_keys": w.new_keys[t, :, b].double().cpu().numpy(),
                  "new_values": w.new_values[t, :, b].double().cpu().numpy()} for t in range(T)]
        orc = O.replay([k[b].double().cpu().numpy() for k in w.prefill_keys],
                       [v[b].double().cpu().numpy() for v in w.prefill_values],
                       [wq.double().cpu().numpy() for wq in w.w_q], steps, w.labels, bits=bits, n_local=64,
                       n_topk=n_topk, d_s=8, compute_exact=False)
        for t in range(T):
            for l in range(L):
                o = outs[t][l].reshape(B, hq, d)[b]
                assert rel_err(o, orc.outputs[t][l]) <= REL_TOL, (name, b, t, l)
                if w.labels[l] == "s":
                    idx, cnt, _ = sels[t][l]
                    for kvh in range(h):
                        u = b * h + kvh
                        assert np.array_equal(idx[u, :cnt[u]], orc.selected[(l, t)][kvh]), (name, b, t, l, kvh)
    assert G in (4, 7, 8)


def test_engine_config1_shapes(tkv):
    """BASELINE config 1 shapes (Llama-8B heads, 4k, 1 Q 1-bit + 1 S layer,
    n_topk=128) on synthetic inputs against the oracle replay."""
    from paper_2505_19586_b200.synth import make_workload

    w = make_workload(2, (0,), 32, 8, 128, 4096, 4, seed=7)
    cfg = tkv.EngineConfig(bits=1, n_local=64, n_topk=128, critical_channels=8)
    model = tkv.ModelConfig(2, 32, 8, 128, 4096)
    eng = tkv.DecodeEngine(model, w.labels, cfg, max_steps=4)
    w_q_np = []
    for l in range(2):
        wq = w.w_q[l] if w.w_q[l] is not None else torch.zeros(32, 4096, 128, dtype=torch.float16, device="cuda")
        eng.prefill(l, w.prefill_keys[l], w.prefill_values[l], wq)
        w_q_np.append(wq.double().cpu().numpy())
    steps = [{"hidden": w.hidden[t, :, 0].double().cpu().numpy(), "queries": w.queries[t, :, 0].double().cpu().numpy(),
              "new_keys": w.new_keys[t, :, 0].double().cpu().numpy(),
              "new_values": w.new_values[t, :, 0].double().cpu().numpy()} for t in range(4)]
    orc = O.replay([k[0].double().cpu().numpy() for k in w.prefill_keys],
                   [v[0].double().cpu().numpy() for v in w.prefill_values], w_q_np, steps, w.labels,
                   compute_exact=False)
    eng.record_selection = True
    for t in range(4):
        out = eng.step(w.hidden[t], w.queries[t], w.new_keys[t], w.new_values[t]).cpu().numpy()
        for l in range(2):
            assert rel_err(out[l], orc.outputs[t][l]) <= REL_TOL
        idx, cnt, _ = (x.cpu().numpy() for x in eng.last_selection[1])
        for kvh in range(8):
            assert np.array_equal(idx[kvh, :cnt[kvh]], orc.selected[(1, t)][kvh])
