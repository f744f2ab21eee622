"""The reference-signature surface (paper_2505_19586_b200/hybridkv.py) against
the reference's semantics: each test restates one of the reference's own
test properties (pkg/tests/test_quantizer.py, test_retriever.py,
test_memsim.py, test_identifier.py) with the hybridkv names bound to this
package, and checks values against the float64 oracle (whose byte streams
and selections are pinned to the reference in tests/test_oracle_golden.py).

Bars: GQT1 bytes identical; index sets identical (ties included); float64
results within 1e-12 relative of the oracle where both compute in float64
from fp16-exact inputs; reconstructions from fp16 blob parameters within the
reference's own round-trip tolerance (rtol 2e-3, atol 1e-2)."""

import struct
from pathlib import Path

import numpy as np
import pytest

import cases
from oracle import tailorkv_oracle as O

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def H():
    import paper_2505_19586_b200.hybridkv as hybridkv

    return hybridkv


def f16(x):
    return np.asarray(x, np.float64).astype(np.float16).astype(np.float64)


SHAPES = [(133, 128, 1, 64), (200, 64, 2, 32), (77, 32, 1, 16), (64, 128, 2, 64), (300, 256, 1, 128),
          (5, 32, 2, 16)]


def _ref_tensor(m, axis, bits, g):
    return O.quantize_keys(m, bits, g) if axis == "keys" else O.quantize_values(m, bits, g)


@pytest.mark.parametrize("axis", ["keys", "values"])
@pytest.mark.parametrize("n,d,bits,g", SHAPES, ids=str)
def test_group_quantized_tensor_matches_reference_codec(H, n, d, bits, g, axis):
    rng = np.random.default_rng(n * d + bits)
    m = f16(rng.normal(size=(n, d)))
    ax = H.GroupAxis.PER_CHANNEL if axis == "keys" else H.GroupAxis.PER_TOKEN
    t = H.GroupQuantizedTensor.from_matrix(m, ax, bits, g)
    ref = _ref_tensor(m, axis, bits, g)
    blob = t.to_bytes()
    assert blob == ref.to_bytes()
    assert t.logical_shape == (n, d)
    assert t.num_complete_rows == ref.codes.shape[0]
    assert t.num_groups == ref.lo.size
    plen = struct.unpack("<I", blob[20:24])[0]
    assert t.packed_codes().tobytes() == blob[24:24 + plen]
    np.testing.assert_allclose(t.dequantize(), ref.dequantize(), rtol=1e-6, atol=1e-6)
    if axis == "keys":
        np.testing.assert_array_equal(t.residual, ref.residual)
    for i in (0, t.num_groups // 2, t.num_groups - 1) if t.num_groups else ():
        p = t.group_params(i)
        assert p.zero_point == ref.lo.reshape(-1)[i] and p.scale == ref.scale.reshape(-1)[i]
    with pytest.raises(H.ParameterError):
        t.group_params(t.num_groups)


def _blob_dequant(blob):
    """Reconstruction from a GQT1 blob's own fp16 parameters (what the
    reference's from_bytes(...).dequantize() returns), restated here."""
    _, bits, axis, g, rows, d, res, plen = struct.unpack("<4sBBHIIII", blob[:24])
    codes = O.unpack_codes(np.frombuffer(blob[24:24 + plen], np.uint8), bits, rows * d)
    gr, gc = (rows // g, d) if axis == 1 else (rows, -(-d // g))
    off = 24 + plen
    zp = np.frombuffer(blob[off:off + 2 * gr * gc], "<f2").astype(np.float64).reshape(gr, gc)
    sc = np.frombuffer(blob[off + 2 * gr * gc:off + 4 * gr * gc], "<f2").astype(np.float64).reshape(gr, gc)
    rs = np.frombuffer(blob[off + 4 * gr * gc:off + 4 * gr * gc + 2 * res * d], "<f2").astype(np.float64)
    if axis == 1:
        c = codes.reshape(gr, d, g).transpose(0, 2, 1).reshape(rows, d)
        x = c * np.repeat(sc, g, axis=0) + np.repeat(zp, g, axis=0)
        return np.vstack([x, rs.reshape(res, d)])
    c = codes.reshape(rows, d)
    cols = np.arange(d) // g
    return c * sc[:, cols] + zp[:, cols]


@pytest.mark.parametrize("axis", ["keys", "values"])
@pytest.mark.parametrize("n,d,bits,g", SHAPES, ids=str)
def test_gqt1_import_roundtrip(H, n, d, bits, g, axis):
    """GroupQuantizedTensor.from_bytes into HBM (quantizer.py:383-422): a blob
    of the reference codec re-exports byte-identically, reconstructs within
    the reference's round-trip tolerance, and decodes like the original."""
    rng = np.random.default_rng(7 * n + d)
    m = f16(rng.normal(size=(n, d)) * 3.0 + 1.0)
    blob = _ref_tensor(m, axis, bits, g).to_bytes()
    t = H.GroupQuantizedTensor.from_bytes(blob)
    assert t.axis is (H.GroupAxis.PER_CHANNEL if axis == "keys" else H.GroupAxis.PER_TOKEN)
    assert t.to_bytes() == blob
    np.testing.assert_allclose(t.dequantize(), _blob_dequant(blob), rtol=2e-3, atol=1e-2)
    q = rng.normal(size=d)
    if axis == "keys" and n >= 1:
        np.testing.assert_allclose(H.qgemv_scores(q, t), t.dequantize() @ q, rtol=1e-3, atol=1e-6)
    if axis == "values":
        w = rng.uniform(size=n)
        w /= w.sum()
        np.testing.assert_allclose(H.qgemv_output(w, t), w @ t.dequantize(), rtol=1e-3, atol=1e-6)


def test_gqt1_import_rejects_bad_blobs(H):
    m = f16(np.random.default_rng(1).normal(size=(64, 32)))
    blob = O.quantize_values(m, 1, 32).to_bytes()
    with pytest.raises(H.EncodingError):
        H.GroupQuantizedTensor.from_bytes(blob[:len(blob) // 2])
    with pytest.raises(H.EncodingError):
        H.GroupQuantizedTensor.from_bytes(b"XQT1" + blob[4:])
    with pytest.raises(H.EncodingError):
        H.GroupQuantizedTensor.from_bytes(blob[:10])


@pytest.mark.parametrize("bits", [1, 2])
@pytest.mark.parametrize("axis", ["keys", "values"])
def test_incremental_append_equals_batch(H, axis, bits):
    rng = np.random.default_rng(11 + bits)
    m = f16(rng.normal(size=(150, 64)))
    ax = H.GroupAxis.PER_CHANNEL if axis == "keys" else H.GroupAxis.PER_TOKEN
    t = H.GroupQuantizedTensor.from_matrix(m[:37], ax, bits, 16)
    t.append_rows(m[37:80])
    t.append_rows(m[80])
    t.append_rows(m[81:])
    assert t.to_bytes() == _ref_tensor(m, axis, bits, 16).to_bytes()


@pytest.mark.parametrize("n", [40, 5000, 131072])
def test_qgemv_matches_reference(H, n):
    rng = np.random.default_rng(n)
    K = f16(rng.normal(size=(n, 128)) * 0.3)
    V = f16(rng.normal(size=(n, 128)))
    kt = H.GroupQuantizedTensor.from_matrix(K, H.GroupAxis.PER_CHANNEL, 1, 64)
    vt = H.GroupQuantizedTensor.from_matrix(V, H.GroupAxis.PER_TOKEN, 1, 64)
    q = rng.normal(size=128)
    w = rng.uniform(size=n)
    w /= w.sum()
    np.testing.assert_allclose(H.qgemv_scores(q, kt), O.qgemv_scores(q, O.quantize_keys(K, 1, 64)), rtol=1e-12,
                               atol=1e-12)
    np.testing.assert_allclose(H.qgemv_output(w, vt), O.qgemv_output(w, O.quantize_values(V, 1, 64)), rtol=1e-12,
                               atol=1e-13)
    with pytest.raises(H.ShapeError):
        H.qgemv_scores(q, vt)
    with pytest.raises(H.ShapeError):
        H.qgemv_output(w, kt)


def test_scalar_like_cases(H):
    # identical tokens with uniform weights reproduce the token; one-hot weights pick one row
    row = np.arange(32.0)
    t = H.GroupQuantizedTensor.from_matrix(np.tile(row, (5, 1)), H.GroupAxis.PER_TOKEN, 1, 16)
    np.testing.assert_allclose(H.qgemv_output(np.full(5, 0.2), t), t.dequantize()[0], atol=1e-12)
    w = np.zeros(5)
    w[3] = 1.0
    np.testing.assert_allclose(H.qgemv_output(w, t), t.dequantize()[3], atol=1e-12)
    # all-zero keys: zero logits
    z = H.GroupQuantizedTensor.from_matrix(np.zeros((64, 32)), H.GroupAxis.PER_CHANNEL, 2, 16)
    np.testing.assert_array_equal(H.qgemv_scores(np.ones(32), z), np.zeros(64))


def test_quantize_layer_kv_append_and_decode(H):
    rng = np.random.default_rng(5)
    h, n, d, G = 4, 1000, 128, 4
    K = f16(rng.normal(size=(h, n, d)) * 0.2)
    V = f16(rng.normal(size=(h, n, d)))
    cache = H.LayerKV.from_arrays(K, V)
    q = H.quantize_layer_kv(cache, 1, 64)
    assert q.num_heads == h and q.seq_len == n
    kq, vq = O.quantize_layer(K, V, 1, 64)
    for u in range(h):
        assert q.keys[u].to_bytes() == kq[u].to_bytes()
        assert q.values[u].to_bytes() == vq[u].to_bytes()
    for _ in range(70):  # across a key-group boundary
        nk, nv = f16(rng.normal(size=(h, d)) * 0.2), f16(rng.normal(size=(h, d)))
        q.append_token(nk, nv)
        cache.append(nk, nv)
        for u in range(h):
            kq[u].append(nk[u])
            vq[u].append(nv[u])
    assert q.seq_len == n + 70 == cache.seq_len
    for u in range(h):
        assert q.keys[u].to_bytes() == kq[u].to_bytes()
        assert q.values[u].to_bytes() == vq[u].to_bytes()
    queries = f16(rng.normal(size=(h * G, d)))
    out = q.decode(queries)
    ref = O.quant_layer_decode(queries, kq, vq)
    for a, b in zip(out, ref):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 2e-3
    with pytest.raises(H.EmptyCacheError):
        H.quantize_layer_kv(H.LayerKV(2, 64), 1, 64)
    with pytest.raises(H.ShapeError):
        q.append_token(np.zeros((h, d + 1)), np.zeros((h, d + 1)))


def test_layer_kv_container(H):
    c = H.LayerKV(2, 32)
    assert c.seq_len == 0 and c.keys.shape == (2, 0, 32)
    for i in range(40):
        H.append_kv(c, np.full((2, 32), float(i)), np.full((2, 32), -float(i)))
    assert c.seq_len == 40 and c.keys[1, 39, 0] == 39.0 and c.values[0, 7, 5] == -7.0
    with pytest.raises(H.ShapeError):
        c.append(np.zeros((3, 32)), np.zeros((3, 32)))
    with pytest.raises(H.NumericError):
        c.append(np.full((2, 32), np.nan), np.zeros((2, 32)))
    with pytest.raises(H.ShapeError):
        H.LayerKV.from_arrays(np.zeros((2, 3, 4)), np.zeros((2, 3, 5)))


def test_retriever_functions_match_reference(H):
    rng = np.random.default_rng(9)
    hq, hid, d, G = 8, 1024, 128, 4
    w_q = f16(rng.normal(size=(hq, hid, d)) / np.sqrt(hid))
    h = f16(rng.normal(size=hid))
    est = H.estimate_query(w_q, h, source_layer=3)
    assert est.source_layer == 3
    np.testing.assert_allclose(est.q_hat, O.estimate_query(w_q, h), rtol=2e-5, atol=1e-6)
    chmax = np.abs(rng.normal(size=d)) + 0.1
    qg = est.q_hat[:G]
    gs = H.group_channel_scores(qg, chmax)
    np.testing.assert_array_equal(gs, O.group_channel_scores(qg, chmax))
    np.testing.assert_array_equal(H.channel_scores_from_max(qg[0], chmax), np.abs(qg[0]) * chmax)
    # channel ties break toward the lower index (retriever.py:161)
    tied = np.array([1.0, 3.0, 3.0, 0.5, 3.0, 2.0, 2.0, 0.0])
    for ds in (1, 2, 3, 4, 6, 8):
        sel = H.select_critical_channels(tied, ds)
        np.testing.assert_array_equal(sel.selected, O.select_channels(tied, ds))
    sel = H.select_critical_channels(gs, 8)
    np.testing.assert_array_equal(sel.selected, O.select_channels(gs, 8))
    with pytest.raises(H.ParameterError):
        H.select_critical_channels(gs, 0)
    # proxy scores, top-k (ties to the more recent index), sparse attention
    n = 4000
    keys = f16(rng.normal(size=(n, d)))
    values = f16(rng.normal(size=(n, d)))
    qry = f16(rng.normal(size=(G, d)))
    crit = keys[:, sel.selected]
    sc = H.approx_scores(qry[:, sel.selected], crit)
    np.testing.assert_allclose(sc, O.approx_scores(qry[:, sel.selected], crit), rtol=1e-12, atol=1e-12)
    scr = np.round(sc)  # heavy exact ties
    cfg = H.RetrievalConfig(n_local=16, n_topk=100, d_s=8)
    chosen = H.select_topk_tokens(scr, cfg)
    np.testing.assert_array_equal(chosen, O.select_tokens(scr, 16, 100))
    out = H.sparse_attention(qry[0], keys, values, chosen)
    np.testing.assert_allclose(out, O.sparse_attention(qry[0], keys, values, chosen), rtol=1e-12, atol=1e-13)
    with pytest.raises(H.EmptyCacheError):
        H.sparse_attention(qry[0], keys, values, np.array([], dtype=int))
    with pytest.raises(H.ParameterError):
        H.sparse_attention(qry[0], keys, values, np.array([n]))
    wts = H.attention_weights(qry[0], keys)
    np.testing.assert_allclose(wts, O.attention_weights(qry[0], keys), rtol=1e-12, atol=1e-15)
    assert abs(wts.sum() - 1.0) < 1e-12
    tw = H.top_weight_tokens(np.round(wts * 1e3) / 1e3, 50)
    np.testing.assert_array_equal(tw, O.top_weight_tokens(np.round(wts * 1e3) / 1e3, 50))
    assert H.recall_at_k(chosen, tw) == O.recall_at_k(chosen, tw)
    np.testing.assert_allclose(H.exact_attention(qry[1], keys, values), O.attention_weights(qry[1], keys) @ values,
                               rtol=1e-12, atol=1e-13)
    cache = H.LayerKV.from_arrays(np.stack([keys, keys[::-1]]), np.stack([values, values[::-1]]))
    qs = f16(rng.normal(size=(8, d)))
    np.testing.assert_allclose(H.layer_attention(qs, cache), O.exact_layer_attention(qs, cache.keys, cache.values),
                               rtol=1e-12, atol=1e-13)
    with pytest.raises(H.ShapeError):
        H.attention_weights(qry[0][:5], keys)


def test_host_pool_and_transfers(H):
    """HostPool on the pinned store (memsim.py:76-135), transfers and their
    byte accounting (memsim.py:196-252; the reference's 24,000 / 65,536 B)."""
    rng = np.random.default_rng(4)
    K = f16(rng.normal(size=(2, 1000, 32)))
    V = f16(rng.normal(size=(2, 1000, 32)))
    pool = H.HostPool()
    pool.offload_layer(3, H.LayerKV.from_arrays(K, V))
    assert pool.has_layer(3) and not pool.has_layer(0) and pool.seq_len(3) == 1000
    with pytest.raises(H.SchedulingError):
        pool.offload_layer(3, H.LayerKV.from_arrays(K, V))
    idx = np.array([999, 0, 17, 17, 500])
    k, v = pool.gather(3, 1, idx)
    np.testing.assert_array_equal(k, K[1][idx])
    np.testing.assert_array_equal(v, V[1][idx])
    k0, v0 = pool.gather(3, 0, np.array([], dtype=int))
    assert k0.shape == (0, 32)
    with pytest.raises(H.ParameterError):
        pool.gather(3, 0, np.array([1000]))
    with pytest.raises(H.ParameterError):
        pool.gather(7, 0, np.array([0]))
    np.testing.assert_array_equal(pool.channel_abs_max(3), np.abs(K).max(axis=1))
    nk = f16(rng.normal(size=(2, 32)) * 50)
    pool.append(3, nk, f16(rng.normal(size=(2, 32))))
    assert pool.seq_len(3) == 1001
    np.testing.assert_array_equal(pool.channel_abs_max(3), np.maximum(np.abs(K).max(axis=1), np.abs(nk)))
    np.testing.assert_array_equal(pool.gather(3, 0, np.array([1000]))[0][0], nk[0])
    cols = pool.gather_key_columns(3, 1, np.array([1, 4, 6]))
    np.testing.assert_array_equal(cols[:1000], K[1][:, [1, 4, 6]])
    buffers = H.DeviceBuffers(2, 32)
    req = H.prefetch_critical_keys(pool, 3, [np.arange(12), np.arange(12)], buffers, step=0)
    assert req.nbytes == 2 * 1001 * 12 * 2 and req.label == "prefetch"
    content = buffers.read_slot(0)
    np.testing.assert_array_equal(content[1][1][:1000], K[1][:, :12])
    with pytest.raises(H.SchedulingError):
        buffers.read_slot(1)
    buffers.begin_prefetch(1)
    with pytest.raises(H.SchedulingError):
        buffers.begin_prefetch(3)
    single = H.HostPool()
    single.offload_layer(0, H.LayerKV.from_arrays(f16(rng.normal(size=(1, 1000, 32))),
                                                  f16(rng.normal(size=(1, 1000, 32)))))
    assert H.prefetch_critical_keys(single, 0, [np.arange(12)], H.DeviceBuffers(1, 32), step=0).nbytes == 24_000
    big = H.HostPool()
    big.offload_layer(0, H.LayerKV.from_arrays(f16(rng.normal(size=(1, 200, 128))),
                                               f16(rng.normal(size=(1, 200, 128)))))
    rows, req = H.fetch_topk(big, 0, [np.arange(128)], None, step=0)
    assert req.nbytes == 65_536 and rows[0][0].shape == (128, 128)
    _, req0 = H.fetch_topk(pool, 3, [np.array([], dtype=int)] * 2, None, step=0)
    assert req0.nbytes == 0


def test_sparse_error_and_calibrate_trace(H):
    rng = np.random.default_rng(2)
    logits = rng.normal(size=5000) * 3
    w = np.exp(logits - logits.max())
    w /= w.sum()
    for k in (1, 250, 4999, 5000):
        assert H.sparse_error(w, k) == pytest.approx(O.sparse_error(w, k), rel=1e-12, abs=1e-15)
    with pytest.raises(H.ParameterError):
        H.sparse_error(w, 0)
    trace = H.read_trace(GOLD / "tiny_trace.hkv")
    ref = O.read_trace_file(GOLD / "tiny_trace.hkv")
    assert trace.prefill_len == ref["prefill_keys"][0].shape[1] and trace.num_steps == len(ref["steps"])
    np.testing.assert_array_equal(trace.prefill[1].keys, ref["prefill_keys"][1])
    np.testing.assert_array_equal(trace.steps[-1].queries, ref["steps"][-1]["queries"])
    k = H.default_probe_k(trace.prefill_len)
    n_q = min(32, ref["prefill_queries"][0].shape[1])
    probe = H.SparsityProbe(k=k, n_q=n_q, tau=0.2)
    prof = H.calibrate(trace, probe)
    orc = O.calibrate(ref["prefill_queries"], ref["prefill_keys"], k, n_q=n_q, tau=0.2)
    for p, (hs, m, label) in zip(prof, orc):
        np.testing.assert_allclose(p.per_head_scores, hs, rtol=1e-5, atol=1e-6)
        assert p.label.value == label
    with pytest.raises(H.ParameterError):
        H.calibrate(trace, H.SparsityProbe(k=trace.prefill_len + 1, n_q=n_q))
