"""Pin the CPU oracle to the reference: KATs from the reference's own tests
plus golden vectors produced by running the reference (tests/golden)."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import cases
from oracle import tailorkv_oracle as O

GOLD = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLD / "golden.json").read_text())
KER = np.load(GOLD / "kernels.npz")


def sha(b):
    return hashlib.sha256(b).hexdigest()


# -- known-answer tests restated from the reference suite --------------------


def test_bit_order_kats():
    # test_quantizer.py:118-124
    assert O.pack_codes([1, 0, 1, 1, 0, 0, 0, 1], 1).tolist() == [0b10001101]
    assert O.pack_codes([3, 0, 1, 2], 2).tolist() == [0b10010011]


def test_param_kats():
    # test_quantizer.py:41-52
    assert O.group_scale(0.0, 3.0, 2) == 1.0
    assert O.group_scale(-1.0, 3.0, 1) == 4.0
    assert O.group_scale(5.0, 5.0, 1) == 1.0
    assert O.encode([-1.0, 3.0], -1.0, 4.0, 1).tolist() == [0, 1]


def test_key_stream_order_kat():
    # test_quantizer.py:196-202
    t = O.quantize_keys(np.arange(8.0).reshape(4, 2), 1, 2)
    assert O.unpack_codes(O.pack_codes(t.code_stream(), 1), 1, 8).tolist() == [0, 1] * 4


def test_channel_score_kats():
    # test_retriever.py:53-77, 84-103
    assert O.group_channel_scores(np.array([1.0, -3.0, 0.5]), np.array([2.0, 1.0, 4.0])).tolist() == [2.0, 3.0, 2.0]
    assert O.group_channel_scores(np.array([[1.0, -1.0], [-2.0, 3.0]]), np.array([1.0, 2.0])).tolist() == [3.0, 8.0]
    assert O.select_channels(np.array([5.0, 5.0, 1.0]), 1).tolist() == [0]
    assert O.select_channels(np.array([1.0, 9.0, 3.0, 8.0]), 2).tolist() == [1, 3]


def test_topk_kats():
    # test_retriever.py:151-171
    assert O.select_tokens(np.zeros(10), 2, 3).tolist() == [5, 6, 7, 8, 9]
    assert O.select_tokens(np.ones(10), 4, 8).tolist() == list(range(10))


def test_pack_roundtrip_random():
    rng = np.random.default_rng(1)
    for bits in (1, 2):
        c = rng.integers(0, 2**bits, size=10_001).astype(np.uint8)
        assert np.array_equal(O.unpack_codes(O.pack_codes(c, bits), bits, c.size), c)


# -- golden vectors from the reference ---------------------------------------


@pytest.mark.parametrize("case", cases.PACK_CASES, ids=lambda c: c["name"])
def test_pack_golden(case):
    k, v = cases.pack_inputs(case)
    g = META["pack"][case["name"]]
    with np.errstate(over="ignore"):
        kb = O.quantize_keys(k, case["bits"], case["g"]).to_bytes()
        vb = O.quantize_values(v, case["bits"], case["g"]).to_bytes()
    assert sha(kb) == g["keys_sha256"] and len(kb) == g["keys_len"]
    assert sha(vb) == g["values_sha256"] and len(vb) == g["values_len"]


def test_incremental_append_matches_batch():
    # test_quantizer.py:204-222 restated on the oracle
    rng = np.random.default_rng(5)
    k = cases.f16(rng.normal(size=(70, 8)))
    t = O.quantize_keys(k[:69], 1, 16)
    t.append(k[69])
    full = O.quantize_keys(k, 1, 16)
    assert t.to_bytes() == full.to_bytes()


@pytest.mark.parametrize("case", cases.DECODE_CASES, ids=lambda c: c["name"])
def test_quant_decode_golden(case):
    keys, values, queries = cases.decode_inputs(case)
    kq, vq = O.quantize_layer(keys, values, case["bits"], case["g"])
    out = O.quant_layer_decode(queries, kq, vq)
    np.testing.assert_allclose(out, KER[case["name"] + "/out"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(O.qgemv_scores(queries[0], kq[0]), KER[case["name"] + "/logits0"],
                               rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("case", cases.TOPK_CASES, ids=lambda c: c["name"])
def test_topk_golden(case):
    sel = O.select_tokens(cases.topk_scores(case), case["n_local"], case["n_topk"])
    assert np.array_equal(sel, KER[case["name"]])


@pytest.mark.parametrize("case", cases.CHANNEL_CASES, ids=lambda c: c["name"])
def test_channels_golden(case):
    qhat, chmax = cases.channel_inputs(case)
    sel = O.select_channels(O.group_channel_scores(qhat, chmax), case["d_s"])
    assert np.array_equal(sel, KER[case["name"]])


def test_calibrate_golden():
    for c in cases.CALIB_CASES:
        pq, pk = cases.calib_inputs(c)
        g = META["calibrate"][c["name"]]
        got = O.calibrate(list(pq), list(pk), g["k"], n_q=c["n_q"], tau=c["tau"])
        for (hs, m, lab), ref in zip(got, g["layers"]):
            np.testing.assert_allclose(hs, ref["scores"], rtol=1e-12)
            assert lab == ref["label"]


def load_pipeline_trace():
    z = np.load(GOLD / "pipeline_trace.npz")
    T = z["queries"].shape[0]
    steps = [{"hidden": z["hidden"][t].astype(np.float64), "queries": z["queries"][t].astype(np.float64),
              "new_keys": z["new_keys"][t].astype(np.float64),
              "new_values": z["new_values"][t].astype(np.float64)} for t in range(T)]
    return z, steps


@pytest.mark.parametrize("run", list(cases.PIPELINE_CONFIGS), ids=str)
def test_replay_matches_reference_pipeline(run):
    z, steps = load_pipeline_trace()
    ref = META["pipeline"]["runs"][run]
    cfg = {"bits": 1, "g": 64, "n_local": 64, "n_topk": 128, "d_s": 8}
    rc = ref["config"]
    cfg.update({k2: rc[k1] for k1, k2 in (("bits", "bits"), ("n_local", "n_local"),
                                          ("n_topk", "n_topk"), ("critical_channels", "d_s"))
                if k1 in rc})
    labels = ["q" if lab == "quantization_friendly" else "s" for lab in ref["labels"]]
    res = O.replay(list(z["prefill_keys"].astype(np.float64)), list(z["prefill_values"].astype(np.float64)),
                   list(z["w_q"].astype(np.float64)), steps, labels, **cfg)
    for rec in ref["retrieval"]:
        l, t = rec["layer"], rec["step"]
        for kvh, ph in enumerate(rec["per_head"]):
            assert res.channels[(l, t)][kvh].tolist() == ph["channels"]
            assert np.array_equal(res.selected[(l, t)][kvh], cases.hex_to_indices(ph["selected_hex"]))
            assert res.fetched[(l, t)][kvh] == ph["fetched"]
    for t in range(len(steps)):
        for l in range(len(labels)):
            a, b = res.outputs[t][l].reshape(-1), res.exact[t][l].reshape(-1)
            cos = float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b)))
            assert abs(cos - ref["cosine"][l][t]) < 1e-9


def test_trace_reader_pins_reference_writer():
    tr = O.read_trace_file(GOLD / "tiny_trace.hkv")
    m = META["pipeline"]["tiny_trace"]
    assert tr["prefill_keys"][0][0, 0, 0] == m["first_key"]
    assert tr["steps"][-1]["new_values"][-1, -1, -1] == m["last_new_value"]
    assert abs(sum(w.sum() for w in tr["w_q"]) - m["w_q_sum"]) < 1e-9


def test_byte_formulas():
    # Table-2 bytes at config 2 (test_memsim.py:379-399): 50,331,648 per layer
    assert O.quant_layer_bytes(131072, 8, 128, 1, 64) == 50_331_648
    assert O.scorer_bytes(131072, 8, 8) == 16_777_216
    assert O.gather_bytes(2621 * 8, 128) == 10_735_616


def test_package_trace_reader_matches_oracle_reader():
    """The engine's HKVTRACE loader (fp16 tensors, no float64 round trip)
    returns the same arrays as the oracle's restatement of trace.py."""
    from paper_2505_19586_b200.trace import load_trace

    ref = O.read_trace_file(GOLD / "tiny_trace.hkv")
    tr = load_trace(GOLD / "tiny_trace.hkv")
    for l in range(len(ref["prefill_keys"])):
        assert np.array_equal(tr.prefill_keys[l].double().numpy(), ref["prefill_keys"][l])
        assert np.array_equal(tr.prefill_values[l].double().numpy(), ref["prefill_values"][l])
        assert np.array_equal(tr.w_q[l].double().numpy(), ref["w_q"][l])
    for t, st in enumerate(ref["steps"]):
        assert np.array_equal(tr.queries[t].double().numpy(), st["queries"])
        assert np.array_equal(tr.new_values[t].double().numpy(), st["new_values"])
        assert np.array_equal(tr.hidden[t].double().numpy(), st["hidden"])


def test_package_trace_reader_errors(tmp_path):
    from paper_2505_19586_b200.errors import TraceFormatError
    from paper_2505_19586_b200.trace import load_trace

    blob = (GOLD / "tiny_trace.hkv").read_bytes()
    bad = tmp_path / "bad_magic.hkv"
    bad.write_bytes(b"NOTATRACE" + blob[9:])
    with pytest.raises(TraceFormatError):
        load_trace(bad)
    tampered = tmp_path / "tampered.hkv"
    tampered.write_bytes(blob[:-2] + bytes([blob[-2] ^ 1, blob[-1]]))
    with pytest.raises(TraceFormatError):
        load_trace(tampered)


def test_timeline_model_matches_reference_golden():
    """tools/timeline_model.py (the reference's decode-step timeline model, memsim.py:339-602)
    reproduces the reference's schedule: every event start, total time, overlap and stall
    (tests/golden/timeline.json, made by tests/golden/make_timeline_golden.py)."""
    import json
    from pathlib import Path

    from tools import timeline_model as T

    cases = json.loads((Path(__file__).parent / "golden" / "timeline.json").read_text())
    for c in cases:
        ev = T.build_timeline(c["labels"], T.LayerCosts(tuple(c["compute"]), c["estimate"], c["score"]),
                              T.LinkModel(c["bandwidth"], c["latency"]), c["prefetch"], c["fetch"])
        assert [e.label for e in ev] == c["labels_ev"]
        r = T.simulate(ev)
        assert np.allclose([e.start for e in ev], c["starts"], rtol=0, atol=1e-15)
        assert r.total_seconds == pytest.approx(c["total"], abs=1e-15)
        assert r.overlap_fraction == pytest.approx(c["overlap"], abs=1e-12)
        assert r.stall_seconds == pytest.approx(c["stall"], abs=1e-15)
        for k, v in c["per_layer"].items():
            assert r.per_layer[int(k)] == pytest.approx(v, abs=1e-15)


def test_timeline_measured_step_model():
    """measured_step: the reference model has one compute engine, so its estimate passes serialise
    with the layers (this engine runs them on a side stream: estimate 0 models that); PCIe bytes
    on the link add their time to the chain they gate."""
    from tools import timeline_model as T

    labels = ["q", "q"] + ["s"] * 30
    serial = T.measured_step(labels, 45e-6, 43e-6, 37e-6, 0, 50e9)
    assert serial["step_seconds"] == pytest.approx(2 * 45e-6 + 30 * (43e-6 + 37e-6), rel=1e-9)
    base = T.measured_step(labels, 45e-6, 43e-6, 0.0, 0, 50e9)
    assert base["step_seconds"] == pytest.approx(2 * 45e-6 + 30 * 43e-6, rel=1e-9)
    more = T.measured_step(labels, 45e-6, 43e-6, 0.0, 29_000, 50e9)
    assert more["step_seconds"] == pytest.approx(base["step_seconds"] + 30 * 29_000 / 50e9, rel=1e-9)


def test_select_tokens_sinks_extension():
    """The sink extension reduces to the reference rule at n_sink = 0 and
    always keeps [0, n_sink) plus exactly n_topk others outside the window."""
    rng = np.random.default_rng(4)
    s = np.round(rng.normal(size=3000))
    assert np.array_equal(O.select_tokens_sinks(s, 16, 200, 0), O.select_tokens(s, 16, 200))
    sel = O.select_tokens_sinks(s, 16, 200, 5)
    assert sel.size == 16 + 200 + 5 and np.all(sel[:5] == np.arange(5))
    rest = sel[(sel >= 5) & (sel < 3000 - 16)]
    assert np.array_equal(rest, np.sort(O.select_tokens(s[5:], 16, 200)[:200] + 5))
    assert np.array_equal(O.select_tokens_sinks(s[:100], 16, 50, 40), np.arange(100))
