"""Generate golden vectors by running the REFERENCE package (hybridkv).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports ``hybridkv`` read-only from /root/reference/pkg/src and writes
small fixtures next to this file.  The GPU box never runs this script; the
fixtures it produced are committed.  Inputs are regenerated from seeds by
``tests/golden/cases.py`` (shared with the tests) so only outputs and
digests are stored.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import cases  # noqa: E402
from hybridkv import quantizer as Rq  # noqa: E402
from hybridkv import retriever as Rr  # noqa: E402
from hybridkv import identifier as Ri  # noqa: E402
from hybridkv.kv_model import LayerKV  # noqa: E402
from hybridkv.pipeline import PipelineConfig, _stable_softmax, run_pipeline  # noqa: E402
from hybridkv.trace import SyntheticSpec, dense, gen_trace, sparse, write_trace  # noqa: E402


def sel_hex(selected) -> str:
    """Selected token set as a little-endian bitmap in hex (compact fixture)."""
    return cases.indices_to_hex(selected)


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def pack_cases() -> dict:
    out = {}
    for c in cases.PACK_CASES:
        k, v = cases.pack_inputs(c)
        kt = Rq.GroupQuantizedTensor.from_matrix(k, Rq.GroupAxis.PER_CHANNEL, c["bits"], c["g"])
        vt = Rq.GroupQuantizedTensor.from_matrix(v, Rq.GroupAxis.PER_TOKEN, c["bits"], c["g"])
        kb, vb = kt.to_bytes(), vt.to_bytes()
        out[c["name"]] = {
            "keys_sha256": sha(kb), "keys_len": len(kb),
            "values_sha256": sha(vb), "values_len": len(vb),
            "keys_packed_sha256": sha(kt.packed_codes().tobytes()),
            "values_packed_sha256": sha(vt.packed_codes().tobytes()),
            "key_residual_rows": int(kt.residual.shape[0]),
        }
    return out


def decode_cases() -> dict:
    arrs = {}
    for c in cases.DECODE_CASES:
        keys, values, queries = cases.decode_inputs(c)
        q = Rq.quantize_layer_kv(LayerKV.from_arrays(keys, values), c["bits"], c["g"])
        hq, d = queries.shape
        grp = hq // keys.shape[0]
        out = np.empty_like(queries)
        logits0 = None
        for qh in range(hq):
            kvh = qh // grp
            logits = Rq.qgemv_scores(queries[qh], q.keys[kvh])
            if qh == 0:
                logits0 = logits
            w = _stable_softmax(logits / np.sqrt(d))
            out[qh] = Rq.qgemv_output(w, q.values[kvh])
        arrs[c["name"] + "/out"] = out
        arrs[c["name"] + "/logits0"] = logits0
    return arrs


def topk_cases() -> tuple[dict, dict]:
    arrs, meta = {}, {}
    for c in cases.TOPK_CASES:
        scores = cases.topk_scores(c)
        cfg = Rr.RetrievalConfig(n_local=c["n_local"], n_topk=c["n_topk"])
        arrs[c["name"]] = Rr.select_topk_tokens(scores, cfg)
    for c in cases.CHANNEL_CASES:
        qhat, chmax = cases.channel_inputs(c)
        s = Rr.group_channel_scores(qhat, chmax)
        arrs[c["name"]] = Rr.select_critical_channels(s, c["d_s"]).selected
    return arrs, meta


def pipeline_cases() -> tuple[dict, dict]:
    spec = SyntheticSpec(
        modes=(dense(), sparse(4, 0.99), sparse(4, 0.99)),
        num_query_heads=4, num_kv_heads=2, head_dim=64,
        prefill_len=136, num_steps=72, seed=2505,
    )
    trace = gen_trace(spec)
    arrs = {
        "prefill_keys": np.stack([p.keys for p in trace.prefill]).astype(np.float16),
        "prefill_values": np.stack([p.values for p in trace.prefill]).astype(np.float16),
        "prefill_queries_tail": np.stack([q[:, -32:, :] for q in trace.prefill_queries]).astype(np.float16),
        "w_q": np.stack(trace.w_q).astype(np.float16),
        "hidden": np.stack([s.hidden for s in trace.steps]).astype(np.float16),
        "queries": np.stack([s.queries for s in trace.steps]).astype(np.float16),
        "new_keys": np.stack([s.new_keys for s in trace.steps]).astype(np.float16),
        "new_values": np.stack([s.new_values for s in trace.steps]).astype(np.float16),
    }
    meta = {"spec": spec.to_dict(), "runs": {}}
    for name, cfg in cases.PIPELINE_CONFIGS.items():
        report = run_pipeline(trace, PipelineConfig(**cfg))
        meta["runs"][name] = {
            "config": cfg,
            "labels": report.labels,
            "profiles": report.profiles,
            "cosine": report.cosine,
            "max_abs_err": report.max_abs_err,
            "recall": report.recall,
            "selected_mass": report.selected_mass,
            "retrieval": [
                {"layer": r["layer"], "step": r["step"],
                 "per_head": [{"channels": ph["channels"], "fetched": ph["fetched"],
                               "selected_hex": sel_hex(ph["selected"])} for ph in r["per_head"]]}
                for r in report.retrieval
            ],
        }
    # a tiny HKVTRACE file to pin the trace reader (trace.py:105-228)
    tiny = gen_trace(SyntheticSpec(modes=(dense(), sparse(2, 0.99)), num_query_heads=2,
                                   num_kv_heads=1, head_dim=32, prefill_len=24, num_steps=2, seed=5))
    write_trace(tiny, HERE / "tiny_trace.hkv")
    meta["tiny_trace"] = {
        "first_key": float(tiny.prefill[0].keys[0, 0, 0]),
        "last_new_value": float(tiny.steps[-1].new_values[-1, -1, -1]),
        "w_q_sum": float(sum(w.sum() for w in tiny.w_q)),
    }
    return arrs, meta


def calibrate_cases() -> tuple[dict, dict]:
    arrs, meta = {}, {}
    for c in cases.CALIB_CASES:
        pq, pk = cases.calib_inputs(c)
        k = Ri.default_probe_k(pk.shape[2])
        per_layer = []
        for l in range(pk.shape[0]):
            hq, n, _ = pq[l].shape
            grp = hq // pk.shape[1]
            hs = [Ri.dense_preference_score(pq[l][qh, n - c["n_q"]:], pk[l][qh // grp], k)
                  for qh in range(hq)]
            prof = Ri.classify_layer(l, hs, c["tau"])
            per_layer.append({"scores": list(prof.per_head_scores), "score": prof.score,
                              "label": prof.label.value})
        meta[c["name"]] = {"k": k, "layers": per_layer}
    return arrs, meta


def main() -> None:
    meta = {"pack": pack_cases()}
    arrs = decode_cases()
    a, _ = topk_cases()
    arrs.update(a)
    np.savez_compressed(HERE / "kernels.npz", **arrs)
    pa, pm = pipeline_cases()
    np.savez_compressed(HERE / "pipeline_trace.npz", **pa)
    meta["pipeline"] = pm
    _, cm = calibrate_cases()
    meta["calibrate"] = cm
    (HERE / "golden.json").write_text(json.dumps(meta, sort_keys=True, separators=(",", ":")))
    print("wrote", sorted(p.name for p in HERE.iterdir()))


if __name__ == "__main__":
    main()
