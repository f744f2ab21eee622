"""CPU oracle for the TailorKV decode hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``hybridkv``
(``/root/reference/pkg/src/hybridkv``) for exactly the functions on the hot
path named in SURVEY.md section 8(a).  It exists to *check* the B200 engine:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` leg may import it;
* the product package ``paper_2505_19586_b200`` never imports it and has no
  CPU fallback (its ops raise when the CUDA library is missing).

Parity pinning: every function below is checked against the reference's own
known-answer tests and against golden vectors produced by importing the
reference in the build container (``tests/golden/make_golden.py`` ->
``tests/golden/*.npz`` / ``*.json``; see ``tests/test_oracle_golden.py``).

Arithmetic follows the reference: float64 everywhere, inputs are fp16-exact
values (``kv_model.py:8-10``, ``trace.py:505-513``).  Each function cites the
reference lines it restates.
"""

from __future__ import annotations

import hashlib
import math
import struct
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# Codec (quantizer.py:66-117)
# ---------------------------------------------------------------------------


def round_half_away(x):
    """Round half away from zero (``quantizer.py:66-68``)."""
    x = np.asarray(x, dtype=np.float64)
    return np.sign(x) * np.floor(np.abs(x) + 0.5)


def group_scale(lo, hi, bits):
    """``(hi-lo)/(2^b-1)``, with a degenerate range mapped to 1.0
    (``quantizer.py:91-96``, ``:266-267``, ``:285-286``)."""
    s = (np.asarray(hi, np.float64) - np.asarray(lo, np.float64)) / float((1 << bits) - 1)
    return np.where(s == 0.0, 1.0, s)


def encode(x, lo, s, bits):
    """Codes ``clip(round_half_away((x-lo)/s), 0, 2^b-1)`` (``quantizer.py:99-107``)."""
    v = (np.asarray(x, np.float64) - lo) / s
    return np.clip(round_half_away(v), 0, (1 << bits) - 1).astype(np.uint8)


# ---------------------------------------------------------------------------
# Bit packing (quantizer.py:125-179)
# ---------------------------------------------------------------------------


def packed_size(count: int, bits: int) -> int:
    """``ceil(count*bits/8)`` (``quantizer.py:125-127``)."""
    return (count * bits + 7) // 8


def pack_codes(codes, bits: int) -> np.ndarray:
    """LSB-first packing: code i occupies bits [i*b, i*b+b) of the stream
    (``quantizer.py:130-151``; b=1 is ``np.packbits(bitorder='little')``)."""
    codes = np.asarray(codes, dtype=np.uint8).reshape(-1)
    per_byte = 8 // bits
    n = codes.size
    padded = np.zeros(((n + per_byte - 1) // per_byte) * per_byte, dtype=np.uint16)
    padded[:n] = codes
    lanes = padded.reshape(-1, per_byte)
    shifts = (np.arange(per_byte, dtype=np.uint16) * bits)
    return (lanes << shifts).sum(axis=1).astype(np.uint8)


def unpack_codes(data, bits: int, count: int) -> np.ndarray:
    """Inverse of :func:`pack_codes` (``quantizer.py:154-179``)."""
    data = np.asarray(data, dtype=np.uint8).reshape(-1)
    if data.size != packed_size(count, bits):
        raise ValueError("packed length does not match code count")
    per_byte = 8 // bits
    shifts = np.arange(per_byte, dtype=np.uint8) * bits
    out = (data[:, None] >> shifts) & ((1 << bits) - 1)
    return out.reshape(-1)[:count].astype(np.uint8)


# ---------------------------------------------------------------------------
# Group-quantized tensors (quantizer.py:187-422, 430-497)
# ---------------------------------------------------------------------------


@dataclass
class QTensor:
    """One KV head's quantized matrix (restates ``GroupQuantizedTensor``).

    ``axis`` is ``"channel"`` (keys: groups of g tokens within a channel,
    float residual for trailing rows) or ``"token"`` (values: groups of g
    channels within a token, ragged last block allowed, no residual).
    ``codes`` is unpacked ``[rows, d]``; ``lo``/``scale`` are the float64
    group grids (``quantizer.py:211-216``).
    """

    axis: str
    bits: int
    g: int
    d: int
    codes: np.ndarray = None
    lo: np.ndarray = None
    scale: np.ndarray = None
    residual: np.ndarray = None

    def __post_init__(self):
        cols = self.d if self.axis == "channel" else -(-self.d // self.g)
        if self.codes is None:
            self.codes = np.zeros((0, self.d), np.uint8)
            self.lo = np.zeros((0, cols))
            self.scale = np.zeros((0, cols))
            self.residual = np.zeros((0, self.d))

    @property
    def rows(self) -> int:
        return self.codes.shape[0]

    @property
    def length(self) -> int:
        return self.rows + self.residual.shape[0]

    # -- append (quantizer.py:238-293) ------------------------------------
    def append(self, rows) -> None:
        rows = np.asarray(rows, np.float64)
        if rows.ndim == 1:
            rows = rows[None, :]
        if self.axis == "token":
            self._append_token_groups(rows)
        else:
            self._append_channel_groups(rows)

    def _append_token_groups(self, rows):
        # quantizer.py:252-275 -- per token, blocks of g channels
        if rows.shape[0] == 0:
            return
        nb = -(-self.d // self.g)
        lo = np.empty((rows.shape[0], nb))
        sc = np.empty((rows.shape[0], nb))
        codes = np.empty(rows.shape, np.uint8)
        for b in range(nb):
            c0, c1 = b * self.g, min((b + 1) * self.g, self.d)
            blk = rows[:, c0:c1]
            lo[:, b] = blk.min(axis=1)
            sc[:, b] = group_scale(lo[:, b], blk.max(axis=1), self.bits)
            codes[:, c0:c1] = encode(blk, lo[:, b : b + 1], sc[:, b : b + 1], self.bits)
        self.codes = np.vstack([self.codes, codes])
        self.lo = np.vstack([self.lo, lo])
        self.scale = np.vstack([self.scale, sc])

    def _append_channel_groups(self, rows):
        # quantizer.py:277-293 -- complete g-token groups leave the residual
        pend = np.vstack([self.residual, rows])
        full = (pend.shape[0] // self.g) * self.g
        if full:
            blk = pend[:full].reshape(-1, self.g, self.d)
            lo = blk.min(axis=1)
            sc = group_scale(lo, blk.max(axis=1), self.bits)
            codes = encode(blk, lo[:, None, :], sc[:, None, :], self.bits)
            self.codes = np.vstack([self.codes, codes.reshape(-1, self.d)])
            self.lo = np.vstack([self.lo, lo])
            self.scale = np.vstack([self.scale, sc])
        self.residual = pend[full:].copy()

    # -- stream + export (quantizer.py:327-380) ---------------------------
    def code_stream(self) -> np.ndarray:
        """Keys: (block, channel, token) order; values: row-major
        (``quantizer.py:327-333``)."""
        if self.axis == "token":
            return self.codes.reshape(-1)
        nb = self.rows // self.g
        return self.codes.reshape(nb, self.g, self.d).transpose(0, 2, 1).reshape(-1)

    def dequantize(self) -> np.ndarray:
        """``code*s+lo`` per group plus the residual (``quantizer.py:335-352``)."""
        if self.axis == "token":
            out = np.empty(self.codes.shape)
            for b in range(self.lo.shape[1]):
                c0, c1 = b * self.g, min((b + 1) * self.g, self.d)
                out[:, c0:c1] = self.codes[:, c0:c1] * self.scale[:, b : b + 1] + self.lo[:, b : b + 1]
        else:
            nb = self.rows // self.g
            c = self.codes.reshape(nb, self.g, self.d).astype(np.float64)
            out = (c * self.scale[:, None, :] + self.lo[:, None, :]).reshape(self.rows, self.d)
        return np.vstack([out, self.residual])

    def to_bytes(self) -> bytes:
        """GQT1 blob: ``<4sBBHIIII`` header, packed codes, zero-points fp16,
        scales fp16, residual fp16 (``quantizer.py:358-380``)."""
        packed = pack_codes(self.code_stream(), self.bits).tobytes()
        hdr = struct.pack(
            "<4sBBHIIII", b"GQT1", self.bits, 1 if self.axis == "channel" else 2,
            self.g, self.rows, self.d, self.residual.shape[0], len(packed),
        )
        return (hdr + packed + self.lo.astype("<f2").tobytes()
                + self.scale.astype("<f2").tobytes() + self.residual.astype("<f2").tobytes())


def quantize_keys(k, bits, g) -> QTensor:
    """Per-channel key quantization of one head (``quantizer.py:489-492``)."""
    t = QTensor("channel", bits, g, np.asarray(k).shape[1])
    t.append(k)
    return t


def quantize_values(v, bits, g) -> QTensor:
    """Per-token value quantization of one head (``quantizer.py:493-496``)."""
    t = QTensor("token", bits, g, np.asarray(v).shape[1])
    t.append(v)
    return t


def quantize_layer(keys, values, bits, g):
    """``quantize_layer_kv`` (``quantizer.py:479-497``): lists over KV heads."""
    keys = np.asarray(keys, np.float64)
    values = np.asarray(values, np.float64)
    if keys.shape[1] == 0:
        raise ValueError("cannot quantize an empty cache")
    return ([quantize_keys(keys[h], bits, g) for h in range(keys.shape[0])],
            [quantize_values(values[h], bits, g) for h in range(values.shape[0])])


# ---------------------------------------------------------------------------
# Quantized GEMVs (quantizer.py:505-558) and the Q-layer step (pipeline.py:327-337)
# ---------------------------------------------------------------------------


def qgemv_scores(q, kt: QTensor) -> np.ndarray:
    """Unscaled logits ``codes @ (q*s) + lo@q`` per token block, residual rows
    at full precision (``quantizer.py:505-533``)."""
    q = np.asarray(q, np.float64).reshape(-1)
    parts = []
    nb = kt.rows // kt.g
    if nb:
        c = kt.codes.reshape(nb, kt.g, kt.d).astype(np.float64)
        parts.append((np.einsum("bgd,bd->bg", c, kt.scale * q[None, :])
                      + (kt.lo @ q)[:, None]).reshape(-1))
    if kt.residual.shape[0]:
        parts.append(kt.residual @ q)
    return np.concatenate(parts) if parts else np.zeros(0)


def qgemv_output(w, vt: QTensor) -> np.ndarray:
    """``(w*s) @ codes + w@lo`` per channel block (``quantizer.py:536-558``)."""
    w = np.asarray(w, np.float64).reshape(-1)
    out = np.empty(vt.d)
    c = vt.codes.astype(np.float64)
    for b in range(vt.scale.shape[1]):
        c0, c1 = b * vt.g, min((b + 1) * vt.g, vt.d)
        out[c0:c1] = (w * vt.scale[:, b]) @ c[:, c0:c1] + w @ vt.lo[:, b]
    return out


def stable_softmax(x) -> np.ndarray:
    """Max-subtracted softmax (``pipeline.py:153-156``)."""
    e = np.exp(x - x.max())
    return e / e.sum()


def quant_layer_decode(queries, kq, vq) -> np.ndarray:
    """One quantization-friendly layer step (``pipeline.py:331-337``):
    per query head, logits over the quantized keys of its KV head,
    ``/sqrt(d)``, softmax, then the quantized value GEMV."""
    queries = np.asarray(queries, np.float64)
    hq, d = queries.shape
    grp = hq // len(kq)
    out = np.empty_like(queries)
    for qh in range(hq):
        kvh = qh // grp  # kv_model.py:71-73
        w = stable_softmax(qgemv_scores(queries[qh], kq[kvh]) / np.sqrt(d))
        out[qh] = qgemv_output(w, vq[kvh])
    return out


# ---------------------------------------------------------------------------
# Exact attention (kv_model.py:169-213)
# ---------------------------------------------------------------------------


def attention_weights(q, keys) -> np.ndarray:
    """``softmax(K q / sqrt(d))`` with max subtraction (``kv_model.py:169-194``)."""
    q = np.asarray(q, np.float64).reshape(-1)
    logits = np.asarray(keys, np.float64) @ q / np.sqrt(q.shape[0])
    logits = logits - logits.max()
    w = np.exp(logits)
    return w / w.sum()


def exact_layer_attention(queries, keys, values) -> np.ndarray:
    """All-head exact attention with the GQA map (``kv_model.py:216-242``)."""
    queries = np.asarray(queries, np.float64)
    grp = queries.shape[0] // keys.shape[0]
    return np.stack([attention_weights(queries[qh], keys[qh // grp]) @ values[qh // grp]
                     for qh in range(queries.shape[0])])


# ---------------------------------------------------------------------------
# Two-stage retrieval (retriever.py:84-226)
# ---------------------------------------------------------------------------


def estimate_query(w_q, hidden) -> np.ndarray:
    """``q_hat[h,k] = sum_d hidden[d] W_q[h,d,k]`` (``retriever.py:84-108``)."""
    return np.einsum("d,hdk->hk", np.asarray(hidden, np.float64), np.asarray(w_q, np.float64))


def group_channel_scores(q_hat_group, chmax) -> np.ndarray:
    """``(sum over group |q_hat|) * max|K|`` (``retriever.py:111-119, 138-148``)."""
    qg = np.asarray(q_hat_group, np.float64)
    if qg.ndim == 1:
        qg = qg[None, :]
    return np.abs(qg).sum(axis=0) * np.asarray(chmax, np.float64)


def select_channels(scores, d_s) -> np.ndarray:
    """Top ``d_s`` channels, ties to the lower index, sorted ascending
    (``retriever.py:151-163``)."""
    scores = np.asarray(scores, np.float64)
    idx = np.arange(scores.size)
    order = sorted(idx.tolist(), key=lambda c: (-scores[c], c))
    return np.sort(np.asarray(order[:d_s], dtype=np.int64))


def approx_scores(q_group_sel, key_cols) -> np.ndarray:
    """``K[:, sel] @ sum_group q[sel]`` -- unscaled (``retriever.py:166-189``)."""
    qg = np.asarray(q_group_sel, np.float64)
    if qg.ndim == 1:
        qg = qg[None, :]
    return np.asarray(key_cols, np.float64) @ qg.sum(axis=0)


def select_tokens(scores, n_local, n_topk) -> np.ndarray:
    """Last ``n_local`` tokens plus the top ``n_topk`` older ones by
    (score desc, index desc), sorted ascending; everything when
    ``n <= n_local + n_topk`` (``retriever.py:192-211``)."""
    scores = np.asarray(scores, np.float64).reshape(-1)
    n = scores.size
    if n == 0:
        raise ValueError("token selection over an empty cache")
    if n <= n_local + n_topk:
        return np.arange(n)
    start = n - n_local
    cand = np.arange(start)
    # stable sort on (-score, -index): argsort of -index first then stable by -score
    by_idx = cand[::-1]
    order = by_idx[np.argsort(-scores[by_idx], kind="stable")]
    return np.sort(np.concatenate([order[:n_topk], np.arange(start, n)]))


def select_tokens_sinks(scores, n_local, n_topk, n_sink) -> np.ndarray:
    """EXTENSION (not in the reference; north_star's "sink/local-window
    tokens"): ``select_tokens`` with tokens [0, n_sink) always selected and
    the Top-K taken over [n_sink, n - n_local) by the same rule (score desc,
    index desc).  n_sink = 0 is exactly ``select_tokens``
    (``retriever.py:192-211``)."""
    s = np.asarray(scores, np.float64)
    n = s.size
    if n_sink == 0:
        return select_tokens(s, n_local, n_topk)
    if n <= n_local + n_topk + n_sink:
        return np.arange(n)
    ls = n - n_local
    cand = np.arange(n_sink, ls)
    top = cand[np.lexsort((-cand, -s[cand]))[:n_topk]]
    return np.sort(np.concatenate([np.arange(n_sink), top, np.arange(ls, n)]))


def sparse_attention(q, keys, values, selected) -> np.ndarray:
    """Exact softmax attention over the selected rows (``retriever.py:214-226``)."""
    sel = np.asarray(selected, np.intp)
    return attention_weights(q, keys[sel]) @ values[sel]


def top_weight_tokens(weights, k) -> np.ndarray:
    """Exact top-k by (weight desc, index desc) (``retriever.py:229-242``)."""
    w = np.asarray(weights, np.float64)
    idx = np.arange(w.size)[::-1]
    order = idx[np.argsort(-w[idx], kind="stable")]
    return np.sort(order[:k])


def recall_at_k(selected, exact) -> float:
    """``|sel ∩ exact| / |exact|`` (``retriever.py:245-252``)."""
    return np.intersect1d(selected, exact).size / np.asarray(exact).size


# ---------------------------------------------------------------------------
# Layer classification (identifier.py:58-187)
# ---------------------------------------------------------------------------


def default_probe_k(n: int) -> int:
    """5 % of the sequence, at least one (``identifier.py:58-60``)."""
    return max(1, int(math.ceil(0.05 * n)))


def sparse_error(weights, k) -> float:
    """``1 - (sum of the k largest weights)`` (``identifier.py:89-107``)."""
    w = np.asarray(weights, np.float64)
    kept = w.sum() if k == w.size else np.sort(w)[w.size - k:].sum()
    return float(1.0 - kept)


def dense_preference_score(recent_queries, keys, k) -> float:
    """Mean sparse error of each probe query (``identifier.py:110-132``)."""
    rq = np.asarray(recent_queries, np.float64)
    return sum(sparse_error(attention_weights(r, keys), k) for r in rq) / rq.shape[0]


def calibrate(prefill_queries, prefill_keys, k, n_q=32, tau=0.2):
    """Per layer: mean over query heads of the dense preference of the last
    ``n_q`` prefill queries against all prefill keys of the head's KV head,
    quantization-friendly iff mean > tau (``identifier.py:135-187``).

    Returns ``[(per_head_scores, score, label)]`` with labels
    ``"quantization_friendly"`` / ``"sparsity_friendly"``.
    """
    out = []
    for Q, K in zip(prefill_queries, prefill_keys):
        hq, n, _ = Q.shape
        grp = hq // K.shape[0]
        hs = [dense_preference_score(Q[qh, n - n_q:], K[qh // grp], k) for qh in range(hq)]
        m = float(np.mean(hs))
        out.append((hs, m, "quantization_friendly" if m > tau else "sparsity_friendly"))
    return out


# ---------------------------------------------------------------------------
# Decode replay (pipeline.py:203-413), returning outputs as well as selections
# ---------------------------------------------------------------------------


@dataclass
class ReplayResult:
    outputs: list = field(default_factory=list)    # [t][l] -> [hq, d]
    exact: list = field(default_factory=list)      # [t][l] -> [hq, d]
    selected: dict = field(default_factory=dict)   # (l, t) -> [h] arrays
    channels: dict = field(default_factory=dict)   # (l, t) -> [h] arrays
    fetched: dict = field(default_factory=dict)    # (l, t) -> [h] counts


def replay(prefill_keys, prefill_values, w_q, steps, labels, *, bits=1, g=64,
           n_local=64, n_topk=128, d_s=8, compute_exact=True) -> ReplayResult:
    """Replay decode steps through the hybrid scheme (``pipeline.py:243-413``).

    ``prefill_keys/values``: per layer ``[h, n0, d]``; ``w_q``: per layer
    ``[hq, hidden, d]``; ``steps``: list of dicts with ``hidden [L, hidden]``,
    ``queries [L, hq, d]``, ``new_keys/new_values [L, h, d]``; ``labels``:
    per layer ``"q"`` or ``"s"``.  Semantics kept: attend before append,
    stage 1 from ``hidden[l-1]`` (``hidden[0]`` at l=0), running channel max
    over all tokens, fetch only indices below the local window.
    """
    L = len(labels)
    h, n0, d = np.asarray(prefill_keys[0]).shape
    hq = np.asarray(steps[0]["queries"]).shape[1]
    grp = hq // h
    d_s = min(d_s, d)  # pipeline.py:244
    K = [np.asarray(prefill_keys[l], np.float64).copy() for l in range(L)]
    V = [np.asarray(prefill_values[l], np.float64).copy() for l in range(L)]
    qc = {l: quantize_layer(K[l], V[l], bits, g) for l in range(L) if labels[l] == "q"}
    chmax = {l: np.abs(K[l]).max(axis=1) for l in range(L) if labels[l] == "s"}  # memsim.py:93
    res = ReplayResult()
    for t, st in enumerate(steps):
        outs, exs = [], []
        for l in range(L):
            qs = np.asarray(st["queries"][l], np.float64)
            if compute_exact:
                exs.append(exact_layer_attention(qs, K[l], V[l]))
            n_now = K[l].shape[1]
            if labels[l] == "q":
                out = quant_layer_decode(qs, qc[l][0], qc[l][1])
            else:
                hid = st["hidden"][l - 1] if l >= 1 else st["hidden"][0]  # pipeline.py:273
                qhat = estimate_query(w_q[l], hid)
                local_start = max(0, n_now - n_local)
                out = np.empty_like(qs)
                sels, chans, fetched = [], [], []
                for kvh in range(h):
                    ch = select_channels(group_channel_scores(
                        qhat[kvh * grp:(kvh + 1) * grp], chmax[l][kvh]), d_s)
                    qg = qs[kvh * grp:(kvh + 1) * grp]
                    sc = approx_scores(qg[:, ch], K[l][kvh][:, ch])
                    sel = select_tokens(sc, n_local, n_topk)
                    for qh in range(kvh * grp, (kvh + 1) * grp):
                        out[qh] = sparse_attention(qs[qh], K[l][kvh], V[l][kvh], sel)
                    sels.append(sel)
                    chans.append(ch)
                    fetched.append(int((sel < local_start).sum()))
                res.selected[(l, t)] = sels
                res.channels[(l, t)] = chans
                res.fetched[(l, t)] = fetched
            outs.append(out)
            # appends after attention (pipeline.py:405-413)
            nk = np.asarray(st["new_keys"][l], np.float64)
            nv = np.asarray(st["new_values"][l], np.float64)
            K[l] = np.concatenate([K[l], nk[:, None, :]], axis=1)
            V[l] = np.concatenate([V[l], nv[:, None, :]], axis=1)
            if labels[l] == "q":
                for kvh in range(h):
                    qc[l][0][kvh].append(nk[kvh])
                    qc[l][1][kvh].append(nv[kvh])
            else:
                chmax[l] = np.maximum(chmax[l], np.abs(nk))  # memsim.py:109-111
        res.outputs.append(outs)
        res.exact.append(exs)
    return res


# ---------------------------------------------------------------------------
# Byte accounting used by bench.py (memsim.py:641-696, 216-249)
# ---------------------------------------------------------------------------


def quant_layer_bytes(n, h, d, bits, g) -> int:
    """Table-2 bytes of one quantized layer: ``2 n h d (b/16 + 2/g) * 2``
    (``memsim.py:690-692``)."""
    num = 2 * n * h * d * (bits * g + 32) * 2
    return num // (16 * g)


def scorer_bytes(n, h, d_s) -> int:
    """Critical-key slice bytes ``n h d_s * 2`` (``memsim.py:216-223``)."""
    return n * h * d_s * 2


def gather_bytes(rows, d) -> int:
    """Top-K fetch bytes ``2 rows d * 2`` (``memsim.py:249``)."""
    return 2 * rows * d * 2


# ---------------------------------------------------------------------------
# HKVTRACE reader (trace.py:105-228) -- used to feed committed golden traces
# ---------------------------------------------------------------------------


def read_trace_file(path) -> dict:
    """Parse an HKVTRACE file into plain numpy arrays (``trace.py:158-228``)."""
    import json

    blob = open(path, "rb").read()
    if blob[:8] != b"HKVTRACE":
        raise ValueError("bad trace magic")
    ver, hlen = struct.unpack("<II", blob[8:16])
    hdr = json.loads(blob[16:16 + hlen].decode())
    payload = blob[16 + hlen:]
    if hashlib.sha256(payload).hexdigest() != hdr["payload_sha256"]:
        raise ValueError("payload digest mismatch")
    arrs, off = {}, 0
    for s in hdr["sections"]:
        shape = tuple(s["shape"])
        nb = 2 * int(np.prod(shape))
        arrs[s["name"]] = np.frombuffer(payload[off:off + nb], "<f2").astype(np.float64).reshape(shape)
        off += nb
    m = hdr["model"]
    L = m["num_layers"]
    steps = []
    for t in range(hdr["num_steps"]):
        steps.append({k: np.stack([arrs[f"step{t}/layer{l}/{sec}"] for l in range(L)])
                      for k, sec in (("hidden", "hidden"), ("queries", "query"),
                                     ("new_keys", "new_key"), ("new_values", "new_value"))})
    return {
        "model": m, "header": hdr,
        "prefill_keys": [arrs[f"layer{l}/prefill_keys"] for l in range(L)],
        "prefill_values": [arrs[f"layer{l}/prefill_values"] for l in range(L)],
        "prefill_queries": [arrs[f"layer{l}/prefill_queries"] for l in range(L)],
        "w_q": [arrs[f"layer{l}/w_q"] for l in range(L)],
        "steps": steps,
    }
