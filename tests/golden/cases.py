"""Seeded input generators shared by make_golden.py and the tests.

Every input is snapped to the fp16 grid (the reference's storage semantics,
``trace.py:505-513``), so the same values reach the reference (as float64),
the oracle and the CUDA engine (as fp16).
"""

from __future__ import annotations

import numpy as np


def f16(x) -> np.ndarray:
    return np.asarray(x, np.float64).astype(np.float16).astype(np.float64)


# name, n, d, g, bits, seed, dist, gpu (inside the CUDA envelope d%32==0, g in {32,64})
PACK_CASES = [
    dict(name="k1_d128_ragged", n=4096 + 37, d=128, g=64, bits=1, seed=11, dist="normal", gpu=True),
    dict(name="k2_d128_ragged", n=4096 + 37, d=128, g=64, bits=2, seed=12, dist="normal", gpu=True),
    dict(name="k1_d64_exact", n=640, d=64, g=64, bits=1, seed=13, dist="outlier", gpu=True),
    dict(name="k2_d96_ragged_blocks", n=300, d=96, g=64, bits=2, seed=14, dist="normal", gpu=True),
    dict(name="k2_ties", n=256 + 5, d=128, g=64, bits=2, seed=15, dist="ties", gpu=True),
    dict(name="k1_ties", n=256 + 63, d=128, g=64, bits=1, seed=16, dist="ties", gpu=True),
    dict(name="k1_const", n=192 + 1, d=64, g=64, bits=1, seed=17, dist="const", gpu=True),
    dict(name="k2_wide", n=512, d=128, g=64, bits=2, seed=18, dist="wide", gpu=True),
    dict(name="k1_wide", n=512, d=128, g=64, bits=1, seed=19, dist="wide", gpu=True),
    dict(name="k2_g32", n=200, d=64, g=32, bits=2, seed=20, dist="normal", gpu=True),
    dict(name="k1_short", n=37, d=128, g=64, bits=1, seed=21, dist="normal", gpu=True),
    dict(name="k1_tiny_ref", n=21, d=10, g=4, bits=1, seed=9, dist="normal", gpu=False),
    dict(name="k2_tiny_ref", n=21, d=10, g=4, bits=2, seed=9, dist="normal", gpu=False),
]


def _dist(rng, n, d, dist):
    if dist == "normal":
        return rng.normal(size=(n, d))
    if dist == "outlier":
        x = rng.normal(size=(n, d)) * 0.2
        x[:, rng.choice(d, 4, replace=False)] *= 40.0
        return x
    if dist == "ties":
        # values on a coarse grid make (x-lo)/s land exactly on k+0.5
        return rng.integers(-3, 4, size=(n, d)) * 0.5
    if dist == "const":
        x = rng.normal(size=(n, d))
        x[:, ::3] = 1.25
        x[::5, :] = -0.75
        return x
    if dist == "wide":
        mag = 10.0 ** rng.uniform(-5, 4.6, size=(n, d))
        return mag * rng.choice([-1.0, 1.0], size=(n, d))
    raise ValueError(dist)


def pack_inputs(c):
    rng = np.random.default_rng(c["seed"])
    k = f16(_dist(rng, c["n"], c["d"], c["dist"]))
    v = f16(_dist(rng, c["n"], c["d"], c["dist"]))
    return k, v


DECODE_CASES = [
    dict(name="dec_b1_ragged", h=2, hq=8, n=1000, d=128, g=64, bits=1, seed=31, kscale=0.3),
    dict(name="dec_b2_long", h=1, hq=4, n=4133, d=128, g=64, bits=2, seed=32, kscale=0.1),
    dict(name="dec_b1_onegroup", h=2, hq=4, n=64, d=64, g=64, bits=1, seed=33, kscale=1.0),
    dict(name="dec_b1_allresidual", h=2, hq=4, n=37, d=128, g=64, bits=1, seed=34, kscale=1.0),
    dict(name="dec_b2_gqa7", h=2, hq=14, n=700, d=128, g=64, bits=2, seed=35, kscale=0.3),
    dict(name="dec_b1_gqa8", h=1, hq=8, n=2000, d=128, g=64, bits=1, seed=36, kscale=0.05),
]


def decode_inputs(c):
    rng = np.random.default_rng(c["seed"])
    keys = f16(rng.normal(0.0, c["kscale"], size=(c["h"], c["n"], c["d"])))
    values = f16(rng.normal(size=(c["h"], c["n"], c["d"])))
    queries = f16(rng.normal(size=(c["hq"], c["d"])))
    return keys, values, queries


TOPK_CASES = [
    dict(name="topk_normal", n=5000, n_local=64, n_topk=128, dist="normal", seed=41),
    dict(name="topk_ties", n=3000, n_local=16, n_topk=200, dist="ties", seed=42),
    dict(name="topk_zeros", n=1000, n_local=2, n_topk=3, dist="zeros", seed=43),
    dict(name="topk_all", n=150, n_local=64, n_topk=128, dist="normal", seed=44),
    dict(name="topk_neg", n=4096, n_local=0, n_topk=100, dist="neg", seed=45),
    dict(name="topk_signed_zero", n=600, n_local=8, n_topk=50, dist="signed_zero", seed=46),
    dict(name="topk_big", n=131072, n_local=64, n_topk=2621, dist="normal", seed=47),
    dict(name="topk_heavy_ties", n=70000, n_local=64, n_topk=1400, dist="ties", seed=48),
]


def topk_scores(c):
    rng = np.random.default_rng(c["seed"])
    n = c["n"]
    if c["dist"] == "normal":
        return rng.normal(size=n)
    if c["dist"] == "ties":
        return rng.integers(0, 6, size=n).astype(np.float64)
    if c["dist"] == "zeros":
        return np.zeros(n)
    if c["dist"] == "neg":
        return -np.abs(rng.normal(size=n)) - 1.0
    if c["dist"] == "signed_zero":
        s = rng.integers(-2, 3, size=n).astype(np.float64) * 0.0
        s[rng.random(n) < 0.5] = -0.0
        s[rng.choice(n, 20, replace=False)] = 1.0
        return s
    raise ValueError(c["dist"])


CHANNEL_CASES = [
    dict(name="chan_normal", G=4, d=128, d_s=8, seed=51, ties=False),
    dict(name="chan_ties", G=4, d=128, d_s=8, seed=52, ties=True),
    dict(name="chan_gqa7", G=7, d=128, d_s=16, seed=53, ties=False),
]


def channel_inputs(c):
    rng = np.random.default_rng(c["seed"])
    qhat = rng.normal(size=(c["G"], c["d"]))
    chmax = f16(np.abs(rng.normal(size=c["d"])) + 0.1)
    if c["ties"]:
        qhat = np.round(qhat)
        chmax = np.ones(c["d"])
    return qhat, chmax


CALIB_CASES = [
    dict(name="calib_two_layers", L=2, hq=4, h=2, n=256, d=64, n_q=32, tau=0.2, seed=61),
]


def calib_inputs(c):
    rng = np.random.default_rng(c["seed"])
    pq = f16(rng.normal(size=(c["L"], c["hq"], c["n"], c["d"])))
    pk = rng.normal(size=(c["L"], c["h"], c["n"], c["d"]))
    pk[0] *= 0.02  # dense layer: near-uniform attention
    pk[1, :, 10, :] += 3.0 * pq[1, ::2].mean(axis=(0, 1))  # sparse layer: one dominant key
    return pq, f16(pk)


PIPELINE_CONFIGS = {
    "default": {},
    "b2_small": {"bits": 2, "n_local": 16, "n_topk": 32, "critical_channels": 8},
    "pinned_q0": {"q_layers": (0,), "n_local": 8, "n_topk": 24, "critical_channels": 4},
    "all_sparse_fullch": {"q_layers": (), "n_local": 0, "n_topk": 48, "critical_channels": 64},
}


def indices_to_hex(indices) -> str:
    idx = np.asarray(indices, dtype=np.int64)
    n = int(idx.max()) + 1 if idx.size else 0
    bits = np.zeros(((n + 7) // 8) * 8, np.uint8)
    bits[idx] = 1
    return np.packbits(bits, bitorder="little").tobytes().hex()


def hex_to_indices(h: str) -> np.ndarray:
    raw = np.frombuffer(bytes.fromhex(h), np.uint8)
    return np.nonzero(np.unpackbits(raw, bitorder="little"))[0].astype(np.int64)
