"""Stage 1 (retriever.py:84-163: q_hat = h . W_q, group channel scores,
top-d_s channels) on both kernels: SIMT for one or two sequences, the
tensor-core cluster kernel (mma.sync m16n8k16, W_q read once per 16
sequences) for more.  q_hat within rtol 2e-5 of the float64 oracle, channel
sets identical."""

import numpy as np
import pytest
import torch

import cases
from oracle import tailorkv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,hq,H,d,G", [(1, 8, 1024, 128, 4), (3, 8, 1024, 128, 4), (16, 32, 4096, 128, 4),
                                        (19, 8, 2048, 128, 4), (5, 14, 1792, 128, 7), (4, 16, 1024, 64, 8),
                                        (6, 4, 1024, 256, 2)])
def test_stage1_matches_oracle_both_kernels(B, hq, H, d, G):
    import paper_2505_19586_b200 as P

    rng = np.random.default_rng(B * 1000 + hq)
    w_q = cases.f16(rng.normal(size=(hq, H, d)) / np.sqrt(H))
    hid = cases.f16(rng.normal(size=(B, H)))
    hkv = hq // G
    chmax = cases.f16(np.abs(rng.normal(size=(B * hkv, d))) + 0.1)
    qhat = torch.empty((B, hq, d), dtype=torch.float64, device="cuda")
    ch = P.stage1_select(torch.tensor(hid, dtype=torch.float16, device="cuda"),
                         torch.tensor(w_q, dtype=torch.float16, device="cuda"),
                         torch.tensor(chmax, dtype=torch.float32, device="cuda"), G, 8, q_hat=qhat).cpu().numpy()
    qh = qhat.cpu().numpy()
    for b in range(B):
        ref_q = O.estimate_query(w_q, hid[b])
        np.testing.assert_allclose(qh[b], ref_q, rtol=2e-5, atol=1e-6)
        for kvh in range(hkv):
            ref = O.select_channels(O.group_channel_scores(ref_q[kvh * G:(kvh + 1) * G], chmax[b * hkv + kvh]), 8)
            assert np.array_equal(ch[b * hkv + kvh], ref), (b, kvh)


def test_stage1_tensor_core_replay_is_bit_identical():
    """Deterministic reductions (SURVEY 8(b) threading): repeated launches give
    the same q_hat bits (fixed-order cluster reduction, no float atomics)."""
    import paper_2505_19586_b200 as P

    rng = np.random.default_rng(3)
    B, hq, H, d, G = 16, 32, 4096, 128, 4
    w = torch.tensor(cases.f16(rng.normal(size=(hq, H, d)) / 64), dtype=torch.float16, device="cuda")
    h = torch.tensor(cases.f16(rng.normal(size=(B, H))), dtype=torch.float16, device="cuda")
    cm = torch.rand(B * hq // G, d, device="cuda") + 0.1
    outs = []
    for _ in range(3):
        q = torch.empty((B, hq, d), dtype=torch.float64, device="cuda")
        c = P.stage1_select(h, w, cm, G, 8, q_hat=q)
        outs.append((q.clone(), c.clone()))
    for q, c in outs[1:]:
        assert torch.equal(q, outs[0][0]) and torch.equal(c, outs[0][1])
