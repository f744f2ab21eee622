"""Synthetic decode workloads shaped like hybridkv's gen_trace
(trace.py:351-541), generated directly on the GPU so 128k-context inputs take
seconds instead of the reference's O(n * hq * hidden * d) construction.

Structure kept from the reference generator:
* query projections W_q ~ N(0, 1/sqrt(hidden)) with planted outlier channels
  driven by one hidden coordinate each (trace.py:412-445);
* step hidden states h_base + N(0, 0.25) with adjacent-layer drift 0.1
  (trace.py:431-441); queries q = h W_q snapped to fp16 (trace.py:443-445);
* dense layers: keys N(0, 0.05 sqrt(d) / q_rms) (trace.py:458-464);
* sparse layers: keys N(0, 1/sqrt(d)) with the outlier channels carrying 95 %
  of the energy, plus dominant tokens in the first 60 % boosted along the
  group-summed query direction (trace.py:466-502);
* values N(0, 1); everything stored as fp16 (trace.py:505-513);
* ``drift``: the per-step query emphasis wanders across the outlier channels,
  each planted hidden coordinate scaled by lognormal(0, 0.6) every step
  (ChannelOutlierSpec.drift, trace.py:268-275, 434-436).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch


@dataclass
class Workload:
    labels: list            # "q" / "s" per layer
    prefill_keys: list      # per layer [B, h, n, d] fp16 (device)
    prefill_values: list
    w_q: list               # per layer [hq, hidden, d] fp16 (None for q layers when not needed)
    hidden: torch.Tensor    # [T, L, B, hidden] fp16
    queries: torch.Tensor   # [T, L, B, hq, d] fp16
    new_keys: torch.Tensor  # [T, L, B, h, d] fp16
    new_values: torch.Tensor
    h_base: torch.Tensor | None = None       # [hidden] fp32: the step hidden state's mean
    drift_coords: torch.Tensor | None = None  # hidden coordinates of the planted outlier channels
    w_q_all: list | None = None              # fp16 W_q of every layer (query generation for new inputs)


def _step_hidden(h_base, coords, steps, L, batch, randn, drift, gen):
    """Step hidden states (trace.py:431-441): h_base + N(0, 0.25) for layer 0
    (outlier coordinates scaled by lognormal(0, 0.6) per step with drift,
    trace.py:434-436), then adjacent-layer drift 0.1."""
    hidden_dim = h_base.numel()
    hid = torch.empty(steps, L, batch, hidden_dim, device=h_base.device)
    for t in range(steps):
        base = h_base[None, :] + randn(batch, hidden_dim, std=0.25)
        if drift and coords is not None and coords.numel():
            amp = torch.exp(0.6 * torch.randn(batch, coords.numel(), generator=gen, device=h_base.device))
            base[:, coords] *= amp
        hid[t, 0] = base
        for l in range(1, L):
            hid[t, l] = math.sqrt(1 - 0.01) * hid[t, l - 1] + 0.1 * randn(batch, hidden_dim)
    return hid


def make_workload(num_layers: int, q_layers, hq: int, h: int, d: int, n: int, steps: int, batch: int = 1,
                  seed: int = 0, device="cuda", num_outliers: int = 8, ratio: float = 0.95,
                  num_dominant: int = 4, keep_wq_for_q_layers: bool = False, drift: bool = False) -> Workload:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    hidden_dim = hq * d
    G = hq // h
    L = num_layers
    labels = ["q" if l in set(q_layers) else "s" for l in range(L)]

    def randn(*shape, std=1.0):
        return torch.randn(*shape, generator=g, device=device, dtype=torch.float32) * std

    ratio_eff = 1.0 - (1.0 - ratio) * 0.8
    o = num_outliers
    amp = 2.0
    col_mag = math.sqrt(ratio_eff / (1.0 - ratio_eff) * (d - o) / o)
    h_base = randn(hidden_dim)
    w_q, outl, all_coords = [], [], []
    for l in range(L):
        W = randn(hq, hidden_dim, d, std=1.0 / math.sqrt(hidden_dim))
        ch = torch.randperm(d, generator=g, device=device)[:o].sort().values
        coords = torch.randperm(hidden_dim, generator=g, device=device)[: h * o].view(h, o)
        if labels[l] == "s":
            for kvh in range(h):
                for j in range(o):
                    c = int(ch[j])
                    heads = slice(kvh * G, (kvh + 1) * G)
                    W[heads, :, c] *= 0.1
                    W[heads, int(coords[kvh, j]), c] += col_mag / amp
                    h_base[int(coords[kvh, j])] = amp
            all_coords.append(coords.reshape(-1))
        w_q.append(W)
        outl.append(ch)
    coords_all = torch.unique(torch.cat(all_coords)) if all_coords else None
    hid = _step_hidden(h_base, coords_all, steps, L, batch, randn, drift, g)
    hid16 = hid.half()
    queries = torch.empty(steps, L, batch, hq, d, device=device, dtype=torch.float16)
    for l in range(L):
        # q = h W_q in fp32, snapped to fp16
        q = torch.einsum("tbi,hid->tbhd", hid[:, l], w_q[l])
        queries[:, l] = q.half()
    pk, pv = [], []
    new_k = torch.empty(steps, L, batch, h, d, device=device, dtype=torch.float16)
    new_v = randn(steps, L, batch, h, d).half()
    for l in range(L):
        v = randn(batch, h, n, d).half()
        q_ref = queries[:, l].float()  # [T, B, hq, d]
        if labels[l] == "q":
            q_rms = q_ref.pow(2).sum(-1).mean().sqrt().item()
            scale = 0.05 * math.sqrt(d) / max(q_rms, 1e-6)
            k = randn(batch, h, n, d, std=scale)
            nk = randn(steps, batch, h, d, std=scale)
        else:
            ch = outl[l]
            k = randn(batch, h, n, d, std=1.0 / math.sqrt(d))
            nk = randn(steps, batch, h, d, std=1.0 / math.sqrt(d))
            e_out = k[..., ch].pow(2).sum()
            e_rest = k.pow(2).sum() - e_out
            m_k = math.sqrt(ratio_eff / (1 - ratio_eff) * (e_rest / e_out).item())
            k[..., ch] *= m_k
            nk[..., ch] *= m_k
            # dominant tokens boosted along each group's mean query direction
            qg = q_ref.view(steps, batch, h, G, d).sum(3).mean(0)  # [B, h, d]
            direction = qg / qg.norm(dim=-1, keepdim=True)
            align = (q_ref.view(steps, batch, h, G, d) * direction[None, :, :, None, :]).sum(-1)
            a_med = align.clamp_min(1e-3).median().item()
            boost = (math.log(n) + 8.0) * math.sqrt(d) / a_med
            dom = torch.randperm(max(1, int(0.6 * n)), generator=g, device=device)[:num_dominant]
            k[:, :, dom] += boost * direction[:, :, None, :]
        pk.append(k.half())
        pv.append(v)
        new_k[:, l] = nk.half()
    w_all = [w.half() for w in w_q]
    w16 = [w if (labels[l] == "s" or keep_wq_for_q_layers) else None for l, w in enumerate(w_all)]
    return Workload(labels, pk, pv, w16, hid16, queries, new_k, new_v, h_base=h_base, drift_coords=coords_all,
                    w_q_all=w_all)


def step_inputs(wl: Workload, steps: int, drift: bool, seed: int) -> tuple:
    """Fresh decode-step inputs for a prefilled workload: hidden states (with
    or without the reference's per-step outlier drift) and the queries
    q = h W_q they induce; the appended K/V rows are the workload's own.
    Returns (hidden [T, L, B, hidden], queries [T, L, B, hq, d]) fp16."""
    dev = wl.h_base.device
    g = torch.Generator(device=dev)
    g.manual_seed(seed)

    def randn(*shape, std=1.0):
        return torch.randn(*shape, generator=g, device=dev, dtype=torch.float32) * std

    L = len(wl.labels)
    batch = wl.hidden.shape[2]
    hid = _step_hidden(wl.h_base, wl.drift_coords, steps, L, batch, randn, drift, g)
    hq, d = wl.queries.shape[3], wl.queries.shape[4]
    queries = torch.empty(steps, L, batch, hq, d, device=dev, dtype=torch.float16)
    for l in range(L):
        queries[:, l] = torch.einsum("tbi,hid->tbhd", hid[:, l], wl.w_q_all[l].float()).half()
    return hid.half(), queries
