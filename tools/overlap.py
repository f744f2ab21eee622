"""How much of step t's fetched Top-K set was already fetched at step t-1?
(config-2 shapes on the synthetic gen_trace-shaped workload, 4 sparse layers)"""
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2505_19586_b200 as P
from paper_2505_19586_b200.synth import make_workload
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
L, T = 5, 8
w = make_workload(L, (0,), 32, 8, 128, n, T, seed=2505)
cfg = P.EngineConfig(bits=1, n_local=64, n_topk=round(0.02 * n), critical_channels=8)
eng = P.DecodeEngine(P.ModelConfig(L, 32, 8, 128, 4096), w.labels, cfg, max_steps=T)
for l in range(L):
    eng.prefill(l, w.prefill_keys[l], w.prefill_values[l], w.w_q[l] if w.w_q[l] is not None else torch.zeros(32, 4096, 128, dtype=torch.float16, device="cuda"))
eng.record_selection = True
prev = {}
hits = []
for t in range(T):
    eng.step(w.hidden[t], w.queries[t], w.new_keys[t], w.new_values[t])
    for l in range(1, L):
        idx, cnt, fc = (x.cpu().numpy() for x in eng.last_selection[l])
        cur = [set(idx[u, :fc[u]].tolist()) for u in range(8)]
        if l in prev:
            hits.append(np.mean([len(cur[u] & prev[l][u]) / max(1, len(cur[u])) for u in range(8)]))
        prev[l] = cur
print(f"n={n}: fetched-row overlap with the previous step: mean {np.mean(hits):.3f} min {np.min(hits):.3f}")
