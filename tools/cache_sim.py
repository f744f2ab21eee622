"""Hit rate of a windowed HBM row cache (rows selected in any of the last W
steps stay resident) on the bench's synthetic workload, from the selections
the engine records:  python tools/cache_sim.py [layers] [steps]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2505_19586_b200 as P
from paper_2505_19586_b200.synth import make_workload

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
T = int(sys.argv[2]) if len(sys.argv) > 2 else 24
n = 131072
w = make_workload(L, (0,), 32, 8, 128, n, T, seed=2505)
cfg = P.EngineConfig(bits=1, n_local=64, n_topk=2621, critical_channels=8)
eng = P.DecodeEngine(P.ModelConfig(L, 32, 8, 128, 4096), w.labels, cfg, max_steps=T)
for l in range(L):
    eng.prefill(l, w.prefill_keys[l], w.prefill_values[l], w.w_q[l] if w.w_q[l] is not None else torch.zeros(32, 4096, 128, dtype=torch.float16, device="cuda"))
eng.record_selection = True
sels = {}
for t in range(T):
    eng.step(w.hidden[t], w.queries[t], w.new_keys[t], w.new_values[t])
    for l, (idx, cnt, fc) in eng.last_selection.items():
        idx, fc = idx.cpu().numpy(), fc.cpu().numpy()
        for u in range(idx.shape[0]):
            sels[(l, u, t)] = set(idx[u, :fc[u]].tolist())
layers = sorted({k[0] for k in sels})
for W in (1, 2, 4, 8, 16):
    hit = tot = 0
    for l in layers:
        for u in range(8):
            for t in range(W, T):
                cur = sels[(l, u, t)]
                cache = set().union(*[sels[(l, u, s)] for s in range(t - W, t)])
                hit += len(cur & cache)
                tot += len(cur)
    print(f"window {W:2d} steps: hit rate {hit / tot:.3f}  (rows per layer over PCIe {8 * (tot - hit) / (tot / 8) * 2621 / 8 / 8:.0f})")
