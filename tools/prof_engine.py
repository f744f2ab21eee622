"""Steady-state engine steps (config-2 shapes, fewer layers) for ncu and the
fused kernel's phase marks:  python tools/prof_engine.py [layers] [steps]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2505_19586_b200 as P
from paper_2505_19586_b200 import _lib
from paper_2505_19586_b200.synth import make_workload
from tools.fz_phases import enable, show

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
T = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n = 131072
w = make_workload(L, (0,), 32, 8, 128, n, T, seed=2505)
cfg = P.EngineConfig(bits=1, n_local=64, n_topk=2621, critical_channels=8)
eng = P.DecodeEngine(P.ModelConfig(L, 32, 8, 128, 4096), w.labels, cfg, max_steps=T)
for l in range(L):
    eng.prefill(l, w.prefill_keys[l], w.prefill_values[l], w.w_q[l] if w.w_q[l] is not None else torch.zeros(32, 4096, 128, dtype=torch.float16, device="cuda"))
for t in range(T):
    if t == T - 1:
        enable(_lib.load())
    h0, m0 = eng.cache_counters()
    prof = eng.step_profiled(w.hidden[t], w.queries[t], w.new_keys[t], w.new_values[t])
    h1, m1 = eng.cache_counters()
    parts = "  ".join(f"{k} {sum(v) / len(v) * 1e3:.1f} us" for k, v in prof.items())
    print(f"step {t}: {parts}  hits {h1 - h0} misses {m1 - m0}")
show(_lib.load())
