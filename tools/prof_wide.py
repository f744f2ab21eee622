"""Time one sparsity-friendly layer at config-2 shapes (8 KV heads, 128k, G=4,
n_topk 2621, d_s 8, HBM row cache W=4) in isolation: the wide decode against
the cluster kernel, graph-replayed 10 launches at a time, plus the wide
kernel's per-partition phase marks of one launch.
    python tools/prof_wide.py [units] [ctx]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_19586_b200 as P  # noqa: E402
from paper_2505_19586_b200 import _lib  # noqa: E402
from tools.fz_phases import wide_enable, wide_show  # noqa: E402

h = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
G, d, T = 4, 128, 40
g = torch.Generator(device="cuda")
g.manual_seed(0)
k = (torch.randn(h, n, d, generator=g, device="cuda") / d ** 0.5).half()
v = torch.randn(h, n, d, generator=g, device="cuda").half()
cfg = P.RetrievalConfig(64, round(0.02 * n), 8)
kmax = cfg.n_local + cfg.n_topk
lib = _lib.load()
base_q = torch.randn(h * G, d, generator=g, device="cuda")
qsteps = [(base_q + 0.2 * torch.randn(h * G, d, generator=g, device="cuda")).half() for _ in range(T // 10 + 1)]
ch = torch.stack([torch.randperm(d, generator=g, device="cuda")[:8].sort().values for _ in range(h)]).int()


def run(mode):
    _lib.set_sparse_kernel(mode)
    lay = P.OffloadedLayerKV(h, d, n + 64, n, 64, keys_on_device=True, cache_rows=kmax, cache_window=4)
    lay.offload(k, v)
    dws = torch.zeros(int(lib.tkv_sparse_decode_workspace(h, lay.capacity, G, d, kmax)), dtype=torch.uint8,
                      device="cuda")
    idx = torch.zeros((h, kmax), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(h, dtype=torch.int32, device="cuda")
    fc = torch.zeros_like(cnt)
    out = torch.zeros((h * G, d), dtype=torch.float32, device="cuda")
    q = qsteps[0].clone()
    fn = lambda: lay.decode(q, ch, G, cfg, idx, cnt, fc, out, dws, keys_from_device=True)  # noqa: E731
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(10):
            fn()
    ts = []
    for it in range(T // 10):
        q.copy_(qsteps[1 + it])
        s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        gr.replay()
        e0.record()
        torch.cuda.synchronize()
        ts.append(s0.elapsed_time(e0) / 10 * 1e3)
    ts.sort()
    print(f"mode {mode}: {ts[len(ts) // 2]:.2f} us per launch (min {ts[0]:.2f}), hits/misses {lay.cache_counters()}")
    if mode == 1:
        wide_enable(lib)
        gr.replay()
        torch.cuda.synchronize()
        wide_enable(lib, False)
        wide_show(lib, _lib.wide_parts(h))
    _lib.set_sparse_kernel(-1)
    return out.clone(), idx.clone(), cnt.clone()


o0, i0, c0 = run(0)
o1, i1, c1 = run(1)
print("selections equal:", bool(torch.equal(c0, c1)) and all(torch.equal(i0[u, :c0[u]], i1[u, :c1[u]]) for u in range(h)),
      "max |out diff|:", float((o0 - o1).abs().max()), "wide errors:", lib.tkv_debug_wide_error(1))
