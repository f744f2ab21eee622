"""Drive one sparsity-friendly layer at config-2 shapes (128k, 8 KV heads,
G=4, n_topk=2621, d_s=8): the fused decode (one launch) against select then
gather+attend, event-timed, plus stage 1.   python tools/prof_sparse.py [kfh]"""
import sys, torch
sys.path.insert(0, ".")
import paper_2505_19586_b200 as P
from paper_2505_19586_b200 import _lib
n, h, G, d = 131072, 8, 4, 128
kfh = int(sys.argv[1]) if len(sys.argv) > 1 else 1  # 0: K+V over PCIe, 1: K token-major HBM, 2: K from kt
g = torch.Generator(device="cuda"); g.manual_seed(0)
k = (torch.randn(h, n, d, generator=g, device="cuda") / d ** 0.5).half()
v = torch.randn(h, n, d, generator=g, device="cuda").half()
q = torch.randn(h * G, d, generator=g, device="cuda").half()
cfg = P.RetrievalConfig(64, 2621, 8)
lay = P.OffloadedLayerKV(h, d, n + 64, n, 64, keys_on_device=(kfh == 1))
lay.offload(k, v)
ch = torch.stack([torch.randperm(d, generator=g, device="cuda")[:8].sort().values for _ in range(h)]).int()
kmax = cfg.n_local + cfg.n_topk
lib = _lib.load()
ws = torch.zeros(int(lib.tkv_select_workspace(h, lay.capacity)), dtype=torch.uint8, device="cuda")
dws = torch.zeros(int(lib.tkv_sparse_decode_workspace(h, lay.capacity, G, d, kmax)), dtype=torch.uint8, device="cuda")
idx = torch.zeros((h, kmax), dtype=torch.int32, device="cuda")
cnt = torch.zeros(h, dtype=torch.int32, device="cuda"); fc = torch.zeros_like(cnt)
out = torch.zeros((h * G, d), dtype=torch.float32, device="cuda")
aws = torch.zeros(int(lib.tkv_sparse_attn_workspace(h, G, d, kmax)), dtype=torch.uint8, device="cuda")
kd = bool(kfh)
ops = {
    "fused": lambda: lay.decode(q, ch, G, cfg, idx, cnt, fc, out, dws, keys_from_device=kd),
    "select": lambda: lay.select(q, ch, G, cfg, idx, cnt, fc, ws),
    "attend": lambda: lay.attend(q, G, cfg, idx, cnt, out, aws, keys_from_device=kd),
}
m = lambda x: sorted(x)[len(x) // 2] * 1e3
for name, fn in ops.items():
    for _ in range(3): fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()  # graph of 10 launches: no host gaps
    with torch.cuda.graph(gr):
        for _ in range(10): fn()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gr.replay(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) / 10)
    print(f"{name:8s} {m(ts):7.1f} us")
rows = int(fc.sum())
by = rows * d * 2 * (1 if kfh else 2)
print(f"fetched rows {rows}; PCIe bytes {by / 1e6:.2f} MB")
H = 4096
w_q = (torch.randn(h * G, H, d, generator=g, device="cuda") / H ** 0.5).half()
hid = torch.randn(1, H, generator=g, device="cuda").half()
for _ in range(3): P.stage1_select(hid, w_q, lay.chmax, G, 8)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); P.stage1_select(hid, w_q, lay.chmax, G, 8); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"stage1 {m(ts):.1f} us -> {w_q.numel() * 2 / (m(ts) * 1e-6) / 1e9:.0f} GB/s")
from tools.fz_phases import show, enable
from paper_2505_19586_b200 import _lib as _L
enable(_L.load())
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    for _ in range(10): ops["fused"]()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); gr.replay(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) / 10)
print(f"fused with phase marks {m(ts):7.1f} us")
show(_L.load())
