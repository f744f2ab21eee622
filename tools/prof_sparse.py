"""Drive one sparsity-friendly layer at config-2 shapes (128k, 8 KV heads,
G=4, n_topk=2621, d_s=8) for ncu: select (scores + top-k) then gather+attend."""
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
idx = torch.zeros((h, kmax), dtype=torch.int32, device="cuda")
cnt = torch.zeros(h, dtype=torch.int32, device="cuda"); fc = torch.zeros_like(cnt)
out = torch.zeros((h * G, d), dtype=torch.float32, device="cuda")
aws = torch.zeros(int(lib.tkv_sparse_attn_workspace(h, G, d, kmax)), dtype=torch.uint8, device="cuda")
def run():
    lay.select(q, ch, G, cfg, idx, cnt, fc, ws)
    lay.attend(q, G, cfg, idx, cnt, out, aws, keys_from_device=bool(kfh))
for _ in range(3): run()
torch.cuda.synchronize()
ts_s, ts_a = [], []
for _ in range(20):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); lay.select(q, ch, G, cfg, idx, cnt, fc, ws); e[1].record()
    lay.attend(q, G, cfg, idx, cnt, out, aws, keys_from_device=bool(kfh)); e[2].record()
    torch.cuda.synchronize(); ts_s.append(e[0].elapsed_time(e[1])); ts_a.append(e[1].elapsed_time(e[2]))
m = lambda x: sorted(x)[len(x) // 2] * 1e3
rows = int(fc.sum())
print(f"select {m(ts_s):.1f} us; gather+attend {m(ts_a):.1f} us; fetched rows {rows}; "
      f"PCIe bytes {rows * d * 2 * (1 if kfh else 2) / 1e6:.2f} MB -> {rows * d * 2 * (1 if kfh else 2) / (m(ts_a) * 1e-6) / 1e9:.1f} GB/s")
# stage 1 alone: q_hat = h W_q (32 x 4096 x 128) + channel select, float64
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
import ctypes as C
ph = (C.c_ulonglong * 8)()
lay.select(q, ch, G, cfg, idx, cnt, fc, ws); torch.cuda.synchronize()
lib.tkv_debug_select_phases(ph)
t = list(ph)
print("select phases (us): score %.1f minmax %.1f radix %.1f (passes %d) flags %.1f output %.1f" % (
    (t[1]-t[0])/1e3, (t[2]-t[1])/1e3, (t[3]-t[2])/1e3, t[6], (t[4]-t[3])/1e3, (t[5]-t[4])/1e3))
