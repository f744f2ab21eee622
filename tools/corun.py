"""Does stage 1 (side stream, low priority) run beside the sparse decode?
Config-2 shapes: one sparse layer (8 KV heads, 128k, d_s 8) decoded 10x in a
graph on the main stream, stage 1 (W_q 32x4096x128, B=1) 10x in a graph on a
side stream; each alone, then both launched together.
    python tools/corun.py [wide_mode]     (1 wide decode, 0 cluster kernel)"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_19586_b200 as P  # noqa: E402
from paper_2505_19586_b200 import _lib  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
_lib.set_sparse_kernel(mode)
h, n, G, d, hq, H = 8, 131072, 4, 128, 32, 4096
g = torch.Generator(device="cuda")
g.manual_seed(0)
k = (torch.randn(h, n, d, generator=g, device="cuda") / d ** 0.5).half()
v = torch.randn(h, n, d, generator=g, device="cuda").half()
cfg = P.RetrievalConfig(64, 2621, 8)
kmax = cfg.n_local + cfg.n_topk
lib = _lib.load()
lay = P.OffloadedLayerKV(h, d, n + 64, n, 64, keys_on_device=True, cache_rows=kmax, cache_window=4)
lay.offload(k, v)
dws = torch.zeros(int(lib.tkv_sparse_decode_workspace(h, lay.capacity, G, d, kmax)), dtype=torch.uint8, device="cuda")
idx = torch.zeros((h, kmax), dtype=torch.int32, device="cuda")
cnt = torch.zeros(h, dtype=torch.int32, device="cuda")
fc = torch.zeros_like(cnt)
out = torch.zeros((h * G, d), dtype=torch.float32, device="cuda")
q = torch.randn(h * G, d, generator=g, device="cuda").half()
ch = torch.stack([torch.randperm(d, generator=g, device="cuda")[:8].sort().values for _ in range(h)]).int()
NL = 6
w = [(torch.randn(hq, H, d, generator=g, device="cuda") / H ** 0.5).half() for _ in range(NL)]
hid = torch.randn(1, H, generator=g, device="cuda").half()
chmax = torch.rand(h, d, generator=g, device="cuda") + 0.1
main = torch.cuda.Stream(priority=-5)
side = torch.cuda.Stream(priority=0)


def dec():
    lay.decode(q, ch, G, cfg, idx, cnt, fc, out, dws, keys_from_device=True)


def s1(i):
    P.stage1_select(hid, w[i % NL], chmax, G, 8)


for _ in range(3):
    dec()
    s1(0)
torch.cuda.synchronize()
gd, gs = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
with torch.cuda.stream(main):
    with torch.cuda.graph(gd, stream=main):
        for _ in range(10):
            dec()
with torch.cuda.stream(side):
    with torch.cuda.graph(gs, stream=side):
        for i in range(10):
            s1(i)


def timed(run_dec, run_s1, reps=5):
    res = {"dec": [], "s1": []}
    for _ in range(reps):
        torch.cuda.synchronize()
        ev = {kk: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for kk in res}
        if run_dec:
            with torch.cuda.stream(main):
                ev["dec"][0].record(main)
                gd.replay()
                ev["dec"][1].record(main)
        if run_s1:
            with torch.cuda.stream(side):
                ev["s1"][0].record(side)
                gs.replay()
                ev["s1"][1].record(side)
        torch.cuda.synchronize()
        for kk, on in (("dec", run_dec), ("s1", run_s1)):
            if on:
                res[kk].append(ev[kk][0].elapsed_time(ev[kk][1]) * 100)  # us per launch (10 per graph)
    return {kk: sorted(x)[len(x) // 2] for kk, x in res.items() if x}


print("mode", mode, "decode alone:", timed(True, False))
print("mode", mode, "stage1 alone:", timed(False, True))
print("mode", mode, "together   :", timed(True, True))
