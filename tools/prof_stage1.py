"""Stage 1 (q_hat = h . W_q + critical channels) timed alone at the BASELINE
shapes, W_q cold (rotated over NL layer slices > L2), graph of 10 launches.

    python tools/prof_stage1.py            # config 2 (B=1) and config 3 (B=16)
    TKV_STAGE1_SIMT=1 python tools/prof_stage1.py   # the SIMT kernel
"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_19586_b200 as P  # noqa: E402

m = lambda x: sorted(x)[len(x) // 2] * 1e3  # noqa: E731
g = torch.Generator(device="cuda")
g.manual_seed(0)
CASES = [("config2 B=1", 1, 32, 4096, 128, 4), ("config3 B=16", 16, 32, 4096, 128, 4),
         ("config4 B=4 (G=7)", 4, 28, 3584, 128, 7), ("config5 B=1 (G=8)", 1, 64, 8192, 128, 8)]
if len(sys.argv) > 1:
    CASES = [CASES[int(i)] for i in sys.argv[1].split(",")]
for name, B, hq, H, d, G in CASES:
    NL = 8
    hkv = hq // G
    w = [(torch.randn(hq, H, d, generator=g, device="cuda") / H ** 0.5).half() for _ in range(NL)]
    hid = torch.randn(B, H, generator=g, device="cuda").half()
    chmax = torch.rand(B * hkv, d, generator=g, device="cuda") + 0.1
    for i in range(3):
        P.stage1_select(hid, w[i % NL], chmax, G, 8)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for i in range(10):
            P.stage1_select(hid, w[i % NL], chmax, G, 8)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gr.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 10)
    by = hq * H * d * 2
    print(f"stage1 {name:18s} {m(ts):7.1f} us -> {by / (m(ts) * 1e-6) / 1e9:6.0f} GB/s "
          f"({by / (m(ts) * 1e-6) / 1e9 / 6542:.2f} of 6542)")
    if os.environ.get("TKV_STAGE1_DBG") == "3":
        import ctypes as C
        from paper_2505_19586_b200 import _lib
        lib = _lib.load()
        buf = (C.c_ulonglong * 8)()
        lib.tkv_debug_stage1_stamps(buf, 1)
        P.stage1_select(hid, w[0], chmax, G, 8)
        torch.cuda.synchronize()
        lib.tkv_debug_stage1_stamps(buf, 0)
        t0 = buf[0]
        print("  stamps (us from first CTA start): loop end %.2f, cluster done %.2f, last arrive %.2f, fence %.2f, "
              "select end %.2f" % tuple((buf[i] - t0) / 1e3 for i in (1, 2, 3, 4, 5)))
    del w
