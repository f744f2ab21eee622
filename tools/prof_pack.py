"""Prefill pack (quantize_layer_kv) at config-2 shapes: 131,072 tokens x 8 KV
heads x d 128, b = 1 and 2, event-timed over the pack launches only (inputs
already on the device), against the HBM roofline of its algorithmic bytes
(read K and V fp16, write codes + (lo, hi) params).
    python tools/prof_pack.py [n]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_19586_b200 as P  # noqa: E402
from paper_2505_19586_b200 import _lib  # noqa: E402
from paper_2505_19586_b200.quantizer import QuantizedLayerKV  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
h, d, g = 8, 128, 64
gen = torch.Generator(device="cuda")
gen.manual_seed(0)
k = (torch.randn(h, n, d, generator=gen, device="cuda") * 0.3).half()
v = torch.randn(h, n, d, generator=gen, device="cuda").half()
peak = 6515.1
import ctypes as C  # noqa: E402
from paper_2505_19586_b200._lib import ptr, stream_ptr  # noqa: E402
lib = _lib.load()
for bits in (1, 2):
    q = QuantizedLayerKV.from_kv(k, v, bits, g, capacity=n)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(lib.tkv_qcache_pack(C.byref(q.struct), ptr(k), ptr(v), n, 0, stream_ptr()))
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    t = ts[len(ts) // 2]
    rd = 2 * h * n * d * 2
    wr = 2 * h * n * d * bits // 8 + (h * (n // g) * d + h * n * ((d + g - 1) // g)) * 4
    print(f"pack n={n} bits={bits}: {t:.1f} us  read {rd / 1e6:.0f} MB + write {wr / 1e6:.1f} MB -> "
          f"{(rd + wr) / (t * 1e-6) / 1e9:.0f} GB/s ({(rd + wr) / (t * 1e-6) / 1e9 / peak:.2f} of {peak})")
