"""Drive the quantized decode at config-2 shapes (128k, 8 KV heads, G=4) for ncu."""
import sys, torch
sys.path.insert(0, ".")
import paper_2505_19586_b200 as P
n, h, G, d = int(sys.argv[1]) if len(sys.argv) > 1 else 131072, 8, 4, 128
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 1
impl = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = torch.Generator(device="cuda"); g.manual_seed(0)
k = (torch.randn(h, n, d, generator=g, device="cuda") * 0.05).half()
v = torch.randn(h, n, d, generator=g, device="cuda").half()
q = torch.randn(h * G, d, generator=g, device="cuda").half()
c = P.quantize_layer_kv(k, v, bits, 64)
out = c.decode(q, impl=impl)
torch.cuda.synchronize()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(20):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); c.decode(q, out=out, impl=impl); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts = sorted(ts)[2:-2]
ms = sum(ts) / len(ts)
byt = 2 * n * h * d * (bits * 64 + 32) * 2 // (16 * 64)
print(f"n={n} bits={bits} impl={impl} decode {ms*1e3:.1f} us  -> {byt/ms/1e6:.0f} GB/s (L2 flushed)")
