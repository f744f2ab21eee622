import sys, numpy as np
sys.path.insert(0, "tests/golden"); sys.path.insert(0, ".")
import cases, paper_2505_19586_b200 as P
c = [c for c in cases.PACK_CASES if c["name"] == sys.argv[1]][0]
k, v = cases.pack_inputs(c)
q = P.quantize_layer_kv(k[None], v[None], c["bits"], c["g"])
open(f"gpurun_out/{c['name']}_keys.bin", "wb").write(q.to_bytes(0, "keys"))
open(f"gpurun_out/{c['name']}_values.bin", "wb").write(q.to_bytes(0, "values"))
