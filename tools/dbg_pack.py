import sys
sys.path[:0] = ["tests", ".", "tests/golden"]
import numpy as np
import paper_2505_19586_b200 as tkv
from oracle import tailorkv_oracle as O
from test_gpu_parity import _boundary_groups
import cases


def unpack(blob, bits, count):
    nbytes = int(np.frombuffer(blob[20:24], "<u4")[0])
    p = np.frombuffer(blob[24:24 + nbytes], np.uint8)
    per = 8 // bits
    sh = np.arange(per) * bits
    return ((p[:, None] >> sh) & ((1 << bits) - 1)).reshape(-1)[:count]


for bits in (1, 2):
  for g in (16, 64):
    rng = np.random.default_rng(40 + bits + g)
    d, n = 128, 4 * 128 + g + 5
    kg = _boundary_groups(rng, (n // g) * d, g, bits)
    keys = np.zeros((n, d), np.float16)
    keys[: (n // g) * g] = kg.reshape(n // g, d, g).transpose(0, 2, 1).reshape(-1, d)
    keys[(n // g) * g:] = cases.f16(rng.normal(size=(n - (n // g) * g, d)))
    values = _boundary_groups(rng, n * (d // g), g, bits).reshape(n, d)
    q = tkv.quantize_layer_kv(keys[None], values[None], bits, g)
    for which, x in (("keys", keys), ("values", values)):
        ref = (O.quantize_keys if which == "keys" else O.quantize_values)(x, bits, g)
        rs = ref.code_stream()
        gb = q.to_bytes(0, which)
        gs = unpack(gb, bits, rs.size)
        bad = np.nonzero(gs != rs)[0]
        print(bits, g, which, "code mismatches", len(bad), "bytes equal", gb == ref.to_bytes())
        if len(bad) == 0 and gb != ref.to_bytes():
            rb = ref.to_bytes()
            i = next(i for i in range(len(rb)) if rb[i] != gb[i])
            print("   first differing byte", i, "of", len(rb))
        for i in bad[:8]:
            if which == "keys":
                blk, rem = divmod(i, d * g)
                c, tt = divmod(rem, g)
                t = blk * g + tt
                grp = x[blk * g:(blk + 1) * g, c]
            else:
                t, c = divmod(i, d)
                grp = x[t, (c // g) * g:(c // g + 1) * g]
            print("  t", t, "c", c, "x", repr(x[t, c]), hex(x[t, c].view(np.uint16)), "lo", repr(grp.min()), hex(grp.min().view(np.uint16)),
                  "hi", repr(grp.max()), hex(grp.max().view(np.uint16)), "gpu", gs[i], "ref", rs[i])
