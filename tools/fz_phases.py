"""Print the fused sparse kernel's phase timestamps (unit 0, every CTA rank)."""
import ctypes as C

NAMES = {1: "chs", 2: "qsum", 3: "score", 4: "minmax", 5: "hist", 6: "hist-sync", 7: "totals", 8: "scan",
         9: "passes", 10: "band", 11: "band-sync", 12: "rank", 13: "count", 14: "out-sync", 15: "rows",
         16: "gather", 17: "sync", 18: "cta-merge", 19: "merge-sync", 20: "final"}


def enable(lib, on=True):
    lib.tkv_debug_sparse_trace(1 if on else 0)


def show(lib):
    ph = (C.c_ulonglong * (8 * 24))()
    lib.tkv_debug_sparse_phases(ph)
    t = [list(ph)[r * 24:(r + 1) * 24] for r in range(8)]
    t0 = min(x[0] for x in t)
    for r in range(8):
        x = t[r]
        print(f"  rank {r} detail: stats->range {(x[21] - x[4]) / 1e3:.2f} range->cleared {(x[22] - x[21]) / 1e3:.2f} "
              f"loop {(x[23] - x[22]) / 1e3:.2f} tail {(x[5] - x[23]) / 1e3:.2f}")
        parts, prev = [], t[r][0]
        for i in range(1, 21):
            if t[r][i] >= prev and t[r][i] > 0:
                parts.append(f"{NAMES[i]} {(t[r][i] - prev) / 1e3:.1f}")
                prev = t[r][i]
        print(f"rank {r} start+{(t[r][0] - t0) / 1e3:.1f}: " + " ".join(parts) + f" | end {(prev - t0) / 1e3:.1f} us")
