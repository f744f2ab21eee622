"""Print the fused sparse kernel's phase timestamps (unit 0, every CTA rank)."""
import ctypes as C
import os

NAMES = {1: "chs", 2: "qsum", 3: "score", 4: "minmax", 5: "hist", 6: "hist-sync", 7: "totals", 8: "scan",
         9: "passes", 10: "band", 11: "band-sync", 12: "select", 13: "count", 14: "out-sync", 15: "rows",
         16: "gather", 17: "sync", 18: "cta-merge", 19: "merge-sync", 20: "final"}


def enable(lib, on=True):
    lib.tkv_debug_sparse_trace((1 if on else 0) | (int(os.environ.get("TKV_FZ_DBG", "0")) & ~1))
    if on:
        lib.tkv_debug_sparse_upath(None, 1)
        lib.tkv_debug_sparse_launches(None, 1)
        lib.tkv_debug_sparse_pathcount(None, 1)


def show_launches(lib, last=31):
    """Gaps between consecutive sparse-kernel launches (unit 0, rank 0)."""
    raw = (C.c_ulonglong * (128 * 3))()
    cnt = lib.tkv_debug_sparse_launches(raw, 0)
    if cnt <= 1:
        return
    v = list(raw)
    idx = [i % 128 for i in range(max(0, cnt - min(cnt, 128)), cnt)][-last:]
    rows = [(v[i * 3], v[i * 3 + 1], v[i * 3 + 2]) for i in idx]
    gaps = [(rows[k][0] - rows[k - 1][2]) / 1e3 for k in range(1, len(rows))]
    waits = [(r[1] - r[0]) / 1e3 for r in rows]
    durs = [(r[2] - r[1]) / 1e3 for r in rows]
    starts = [(rows[k][1] - rows[k - 1][2]) / 1e3 for k in range(1, len(rows))]
    med = lambda x: sorted(x)[len(x) // 2]  # noqa: E731
    print(f"  launches ({len(rows)} consecutive): end->start median {med(gaps):.2f} us (min {min(gaps):.2f} max "
          f"{max(gaps):.2f}), start->PDL-wait-done median {med(waits):.2f}, end->wait-done median {med(starts):.2f}, "
          f"wait-done->end median {med(durs):.2f} us")
    print("  per launch gap end->wait-done (us): " + " ".join(f"{x:.1f}" for x in starts))


def show_units(lib, units=8):
    raw = (C.c_ulonglong * (64 * 8 * 2))()
    lib.tkv_debug_sparse_units(raw)
    v = list(raw)
    up = (C.c_int * (64 * 4))()
    lib.tkv_debug_sparse_upath(up, 0)
    t0 = min(v[(u * 8 + r) * 2] for u in range(units) for r in range(8))
    for u in range(units):
        st = [v[(u * 8 + r) * 2] for r in range(8)]
        en = [v[(u * 8 + r) * 2 + 1] for r in range(8)]
        print(f"  unit {u}: start +{(min(st) - t0) / 1e3:.1f}..{(max(st) - t0) / 1e3:.1f} us, "
              f"end +{(min(en) - t0) / 1e3:.1f}..{(max(en) - t0) / 1e3:.1f} us  path {up[u * 4]} list {up[u * 4 + 1]} "
              f"rows {up[u * 4 + 2]} pcie rows {up[u * 4 + 3]}")


def show(lib):
    pc = (C.c_uint * 4)()
    lib.tkv_debug_sparse_pathcount(pc, 0)
    print(f"  select paths (units x launches): list attempt 0 {pc[0]}, attempt 1 {pc[1]}, full range {pc[2]}")
    show_launches(lib)
    show_units(lib)
    dbg = (C.c_double * 16)()
    lib.tkv_debug_sparse_attempts(dbg)
    for a in range(2):
        d = list(dbg)[a * 8:(a + 1) * 8]
        print(f"  attempt {a}: above {d[1]:.0f} list {d[2]:.0f} need {d[3]:.0f} ok {d[4]:.0f} center {d[5]:.5g} "
              f"width {d[6]:.4g} sd {d[7]:.4g}")
    ph = (C.c_ulonglong * (8 * 40))()
    lib.tkv_debug_sparse_phases(ph)
    t = [list(ph)[r * 40:(r + 1) * 40] for r in range(8)]
    t0 = min(x[0] for x in t)
    x = t[0]
    clk = (C.c_ulonglong * 16)()
    lib.tkv_debug_sparse_clocks(clk)
    cyc = clk[1] - clk[0]
    if x[20] > x[0] and cyc:
        print(f"  SM clock over the kernel (rank 0): {cyc / ((x[20] - x[0]) / 1e3):.0f} MHz ({cyc} cycles)")
    us = lambda a, b: (x[b] - x[a]) / 1e3  # noqa: E731
    if x[5] and x[22] and x[5] > x[4]:
        print(f"  list path (rank 0): setup {us(4, 9):.2f} passA {us(9, 5):.2f} sync1 {us(5, 6):.2f} "
              f"gather {us(6, 7):.2f} radix {us(7, 8):.2f} band+rank {us(8, 21):.2f} sync2 {us(21, 22):.2f} "
              f"bitmap {us(22, 23):.2f}")
    for r in (0, 7):
        y = t[r]
        if y[24] and y[30]:
            g = lambda a, b: (y[b] - y[a]) / 1e3  # noqa: E731
            print(f"  gather rank {r}: lookups {g(15, 24):.2f} issue-hbm {g(24, 25):.2f} logits {g(25, 27):.2f} "
                  f"(pcie-issued at {g(25, 35):.2f}) wait {g(27, 28):.2f} softmax {g(28, 29):.2f} "
                  f"slots {g(29, 36):.2f} insert {g(36, 30):.2f} rest {g(30, 16):.2f} | "
                  f"logits batch0: loads-issued {g(25, 32):.2f} computed {g(32, 33):.2f}")
    for r in range(8):
        parts, prev = [], t[r][0]
        for i in (1, 2, 3, 4, 12, 13, 14, 15, 16, 17, 18, 19, 20):
            if t[r][i] >= prev and t[r][i] > 0:
                parts.append(f"{NAMES[i]} {(t[r][i] - prev) / 1e3:.1f}")
                prev = t[r][i]
        print(f"rank {r} start+{(t[r][0] - t0) / 1e3:.1f}: " + " ".join(parts) + f" | end {(prev - t0) / 1e3:.1f} us")


WIDE_MARKS = {1: "pdl-wait", 2: "tma", 3: "score", 4: "list", 6: "barrier", 14: "r:sync", 15: "r:hdr",
              16: "r:lists+counts", 17: "r:hist", 18: "r:band", 19: "r:f64", 20: "r:rank", 21: "r:pcount",
              8: "resolve-end", 9: "output", 22: "g:lookup", 23: "g:issue", 24: "g:logits(w0)",
              25: "g:softmax+pv(w0)", 26: "g:insert", 10: "gather-end", 27: "partial", 11: "merge-arrive",
              12: "final-merge", 13: "append"}
WIDE_ORDER = [1, 2, 3, 4, 6, 14, 15, 16, 17, 18, 19, 20, 21, 8, 9, 22, 23, 24, 25, 26, 10, 27, 11, 12, 13]


def wide_enable(lib, on=True):
    lib.tkv_debug_wide_trace(1 if on else 0)
    if on:
        lib.tkv_debug_wide_launches(None, 1)


def wide_launches(lib):
    """[(start, after-wait, end)] of unit 0 for the launches since the last reset (<= 128)."""
    raw = (C.c_ulonglong * (128 * 3))()
    cnt = lib.tkv_debug_wide_launches(raw, 0)
    v = list(raw)
    idx = [i % 128 for i in range(max(0, cnt - min(cnt, 128)), cnt)]
    return [(v[i * 3], v[i * 3 + 1], v[i * 3 + 2]) for i in idx]


def wide_show(lib, parts=18):
    """Per-partition phase marks of unit 0 in the last wide launch, and launch gaps."""
    pc = (C.c_uint * 4)()
    lib.tkv_debug_wide_paths(pc)
    print(f"  wide select paths (units x launches): list 0 {pc[0]}, list 1 {pc[1]}, radix {pc[2]}, exact radix {pc[3]}")
    rows = wide_launches(lib)
    if len(rows) > 1:
        med = lambda x: sorted(x)[len(x) // 2]  # noqa: E731
        per = [(rows[k][2] - rows[k - 1][2]) / 1e3 for k in range(1, len(rows))]
        wait = [(r[1] - r[0]) / 1e3 for r in rows]
        body = [(r[2] - r[1]) / 1e3 for r in rows]
        gap = [(rows[k][1] - rows[k - 1][2]) / 1e3 for k in range(1, len(rows))]
        print(f"  wide launches ({len(rows)}): period median {med(per):.2f} us, start->wait-done {med(wait):.2f}, "
              f"wait-done->end {med(body):.2f}, prev end->wait-done {med(gap):.2f}")
    ue = (C.c_ulonglong * 65)()
    lib.tkv_debug_wide_unit_ends(ue)
    if rows:
        wd = rows[-1][1]
        ends = [(x - wd) / 1e3 for x in list(ue)[:8] if x]
        print("  unit final-merge ends after wait-done (us): " + " ".join(f"{x:.1f}" for x in ends)
              + f"; latest CTA exit (any launch) {(ue[64] - wd) / 1e3:.1f}")
    dbg = (C.c_int * 8)()
    lib.tkv_debug_wide_dbg(dbg)
    print(f"  unit 0 lists: merged {dbg[0]}, in window {dbg[4]}, band {dbg[1]}, need in band {dbg[2]}, "
          f"above all lists {dbg[3]}; first attempt: overflow {dbg[5]} merged {dbg[6]} XL-XH {dbg[7]}")
    mk = (C.c_ulonglong * (32 * 32))()
    lib.tkv_debug_wide_marks(mk)
    t = [list(mk)[p * 32:(p + 1) * 32] for p in range(min(parts, 32))]
    if not any(x[1] for x in t):
        print("  (the wide decode did not run)")
        return
    t0 = min(x[1] for x in t if x[1])
    for p, x in enumerate(t):
        parts_s, prev = [], x[1]
        for i in WIDE_ORDER:
            if i == 1 or not x[i] or x[i] < prev:
                continue
            parts_s.append(f"{WIDE_MARKS[i]} {(x[i] - prev) / 1e3:.2f}")
            prev = x[i]
        print(f"  part {p:2d} start {(x[0] - t0) / 1e3:+.2f} wait-done {(x[1] - t0) / 1e3:+.2f}: " + " ".join(parts_s)
              + f" | end {(prev - t0) / 1e3:.2f} us")
