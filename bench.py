"""TailorKV decode benchmark (BASELINE.json metric: decode ms/token @128k,
Llama-3.1-8B shapes, 2 layers 1-bit quantized + 30 Top-K 2 % offloaded).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N>1 is launched by torchrun; KV heads are sharded over ranks (strong
scaling: every rank decodes its heads of the same token) and each layer's
head outputs are all-gathered with NCCL.  Timing: W untimed steps, then K
steps bracketed by barrier + synchronize, CUDA events on the decode stream,
max over ranks.  Each step reads ~1.6 GB of HBM (> 126 MB L2), so no L2
flush is inserted.  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode ms/token @128k ctx (Llama-3.1-8B shapes) at 1/2/4/8 B200; HBM & PCIe GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cache-warm", type=int, default=100,
                    help="untimed decode steps before everything else, so every timed loop sees the HBM row "
                         "cache's steady state (a 128k-context decode runs for many tokens; the hit rate rises "
                         "over the first ~100 steps)")
    ap.add_argument("--e2e-plain", action="store_true",
                    help="time e2e with the device graph plus separate host copies (the round-1 way) instead of "
                         "the host-I/O graph (A/B of the overlapped copies)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS),
                    help="BASELINE.json config (2 = the headline; 3-5 run the same engine at their shapes)")
    ap.add_argument("--ctx", type=int, default=None, help="override the config's context length")
    ap.add_argument("--topk-frac", type=float, default=None, help="override the config's Top-K fraction")
    ap.add_argument("--keys-over-pcie", action="store_true",
                    help="headline with K and V rows both gathered over PCIe (the reference's fetch_topk transfer)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--single-copy-keys", action="store_true",
                    help="no token-major HBM key copy: key rows are gathered from the scorer's channel-major copy")
    ap.add_argument("--unfused", action="store_true", help="sparse layers as two launches (select, gather+attend)")
    ap.add_argument("--phases", action="store_true", help="print the fused sparse kernel's phase marks (unit 0)")
    ap.add_argument("--no-fidelity", action="store_true", help="skip the one-step recall/cosine evaluation")
    ap.add_argument("--serial-stage1", action="store_true", help="stage 1 runs in line, not overlapped")
    ap.add_argument("--no-l2-prefetch", action="store_true", help="stage 1 does not prefetch the scorer columns")
    ap.add_argument("--cache-steps", type=int, default=4,
                    help="HBM row cache window: a value row stays resident until unselected for this many steps (0: off)")
    ap.add_argument("--seed", type=int, default=2505)
    ap.add_argument("--shard-of", type=int, default=1,
                    help="run rank 0's share of an N-GPU kv-head shard on this GPU without the all-gather "
                         "(per-GPU work of the multi-GPU configuration; not the headline)")
    args = ap.parse_args()
    c = CONFIGS[args.config]
    args.ctx = c["ctx"] if args.ctx is None else args.ctx
    args.topk_frac = c["topk"] if args.topk_frac is None else args.topk_frac
    args.batch, args.bits, args.q_layers, args.model = c["batch"], c["bits"], c["q_layers"], c["model"]
    return args


# BASELINE.json configs.  Where BASELINE.json leaves the quantized-layer set or
# the Top-K fraction open, SURVEY.md 8(d) fixes them (stated in the workload name).
CONFIGS = {
    2: {"model": "LLAMA31_8B", "label": "Llama-3.1-8B", "ctx": 131072, "batch": 1, "q_layers": (0, 1), "bits": 1,
        "topk": 0.02},
    3: {"model": "LLAMA31_8B", "label": "Llama-3.1-8B", "ctx": 32768, "batch": 16, "q_layers": (0, 1), "bits": 2,
        "topk": 0.03},
    4: {"model": "QWEN25_7B", "label": "Qwen2.5-7B", "ctx": 131072, "batch": 4, "q_layers": (0,), "bits": 1,
        "topk": 0.01},
    5: {"model": "LLAMA31_70B", "label": "Llama-3.1-70B", "ctx": 131072, "batch": 1, "q_layers": (0, 1), "bits": 1,
        "topk": 0.02},
}


def model_of(args):
    from paper_2505_19586_b200 import kv_model
    return getattr(kv_model, args.model)


def metric_of(args):
    return METRIC if args.config == 2 else f"decode ms/token, BASELINE config {args.config}"


# ---------------------------------------------------------------------------
# CPU reference (oracle port of hybridkv) on the host cores
# ---------------------------------------------------------------------------
class CpuReference:
    """The reference algorithm (oracle port of hybridkv, numpy float64) at the
    config's full shapes on host cores: one quantization-friendly layer
    (quantize_layer_kv + per-step qgemv decode + append_token) and one
    sparsity-friendly layer (stage 1, critical-key prefetch, approx scores,
    top-k, fetch_topk, sparse attention, append) at the full context.  A
    decode step runs the model's layer sequence over these two layers'
    caches (n_Q quantized + n_S Top-K layers; every layer costs the same
    as its kind's representative, the contents do not change the work);
    B sequences are B independent replays (the reference has no batch
    dimension)."""

    def __init__(self, args, n_topk: int):
        import numpy as np

        from oracle import tailorkv_oracle as O

        self.O, self.np = O, np
        model = model_of(args)
        self.args, self.n_topk = args, n_topk
        ctx, bits = args.ctx, args.bits
        rng = np.random.default_rng(1)
        h, hq, d, H = model.num_kv_heads, model.num_query_heads, model.head_dim, model.hidden_dim
        self.h, self.G, self.ctx = h, hq // h, ctx
        self.n_q = len(args.q_layers)
        self.n_s = model.num_layers - self.n_q

        def f16n(shape, std=1.0):
            return (rng.standard_normal(size=shape, dtype=np.float32) * std).astype(np.float16).astype(np.float64)

        kq, vq = f16n((h, ctx, d), 0.05), f16n((h, ctx, d))
        self.new_q = (kq[:, -1].copy(), vq[:, -1].copy())
        self.qk, self.qv = O.quantize_layer(kq, vq, bits, 64)
        del kq, vq
        self.qs = f16n((hq, d))
        self.ks = f16n((h, ctx, d), 1 / math.sqrt(d))
        self.vs = f16n((h, ctx, d))
        self.w_q = f16n((hq, H, d), 1 / math.sqrt(H))
        self.hid = f16n((H,))
        self.chmax = np.abs(self.ks).max(axis=1)

    def q_layer(self):
        O = self.O
        O.quant_layer_decode(self.qs, self.qk, self.qv)
        for u in range(self.h):  # append_token (quantizer.py:445-451)
            self.qk[u].append(self.new_q[0][u])
            self.qv[u].append(self.new_q[1][u])

    def s_layer(self):
        O, np, G, ks, vs = self.O, self.np, self.G, self.ks, self.vs
        qhat = O.estimate_query(self.w_q, self.hid)
        local_start = self.ctx - 64
        for u in range(self.h):
            ch = O.select_channels(O.group_channel_scores(qhat[u * G:(u + 1) * G], self.chmax[u]), 8)
            crit = ks[u][:, ch].copy()                  # prefetch_critical_keys (memsim.py:205-225)
            sc = O.approx_scores(self.qs[u * G:(u + 1) * G][:, ch], crit)
            sel = O.select_tokens(sc, 64, self.n_topk)
            far = sel[sel < local_start]
            kf, vf = ks[u][far].copy(), vs[u][far].copy()  # fetch_topk (memsim.py:228-252)
            ksel = np.concatenate([kf, ks[u][sel[sel >= local_start]]])
            vsel = np.concatenate([vf, vs[u][sel[sel >= local_start]]])
            for j in range(G):
                O.attention_weights(self.qs[u * G + j], ksel) @ vsel

    def layer_times(self) -> tuple[float, float]:
        """Seconds of one quantized and one Top-K layer (one sample each)."""
        t0 = time.perf_counter()
        self.q_layer()
        t1 = time.perf_counter()
        self.s_layer()
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1

    def step(self) -> float:
        """One full decode step of one sequence (all layers), seconds."""
        t0 = time.perf_counter()
        for _ in range(self.n_q):
            self.q_layer()
        for _ in range(self.n_s):
            self.s_layer()
        return time.perf_counter() - t0


def cpu_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        return max([p.get("num_threads", 1) for p in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def cpu_reference_ms(args, n_topk: int) -> tuple[float, dict]:
    """Bounded in-run CPU baseline: one sample of each layer kind at the full
    context, combined as n_Q T_Q + n_S T_S per token (times B)."""
    ref = CpuReference(args, n_topk)
    tq, ts = ref.layer_times()
    ms = (ref.n_q * tq + ref.n_s * ts) * args.batch * 1e3
    return ms, {"q_layer_ms": tq * 1e3, "s_layer_ms": ts * 1e3, "threads": cpu_threads()}


def cpu_sample_text(args, prefix=""):
    model = model_of(args)
    n_q = len(args.q_layers)
    return (f"{prefix}1 quantized layer + 1 Top-K layer, both at the full {args.ctx}-token context, timed once; "
            f"token = {n_q} Q + {model.num_layers - n_q} S layers"
            + (f", x{args.batch} sequences (independent replays)" if args.batch > 1 else "")
            + "; oracle port of hybridkv (numpy float64)")


def run_reference(args, rank):
    """--impl reference: full decode steps of the reference algorithm on the
    host cores (rank 0 only).  Each timed step runs every layer of the model
    for one sequence (B sequences = B x that time); at most 1 warm-up and 2
    timed steps whatever --steps/--warmup ask (a step is ~15 s of CPU work at
    128k), and the line reports the counts actually run."""
    if rank != 0:
        return
    import numpy as np

    n_topk = round(args.topk_frac * args.ctx)
    t_setup = time.perf_counter()
    ref = CpuReference(args, n_topk)
    setup_s = time.perf_counter() - t_setup
    warm, reps = min(args.warmup, 1), max(1, min(args.steps, 2))
    times = []
    for i in range(warm + reps):
        t = ref.step()
        if i >= warm:
            times.append(t * args.batch * 1e3)
    v = float(np.mean(times))
    sample = (f"{reps} timed full decode steps after {warm} warm-up (every layer of the model at the full context, "
              f"one sequence" + (f", x{args.batch} for the batch of independent replays" if args.batch > 1 else "")
              + "); oracle port of hybridkv (numpy float64)")
    line = {
        "impl": "reference", "metric": metric_of(args), "value": v, "unit": "ms/token", "n_gpus": args.gpus,
        "steps": reps, "warmup": warm, "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": v, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, n_topk, args.gpus),
        "cpu_baseline": {"value": v, "unit": "ms/token", "cores": cpu_threads(), "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "ms/token", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": setup_s,
    }
    print(json.dumps(line), flush=True)


def workload_config(args, n_topk, world=1):
    m = model_of(args)
    c = CONFIGS[args.config]
    nq = len(args.q_layers)
    qset = "{" + ",".join(map(str, args.q_layers)) + "}"
    return {
        "workload": f"config{args.config}: {c['label']} shapes, {m.num_layers} layers (Q={qset} {args.bits}-bit g=64, "
                    f"{m.num_layers - nq} Top-K layers), ctx={args.ctx}, batch={args.batch}, n_topk={n_topk} "
                    f"({args.topk_frac:.0%}), n_local=64, d_s=8",
        "ctx": args.ctx, "batch": args.batch, "layers": m.num_layers, "q_layers": list(args.q_layers),
        "bits": args.bits, "group_size": 64, "n_topk": n_topk, "n_local": 64, "d_s": 8,
        "kv_heads": m.num_kv_heads, "q_heads": m.num_query_heads, "head_dim": m.head_dim,
        "parallelism": (f"kv-head shard x{world}" if getattr(args, "shard_of", 1) <= 1 else
                        f"rank 0's share of a kv-head shard x{args.shard_of} on one GPU, all-gather not run"),
        "key_rows_from": "host (PCIe)" if args.keys_over_pcie else "hbm (scorer copy); value rows over PCIe",
        "l2": "inputs larger than L2 (every step reads > 1 GB of HBM)",
        "cache_warm_steps": getattr(args, "cache_warm", 0),
    }


# ---------------------------------------------------------------------------
# measurement helpers
# ---------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML every 20 ms while the
    timed region runs (nvidia-smi's query fields, in-process)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.max_mhz = None

    def _run(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                try:
                    r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((sm, r))
                self._stop.wait(0.02)
        except Exception as exc:  # pragma: no cover
            self.samples.append((None, 0))
            self.error = str(exc)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        import statistics

        sm = [s for s, _ in self.samples if s is not None]
        reasons = sorted({k for _, r in self.samples for k, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm)}


def pcie_peaks(torch, lib_mod, device):
    """Measured H2D peaks on this box: pinned cudaMemcpyAsync of 256 MiB and
    a UVA zero-copy kernel reading random 512-byte rows."""
    import ctypes as C

    from paper_2505_19586_b200.hoststore import PinnedArena, gpu_numa_node

    nbytes = 256 << 20
    host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dev = torch.empty(nbytes, dtype=torch.uint8, device=device)
    for _ in range(2):
        dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        dev.copy_(host, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    memcpy_gbs = 5 * nbytes / (a.elapsed_time(b) * 1e-3) / 1e9
    arena = PinnedArena(1 << 30, gpu_numa_node(device.index or 0))
    rows_total = (1 << 30) // 512
    g = torch.Generator(device=device)
    g.manual_seed(0)
    nrows = 200_000
    rows = torch.randint(0, rows_total, (nrows,), generator=g, device=device, dtype=torch.int32)
    sink = torch.zeros(1, device=device)
    lib = lib_mod.load()
    for _ in range(2):
        lib.tkv_uva_read_probe(arena.addr, 1 << 30, 512, rows.data_ptr(), nrows, sink.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    a.record()
    for _ in range(5):
        lib.tkv_uva_read_probe(arena.addr, 1 << 30, 512, rows.data_ptr(), nrows, sink.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    b.record()
    torch.cuda.synchronize()
    uva_gbs = 5 * nrows * 512 / (a.elapsed_time(b) * 1e-3) / 1e9
    rows256 = rows * 2
    a.record()
    for _ in range(5):
        lib.tkv_uva_read_probe(arena.addr, 1 << 30, 256, rows256.data_ptr(), nrows, sink.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    b.record()
    torch.cuda.synchronize()
    uva256_gbs = 5 * nrows * 256 / (a.elapsed_time(b) * 1e-3) / 1e9
    arena.close()
    del host, dev
    return memcpy_gbs, uva_gbs, uva256_gbs


def relaunch(args) -> int:
    """``bench.py --gpus N`` run without a launcher: start N ranks with
    torch.distributed.run on this node (127.0.0.1) and pass rank 0's line
    through."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    import paper_2505_19586_b200 as P
    from paper_2505_19586_b200 import _lib
    from paper_2505_19586_b200.synth import make_workload

    _lib.load()
    model = model_of(args)
    B = args.batch
    L, n = model.num_layers, args.ctx
    n_topk = round(args.topk_frac * n)
    cfg = P.EngineConfig(bits=args.bits, group_size=64, n_local=64, n_topk=n_topk, critical_channels=8,
                         keys_from_hbm=not args.keys_over_pcie, fused_sparse=not args.unfused,
                         token_major_keys=not args.single_copy_keys,
                         row_cache=args.cache_steps > 0, row_cache_steps=max(1, args.cache_steps),
                         scorer_l2_prefetch=not args.no_l2_prefetch, overlap_stage1=not args.serial_stage1)
    W, K = args.warmup, args.steps
    PROF = 2
    total = args.cache_warm + W + 3 * K + 2 * PROF + 2 * min(K, 20) + 24
    t_setup = time.time()
    wl = make_workload(L, args.q_layers, model.num_query_heads, model.num_kv_heads, model.head_dim, n, total,
                       batch=B, seed=args.seed, device=device)
    if args.shard_of > 1:  # one rank's share of an N-GPU run, collective not run (see --help)
        eng = P.DecodeEngine(model, wl.labels, cfg, batch=B, max_steps=total, rank=0, world_size=args.shard_of,
                             process_group="none", device=device)
    else:
        eng = P.DecodeEngine(model, wl.labels, cfg, batch=B, max_steps=total, rank=rank, world_size=world,
                             device=device)
    if os.environ.get("TKV_FZ_DBG"):  # experiments in the sparse kernel (debug bits)
        _lib.load().tkv_debug_sparse_trace(int(os.environ["TKV_FZ_DBG"]) & ~1)
    if os.environ.get("TKV_AIM"):  # tuning: first aimed range half-width (score sd)
        import ctypes
        _lib.load().tkv_debug_sparse_aim(ctypes.c_float(float(os.environ["TKV_AIM"])))
    for l in range(L):
        eng.prefill(l, wl.prefill_keys[l], wl.prefill_values[l], wl.w_q[l])
        wl.prefill_keys[l] = wl.prefill_values[l] = None
    torch.cuda.synchronize()
    setup_s = time.time() - t_setup

    step_i = 0

    def inputs(t):
        return wl.hidden[t], wl.queries[t], wl.new_keys[t], wl.new_values[t]

    # per-kernel profile: the step graph captured with an event-record node
    # around every kernel group, replayed like the timed graph (no host gaps)
    def profile_mode():
        nonlocal step_i
        eng.capture_profiled()
        res = {}
        c0 = eng.cache_counters()
        for _ in range(PROF):
            eng.load_step(*inputs(step_i))
            for k, v in eng.replay_profiled().items():
                res.setdefault(k, []).extend(v)
            step_i += 1
        c1 = eng.cache_counters()
        return res, c1[0] - c0[0], c1[1] - c0[1]

    n_sparse = sum(1 for x in wl.labels if x == "s")
    # row-cache warm-up: untimed decode steps before any timed loop
    eng.capture()
    for _ in range(args.cache_warm):
        eng.step(*inputs(step_i)); step_i += 1
    torch.cuda.synchronize()
    # variant: the other key-row source, graph-timed for K steps, then profiled
    eng.keys_from_hbm = args.keys_over_pcie
    eng.capture()
    for _ in range(2):
        eng.step(*inputs(step_i)); step_i += 1
    torch.cuda.synchronize()
    sv, ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sv.record()
    for _ in range(K):
        eng.step(*inputs(step_i)); step_i += 1
    ev.record()
    torch.cuda.synchronize()
    ms_variant = sv.elapsed_time(ev) / K
    prof_alt, _, _ = profile_mode()

    eng.keys_from_hbm = not args.keys_over_pcie
    eng.capture()
    for _ in range(W):
        eng.step(*inputs(step_i)); step_i += 1
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- end-to-end first (the HBM row cache is colder than in the device-resident loop after it):
    # pinned host inputs in, outputs back to host, every step, through DecodeEngine.step_host: the
    # host-I/O graph copies the inputs in (first two layers' slices, then the rest) and the outputs back
    # (all but the last L/8 layers as soon as those are done, then the tail), on a copy stream beside
    # the layers ----
    host_in = [tuple(x.cpu().pin_memory() for x in inputs(step_i + k)) for k in range(K + 2)]
    h2d = sum(x.numel() * x.element_size() for x in host_in[0])  # every rank receives the full step input
    if args.e2e_plain:
        host_out = torch.empty(eng.out.shape, dtype=torch.float32).pin_memory()
        run_host = lambda x: (eng.step(*x), host_out.copy_(eng.out, non_blocking=True))  # noqa: E731
    else:
        eng.capture(host_io=True)
        host_out = eng.host_out
        run_host = lambda x: eng.step_host(*x)  # noqa: E731
    d2h = host_out.numel() * host_out.element_size()
    for k in range(2):  # the first replays of the graph, untimed
        run_host(host_in[k]); step_i += 1
    barrier(); torch.cuda.synchronize()
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ec0 = eng.cache_counters()
    s2.record()
    for k in range(K):
        run_host(host_in[2 + k]); step_i += 1
    e2.record()
    torch.cuda.synchronize(); barrier()
    ms_e2e = s2.elapsed_time(e2) / K
    ec1 = eng.cache_counters()
    e2e_hit = (ec1[0] - ec0[0]) / max(1, (ec1[0] - ec0[0]) + (ec1[1] - ec0[1]))
    del host_in
    eng.capture()  # device-resident graph for the loops below

    # ---- device-resident timing (value) ----
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tc0 = eng.cache_counters()
    with ClockSampler(local) as clocks:
        barrier(); torch.cuda.synchronize()
        start.record()
        for _ in range(K):
            eng.step(*inputs(step_i)); step_i += 1
        end.record()
        torch.cuda.synchronize(); barrier()
    ms = start.elapsed_time(end) / K
    t_hits, t_misses = eng.cache_counters()
    t_hits, t_misses = t_hits - tc0[0], t_misses - tc0[1]

    # ---- sparse-layer period inside the timed graph (PDL kept): per-launch globaltimer stamps of the
    # fused kernel (unit 0, CTA rank 0) over one more plain-graph step ----
    lib = _lib.load()
    trace_mode = int(os.environ.get("TKV_FZ_DBG", "0")) & ~1
    from tools.fz_phases import wide_enable, wide_launches
    lib.tkv_debug_sparse_launches(None, 1)
    lib.tkv_debug_sparse_trace(1 | trace_mode)
    wide_enable(lib)
    eng.step(*inputs(step_i)); step_i += 1
    torch.cuda.synchronize()
    lib.tkv_debug_sparse_trace(trace_mode)
    wide_enable(lib, False)
    import ctypes as C
    raw = (C.c_ulonglong * (128 * 3))()
    cnt = lib.tkv_debug_sparse_launches(raw, 0)
    stamps = [(raw[i * 3], raw[i * 3 + 1], raw[i * 3 + 2]) for i in range(min(cnt, 128))]
    path = lib.tkv_debug_sparse_path()  # what the dispatch chose: cluster size, 0 wide, -1 unfused
    if path == 0:  # the wide decode
        stamps = wide_launches(lib)
        sparse_kernel = f"wide (sparse_wide_kernel, {_lib.wide_parts(eng.units)} CTAs per unit)"
    elif path > 0:
        sparse_kernel = f"cluster (sparse_fused_kernel, one {path}-CTA cluster per unit)"
        if path != 8:
            stamps = []  # (the launch stamps are recorded by the 8-CTA build only)
    else:
        sparse_kernel = "unfused (select, gather + attention, append)"
        stamps = []
    plain = None
    if len(stamps) >= 2 and not args.unfused:
        ends = [x[2] for x in stamps]
        period = (ends[-1] - ends[0]) / (len(ends) - 1) / 1e6          # ms between consecutive layer ends
        body = sorted((x[2] - x[1]) / 1e6 for x in stamps)[len(stamps) // 2]  # PDL wait -> end, median
        plain = {"period_ms": period, "body_ms": body, "launches": len(stamps)}

    # fidelity of one eager step against exact attention over all tokens (GPU, outside the timing)
    fidelity = None
    if not args.no_fidelity:
        eng.record_selection = True
        graph, eng.graph = eng.graph, None
        eng.step(*inputs(step_i)); step_i += 1
        fl = [eng.layer_fidelity(l) for l in range(L) if wl.labels[l] == "s"]
        eng.graph, eng.record_selection = graph, False
        fidelity = {"layers": len(fl), "recall_mean": sum(f["recall"] for f in fl) / len(fl),
                    "recall_min": min(f["recall"] for f in fl),
                    "selected_mass_mean": sum(f["selected_mass"] for f in fl) / len(fl),
                    "cosine_min": min(f["cosine"] for f in fl),
                    "note": "one step, Top-K layers, vs exact softmax attention over all tokens "
                            "(pipeline.py:316-403 metrics, computed on the GPU)"}

    # per-kernel profile of the main mode, steady state (after the timed steps)
    if args.phases:
        from tools.fz_phases import enable
        enable(_lib.load())
    prof, hits, misses = profile_mode()
    if args.phases and rank == 0:
        from tools.fz_phases import show, show_launches
        _lib.load().tkv_debug_sparse_trace(int(os.environ.get("TKV_FZ_DBG", "0")) & ~1)
        show(_lib.load())
        # launch gaps inside the plain (timed) graph: one more step with the trace on
        enable(_lib.load())
        eng.step(*inputs(step_i)); step_i += 1
        torch.cuda.synchronize()
        _lib.load().tkv_debug_sparse_trace(int(os.environ.get("TKV_FZ_DBG", "0")) & ~1)
        print("plain graph:")
        show_launches(_lib.load())
        from tools.fz_phases import wide_enable, wide_show
        wide_enable(_lib.load())
        eng.step(*inputs(step_i)); step_i += 1
        torch.cuda.synchronize()
        wide_enable(_lib.load(), False)
        print("plain graph, wide decode:")
        wide_show(_lib.load(), _lib.wide_parts(eng.units))
    fetch_rows = int(eng.fetch_count.sum().item())
    cached_rows = hits / (PROF * n_sparse)     # per launch, served from the HBM row cache
    pcie_rows = misses / (PROF * n_sparse)     # per launch, fetched over PCIe

    def timed(steps, src):
        """Graph-replayed steps from ``src(k)`` inputs: (ms/token, hit rate, PCIe value rows per launch)."""
        nonlocal step_i
        eng.capture()
        for k in range(2):
            eng.step(*src(k)); step_i += 1
        torch.cuda.synchronize()
        c0 = eng.cache_counters()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(steps):
            eng.step(*src(2 + k)); step_i += 1
        b.record()
        torch.cuda.synchronize()
        c1 = eng.cache_counters()
        hh, mm = c1[0] - c0[0], c1[1] - c0[1]
        return a.elapsed_time(b) / steps, hh / max(1, hh + mm), mm / max(1, steps * n_sparse)

    # ---- the same engine with the row cache off (every selected far value row over PCIe) ----
    KX = min(K, 20)
    cache_off = None
    if cfg.row_cache and not args.keys_over_pcie:
        eng.set_row_cache(False)
        base = step_i
        ms_off, _, _ = timed(KX, lambda k: inputs(base + k))
        eng.set_row_cache(True)
        cache_off = {"ms_per_token": ms_off, "steps": KX,
                     "note": "row cache switched off on the same engine and inputs: every selected far value row "
                             "crosses PCIe each step (key rows still from HBM)"}
    # ---- drift workload: the reference's ChannelOutlierSpec(drift=True) step inputs (trace.py:434-436) ----
    from paper_2505_19586_b200.synth import step_inputs
    d_hid, d_q = step_inputs(wl, KX + 2, drift=True, seed=args.seed + 1)
    base = step_i
    ms_drift, hit_drift, pcie_drift = timed(KX, lambda k: (d_hid[k], d_q[k], wl.new_keys[base + k],
                                                           wl.new_values[base + k]))
    drift = {"ms_per_token": ms_drift, "steps": KX, "row_cache_hit_rate": hit_drift,
             "pcie_value_rows_per_launch": pcie_drift,
             "note": "same prefilled caches; step hidden states with the reference's per-step lognormal(0, 0.6) "
                     "scaling of the planted outlier coordinates (synth.step_inputs, trace.py:268-275, 434-436), "
                     "queries q = h W_q; the row cache carries over from the stationary steps"}
    del d_hid, d_q

    if world > 1:
        t = torch.tensor([ms, ms_e2e], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e = t.tolist()

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_key = next((k for k in peaks if "hbm" in k.lower() and isinstance(peaks[k], (int, float))), None)
    hbm_peak = float(peaks[hbm_key]) if hbm_key else 6552.0
    hbm_src = f"MEASURED_PEAKS.json:{hbm_key}" if hbm_key else "BASELINE.md measured copy peak (MEASURED_PEAKS.json absent)"
    memcpy_gbs, uva_gbs, uva256_gbs = pcie_peaks(torch, _lib, device)

    def mean(x):
        return sum(x) / len(x) if x else float("nan")

    U = eng.units
    quant_ms = mean(prof.get("quant_decode", []))
    stage1_ms = mean(prof.get("stage1", []))
    if args.unfused:
        sparse_ms = mean(prof.get("select", [])) + mean(prof.get("gather_attend", []))
        alt_ms = mean(prof_alt.get("select", [])) + mean(prof_alt.get("gather_attend", []))
    else:
        sparse_ms = mean(prof.get("sparse_decode", []))
        alt_ms = mean(prof_alt.get("sparse_decode", []))
    sparse_node_ms = sparse_ms
    if plain is not None:
        # the layer period inside the timed (plain) graph: consecutive sparse launches' end-to-end spacing,
        # so n_S x period + the quantized layers fits in ms_per_step (event nodes break the PDL overlap)
        sparse_ms = plain["period_ms"]
    append_ms = mean(prof.get("sparse_append", []))
    from oracle import tailorkv_oracle as O  # byte formulas only (memsim.py accounting)
    d = model.head_dim
    # PCIe bytes of one sparse-layer launch: K+V rows (memsim.py:249, no row cache) or, in the
    # default mode, the value rows that missed the HBM row cache (counted by the kernel)
    gather_bytes = O.gather_bytes(fetch_rows, d) if args.keys_over_pcie else int(pcie_rows * d * 2)
    alt_bytes = O.gather_bytes(fetch_rows, d) if not args.keys_over_pcie else fetch_rows * d * 2
    quant_bytes = O.quant_layer_bytes(n, U, d, args.bits, 64)
    scorer_bytes = O.scorer_bytes(n, U, 8)
    # HBM bytes of the same launch: scorer columns + key rows (+ cached value rows)
    sparse_hbm = scorer_bytes + (0 if args.keys_over_pcie else int(fetch_rows * d * 2 + cached_rows * d * 2))
    wq_bytes = eng.hq_r * model.hidden_dim * d * 2
    rooflines = {
        # HBM is the resource the kernel moves most bytes through (scorer columns, key rows, cached
        # value rows); the PCIe leg (value rows that missed the row cache) is reported beside it
        "sparse_decode": {"bound": "hbm", "achieved": sparse_hbm / (sparse_ms * 1e-3) / 1e9,
                          "peak": hbm_peak, "unit": "GB/s", "ms": sparse_ms, "bytes": sparse_hbm,
                          "peak_source": hbm_src,
                          "pcie_bytes": gather_bytes, "pcie_gbs": gather_bytes / (sparse_ms * 1e-3) / 1e9,
                          "pcie_peak": memcpy_gbs,
                          "pcie_peak_source": "measured pinned cudaMemcpyAsync H2D 256 MiB, this run",
                          "kernel": (f"{sparse_kernel}: scores + top-k + gather + attention + append"
                                     if not args.unfused else "select + sparse_attn"),
                          "timing": ("layer period in the plain timed graph: (end of the last sparse launch - end of "
                                     "the first) / (launches - 1), globaltimer stamps of unit 0"
                                     if plain is not None else "graph event nodes"),
                          "body_ms": plain["body_ms"] if plain else None, "graph_node_ms": sparse_node_ms},
        "quant_decode": {"bound": "hbm", "achieved": quant_bytes / (quant_ms * 1e-3) / 1e9, "peak": hbm_peak,
                         "unit": "GB/s", "ms": quant_ms, "bytes": quant_bytes, "peak_source": hbm_src},
        "stage1": {"bound": "hbm", "achieved": wq_bytes / (stage1_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                   "ms": stage1_ms, "bytes": wq_bytes, "peak_source": hbm_src},
    }
    if append_ms == append_ms:  # (separate append launch: unfused path)
        rooflines["sparse_append"] = {"ms": append_ms}
    for r in rooflines.values():
        if "achieved" in r:
            r["frac"] = r["achieved"] / r["peak"]
    rooflines["sparse_decode"]["pcie_frac"] = rooflines["sparse_decode"]["pcie_gbs"] / memcpy_gbs
    dom = rooflines["sparse_decode"]
    # DRAM traffic per launch from the committed ncu --set full capture of the same kernels
    traffic = {}
    tpath = ROOT / "profiles" / "r2" / "r2_ncu_traffic.json"
    if tpath.exists():
        traffic = json.loads(tpath.read_text())
    def _traffic(name):
        t = traffic.get(name)
        return None if t is None else t["dram_bytes_read"] + t["dram_bytes_write"]
    rooflines["quant_decode"]["traffic"] = _traffic("quant_decode_pipe_kernel") or _traffic("quant_decode_imma_kernel")
    # (stage 1's DRAM bytes include the 16.8 MB L2 prefetch of the next layer's scorer columns it issues)
    rooflines["stage1"]["traffic"] = _traffic("stage1_fused_kernel") if args.batch <= 2 else None
    # f4: the reference's decode-step timeline model (memsim.py:339-602) driven by the costs measured above
    from tools.timeline_model import measured_step
    bw = memcpy_gbs * 1e9
    tl_serial = measured_step(wl.labels, quant_ms * 1e-3, sparse_ms * 1e-3, stage1_ms * 1e-3, gather_bytes, bw)
    tl_side = measured_step(wl.labels, quant_ms * 1e-3, sparse_ms * 1e-3, 0.0, gather_bytes, bw)
    tl_ref = measured_step(wl.labels, quant_ms * 1e-3, sparse_ms * 1e-3, stage1_ms * 1e-3,
                           O.gather_bytes(fetch_rows, d), bw, prefetch_bytes=scorer_bytes)
    timeline_model = {
        "measured_ms": ms,
        "model_ms": tl_side["step_seconds"] * 1e3,
        "model_serial_estimate_ms": tl_serial["step_seconds"] * 1e3,
        "model_reference_transfers_ms": tl_ref["step_seconds"] * 1e3,
        "model_reference_transfers_overlap": tl_ref["overlap_fraction"],
        "model_reference_transfers_stall_ms": tl_ref["stall_seconds"] * 1e3 / 4,
        "note": "tools/timeline_model.py (the reference model, golden-tested) fed with this run's per-kernel "
                "times (graph-node events) and PCIe bytes: model_ms runs stage 1 concurrently (side stream), "
                "model_serial_estimate_ms on the one compute engine the reference assumes, "
                "model_reference_transfers_ms with the reference's per-step critical-key prefetch and K+V Top-K "
                "fetch over the measured H2D bandwidth",
    }
    # resident bytes against the reference's closed-form footprints (memsim.py:641-706)
    res = eng.resident_bytes()
    h_all = model.num_kv_heads * B
    orig = 2 * L * n * h_all * d * 2
    n_q = len(args.q_layers)
    ref_hybrid = (2 * n_q * n * h_all * d * 2 * (args.bits / 16 + 2 / 64)      # hybridkv_q
                  + n_sparse * 2 * n * h_all * 8 * 2                           # hybridkv_s (d_s = 8)
                  + n_sparse * 64 * 2 * h_all * d * 2)                         # local windows
    memory = {"resident": res,
              "reference_original_bytes": orig, "reference_hybrid_device_bytes": int(ref_hybrid),
              "reference_host_kv_bytes": n_sparse * 2 * n * h_all * d * 2,
              "note": "hbm: this rank's device allocations by structure; the reference model keeps 2*n*h*d_s key "
                      "columns per sparse layer on the device (hybridkv_s) and re-sends them every step, this "
                      "engine keeps all keys resident (channel-major for the scorer, plus a token-major copy "
                      "unless EngineConfig.token_major_keys=False) so nothing but missed value rows crosses PCIe"}
    line = {
        "metric": metric_of(args), "value": ms, "unit": "ms/token", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": f"fp16 storage / {args.bits}-bit codes, fp32 accumulate",
        "data": "synthetic (gen_trace-shaped, GPU-generated)",
        "config": workload_config(args, n_topk, world),
        "roofline": {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"], "unit": "GB/s",
                     "frac": dom["frac"], "traffic": _traffic("sparse_fused_kernel") if not args.unfused else None,
                     "traffic_note": "DRAM bytes per launch of the cluster kernel (ncu --set full capture of a "
                                     "main-mode launch, profiles/r2/r2_ncu_traffic.json): 29.9 MB against 27.5 MB "
                                     "algorithmic",
                     "bound_note": "the launch is a chain of ~15 dependent, latency-bound phases (scores, select, "
                                   "gather, attention, merges) plus its instruction fetch (121 KB of SASS per launch); "
                                   "it takes ~43 us whatever the work per CTA (DESIGN.md 4.7, profiles/r2/"
                                   "r2_kernels.md), far from the HBM roofline; the PCIe leg is "
                                   "rooflines.sparse_decode.pcie_*",
                     "kernel": dom["kernel"], "timing": dom["timing"]},
        "rooflines": rooflines,
        "row_cache": {"window_steps": cfg.row_cache_steps, "slots_per_head": (eng.retrieval.n_local + eng.retrieval.n_topk) * cfg.row_cache_steps,
                      "timed_region_hit_rate": t_hits / max(1, t_hits + t_misses),
                      "timed_region_pcie_value_bytes_per_token": t_misses * model.head_dim * 2 / K,
                      "rows_per_launch_from_hbm_cache": cached_rows, "rows_per_launch_over_pcie": pcie_rows,
                      "note": "value rows selected in the last window_steps steps stay in HBM; exact (rows never change)"},
        "pcie": {"memcpy_h2d_gbs": memcpy_gbs, "uva_512B_rows_gbs": uva_gbs, "uva_256B_rows_gbs": uva256_gbs,
                 "gather_bytes_per_token": gather_bytes * n_sparse, "fetched_rows_per_layer": fetch_rows,
                 "reference_fetch_topk_bytes_per_token": O.gather_bytes(fetch_rows, model.head_dim) * n_sparse},
        "e2e": {"value": ms_e2e, "unit": "ms/token", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "row_cache_hit_rate": e2e_hit,
                "note": "DecodeEngine.step_host: pinned host inputs copied in and the outputs copied back to pinned "
                        "host memory every step by the host-I/O graph (copies on a copy stream, overlapped with "
                        "the layers: the first two layers' inputs first; outputs in two pieces, the last L/8 "
                        "layers' at the end); runs "
                        "on the K steps right after the warm-up, BEFORE the device-resident ones; both loops run "
                        "after cache_warm_steps untimed steps (the row cache's hit rate rises over the first "
                        "~100 steps)"},
        "cache_off": cache_off,
        "drift": drift,
        "memory": memory,
        "variant": {"key_rows_from": "hbm" if args.keys_over_pcie else "host (PCIe, the reference's fetch_topk transfer)",
                    "ms_per_token": ms_variant, "sparse_decode_ms": alt_ms,
                    "pcie_gbs": alt_bytes / (alt_ms * 1e-3) / 1e9, "pcie_bytes": alt_bytes,
                    "pcie_frac": alt_bytes / (alt_ms * 1e-3) / 1e9 / memcpy_gbs},
        "fidelity": fidelity,
        "timeline_model": timeline_model,
        "gpu_launches": eng.kernels_per_step() * K,
        "clocks": clocks.summary(),
        "plain_graph_sparse_trace": plain,
        "setup_s": setup_s,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cms, info = cpu_reference_ms(args, n_topk)
        line["cpu_baseline"] = {"value": cms, "unit": "ms/token", "cores": info["threads"], "kind": "port",
                                "sample": cpu_sample_text(args), "detail": info}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
