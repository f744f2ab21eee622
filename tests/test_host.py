"""CPU tests: C-ABI exports, shard planning, and the N>1 exchange step on gloo."""

import os
import re
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import tailorkv_oracle as O

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_header_symbol():
    from paper_2505_19586_b200 import _lib

    lib = _lib.load()
    hdr = (ROOT / "include" / "tailorkv.h").read_text()
    declared = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(tkv_\w+)\s*\(", hdr, flags=re.M))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.exported_symbols())
    assert lib.tkv_abi_version() == 1


def test_status_codes_map_to_reference_exceptions():
    from paper_2505_19586_b200 import _lib, errors

    for code, cls in [(1, errors.ShapeError), (2, errors.ParameterError), (3, errors.EmptyCacheError),
                      (4, errors.NumericError), (5, errors.EncodingError), (6, errors.SchedulingError)]:
        with pytest.raises(cls):
            _lib.check(code)


def test_qcache_sizes_validation_without_gpu():
    import ctypes as C

    from paper_2505_19586_b200 import _lib
    from paper_2505_19586_b200.errors import ParameterError, ShapeError

    lib = _lib.load()
    sizes = (C.c_int64 * 6)()
    tile = C.c_int32()
    assert lib.tkv_qcache_sizes(8, 128, 1, 64, 131072, sizes, C.byref(tile)) == 0
    # Table 2 accounting: codes + 16-bit (lo,hi) per group = 50,331,648 B per layer
    codes = sizes[0] + sizes[3]
    params = sizes[1] + sizes[4]
    assert codes + params == O.quant_layer_bytes(131072, 8, 128, 1, 64)
    with pytest.raises(ParameterError):
        _lib.check(lib.tkv_qcache_sizes(8, 128, 3, 64, 131072, sizes, C.byref(tile)))
    with pytest.raises(ShapeError):
        _lib.check(lib.tkv_qcache_sizes(8, 100, 1, 64, 131072, sizes, C.byref(tile)))


@pytest.mark.parametrize("batch,heads,world", [(1, 8, 1), (1, 8, 2), (1, 8, 8), (16, 8, 2), (16, 8, 8),
                                               (4, 4, 8), (1, 8, 4)])
def test_shard_plan_covers_units_once(batch, heads, world):
    from paper_2505_19586_b200.engine import shard_plan

    plan = shard_plan(batch, heads, world)
    seen = np.zeros((batch, heads), int)
    for s in plan:
        seen[s.b0:s.b0 + s.batch, s.k0:s.k0 + s.kv_heads] += 1
    assert (seen == 1).all()


def test_shard_plan_rejects_uneven():
    from paper_2505_19586_b200.engine import shard_plan
    from paper_2505_19586_b200.errors import ConfigError

    with pytest.raises(ConfigError):
        shard_plan(1, 8, 3)


def _gloo_worker(rank, world, port, batch, heads, G, d, seed, q):
    import torch.distributed as dist

    from paper_2505_19586_b200.engine import assemble, shard_plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(seed)
        n = 300
        keys = rng.normal(size=(batch, heads, n, d))
        values = rng.normal(size=(batch, heads, n, d))
        queries = rng.normal(size=(batch, heads * G, d))
        plan = shard_plan(batch, heads, world)
        s = plan[rank]
        # each rank computes only its heads (oracle exact attention stands in
        # for the per-rank kernel output), then the per-layer exchange step
        local = np.stack([O.exact_layer_attention(queries[b, s.k0 * G:(s.k0 + s.kv_heads) * G],
                                                  keys[b, s.k0:s.k0 + s.kv_heads], values[b, s.k0:s.k0 + s.kv_heads])
                          for b in range(s.b0, s.b0 + s.batch)])
        t = torch.from_numpy(local.reshape(-1, d)).float()
        out = torch.zeros(world * t.shape[0], d)
        dist.all_gather_into_tensor(out, t)
        parts = [out.view(world, -1, d)[r].reshape(p.batch, p.kv_heads * G, d) for r, p in enumerate(plan)]
        full = assemble(parts, plan, batch, heads).numpy()
        ref = np.stack([O.exact_layer_attention(queries[b], keys[b], values[b]) for b in range(batch)])
        q.put((rank, float(np.abs(full - ref).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch,heads,G", [(1, 8, 4), (4, 4, 7)])
def test_head_sharded_allgather_gloo(batch, heads, G):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + batch
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, batch, heads, G, 32, 7, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(err < 1e-5 for _, err in res), res


def test_bench_configs_match_baseline():
    """bench.py --config 2..5 carry BASELINE.json's shapes (SURVEY.md 8(d) fills the open
    choices), and every config's units split over the GPU counts the metric names."""
    import json
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    import bench
    from paper_2505_19586_b200 import kv_model
    from paper_2505_19586_b200.engine import shard_plan

    base = json.loads((root / "BASELINE.json").read_text())
    assert len(base["configs"]) == 5
    expect = {2: (32, 8, 131072, 1, 2621), 3: (32, 8, 32768, 16, 983), 4: (28, 4, 131072, 4, 1311),
              5: (80, 8, 131072, 1, 2621)}
    for c, (L, h, n, B, topk) in expect.items():
        args = type("A", (), {})()
        cfg = bench.CONFIGS[c]
        args.config, args.ctx, args.topk_frac = c, cfg["ctx"], cfg["topk"]
        args.batch, args.bits, args.q_layers, args.model = cfg["batch"], cfg["bits"], cfg["q_layers"], cfg["model"]
        args.gpus, args.keys_over_pcie = 1, False
        m = getattr(kv_model, cfg["model"])
        assert (m.num_layers, m.num_kv_heads, cfg["ctx"], cfg["batch"]) == (L, h, n, B)
        w = bench.workload_config(args, round(cfg["topk"] * n))
        assert w["n_topk"] == topk and w["layers"] == L and w["batch"] == B
        assert w["workload"].startswith(f"config{c}:")
        for world in (1, 2, 4, 8):
            plan = shard_plan(B, h, world)
            assert sum(p.batch * p.kv_heads for p in plan) == B * h
    assert bench.metric_of(type("A", (), {"config": 2})()) == base["metric"]


@pytest.mark.parametrize("batch,heads,world", [(1, 8, 8), (1, 8, 2), (16, 8, 8), (4, 4, 8), (2, 4, 2)])
def test_step_inputs_full_or_presharded(batch, heads, world):
    """DecodeEngine.load_step accepts full inputs or the rank's slice; a
    pre-sharded batch-1 input is not sliced a second time."""
    from paper_2505_19586_b200.engine import shard_plan, slice_step_input

    L, G, d = 3, 4, 8
    q = torch.arange(L * batch * heads * G * d, dtype=torch.float32).view(L, batch, heads * G, d)
    kv = torch.arange(L * batch * heads * d, dtype=torch.float32).view(L, batch, heads, d)
    for s in shard_plan(batch, heads, world):
        want_q = q[:, s.b0:s.b0 + s.batch, s.k0 * G:(s.k0 + s.kv_heads) * G]
        want_kv = kv[:, s.b0:s.b0 + s.batch, s.k0:s.k0 + s.kv_heads]
        assert torch.equal(slice_step_input(q, s, batch, heads, G, world), want_q)
        assert torch.equal(slice_step_input(kv, s, batch, heads, 1, world), want_kv)
        # already the rank's slice: unchanged
        assert torch.equal(slice_step_input(want_q, s, batch, heads, G, world), want_q)
        assert torch.equal(slice_step_input(want_kv, s, batch, heads, 1, world), want_kv)
