"""Golden outputs of the reference's timeline model (hybridkv/memsim.py:339-602).

Run in the build container (imports hybridkv read-only from /root/reference):

    python tests/golden/make_timeline_golden.py

Writes tests/golden/timeline.json: per case the inputs and the reference's
total time, overlap fraction, stall time, per-layer sums and event starts.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from hybridkv import memsim as M  # noqa: E402
from hybridkv.identifier import LayerKind  # noqa: E402


def case(seed, L, steps, sparse_frac):
    rng = np.random.default_rng(seed)
    labels = ["s" if rng.random() < sparse_frac else "q" for _ in range(L)]
    compute = [float(x) for x in rng.uniform(1e-4, 1e-3, L)]
    est, score = float(rng.uniform(0, 3e-4)), float(rng.uniform(0, 3e-4))
    bw, lat = float(rng.uniform(4e9, 64e9)), float(rng.uniform(0, 5e-6))
    pre = [[int(rng.integers(0, 20_000_000)) if x == "s" else 0 for x in labels] for _ in range(steps)]
    fet = [[int(rng.integers(0, 12_000_000)) if x == "s" else 0 for x in labels] for _ in range(steps)]
    kinds = [LayerKind.SPARSITY_FRIENDLY if x == "s" else LayerKind.QUANTIZATION_FRIENDLY for x in labels]
    tl = M.build_timeline(kinds, M.LayerCosts(tuple(compute), est, score), M.LinkModel(bw, lat), pre, fet)
    r = M.simulate(tl)
    return {"labels": labels, "compute": compute, "estimate": est, "score": score, "bandwidth": bw, "latency": lat,
            "prefetch": pre, "fetch": fet, "total": r.total_seconds, "overlap": r.overlap_fraction,
            "stall": r.stall_seconds, "per_layer": {str(k): v for k, v in r.per_layer.items()},
            "starts": [e.start for e in tl.events], "labels_ev": [e.label for e in tl.events]}


cases = [case(1, 4, 3, 0.5), case(2, 8, 4, 0.8), case(3, 6, 2, 1.0), case(4, 5, 5, 0.0), case(5, 32, 3, 0.94)]
(HERE / "timeline.json").write_text(json.dumps(cases))
print("wrote", len(cases), "cases")
