"""Decode-step timeline model (hybridkv/memsim.py:255-602), fed with measured costs.

The reference predicts a decode step with a two-resource event DAG: one
compute engine and one host->device link, earliest-start list scheduling,
and a double-buffered critical-key slot per sparse layer.  This module keeps
that model's API (``LinkModel``, ``LayerCosts``, ``build_timeline``,
``simulate``) so reference scripts can run against it, and adds
``measured_step`` which builds the DAG from the per-kernel times and PCIe
bytes bench.py measures on the GPU.  It is host-side
analysis code: nothing here runs on the decode path.
"""

from __future__ import annotations

import enum
import heapq
from dataclasses import dataclass, field
from typing import Sequence

from paper_2505_19586_b200.errors import ParameterError, SchedulingError, ShapeError


@dataclass(frozen=True)
class LinkModel:
    """duration = base_latency + bytes / bandwidth; empty transfers take no time (memsim.py:45-63)."""

    bandwidth: float
    base_latency: float = 0.0

    def __post_init__(self) -> None:
        if self.bandwidth <= 0:
            raise ParameterError(f"bandwidth must be positive, got {self.bandwidth}")
        if self.base_latency < 0:
            raise ParameterError(f"base_latency must be >= 0, got {self.base_latency}")

    def transfer_seconds(self, nbytes: int) -> float:
        if nbytes < 0:
            raise ParameterError("transfer size must be >= 0")
        return 0.0 if nbytes == 0 else self.base_latency + nbytes / self.bandwidth


@dataclass(frozen=True)
class LayerCosts:
    """Per-layer compute seconds plus the estimate / score pass costs (memsim.py:318-331)."""

    compute: tuple[float, ...]
    estimate: float = 0.0
    score: float = 0.0

    def __post_init__(self) -> None:
        if min(self.compute, default=0.0) < 0 or self.estimate < 0 or self.score < 0:
            raise ParameterError("costs must be non-negative")


class EventKind(str, enum.Enum):
    COMPUTE = "compute"
    TRANSFER = "transfer"


@dataclass
class TimelineEvent:
    id: int
    kind: EventKind
    layer: int
    step: int
    label: str
    duration: float
    depends_on: list[int] = field(default_factory=list)
    start: float | None = None
    writes_slot: tuple[int, int] | None = None
    reads_slot: tuple[int, int] | None = None

    @property
    def end(self) -> float:
        if self.start is None:
            raise SchedulingError("event has not been scheduled")
        return self.start + self.duration


@dataclass
class SimulationResult:
    events: list[TimelineEvent]
    total_seconds: float
    per_layer: dict[int, dict[str, float]]
    overlap_fraction: float
    stall_seconds: float

    def to_dict(self) -> dict:
        return {"total_seconds": self.total_seconds,
                "per_layer": {str(k): dict(v) for k, v in sorted(self.per_layer.items())},
                "overlap_fraction": self.overlap_fraction, "stall_seconds": self.stall_seconds}


def _sparse(label) -> bool:
    return str(getattr(label, "value", label)) in ("s", "sparsity_friendly", "sparse")


def build_timeline(labels: Sequence, costs: LayerCosts, link: LinkModel, prefetch_bytes: Sequence[Sequence[int]],
                   fetch_bytes: Sequence[Sequence[int]]) -> list[TimelineEvent]:
    """Event DAG of ``len(prefetch_bytes)`` decode steps (memsim.py:339-459).

    Sparse layer l: estimate (ready once layer l-1's input hidden state
    exists) -> critical-key prefetch into slot t % 2 (after the score that
    read that slot two steps earlier) -> score (also after layer l's input)
    -> Top-K fetch -> compute.  Quantized layers: compute after their input.
    Estimates of layers 0 and 1 are issued at step start, then the estimate
    of layer l+2 right after layer l's events.
    """
    L = len(labels)
    if len(costs.compute) != L:
        raise ShapeError(f"{len(costs.compute)} compute costs for {L} layers")
    if len(fetch_bytes) != len(prefetch_bytes):
        raise ShapeError("prefetch_bytes and fetch_bytes must cover the same steps")
    ev: list[TimelineEvent] = []
    main: dict[tuple[int, int], int] = {}
    scores: dict[tuple[int, int], int] = {}

    def new(kind, layer, step, label, dur, deps, writes=None, reads=None) -> int:
        ev.append(TimelineEvent(len(ev), kind, layer, step, label, dur, [d for d in deps if d is not None],
                                writes_slot=writes, reads_slot=reads))
        return len(ev) - 1

    def input_of(t, l):  # the event publishing layer l's input hidden state
        if l >= 1:
            return main.get((t, l - 1))
        return main.get((t - 1, L - 1)) if t >= 1 else None

    for t in range(len(prefetch_bytes)):
        est: dict[int, int] = {}

        def estimate(l):
            if l < L and _sparse(labels[l]):
                est[l] = new(EventKind.COMPUTE, l, t, "estimate", costs.estimate, [input_of(t, max(l - 1, 0))])

        estimate(0)
        estimate(1)
        for l in range(L):
            if _sparse(labels[l]):
                slot = (l, t % 2)
                pre = new(EventKind.TRANSFER, l, t, "prefetch", link.transfer_seconds(int(prefetch_bytes[t][l])),
                          [est[l], scores.get((t - 2, l))], writes=slot)
                sc = new(EventKind.COMPUTE, l, t, "score", costs.score, [pre, input_of(t, l)], reads=slot)
                scores[(t, l)] = sc
                fe = new(EventKind.TRANSFER, l, t, "topk_fetch", link.transfer_seconds(int(fetch_bytes[t][l])), [sc])
                main[(t, l)] = new(EventKind.COMPUTE, l, t, "compute", costs.compute[l], [fe, input_of(t, l)])
            else:
                main[(t, l)] = new(EventKind.COMPUTE, l, t, "compute", costs.compute[l], [input_of(t, l)])
            estimate(l + 2)
    return ev


def _merged(spans):
    out = []
    for lo, hi in sorted(spans):
        if out and lo <= out[-1][1]:
            out[-1][1] = max(out[-1][1], hi)
        else:
            out.append([lo, hi])
    return out


def simulate(events: list[TimelineEvent]) -> SimulationResult:
    """Earliest-start list scheduling, one exclusive compute engine and one
    exclusive link, ready events admitted in (ready time, id) order
    (memsim.py:510-602); checks dependencies and the double-buffer exclusion."""
    by_id = {e.id: e for e in events}
    kids: dict[int, list[int]] = {e.id: [] for e in events}
    pending = {}
    for e in events:
        pending[e.id] = len(e.depends_on)
        for d in e.depends_on:
            if d not in kids:
                raise SchedulingError(f"event {e.id} depends on unknown event {d}")
            kids[d].append(e.id)
    ready = {e.id: 0.0 for e in events}
    heap = [(0.0, e.id) for e in events if not e.depends_on]
    heapq.heapify(heap)
    free = {EventKind.COMPUTE: 0.0, EventKind.TRANSFER: 0.0}
    done = 0
    while heap:
        r, i = heapq.heappop(heap)
        e = by_id[i]
        e.start = max(r, free[e.kind])
        free[e.kind] = e.end
        done += 1
        for k in kids[i]:
            ready[k] = max(ready[k], e.end)
            pending[k] -= 1
            if pending[k] == 0:
                heapq.heappush(heap, (ready[k], k))
    if done != len(events):
        raise SchedulingError("cyclic dependency in timeline")
    for e in events:
        if any(e.start < by_id[d].end - 1e-12 for d in e.depends_on):
            raise SchedulingError("dependency violated by scheduler")
    for w in events:
        if w.writes_slot is None or w.duration <= 0:
            continue
        for r in events:
            if r.reads_slot == w.writes_slot and r.duration > 0 and w.start < r.end and r.start < w.end:
                raise SchedulingError(f"slot {w.writes_slot} written by event {w.id} while read by event {r.id}")
    per_layer: dict[int, dict[str, float]] = {}
    for e in events:
        b = per_layer.setdefault(e.layer, {"compute": 0.0, "transfer": 0.0})
        b["compute" if e.kind is EventKind.COMPUTE else "transfer"] += e.duration
    comp = _merged([(e.start, e.end) for e in events if e.kind is EventKind.COMPUTE and e.duration > 0])
    xfer = _merged([(e.start, e.end) for e in events if e.kind is EventKind.TRANSFER and e.duration > 0])
    overlap, i, j = 0.0, 0, 0
    while i < len(comp) and j < len(xfer):
        overlap += max(0.0, min(comp[i][1], xfer[j][1]) - max(comp[i][0], xfer[j][0]))
        if comp[i][1] <= xfer[j][1]:
            i += 1
        else:
            j += 1
    xfer_total = sum(hi - lo for lo, hi in xfer)
    stall = 0.0
    for e in events:
        if e.label == "score":
            pre = max((by_id[d].end for d in e.depends_on if by_id[d].label == "prefetch"), default=0.0)
            other = max((by_id[d].end for d in e.depends_on if by_id[d].label != "prefetch"), default=0.0)
            stall += max(0.0, pre - other)
    return SimulationResult(events, max((e.end for e in events), default=0.0), per_layer,
                            overlap / xfer_total if xfer_total > 0 else 0.0, stall)


def measured_step(labels: Sequence[str], quant_s: float, sparse_s: float, stage1_s: float, fetch_bytes: int,
                  h2d_bandwidth: float, steps: int = 4, prefetch_bytes: int = 0) -> dict:
    """The reference's model driven by this engine's measured costs.

    ``quant_s``: one quantized layer's decode; ``sparse_s``: one fused sparse
    launch (score + select + gather + attention, modelled as the layer's
    compute -- the fused kernel has no separate score event); ``stage1_s``:
    the estimate pass; ``fetch_bytes``: PCIe bytes per sparse layer (value
    rows that missed the HBM row cache); ``prefetch_bytes``: critical-key
    bytes per sparse layer (0 here: the keys are resident in HBM; the
    reference design moves n*h*d_s*2).  Returns the simulated per-step time
    and the overlap / stall statistics of the steady-state steps."""
    L = len(labels)
    costs = LayerCosts(tuple(sparse_s if _sparse(x) else quant_s for x in labels), estimate=stage1_s, score=0.0)
    link = LinkModel(h2d_bandwidth)
    pb = [[prefetch_bytes if _sparse(x) else 0 for x in labels] for _ in range(steps)]
    fb = [[fetch_bytes if _sparse(x) else 0 for x in labels] for _ in range(steps)]
    res = simulate(build_timeline(labels, costs, link, pb, fb))
    ends = [max(e.end for e in res.events if e.step == t) for t in range(steps)]
    per_step = (ends[-1] - ends[0]) / (steps - 1) if steps > 1 else ends[0]
    return {"step_seconds": per_step, "total_seconds": res.total_seconds,
            "overlap_fraction": res.overlap_fraction, "stall_seconds": res.stall_seconds, "layers": L}
