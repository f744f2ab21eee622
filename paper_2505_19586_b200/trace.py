"""HKVTRACE reader that feeds the engine.

Parses the reference's trace container (hybridkv/trace.py:105-228: magic,
little-endian (version, header length), a JSON header with the model, labels,
section list and payload SHA-256, then the fp16 payload) and hands the
sections to the GPU without any float64 round trip: the payload is staged in
pinned memory and copied to the device in one H2D transfer, and every section
is a view of that buffer.  Error behaviour follows trace.py:151-228
(TraceFormatError on bad magic, version, header, digest or section sizes).
"""

from __future__ import annotations

import hashlib
import json
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .errors import TraceFormatError

_MAGIC = b"HKVTRACE"
_VERSION = 1


@dataclass
class DeviceTrace:
    """A decode trace as fp16 tensors (on the device unless loaded on the CPU)."""

    header: dict
    labels: list            # per layer: "quantization_friendly" / "sparsity_friendly" (empty if unlabelled)
    prefill_keys: list      # per layer [h, n, d]
    prefill_values: list
    prefill_queries: list   # per layer [hq, n_q, d] (the calibration probe's queries)
    w_q: list               # per layer [hq, hidden, d]
    hidden: torch.Tensor    # [T, L, hidden]
    queries: torch.Tensor   # [T, L, hq, d]
    new_keys: torch.Tensor  # [T, L, h, d]
    new_values: torch.Tensor

    @property
    def num_steps(self) -> int:
        return self.hidden.shape[0]

    def step_inputs(self, t: int):
        """Inputs of step t in DecodeEngine.step's layout (batch of one)."""
        return (self.hidden[t][:, None], self.queries[t][:, None], self.new_keys[t][:, None],
                self.new_values[t][:, None])


def _header(blob: bytes) -> tuple[dict, bytes]:
    prefix = len(_MAGIC) + 8
    if len(blob) < prefix or blob[:len(_MAGIC)] != _MAGIC:
        raise TraceFormatError("not a trace file (bad magic)")
    version, hlen = struct.unpack("<II", blob[len(_MAGIC):prefix])
    if version != _VERSION:
        raise TraceFormatError(f"unsupported trace format version {version}")
    if len(blob) < prefix + hlen:
        raise TraceFormatError("trace header truncated")
    try:
        header = json.loads(blob[prefix:prefix + hlen].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise TraceFormatError(f"trace header is not valid JSON: {exc}") from exc
    return header, blob[prefix + hlen:]


def load_trace(path, device=None) -> DeviceTrace:
    """Read an HKVTRACE file; ``device`` None keeps the tensors on the CPU."""
    blob = Path(path).read_bytes()
    header, payload = _header(blob)
    if hashlib.sha256(payload).hexdigest() != header.get("payload_sha256"):
        raise TraceFormatError("trace payload digest mismatch")
    sections = header["sections"]
    total = sum(2 * int(np.prod(s["shape"])) for s in sections)
    if total != len(payload):
        raise TraceFormatError(f"payload holds {len(payload)} bytes, sections describe {total}")
    host = torch.frombuffer(bytearray(payload), dtype=torch.float16)
    if device is not None:
        dev = torch.device(device)
        buf = torch.empty(host.numel(), dtype=torch.float16, device=dev)
        buf.copy_(host.pin_memory(), non_blocking=True)
    else:
        buf = host
    arrs, off = {}, 0
    for s in sections:
        cnt = int(np.prod(s["shape"]))
        arrs[s["name"]] = buf[off:off + cnt].view(*s["shape"])
        off += cnt
    m = header["model"]
    L, T = m["num_layers"], header["num_steps"]

    def stack(sec):
        return torch.stack([torch.stack([arrs[f"step{t}/layer{l}/{sec}"] for l in range(L)]) for t in range(T)])

    return DeviceTrace(
        header=header, labels=list(header.get("labels") or []),
        prefill_keys=[arrs[f"layer{l}/prefill_keys"] for l in range(L)],
        prefill_values=[arrs[f"layer{l}/prefill_values"] for l in range(L)],
        prefill_queries=[arrs[f"layer{l}/prefill_queries"] for l in range(L)],
        w_q=[arrs[f"layer{l}/w_q"] for l in range(L)],
        hidden=stack("hidden"), queries=stack("query"), new_keys=stack("new_key"), new_values=stack("new_value"),
    )
