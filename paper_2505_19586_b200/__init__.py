"""B200-native TailorKV decode engine (arXiv 2505.19586).

A drop-in for the decode hot path of the reference package ``hybridkv``
(/root/reference/pkg/src/hybridkv): layer classification, the
prefill/compress call and the per-layer decode-attention call, executed by
hand-written sm_100a CUDA kernels behind a C ABI (include/tailorkv.h).
There is no CPU fallback.
"""

from .errors import (
    ConfigError,
    EmptyCacheError,
    EncodingError,
    NumericError,
    ParameterError,
    SchedulingError,
    ShapeError,
    TraceFormatError,
)
from .kv_model import ModelConfig
from .identifier import LayerKind, SparsityProbe, calibrate, classify_layer, default_probe_k, dense_preference_score
from .quantizer import QuantizedLayerKV, qgemv_output, qgemv_scores, quantize_layer_kv
from .retriever import RetrievalConfig, select_topk_tokens, stage1_select
from .hoststore import OffloadedLayerKV
from .engine import DecodeEngine, EngineConfig, assemble, shard_plan
from .fidelity import sparse_layer_fidelity
from .trace import DeviceTrace, load_trace

__version__ = "0.1.0"

__all__ = [
    "ConfigError", "EmptyCacheError", "EncodingError", "NumericError", "ParameterError", "SchedulingError",
    "ShapeError", "TraceFormatError", "ModelConfig", "LayerKind", "SparsityProbe", "calibrate", "classify_layer",
    "default_probe_k", "dense_preference_score", "QuantizedLayerKV", "qgemv_output", "qgemv_scores",
    "quantize_layer_kv", "RetrievalConfig", "select_topk_tokens", "stage1_select", "OffloadedLayerKV",
    "DecodeEngine", "EngineConfig", "assemble", "shard_plan", "sparse_layer_fidelity", "DeviceTrace", "load_trace",
    "__version__",
]
