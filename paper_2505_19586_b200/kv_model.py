"""Model dimensions (hybridkv/kv_model.py:22-73), host-side only."""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError


@dataclass(frozen=True)
class ModelConfig:
    """Attention dimensions; same fields and checks as the reference."""

    num_layers: int
    num_query_heads: int
    num_kv_heads: int
    head_dim: int
    hidden_dim: int
    element_bytes: int = 2

    def __post_init__(self) -> None:
        if self.num_layers < 1:
            raise ConfigError(f"num_layers must be >= 1, got {self.num_layers}")
        if self.head_dim < 1:
            raise ConfigError(f"head_dim must be >= 1, got {self.head_dim}")
        if self.num_kv_heads < 1 or self.num_query_heads < 1:
            raise ConfigError("head counts must be >= 1")
        if self.num_query_heads % self.num_kv_heads:
            raise ConfigError(f"num_query_heads ({self.num_query_heads}) must be divisible by "
                              f"num_kv_heads ({self.num_kv_heads})")
        if self.hidden_dim != self.num_query_heads * self.head_dim:
            raise ConfigError(f"hidden_dim ({self.hidden_dim}) must equal num_query_heads * head_dim")
        if self.element_bytes != 2:
            raise ConfigError("storage is 16-bit float semantics; element_bytes must be 2")

    @property
    def queries_per_kv_head(self) -> int:
        return self.num_query_heads // self.num_kv_heads

    def kv_head_for(self, query_head: int) -> int:
        """KV head read by a query head (kv_model.py:71-73)."""
        return query_head // self.queries_per_kv_head


# Shapes named by BASELINE.json configs
LLAMA31_8B = ModelConfig(num_layers=32, num_query_heads=32, num_kv_heads=8, head_dim=128, hidden_dim=4096)
QWEN25_7B = ModelConfig(num_layers=28, num_query_heads=28, num_kv_heads=4, head_dim=128, hidden_dim=3584)
LLAMA31_70B = ModelConfig(num_layers=80, num_query_heads=64, num_kv_heads=8, head_dim=128, hidden_dim=8192)
