"""B200-native SageAttention2++ (arXiv 2505.21136): sm_100a INT8 QK^T + FP8 PV attention.

Public API:
    sageattn(q, k, v, tensor_layout="HND", is_causal=False, sm_scale=None)   north-star drop-in
    torch.ops.sa2pp.sageattn(q, k, v, tensor_layout, is_causal, sm_scale)    the same as a custom op
    attention_quantized(q, k, v, AttentionConfig) -> RunReport               lpattn operator mirror
    quantize(q, k, v)                                                        prepass only
    AttentionConfig, RangeConfig, RangeConfigError                           lpattn config mirror
"""

from .config import TABLE2_PAIRS, AttentionConfig, RangeConfig, RangeConfigError
from .api import (HostPipeline, QuantizedTensors, RunReport, attention_quantized, compare, new_report,
                  quantize, read_report, sageattn, sageattn_host)
from .ops import sageattn_op  # registers torch.ops.sa2pp.sageattn

__version__ = "1.0.0"
__all__ = [
    "sageattn", "sageattn_op", "read_report", "sageattn_host", "HostPipeline", "attention_quantized", "quantize", "compare", "new_report",
    "AttentionConfig", "RangeConfig", "RangeConfigError", "TABLE2_PAIRS",
    "QuantizedTensors", "RunReport",
]
