"""Pipeline configuration, mirroring the reference's AttentionConfig / RangeConfig.

Same field names, defaults and error behaviour as lpattn
(attention.py:58-95, quantization.py:24-68), so code written against the
reference constructs these unchanged.  Validation here is host logic only;
the C ABI re-checks the same rules (sa2pp_check_problem).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Optional

FP16_MAX = 65504.0
MMA_K_GROUP = 32
RANGE_PRODUCT_LIMIT = FP16_MAX / MMA_K_GROUP  # 2047.0 (quantization.py:26)
#: Table 2 range pairs of the paper, all safe at buffering depth 2.
TABLE2_PAIRS = ((448.0, 2.25), (224.0, 4.5), (112.0, 9.0))


class RangeConfigError(ValueError):
    """The requested quantization ranges can overflow the FP16 accumulator."""


@dataclass(frozen=True)
class RangeConfig:
    """Target magnitudes p_r (exponentiated scores) and v_r (values)."""

    p_r: float
    v_r: float
    buffering_depth: int = 2
    expect_overflow: bool = False

    def __post_init__(self):
        if self.p_r <= 0 or self.v_r <= 0:
            raise RangeConfigError("p_r and v_r must be positive")
        if self.buffering_depth not in (1, 2):
            raise RangeConfigError(f"buffering_depth must be 1 or 2, got {self.buffering_depth}")
        if not self.expect_overflow and self.product > self.bound:
            raise RangeConfigError(
                f"p_r*v_r = {self.product:g} > {self.bound:g} "
                f"(FP16 accumulator bound at buffering depth {self.buffering_depth})")

    @property
    def product(self) -> float:
        return self.p_r * self.v_r

    @property
    def bound(self) -> float:
        return RANGE_PRODUCT_LIMIT / self.buffering_depth


@dataclass(frozen=True)
class AttentionConfig:
    """Problem shape plus every knob of the quantized pipeline (attention.py:58-95)."""

    seq_len: int
    head_dim: int
    num_heads: int = 1
    block_q: int = 128
    block_k: int = 64
    qk_bits: int = 8
    range: RangeConfig = field(default_factory=lambda: RangeConfig(224.0, 4.5, 2))
    causal: bool = False
    smoothing: bool = True
    softmax_scale: Optional[float] = None
    pv_accumulator: str = "fp16"

    def __post_init__(self):
        if min(self.seq_len, self.head_dim, self.num_heads) < 1:
            raise ValueError("seq_len, head_dim and num_heads must be positive")
        if min(self.block_q, self.block_k) < 1:
            raise ValueError("tile sizes must be positive")
        if self.qk_bits not in (4, 8):
            raise ValueError("qk_bits must be 4 or 8")
        if self.pv_accumulator not in ("fp16", "fp32"):
            raise ValueError("pv_accumulator must be 'fp16' or 'fp32'")

    @property
    def scale(self) -> float:
        if self.softmax_scale is not None:
            return self.softmax_scale
        return 1.0 / math.sqrt(self.head_dim)

    def with_range(self, range_config: RangeConfig) -> "AttentionConfig":
        return replace(self, range=range_config)
