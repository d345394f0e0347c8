"""Per-step analytic counters (reference tensor.py:35-58), same formulas, so the
B200 path reports the attention-score FLOPs and score footprint the
reference's cost model (costs.py:98) and tests compare against."""

from __future__ import annotations

from dataclasses import dataclass


@dataclass
class StepCounters:
    matmul_flops: int = 0
    attn_score_flops: int = 0
    attn_score_elements_peak: int = 0

    def add_matmul(self, m: int, k: int, n: int) -> None:
        self.matmul_flops += 2 * m * k * n

    def add_score_flops(self, m: int, k: int, n: int) -> None:
        self.attn_score_flops += 2 * m * k * n

    def record_score_footprint(self, elements: int) -> None:
        if elements > self.attn_score_elements_peak:
            self.attn_score_elements_peak = elements
