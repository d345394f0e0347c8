"""Position-keyed dropout: the reference's counter-based masks.

nnops.py:30-166: every keep decision is a pure function of (seed, layer, site,
sample, [head,] global position, column) through a splitmix64-style mix, so a
mask is the same whichever rank computes it and is recomputed (never stored)
in the backward.  The host derives the per-site keys; the kernels derive row
keys and words (``drop_mix`` in csrc/common.cuh) and compare integer bits with
``thresh = ceil(rate * 2**53)``, which is exactly nnops.keep_mask's
``(word >> 11) * 2**-53 >= rate``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

from ._native import DropoutDesc

DROPOUT_TAGS = {"embed": 1, "attn_score": 2, "attn_out": 3, "ffn_hidden": 4, "ffn_out": 5}  # nnops.py:32-38

_M64 = (1 << 64) - 1
_GOLDEN, _MIX_A, _MIX_B = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def mix_key(h: int, word: int) -> int:
    """nnops.mix_key: fold ``word`` into the 64-bit hash state ``h``."""
    z = (h + word * _GOLDEN) & _M64
    z = ((z ^ (z >> 30)) * _MIX_A) & _M64
    z = ((z ^ (z >> 27)) * _MIX_B) & _M64
    return z ^ (z >> 31)


@dataclass(frozen=True)
class DropoutPolicy:
    """nnops.DropoutPolicy (nnops.py:67-104): the seed is the only state."""

    rate: float
    seed: int = 0
    enabled: bool = True

    def __post_init__(self) -> None:
        if not 0.0 <= self.rate < 1.0:
            raise ValueError(f"dropout rate must be in [0, 1), got {self.rate}")

    @classmethod
    def off(cls) -> "DropoutPolicy":
        return cls(rate=0.0, enabled=False)

    def at_step(self, step: int) -> "DropoutPolicy":
        return replace(self, seed=mix_key(self.seed & _M64, step + 1))

    def fork(self, lane: int) -> "DropoutPolicy":
        return replace(self, seed=mix_key(mix_key(self.seed & _M64, 0x666F726B), lane + 1))

    @property
    def active(self) -> bool:
        return self.enabled and self.rate > 0.0

    # ---- device descriptors
    def site_key(self, layer: int, tag: str) -> int:
        """nnops._site_key (nnops.py:107-112)."""
        try:
            tag_id = DROPOUT_TAGS[tag]
        except KeyError:
            raise ValueError(f"unknown dropout tag {tag!r}") from None
        return mix_key(mix_key(self.seed & _M64, tag_id), layer + 1)

    @property
    def thresh(self) -> int:
        return math.ceil(self.rate * 2.0 ** 53)

    @property
    def scale(self) -> float:
        return 1.0 / (1.0 - self.rate)

    def desc(self, layer: int, tag: str = "attn_score") -> DropoutDesc:
        """lss_dropout descriptor of one site (inactive when the policy is off)."""
        d = DropoutDesc()
        if self.active:
            d.site_key, d.thresh, d.scale, d.active = self.site_key(layer, tag), self.thresh, self.scale, 1
        return d


def as_policy(policy) -> DropoutPolicy:
    """Accept None, our policy, or any object with rate / seed / enabled (e.g. the
    reference's nnops.DropoutPolicy)."""
    if policy is None:
        return DropoutPolicy.off()
    if isinstance(policy, DropoutPolicy):
        return policy
    return DropoutPolicy(getattr(policy, "rate", 0.0), getattr(policy, "seed", 0), getattr(policy, "enabled", True))
