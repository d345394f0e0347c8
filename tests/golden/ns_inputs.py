"""Seeded inputs of the north-star-shape golden cases (E=1024, 16 heads).

Shared by ``make_golden.py`` (which feeds them to the REAL reference in the dev
container) and the tests (which rebuild them on the GPU box, where the
reference is absent), so the fixtures only have to store outputs.  numpy's
PCG64 ``default_rng`` streams (standard_normal / uniform) are stable across
numpy versions >= 1.17; every array is rounded to float32, the precision the
B200 path takes its fp32 inputs in.
"""

from __future__ import annotations

import math

import numpy as np

ATTN_NAMES = ("ln1_gain", "ln1_bias", "wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo")


def ns_inputs(seq: int, embed: int, batch: int = 1, seed: int = 0):
    """(x, grad_y, params) for one attention sublayer: U(+-1/sqrt(E)) weights as
    model.init_params (model.py:179-224), plus non-trivial LN affine and biases
    so that every gradient is exercised."""
    rng = np.random.default_rng(seed)
    bound = 1.0 / math.sqrt(embed)
    f32 = lambda a: np.asarray(a, np.float32)  # noqa: E731
    p = {}
    for n in ("wq", "wk", "wv", "wo"):
        p[n] = f32(rng.uniform(-bound, bound, (embed, embed)))
    for n in ("bq", "bk", "bv", "bo"):
        p[n] = f32(0.05 * rng.standard_normal(embed))
    p["ln1_gain"] = f32(1.0 + 0.1 * rng.standard_normal(embed))
    p["ln1_bias"] = f32(0.1 * rng.standard_normal(embed))
    x = f32(rng.standard_normal((batch, seq, embed)))
    gy = f32(rng.standard_normal((batch, seq, embed)))
    return x, gy, p


# stored row / weight-row subsets of the NS fixtures (the full tensors are
# 8-16 MB each; the row sums below cover every element)
ROW_STRIDE = 16
WROW_STRIDE = 32
