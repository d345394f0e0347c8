"""CPU oracle for the LSS sequence-distributed attention sublayer.

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``paper_2311_02382_b200``)
imports this module; only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may use it, and
only as the checker / the reference CPU arm, never as the thing measured.

This is a numpy restatement of the reference's algorithm for the hot path
(``/root/reference/pkg/src/seqpar``), written independently from the
definitions, vectorised over (batch, head) instead of the reference's Python
loops.  Every function cites the reference lines it follows.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference
(``seqpar`` imported from ``/root/reference``) on seeded inputs and commits the
outputs under ``tests/golden/``; ``tests/test_oracle.py`` checks this oracle
against those fixtures and against the reference's own known-answer tests
(``tests/test_model.py:17-163`` in the reference).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

LAYERNORM_EPS = 1e-5  # nnops.py:28


class OracleShapeError(ValueError):
    pass


class OracleDegenerateRow(ValueError):
    pass


# --------------------------------------------------------------------------
# L1 primitives (nnops.py)
# --------------------------------------------------------------------------


def layernorm_fwd(x, gain, bias, eps=LAYERNORM_EPS):
    """nnops.py:199-208: y = (x-mu)*inv_std*g + b; cache (xhat, inv_std)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    inv_std = 1.0 / np.sqrt(var + eps)
    xhat = (x - mu) * inv_std
    return xhat * gain + bias, (xhat, inv_std)


def layernorm_bwd(cache, gain, gy):
    """nnops.py:211-227: gx = inv_std*(g - mean(g) - xhat*mean(g*xhat)), g = gy*gain."""
    xhat, inv_std = cache
    red = tuple(range(gy.ndim - 1))
    g_gain = (gy * xhat).sum(axis=red)
    g_bias = gy.sum(axis=red)
    g = gy * gain
    gx = inv_std * (g - g.mean(-1, keepdims=True) - xhat * (g * xhat).mean(-1, keepdims=True))
    return gx, g_gain, g_bias


def linear_fwd(x, w, b):
    """nnops.py:180-183 via model.linear3 (model.py:237-239): y = x @ W + b, W is [in, out]."""
    return x @ w + b


def linear_bwd(x, w, gy):
    """nnops.py:186-193 via model.linear3_bwd (model.py:242-245)."""
    e_in = x.shape[-1]
    x2 = x.reshape(-1, e_in)
    g2 = gy.reshape(-1, gy.shape[-1])
    gx = gy @ w.T
    return gx, x2.T @ g2, g2.sum(axis=0)


# --------------------------------------------------------------------------
# Attention core (model.py:280-359, tensor.py:104-131)
# --------------------------------------------------------------------------


def _split_heads(a, n_heads):
    # (B, rows, E) -> (B, H, rows, d); head h <-> columns [h*d, (h+1)*d) (model.py:309)
    b, r, e = a.shape
    d = e // n_heads
    return a.reshape(b, r, n_heads, d).transpose(0, 2, 1, 3)


def _merge_heads(a):
    b, h, r, d = a.shape
    return a.transpose(0, 2, 1, 3).reshape(b, r, h * d)


def causal_keep(m, t, offset):
    """model.py:301-304: keep[i, j] = j <= offset + i (global query position)."""
    q_pos = np.arange(offset, offset + m)
    return np.arange(t)[None, :] <= q_pos[:, None]


def scores_fwd(q, k, v, offset, n_heads, causal=True):
    """model.py:280-326.  q (B,m,E) local rows at global positions offset..offset+m,
    k/v (B,t,E) whole sequence.  Returns (ctx, P) with P (B,H,m,t) the softmax
    probabilities (the reference's cached ``aw``).  Masked entries are exact
    zeros and a fully-masked row raises (tensor.py:123-130)."""
    bsz, m, e = q.shape
    t = k.shape[1]
    d = e // n_heads
    scale = 1.0 / math.sqrt(d)
    qh, kh, vh = (_split_heads(a, n_heads) for a in (q, k, v))
    s = (qh @ kh.transpose(0, 1, 3, 2)) * scale  # BLAS, as tensor.matmul (tensor.py:91)
    if causal:
        keep = causal_keep(m, t, offset)
        if np.any(keep.sum(axis=1) == 0):
            raise OracleDegenerateRow("softmax row fully masked")
        s = np.where(keep, s, -np.inf)
    s = s - s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p = p / p.sum(axis=-1, keepdims=True)
    ctx = _merge_heads(p @ vh)
    return ctx, p


def scores_bwd(p, q, k, v, grad_ctx, n_heads):
    """model.py:329-359: dP = dO V^T; dV = P^T dO; dS = P*(dP - rowsum(dP*P))*scale;
    dQ = dS K; dK = dS^T Q.  dK/dV span the full key length t (partials of this
    block's query rows)."""
    d = q.shape[2] // n_heads
    scale = 1.0 / math.sqrt(d)
    qh, kh, vh, gh = (_split_heads(a, n_heads) for a in (q, k, v, grad_ctx))
    dp = gh @ vh.transpose(0, 1, 3, 2)
    dv = p.transpose(0, 1, 3, 2) @ gh
    ds = p * (dp - (dp * p).sum(axis=-1, keepdims=True)) * scale
    dq = ds @ kh
    dk = ds.transpose(0, 1, 3, 2) @ qh
    return _merge_heads(dq), _merge_heads(dk), _merge_heads(dv)


def attention_from_definition(q, k, v, offset, n_heads, causal=True):
    """Scalar-loop oracle of the reference's own test (tests/test_model.py:17-37)."""
    bsz, m, e = q.shape
    t = k.shape[1]
    d = e // n_heads
    out = np.zeros_like(q, dtype=np.float64)
    for b in range(bsz):
        for h in range(n_heads):
            lo, hi = h * d, (h + 1) * d
            for i in range(m):
                limit = offset + i + 1 if causal else t
                sc = np.array([float(np.dot(q[b, i, lo:hi], k[b, j, lo:hi])) / math.sqrt(d)
                               for j in range(limit)])
                w = np.exp(sc - sc.max())
                w = w / w.sum()
                out[b, i, lo:hi] = w @ v[b, :limit, lo:hi]
    return out


# --------------------------------------------------------------------------
# Attention half of one LSS layer (model.py:442-448 fwd, 479-486 bwd) with the
# packed-K/V kv_fwd/kv_bwd of sharded.py:144-154 / 192-202.
# --------------------------------------------------------------------------


@dataclass
class AttnParams:
    """The attention-half parameters of model.LayerParams (model.py:83-94)."""
    ln1_gain: np.ndarray
    ln1_bias: np.ndarray
    wq: np.ndarray
    bq: np.ndarray
    wk: np.ndarray
    bk: np.ndarray
    wv: np.ndarray
    bv: np.ndarray
    wo: np.ndarray
    bo: np.ndarray

    GRAD_ORDER = ("ln1_gain", "ln1_bias", "wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo")

    def astype(self, dt):
        return AttnParams(*[getattr(self, n).astype(dt) for n in self.GRAD_ORDER])


def init_attn_params(embed_dim, seed=0, dtype=np.float64):
    """Same draw convention as model.init_params (model.py:179-224) restricted to
    layer 0's attention half: U(+-1/sqrt(E)) weights in draw order q, k, v, out
    AFTER the token and position tables.  Because the tables are drawn first the
    exact stream only matches init_params when vocab/seq_len match, so the
    golden fixtures store the weights they used."""
    rng = np.random.default_rng(seed)
    bound = 1.0 / math.sqrt(embed_dim)
    e = embed_dim

    def u():
        return rng.uniform(-bound, bound, (e, e)).astype(dtype)

    wq, wk, wv, wo = u(), u(), u(), u()
    z = np.zeros(e, dtype=dtype)
    return AttnParams(np.ones(e, dtype=dtype), z.copy(), wq, z.copy(), wk, z.copy(),
                      wv, z.copy(), wo, z.copy())


def attn_rank_fwd(x_seg, p: AttnParams, offset, kv_full, n_heads, causal=True):
    """model.layer_fwd lines 442-448 for one rank: LN1 -> Q -> scores -> out -> residual.
    ``kv_full`` = (k, v) for the whole sequence (the all-gather result)."""
    xh, ln_cache = layernorm_fwd(x_seg, p.ln1_gain, p.ln1_bias)
    q = linear_fwd(xh, p.wq, p.bq)
    k, v = kv_full
    ctx, prob = scores_fwd(q, k, v, offset, n_heads, causal)
    y = x_seg + linear_fwd(ctx, p.wo, p.bo)
    return y, dict(xh=xh, ln=ln_cache, q=q, ctx=ctx, p=prob)


def lss_attention(x, grad_y, p: AttnParams, n_heads, workers, causal=True):
    """Run the attention half of one LSS layer on ``workers`` simulated ranks,
    forward and backward, with the packed-K/V exchange: each rank projects its
    own [K_r|V_r] and all-gathers them in rank order (sharded.py:144-154); the
    backward reduce-scatters [dK|dV] (sharded.py:192-202) and the replicated
    parameter gradients are averaged over the group (sharded.py:219-244).

    x, grad_y: (B, l, E).  Returns dict with y (B,l,E) (rank rows concatenated),
    dx (B,l,E), and the averaged parameter gradients (AttnParams)."""
    bsz, seq, e = x.shape
    if seq % workers:
        raise OracleShapeError(f"sequence length {seq} not divisible by {workers}")  # sharded.py:50-53
    m = seq // workers
    segs = [slice(r * m, (r + 1) * m) for r in range(workers)]  # ShardSpec.offset = rank*block
    # forward: each rank LN1 + own K/V projection, then the rank-ordered gather
    xh = [layernorm_fwd(x[:, s], p.ln1_gain, p.ln1_bias) for s in segs]
    k_parts = [linear_fwd(xh[r][0], p.wk, p.bk) for r in range(workers)]
    v_parts = [linear_fwd(xh[r][0], p.wv, p.bv) for r in range(workers)]
    k_full = np.concatenate(k_parts, axis=1)  # collectives.py:340 (rank order, dim=1)
    v_full = np.concatenate(v_parts, axis=1)
    ys, caches = [], []
    for r, s in enumerate(segs):
        y, c = attn_rank_fwd(x[:, s], p, r * m, (k_full, v_full), n_heads, causal)
        ys.append(y)
        caches.append(c)
    # backward (model.py:479-486 with the unfused kv_bwd of sharded.py:193-202)
    dk_full = np.zeros_like(k_full)
    dv_full = np.zeros_like(v_full)
    per_rank = []
    for r, s in enumerate(segs):
        c = caches[r]
        gy = grad_y[:, s]
        g_ctx, g_wo, g_bo = linear_bwd(c["ctx"], p.wo, gy)
        dq, dk, dv = scores_bwd(c["p"], c["q"], k_full, v_full, g_ctx, n_heads)
        dk_full = dk_full + dk  # reduce_scatter sums contributions (collectives.py:365-367)
        dv_full = dv_full + dv
        per_rank.append((gy, dq, g_wo, g_bo))
    grads_sum = None
    dxs = []
    for r, s in enumerate(segs):
        c = caches[r]
        gy, dq, g_wo, g_bo = per_rank[r]
        gk, gv = dk_full[:, s], dv_full[:, s]  # block r of the sum (collectives.py:368-370)
        gxq, g_wq, g_bq = linear_bwd(c["xh"], p.wq, dq)
        gxk, g_wk, g_bk = linear_bwd(c["xh"], p.wk, gk)
        gxv, g_wv, g_bv = linear_bwd(c["xh"], p.wv, gv)
        gx_ln, g_g, g_b = layernorm_bwd(c["ln"], p.ln1_gain, gxq + gxk + gxv)
        dxs.append(gy + gx_ln)  # grad_in = grad_mid + g_ln1 (model.py:486)
        g = [g_g, g_b, g_wq, g_bq, g_wk, g_bk, g_wv, g_bv, g_wo, g_bo]
        grads_sum = g if grads_sum is None else [a + b for a, b in zip(grads_sum, g)]
    grads = AttnParams(*[a / workers for a in grads_sum])  # all_reduce mean (sharded.py:238)
    return dict(y=np.concatenate(ys, axis=1), dx=np.concatenate(dxs, axis=1), grads=grads,
                k_full=k_full, v_full=v_full)


# --------------------------------------------------------------------------
# Blocked evaluation for the north-star shapes (E=1024, 16 heads, l up to 50112;
# SURVEY §8(c) "row-subset parity").  The reference materialises P per (b, h)
# (model.py:307-325): 16 x 8192^2 fp64 = 8.6 GB at l=8192, 40 GB per rank at
# l=50112.  The functions below evaluate exactly the same formulas one (sample,
# head) and one block of query rows at a time, so only a block of P is ever alive.
# Row-wise softmax makes row blocks independent; dK/dV are sums over query rows
# (model.py:352, 358), accumulated block by block.
# --------------------------------------------------------------------------


def _head_task(qh, kh, vh, gh, q_pos, causal, scale, chunk, key_range, dt):
    """One (sample, head): rows of qh at global positions q_pos against all keys."""
    rows, t = qh.shape[0], kh.shape[0]
    k0, k1 = key_range
    ctx = np.empty((rows, vh.shape[1]), dt)
    lse2 = np.empty(rows, np.float64)
    dq = np.empty_like(ctx) if gh is not None else None
    dk = np.zeros((k1 - k0, kh.shape[1]), dt) if gh is not None else None
    dv = np.zeros((k1 - k0, vh.shape[1]), dt) if gh is not None else None
    for r0 in range(0, rows, chunk):
        r1 = min(rows, r0 + chunk)
        pos = q_pos[r0:r1]
        kend = int(min(t, pos.max() + 1)) if causal else t  # keys past the block's last row are all masked
        if causal and pos.min() < 0:
            raise OracleDegenerateRow("softmax row fully masked")  # tensor.py:123-126
        s = (qh[r0:r1] @ kh[:kend].T) * dt(scale)  # model.py:311
        if causal:
            s = np.where(np.arange(kend)[None, :] <= pos[:, None], s, -np.inf)  # model.py:301-304
        mx = s.max(axis=1, keepdims=True)  # tensor.py:115-117
        p = np.exp(s - mx)
        den = p.sum(axis=1, keepdims=True)
        p /= den
        lse2[r0:r1] = (mx[:, 0].astype(np.float64) + np.log(den[:, 0].astype(np.float64))) / math.log(2.0)
        ctx[r0:r1] = p @ vh[:kend]  # model.py:320
        if gh is None:
            continue
        g = gh[r0:r1]
        dp = g @ vh[:kend].T  # model.py:346
        ds = p * (dp - (dp * p).sum(axis=1, keepdims=True)) * dt(scale)  # model.py:353-356
        dq[r0:r1] = ds @ kh[:kend]  # model.py:357
        hi = min(k1, kend)
        if hi > k0:
            dk[:hi - k0] += ds[:, k0:hi].T @ qh[r0:r1]  # model.py:358
            dv[:hi - k0] += p[:, k0:hi].T @ g  # model.py:349-352 (dropout 0)
    return ctx, lse2, dq, dk, dv


def attention_blocked(q, k, v, offset, n_heads, causal=True, grad_ctx=None, rows=None, key_range=None,
                      chunk=512, dtype=np.float32, threads=None):
    """scores_fwd + scores_bwd (model.py:280-359) block by block.

    q (B, m, E) at global positions offset..offset+m; k/v (B, t, E) the whole
    sequence; ``rows`` (optional index array) selects the query rows to evaluate;
    ``grad_ctx`` (B, len(rows), E) adds the backward.  dK/dV are returned for the
    key rows ``key_range`` = [k0, k1) only (default all) and contain the
    contributions of the selected rows only.  Returns dict(ctx, lse2 (B, H, rows)
    base-2 log-sum-exp, dq, dk, dv).  (Sample, head) pairs run on a thread pool
    (numpy releases the GIL inside BLAS and the ufuncs)."""
    from concurrent.futures import ThreadPoolExecutor

    bsz, m, e = q.shape
    t = k.shape[1]
    d = e // n_heads
    rows = np.arange(m) if rows is None else np.asarray(rows)
    key_range = (0, t) if key_range is None else key_range
    scale = 1.0 / math.sqrt(d)
    dt = np.dtype(dtype).type
    q_pos = offset + rows
    tasks = []
    for b in range(bsz):
        for h in range(n_heads):
            c = slice(h * d, (h + 1) * d)
            gh = None if grad_ctx is None else np.ascontiguousarray(grad_ctx[b, :, c], dtype)
            tasks.append((b, h, np.ascontiguousarray(q[b, rows, c], dtype), np.ascontiguousarray(k[b, :, c], dtype),
                          np.ascontiguousarray(v[b, :, c], dtype), gh))
    n_thr = threads or min(len(tasks), os.cpu_count() or 1)
    with ThreadPoolExecutor(n_thr) as ex:
        res = list(ex.map(lambda a: _head_task(a[2], a[3], a[4], a[5], q_pos, causal, scale, chunk, key_range, dt),
                          tasks))
    n_r, (k0, k1) = len(rows), key_range
    out = dict(ctx=np.empty((bsz, n_r, e), dtype), lse2=np.empty((bsz, n_heads, n_r)))
    if grad_ctx is not None:
        out.update(dq=np.empty((bsz, n_r, e), dtype), dk=np.empty((bsz, k1 - k0, e), dtype),
                   dv=np.empty((bsz, k1 - k0, e), dtype))
    for (b, h, *_), (ctx, lse2, dq, dk, dv) in zip(tasks, res):
        c = slice(h * d, (h + 1) * d)
        out["ctx"][b, :, c] = ctx
        out["lse2"][b, h] = lse2
        if grad_ctx is not None:
            out["dq"][b, :, c] = dq
            out["dk"][b, :, c] = dk
            out["dv"][b, :, c] = dv
    return out


def lss_attention_blocked(x, grad_y, p: AttnParams, n_heads, workers=1, causal=True, dtype=np.float32):
    """:func:`lss_attention` for shapes whose P does not fit in host memory.

    Identical arithmetic with the rank structure folded away: LN1 and the
    projections are row-local, the gathered K/V is the rank-ordered
    concatenation of every rank's own projection (= the projection of the whole
    sequence), each rank's dK/dV partials are summed by the reduce-scatter
    (= the dK/dV of all rows), and the sync averages the per-rank parameter
    gradients (= the gradient of all rows / workers).  Returns the same keys as
    :func:`lss_attention` plus the attention internals (q, k, v, ctx, lse2,
    g_ctx, dq, dk, dv) for kernel-level checks."""
    bsz, seq, e = x.shape
    if seq % workers:
        raise OracleShapeError(f"sequence length {seq} not divisible by {workers}")
    c = lambda a: a.astype(dtype)  # noqa: E731
    x, grad_y, p = c(x), c(grad_y), p.astype(dtype)
    xh, ln = layernorm_fwd(x, p.ln1_gain, p.ln1_bias)
    q, k, v = linear_fwd(xh, p.wq, p.bq), linear_fwd(xh, p.wk, p.bk), linear_fwd(xh, p.wv, p.bv)
    fwd = attention_blocked(q, k, v, 0, n_heads, causal, dtype=dtype)
    ctx = fwd["ctx"]
    y = x + linear_fwd(ctx, p.wo, p.bo)
    g_ctx, g_wo, g_bo = linear_bwd(ctx, p.wo, grad_y)
    bwd = attention_blocked(q, k, v, 0, n_heads, causal, grad_ctx=g_ctx, dtype=dtype)
    dq, dk, dv = bwd["dq"], bwd["dk"], bwd["dv"]
    gxq, g_wq, g_bq = linear_bwd(xh, p.wq, dq)
    gxk, g_wk, g_bk = linear_bwd(xh, p.wk, dk)
    gxv, g_wv, g_bv = linear_bwd(xh, p.wv, dv)
    gx_ln, g_g, g_b = layernorm_bwd(ln, p.ln1_gain, gxq + gxk + gxv)
    grads = AttnParams(*[a / workers for a in (g_g, g_b, g_wq, g_bq, g_wk, g_bk, g_wv, g_bv, g_wo, g_bo)])
    return dict(y=y, dx=grad_y + gx_ln, grads=grads, q=q, k=k, v=v, ctx=ctx, lse2=fwd["lse2"], g_ctx=g_ctx,
                dq=dq, dk=dk, dv=dv)


# --------------------------------------------------------------------------
# FFN half of the layer: model.py:362-390, 449-452, 475-478
# --------------------------------------------------------------------------

GELU_C = math.sqrt(2.0 / math.pi)  # nnops._GELU_C


def gelu_fwd(x):
    """nnops.py:235-237: 0.5 x (1 + tanh(c (x + 0.044715 x^3)))."""
    return 0.5 * x * (1.0 + np.tanh(GELU_C * (x + 0.044715 * x ** 3)))


def gelu_bwd(x, gy):
    """nnops.py:240-245."""
    t = np.tanh(GELU_C * (x + 0.044715 * x ** 3))
    return gy * (0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * GELU_C * (1.0 + 3.0 * 0.044715 * x * x))


@dataclass
class FfnParams:
    """The FFN-half parameters of model.LayerParams (model.py:91-94)."""
    ln2_gain: np.ndarray
    ln2_bias: np.ndarray
    w_in: np.ndarray
    b_in: np.ndarray
    w_out: np.ndarray
    b_out: np.ndarray

    GRAD_ORDER = ("ln2_gain", "ln2_bias", "w_in", "b_in", "w_out", "b_out")

    def astype(self, dt):
        return FfnParams(*[getattr(self, n).astype(dt) for n in self.GRAD_ORDER])


def ffn_half(x_mid, grad_out, f: FfnParams):
    """model.layer_fwd 449-452 (LN2 -> ffn_fwd -> residual) and layer_bwd 475-478
    (ffn_bwd -> LN2 bwd -> grad_mid = grad_out + g_ln2), dropout 0.  Row-local,
    so it runs on the whole (B, l, E) at once; returns (y, grad_mid, grads summed
    over all rows)."""
    yh, ln2 = layernorm_fwd(x_mid, f.ln2_gain, f.ln2_bias)
    h_pre = linear_fwd(yh, f.w_in, f.b_in)  # model.py:375
    h = gelu_fwd(h_pre)  # model.py:376
    y = x_mid + linear_fwd(h, f.w_out, f.b_out)  # model.py:378, 452
    g_h, g_wout, g_bout = linear_bwd(h, f.w_out, grad_out)  # model.py:385
    g_pre = gelu_bwd(h_pre, g_h)  # model.py:387
    g_yh, g_win, g_bin = linear_bwd(yh, f.w_in, g_pre)  # model.py:388
    g_ln2x, g_g2, g_b2 = layernorm_bwd(ln2, f.ln2_gain, g_yh)  # model.py:476
    return y, grad_out + g_ln2x, FfnParams(g_g2, g_b2, g_win, g_bin, g_wout, g_bout)


def lss_layer(x, grad_y, p: AttnParams, f: FfnParams, n_heads, workers, causal=True):
    """The complete pre-norm layer (model.layer_fwd / layer_bwd, model.py:424-499)
    on ``workers`` ranks: the attention half as in :func:`lss_attention`, the FFN
    half rank-local; every gradient averaged over the group (sharded.py:238)."""
    x_mid = lss_attention(x, np.zeros_like(x), p, n_heads, workers, causal)["y"]
    y, grad_mid, fg = ffn_half(x_mid, grad_y, f)
    att = lss_attention(x, grad_mid, p, n_heads, workers, causal)
    return dict(y=y, dx=att["dx"], grads=att["grads"],
                ffn_grads=FfnParams(*[getattr(fg, n) / workers for n in FfnParams.GRAD_ORDER]))


def cross_entropy(logits, targets):
    """nnops.cross_entropy (nnops.py:274-299): mean loss over rows and its logit gradient."""
    n = logits.shape[0]
    shifted = logits - logits.max(axis=1, keepdims=True)
    e = np.exp(shifted)
    se = e.sum(axis=1, keepdims=True)
    loss = float(-np.mean((shifted - np.log(se))[np.arange(n), targets]))
    grad = e / se
    grad[np.arange(n), targets] -= 1.0
    return loss, grad / n


def gpt_forward_backward(P, tokens, targets, n_heads, causal=True, workers=1):
    """model.forward / model.backward (model.py:583-618) for the whole decoder:
    token + position embedding (517-540), the layers (:func:`lss_layer`), final LN +
    head (552-570), mean cross-entropy.  ``P`` is a dict with token_table, pos_table,
    layers [(AttnParams, FfnParams)], final_gain, final_bias, head_w, head_b.
    Returns (loss, grads dict with the same keys; layers as (AttnParams, FfnParams))."""
    b, m = tokens.shape
    x = P["token_table"][tokens] + P["pos_table"][None]
    xs = [x]
    for p, f in P["layers"]:
        x = lss_layer(x, np.zeros_like(x), p, f, n_heads, workers, causal)["y"]
        xs.append(x)
    xf, lnf = layernorm_fwd(x, P["final_gain"], P["final_bias"])
    v = P["head_w"].shape[1]
    logits = (xf @ P["head_w"] + P["head_b"]).reshape(b * m, v)
    loss, glog = cross_entropy(logits, targets.reshape(-1))
    g_xf, g_hw, g_hb = linear_bwd(xf, P["head_w"], glog.reshape(b, m, v))
    g, g_fg, g_fb = layernorm_bwd(lnf, P["final_gain"], g_xf)
    layer_grads = [None] * len(P["layers"])
    for li in range(len(P["layers"]) - 1, -1, -1):
        p, f = P["layers"][li]
        out = lss_layer(xs[li], g, p, f, n_heads, workers, causal)
        g = out["dx"]
        layer_grads[li] = (out["grads"], out["ffn_grads"])
    g_tok = np.zeros_like(P["token_table"])
    np.add.at(g_tok, tokens.reshape(-1), g.reshape(b * m, -1))  # nnops.py:258-262
    return loss, dict(token_table=g_tok, pos_table=g.sum(axis=0), layers=layer_grads, final_gain=g_fg,
                      final_bias=g_fb, head_w=g_hw, head_b=g_hb)


def sgd_step(params, grads, lr):
    """model.sgd_step (model.py:621-623)."""
    return [p - lr * g for p, g in zip(params, grads)]


def adam_step(params, grads, m, v, t, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """optim.adam_step (optim.py:35-53), t 1-based; returns (params, m, v)."""
    m = [beta1 * a + (1.0 - beta1) * g for a, g in zip(m, grads)]
    v = [beta2 * a + (1.0 - beta2) * g * g for a, g in zip(v, grads)]
    out = [p - lr * (a / (1.0 - beta1 ** t)) / (np.sqrt(b / (1.0 - beta2 ** t)) + eps)
           for p, a, b in zip(params, m, v)]
    return out, m, v


# --------------------------------------------------------------------------
# Work accounting (costs.py:98 convention, extended to fwd+bwd)
# --------------------------------------------------------------------------


def attention_pairs(seq, causal):
    return seq * (seq + 1) // 2 if causal else seq * seq


def layer_flops(batch, seq, embed, causal):
    """F = 24*l*E^2 + 12*E*P per sequence."""
    return batch * (24 * seq * embed * embed + 12 * embed * attention_pairs(seq, causal))


def sample_rows(x, grad_y, p, n_heads, offset, rows, causal=True):
    """The bounded CPU sample used as the reference arm: one block of ``rows``
    query rows at global ``offset`` through the attention half forward and
    backward against full-length K/V (whose projection is done outside the
    timed region, as if received from the all-gather).  Returns the time-relevant
    outputs so the caller can keep them alive."""
    s = slice(offset, offset + rows)
    xh_all, _ = layernorm_fwd(x, p.ln1_gain, p.ln1_bias)
    k_full = linear_fwd(xh_all, p.wk, p.bk)
    v_full = linear_fwd(xh_all, p.wv, p.bv)

    def run():
        xh, ln = layernorm_fwd(x[:, s], p.ln1_gain, p.ln1_bias)
        k_own = linear_fwd(xh, p.wk, p.bk)
        v_own = linear_fwd(xh, p.wv, p.bv)
        q = linear_fwd(xh, p.wq, p.bq)
        ctx, prob = scores_fwd(q, k_full, v_full, offset, n_heads, causal)
        y = x[:, s] + linear_fwd(ctx, p.wo, p.bo)
        gy = grad_y[:, s]
        g_ctx, g_wo, g_bo = linear_bwd(ctx, p.wo, gy)
        dq, dk, dv = scores_bwd(prob, q, k_full, v_full, g_ctx, n_heads)
        gxq, g_wq, _ = linear_bwd(xh, p.wq, dq)
        gxk, g_wk, _ = linear_bwd(xh, p.wk, dk[:, s])
        gxv, g_wv, _ = linear_bwd(xh, p.wv, dv[:, s])
        gx, _, _ = layernorm_bwd(ln, p.ln1_gain, gxq + gxk + gxv)
        return y, gy + gx, k_own, v_own

    return run
