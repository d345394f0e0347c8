"""The reference's layer API (seqpar.model) on B200 kernels: the attention half
(the hot path) and the FFN half.

Same names, argument meaning and error behaviour as the reference
(/root/reference/pkg/src/seqpar/model.py) for the hot path:

  ModelConfig (model.py:39-80), LinearParams (nnops.py:172-177),
  linear3 / linear3_bwd (model.py:237-245), norm3 / norm3_bwd (248-257),
  scores_fwd / scores_bwd (280-359), local_kv_fwd / local_kv_bwd (413-421),
  ffn_fwd / ffn_bwd (362-390), layer_fwd / layer_bwd (424-499): the attention
  half always, plus LN2 -> FFN -> residual when the LayerParams carry the FFN
  weights.

Arrays are torch CUDA tensors.  ``precision`` selects the kernel family:
"bf16" (tcgen05 path, bf16 operands / fp32 accumulation, the default) or
"single" (fp32 FFMA check mode).  The residual stream and all gradients are
fp32 in both.  The reference caches the full probability matrix P per
(sample, head); the B200 ScoreCache keeps (ctx, lse) and the backward
recomputes P (flash-attention), so ``cache.attn`` does not exist -- use
``probabilities()`` to materialise P for a check.

Out of scope here: dropout > 0 (raises), embeddings/head --
every BASELINE config runs dropout 0 and the hot path is the attention
sublayer.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import torch

from . import kernels as K
from .dropout import DropoutPolicy, as_policy
from .errors import ShapeError, UnsupportedError

LAYERNORM_EPS = 1e-5


@dataclass(frozen=True)
class ModelConfig:
    """model.py:39-80.  ``precision`` is "bf16" or "single" on the B200 path."""

    embed_dim: int
    n_layers: int
    n_heads: int
    ff_dim: int
    vocab: int
    seq_len: int
    batch: int = 1
    dropout: float = 0.0
    causal: bool = True
    precision: str = "bf16"

    def __post_init__(self) -> None:
        if self.embed_dim < 1 or self.n_heads < 1 or self.ff_dim < 1:
            raise ValueError("model dimensions must be positive")
        if self.embed_dim % self.n_heads != 0:
            raise ShapeError(f"embed_dim {self.embed_dim} is not divisible by n_heads {self.n_heads}")
        if self.n_layers < 0:
            raise ValueError("n_layers must be non-negative")
        if self.vocab < 1 or self.seq_len < 1 or self.batch < 1:
            raise ValueError("vocab, seq_len and batch must be positive")
        if not 0.0 <= self.dropout < 1.0:
            raise ValueError(f"dropout must be in [0, 1), got {self.dropout}")
        K.code(self.precision)  # UnsupportedError for "double"

    @property
    def head_dim(self) -> int:
        return self.embed_dim // self.n_heads

    @property
    def act_dtype(self) -> torch.dtype:
        return K.act_dtype(self.precision)


@dataclass(frozen=True)
class LinearParams:
    """nnops.py:172-177: weight [d_in, d_out], bias [d_out], y = x W + b (fp32)."""

    weight: torch.Tensor
    bias: torch.Tensor


@dataclass
class LayerParams:
    """model.LayerParams (model.py:83-94).  The FFN half (ln2_*, ff_in, ff_out) is
    optional: without it the layer is its attention half (the hot path)."""

    ln1_gain: torch.Tensor
    ln1_bias: torch.Tensor
    attn_q: LinearParams
    attn_k: LinearParams
    attn_v: LinearParams
    attn_out: LinearParams
    ln2_gain: Optional[torch.Tensor] = None
    ln2_bias: Optional[torch.Tensor] = None
    ff_in: Optional[LinearParams] = None
    ff_out: Optional[LinearParams] = None

    @property
    def has_ffn(self) -> bool:
        return self.ff_in is not None

    def named_arrays(self):
        """Same relative order as Parameters.named_arrays (model.py:118-133)."""
        yield "ln1_gain", self.ln1_gain
        yield "ln1_bias", self.ln1_bias
        for n in ("attn_q", "attn_k", "attn_v", "attn_out"):
            p = getattr(self, n)
            yield f"{n}.weight", p.weight
            yield f"{n}.bias", p.bias
        if self.has_ffn:
            yield "ln2_gain", self.ln2_gain
            yield "ln2_bias", self.ln2_bias
            for n in ("ff_in", "ff_out"):
                p = getattr(self, n)
                yield f"{n}.weight", p.weight
                yield f"{n}.bias", p.bias


def layer_params_from_arrays(ln1_gain, ln1_bias, wq, bq, wk, bk, wv, bv, wo, bo, device="cuda", *,
                             ln2_gain=None, ln2_bias=None, w_in=None, b_in=None, w_out=None, b_out=None):
    t = lambda a: torch.as_tensor(a, dtype=torch.float32, device=device).contiguous()  # noqa: E731
    lp = LayerParams(t(ln1_gain), t(ln1_bias), LinearParams(t(wq), t(bq)), LinearParams(t(wk), t(bk)),
                     LinearParams(t(wv), t(bv)), LinearParams(t(wo), t(bo)))
    if w_in is not None:
        lp.ln2_gain, lp.ln2_bias = t(ln2_gain), t(ln2_bias)
        lp.ff_in, lp.ff_out = LinearParams(t(w_in), t(b_in)), LinearParams(t(w_out), t(b_out))
    return lp


def _check_dropout(cfg: ModelConfig, policy) -> None:
    """Dropout (position-keyed masks, dropout.py) runs on the bf16 tcgen05 path; the
    fp32 check mode has no dropout kernels."""
    if as_policy(policy).active and cfg.precision != "bf16":
        raise UnsupportedError("dropout > 0 runs on the bf16 path only (no fp32 check-mode dropout kernels)")


def _dropout(x: torch.Tensor, policy, layer: int, tag: str, offset: int, out=None, residual=None):
    """nnops.dropout_fwd / dropout_bwd on (B, m, C) rows at global positions
    offset..offset+m (model.dropout3 / row_coords, model.py:230-268); identity
    (plus residual) when the policy is off."""
    pol = as_policy(policy)
    if not pol.active:
        if residual is None:
            return x
        return (x.to(torch.float32) + residual) if out is None else out.copy_(x + residual)
    b, m, c = x.shape
    out = out if out is not None else torch.empty_like(x if residual is None else residual)
    return K.dropout_rows(x.contiguous(), out, rows_per_sample=m, offset=offset, site_key=pol.site_key(layer, tag),
                          thresh=pol.thresh, scale=pol.scale, residual=residual)


def _as_act(x: torch.Tensor, cfg: ModelConfig) -> torch.Tensor:
    return x if x.dtype == cfg.act_dtype else x.to(cfg.act_dtype)


class _Precision:
    """Stand-in for an omitted ``cfg``: the kernel family follows the operand's dtype
    (bf16 -> tcgen05 path, fp32 -> fp32 check mode), as the reference's dtype
    policy follows its arrays (tensor.py:24-32)."""

    def __init__(self, x: torch.Tensor):
        self.precision = "bf16" if x.dtype == torch.bfloat16 else "single"
        self.act_dtype = K.act_dtype(self.precision)


def _cfg_or(cfg, x: torch.Tensor):
    return cfg if cfg is not None else _Precision(x)


# ------------------------------------------------------------------ linear / norm


def linear3(x: torch.Tensor, p: LinearParams, cfg: Optional[ModelConfig] = None,
            out_dtype=torch.float32) -> torch.Tensor:
    """model.linear3 (model.py:237-239): x (B, m, E_in) @ W + b -> (B, m, E_out).
    ``cfg`` may be omitted as in the reference: the precision then follows x."""
    cfg = _cfg_or(cfg, x)
    b, m, e = x.shape
    if p.weight.shape[0] != e:
        raise ShapeError(f"matmul inner dims disagree: {tuple(x.shape)} x {tuple(p.weight.shape)}")
    a = _as_act(x, cfg).contiguous()
    w = _as_act(p.weight, cfg).contiguous()
    n = w.shape[1]
    out = torch.empty(b, m, n, dtype=out_dtype, device=x.device)
    # B operand = W stored [d_in][d_out] = [K][N] -> N-major
    K.gemm(a.view(b * m, e), w, b_mn_major=True, bias=p.bias, out=out.view(b * m, n), M=b * m, N=n, K=e)
    return K.checked(out)


def linear3_bwd(x: torch.Tensor, p: LinearParams, grad_y: torch.Tensor, cfg: Optional[ModelConfig] = None):
    """model.linear3_bwd (model.py:242-245) -> (grad_x, grad_W, grad_b), fp32."""
    cfg = _cfg_or(cfg, x)
    b, m, e = x.shape
    n = p.weight.shape[1]
    gy32 = grad_y.to(torch.float32).contiguous().view(b * m, n)
    gy = _as_act(gy32, cfg).contiguous()
    xa = _as_act(x, cfg).contiguous().view(b * m, e)
    w = _as_act(p.weight, cfg).contiguous()
    gx = torch.empty(b * m, e, dtype=torch.float32, device=x.device)
    K.gemm(gy, w, out=gx, M=b * m, N=e, K=n)  # gy . W^T  (W [e][n] is K-major for N=e)
    gw = torch.empty(e, n, dtype=torch.float32, device=x.device)
    K.gemm(xa, gy, a_mn_major=True, b_mn_major=True, out=gw, M=e, N=n, K=b * m)  # x^T . gy
    gb = torch.zeros(n, dtype=torch.float32, device=x.device)
    K.cat_cast_colsum([(gy32, n, n)], b * m, dst=None, colsum=gb)
    K.checked(gx, gw, gb)
    return gx.view(b, m, e), gw, gb


@dataclass
class NormCache:
    x: torch.Tensor
    mean: torch.Tensor
    rstd: torch.Tensor


def norm3(x: torch.Tensor, gain: torch.Tensor, bias: torch.Tensor, cfg: Optional[ModelConfig] = None,
          out_dtype=torch.float32):
    """model.norm3 (model.py:248-251) -> (y, cache)."""
    x = x.to(torch.float32).contiguous()
    y, mean, rstd = K.layernorm_fwd(x, gain, bias, out_dtype=out_dtype)
    return K.checked(y), NormCache(x, mean, rstd)


def norm3_bwd(cache: NormCache, gain: torch.Tensor, grad_y: torch.Tensor, grad_res=None):
    """model.norm3_bwd (model.py:254-257) -> (grad_x, grad_gain, grad_bias).
    ``grad_res`` (optional) is added to grad_x (the residual of model.py:486)."""
    gy = grad_y.to(torch.float32).contiguous()
    return K.layernorm_bwd(gy, cache.x, cache.mean, cache.rstd, gain, grad_res=grad_res)


# ------------------------------------------------------------------ attention core


@dataclass
class ScoreCache:
    """B200 replacement of model.ScoreCache: (ctx, lse) instead of full P."""

    offset: int
    ctx: torch.Tensor
    lse2: torch.Tensor
    k: torch.Tensor = field(repr=False)
    v: torch.Tensor = field(repr=False)
    workers: int = 1
    seg_len: int = 0
    policy: object = None  # dropout policy and layer: the masks are recomputed in the backward
    layer: int = 0


def _kv_rows(k: torch.Tensor):
    """Accept (B, t, E) or the packed segment layout (G, B, seg, E)."""
    if k.dim() == 3:
        return 1, k.shape[1]
    if k.dim() == 4:
        return k.shape[0], k.shape[2]
    raise ShapeError(f"keys must be (B, t, E) or (G, B, seg, E), got {tuple(k.shape)}")


def scores_fwd(q, k, v, offset: int, cfg: ModelConfig, policy=None, layer: int = 0, counters=None):
    """model.scores_fwd (model.py:280-326) -> (ctx, ScoreCache).

    q (B, m, E) holds this block's rows at global positions offset..offset+m;
    k/v hold the whole sequence, (B, t, E), or as G row-segments (G, B, seg, E)
    (e.g. views into the packed all-gather buffer).  Causal rows attend to
    keys at or before their global position."""
    _check_dropout(cfg, policy)
    bsz, m, e = q.shape
    if e != cfg.embed_dim:
        raise ShapeError(f"q has {e} features, config says {cfg.embed_dim}")
    workers, seg = _kv_rows(k)
    t = workers * seg
    if cfg.causal and offset < 0:
        from .errors import DegenerateRowError

        raise DegenerateRowError("negative offset leaves causal rows fully masked")
    qa = _as_act(q, cfg).contiguous()
    ka = k if k.dtype == cfg.act_dtype else k.to(cfg.act_dtype)
    va = v if v.dtype == cfg.act_dtype else v.to(cfg.act_dtype)
    if ka.dim() == 3:
        ka, va = ka.contiguous(), va.contiguous()
    pol = as_policy(policy)
    if pol.active:  # probability dropout inside the flash kernel (nnops.keep_mask keys)
        ctx = torch.empty(bsz, m, e, dtype=qa.dtype, device=qa.device)
        lse = torch.empty(bsz, cfg.n_heads, K.rows_pad(m), dtype=torch.float32, device=qa.device)
        kv = (ka, va) if ka.dim() == 4 else (ka.unsqueeze(0), va.unsqueeze(0))
        K.attn_fwd_partial(qa, kv[0], kv[1], rows=m, row0=0, workers=workers, seg_len=seg, heads=cfg.n_heads,
                           offset=offset, causal=cfg.causal, g_begin=0, g_end=workers, out=ctx, lse2=lse,
                           dropout=pol.desc(layer))
    else:
        ctx, lse = K.attn_fwd(qa, ka, va, workers=workers, seg_len=seg, heads=cfg.n_heads, offset=offset,
                              causal=cfg.causal)
    if counters is not None:  # model.py:312-313, 321-325: 2*m*d*t twice per (b, h)
        bh = bsz * cfg.n_heads
        counters.add_score_flops(m, cfg.head_dim * bh, t)
        counters.add_score_flops(m, t, cfg.head_dim * bh)
        counters.record_score_footprint(bh * m * t)
    return K.checked(ctx), ScoreCache(offset, ctx, lse, ka, va, workers, seg, pol, layer)


def scores_bwd(cache: ScoreCache, q, k, v, grad_ctx, cfg: ModelConfig, policy=None):
    """model.scores_bwd (model.py:329-359) -> (grad_q, grad_k, grad_v), fp32.
    grad_k / grad_v cover the whole key length (this block's partials) in the
    layout k/v were given in."""
    _check_dropout(cfg, policy)
    qa = _as_act(q, cfg).contiguous()
    go = _as_act(grad_ctx, cfg).contiguous()
    workers, seg = cache.workers, cache.seg_len
    bsz, m, e = qa.shape
    ka, va = cache.k, cache.v
    if ka.dim() == 3:
        packed = torch.empty(bsz, seg, 2 * e, dtype=torch.float32, device=qa.device)
    else:
        packed = torch.empty(workers, bsz, seg, 2 * e, dtype=torch.float32, device=qa.device)
    gk, gv = packed[..., :e], packed[..., e:]
    pol = as_policy(cache.policy)
    if pol.active:  # same masks as the forward, recomputed from (seed, layer, b, h, q_pos, k_pos)
        H = cfg.n_heads
        delta = torch.empty(bsz, H, cache.lse2.shape[-1], dtype=torch.float32, device=qa.device)
        K.attn_delta(cache.ctx, go, delta, heads=H, scaled=True)
        gq = torch.zeros(bsz, m, e, dtype=torch.float32, device=qa.device)
        src = dict(q=qa, grad_o=go, grad_q=gq, row0=0, rows=m, pos0=cache.offset, g_begin=0, g_end=workers,
                   lse2=cache.lse2, delta=delta)
        dq64 = None
        if K.deterministic():  # fixed-point dQ: bitwise repeatable
            dq64 = src["grad_q_fixed"] = torch.zeros(bsz, m, e, dtype=torch.int64, device=qa.device)
        kv = (ka, va) if ka.dim() == 4 else (ka.unsqueeze(0), va.unsqueeze(0))
        gk4, gv4 = (gk, gv) if gk.dim() == 4 else (gk.unsqueeze(0), gv.unsqueeze(0))
        K.attn_bwd_sources(kv[0], kv[1], [src], grad_k=gk4, grad_v=gv4, workers=workers, seg_len=seg, heads=H,
                           causal=cfg.causal, dropout=pol.desc(cache.layer))
        if dq64 is not None:
            K.fixed_to_f32(gq, dq64)
        K.checked(gq, packed)
        return gq, gk, gv
    gq, gk, gv = K.attn_bwd(qa, ka, va, cache.ctx, go, cache.lse2, workers=workers, seg_len=seg,
                            heads=cfg.n_heads, offset=cache.offset, causal=cfg.causal, grad_k=gk,
                            grad_v=gv)
    K.checked(gq, packed)
    return gq, gk, gv


def probabilities(cache: ScoreCache, q, cfg: ModelConfig) -> torch.Tensor:
    """Materialise P (B, H, m, t) from (q, k, lse) for checks (the reference's cache.attn)."""
    bsz, m, e = q.shape
    d = cfg.head_dim
    k = cache.k if cache.k.dim() == 3 else cache.k.permute(1, 0, 2, 3).reshape(bsz, -1, e)
    qh = q.float().view(bsz, m, cfg.n_heads, d).transpose(1, 2)
    kh = k.float().reshape(bsz, -1, cfg.n_heads, d).transpose(1, 2)
    s = qh @ kh.transpose(-1, -2) / math.sqrt(d) * (1.0 / math.log(2))
    p = torch.exp2(s - cache.lse2[:, :, :m, None])
    if cfg.causal:
        t = k.shape[1]
        keep = torch.arange(t, device=q.device)[None, :] <= (cache.offset + torch.arange(m, device=q.device))[:, None]
        p = torch.where(keep, p, torch.zeros((), device=q.device))
    return p


# ------------------------------------------------------------------ FFN half


@dataclass
class FfnCache:
    """model.FfnCache (model.py:365-369) without dropout: yh, h_pre, h (operand dtype)."""

    yh: torch.Tensor
    h_pre: torch.Tensor
    h: torch.Tensor  # h_drop (the dropped activation feeds ff_out and its wgrad)
    policy: object = None
    layer: int = 0
    offset: int = 0


def ffn_fwd(yh: torch.Tensor, lp: LayerParams, cfg: ModelConfig, policy=None, layer: int = 0, residual=None,
            offset: int = 0):
    """model.ffn_fwd (model.py:371-378): ff_in -> tanh-GeLU -> ff_out.  The GeLU
    runs in the ff_in GEMM's epilogue (which also keeps the pre-activation for
    the backward); ``residual`` (fp32, optional) is added in the ff_out epilogue
    (model.py:452's x_mid + ff)."""
    _check_dropout(cfg, policy)
    b, m, e = yh.shape
    ff = lp.ff_in.weight.shape[1]
    if lp.ff_in.weight.shape[0] != e or lp.ff_out.weight.shape != (ff, e):
        raise ShapeError(f"ffn weights {tuple(lp.ff_in.weight.shape)} / {tuple(lp.ff_out.weight.shape)} "
                         f"do not match embed {e}")
    ya = _as_act(yh, cfg).contiguous().view(b * m, e)
    ad = cfg.act_dtype
    h_pre = torch.empty(b * m, ff, dtype=ad, device=yh.device)
    h = torch.empty(b * m, ff, dtype=ad, device=yh.device)
    K.gemm(ya, _as_act(lp.ff_in.weight, cfg).contiguous(), b_mn_major=True, bias=lp.ff_in.bias, out=h,
           act="gelu", pre=h_pre, M=b * m, N=ff, K=e)
    pol = as_policy(policy)
    if pol.active:  # model.py:377 (ffn_hidden) and 451 (ffn_out)
        _dropout(h.view(b, m, ff), pol, layer, "ffn_hidden", offset, out=h.view(b, m, ff))
    out = torch.empty(b * m, e, dtype=torch.float32, device=yh.device)
    res = None if residual is None else residual.to(torch.float32).contiguous().view(b * m, e)
    K.gemm(h, _as_act(lp.ff_out.weight, cfg).contiguous(), b_mn_major=True, bias=lp.ff_out.bias, out=out,
           residual=None if pol.active else res, M=b * m, N=e, K=ff)
    if pol.active:
        out = _dropout(out.view(b, m, e), pol, layer, "ffn_out", offset,
                       residual=None if res is None else res.view(b, m, e))
    return out.view(b, m, e), FfnCache(ya, h_pre, h, pol, layer, offset)


def ffn_bwd(cache: FfnCache, lp: LayerParams, grad_out: torch.Tensor, cfg: ModelConfig, policy=None):
    """model.ffn_bwd (model.py:381-390) -> (grad_yh, (ff_in_wg, ff_in_bg, ff_out_wg, ff_out_bg)).
    The GeLU derivative at the stored pre-activation is applied in the epilogue of
    the GEMM that produces grad_h."""
    _check_dropout(cfg, policy)
    b, m, e = grad_out.shape
    M, ff = cache.h.shape
    ad = cfg.act_dtype
    g32 = grad_out.to(torch.float32).contiguous().view(M, e)
    pol = as_policy(cache.policy)
    if pol.active:  # dropout3_bwd(ffn_out), model.py:475
        g32 = _dropout(g32.view(b, m, e), pol, cache.layer, "ffn_out", cache.offset).view(M, e)
    g = torch.empty(M, e, dtype=ad, device=g32.device)
    ff_out_bg = torch.zeros(e, dtype=torch.float32, device=g32.device)
    K.cat_cast_colsum([(g32, e, e)], M, dst=g, colsum=ff_out_bg)
    w_out = _as_act(lp.ff_out.weight, cfg).contiguous()  # [ff][E] = [N][K] for g . W_out^T
    g_pre32 = torch.empty(M, ff, dtype=torch.float32, device=g32.device)
    K.gemm(g, w_out, out=g_pre32, act="gelu_bwd", aux=cache.h_pre, M=M, N=ff, K=e)
    if pol.active:  # dropout_bwd(ffn_hidden), model.py:387 (elementwise: commutes with GeLU')
        _dropout(g_pre32.view(b, m, ff), pol, cache.layer, "ffn_hidden", cache.offset, out=g_pre32.view(b, m, ff))
    ff_out_wg = torch.empty(ff, e, dtype=torch.float32, device=g32.device)
    K.gemm(cache.h, g, a_mn_major=True, b_mn_major=True, out=ff_out_wg, M=ff, N=e, K=M)  # h^T . g
    g_pre = torch.empty(M, ff, dtype=ad, device=g32.device)
    ff_in_bg = torch.zeros(ff, dtype=torch.float32, device=g32.device)
    K.cat_cast_colsum([(g_pre32, ff, ff)], M, dst=g_pre, colsum=ff_in_bg)
    w_in = _as_act(lp.ff_in.weight, cfg).contiguous()  # [E][ff] = [N][K] for g_pre . W_in^T
    grad_yh = torch.empty(M, e, dtype=torch.float32, device=g32.device)
    K.gemm(g_pre, w_in, out=grad_yh, M=M, N=e, K=ff)
    ff_in_wg = torch.empty(e, ff, dtype=torch.float32, device=g32.device)
    K.gemm(cache.yh, g_pre, a_mn_major=True, b_mn_major=True, out=ff_in_wg, M=e, N=ff, K=M)  # yh^T . g_pre
    return grad_yh.view(b, m, e), (ff_in_wg, ff_in_bg, ff_out_wg, ff_out_bg)


# ------------------------------------------------------------------ layer


def local_kv_fwd(xh: torch.Tensor, lp: LayerParams, cfg: Optional[ModelConfig] = None):
    """model.local_kv_fwd (model.py:413-415): project the block itself."""
    cfg = _cfg_or(cfg, xh)
    return linear3(xh, lp.attn_k, cfg, cfg.act_dtype), linear3(xh, lp.attn_v, cfg, cfg.act_dtype), xh


def local_kv_bwd(kv_ctx, lp: LayerParams, grad_k, grad_v, cfg: Optional[ModelConfig] = None):
    """model.local_kv_bwd (model.py:418-421)."""
    gkx, k_wg, k_bg = linear3_bwd(kv_ctx, lp.attn_k, grad_k, cfg)
    gvx, v_wg, v_bg = linear3_bwd(kv_ctx, lp.attn_v, grad_v, cfg)
    return gkx + gvx, k_wg, k_bg, v_wg, v_bg


@dataclass
class LayerCache:
    offset: int
    ln1: NormCache
    xh: torch.Tensor
    kv_ctx: object
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    scores: ScoreCache
    ctx: torch.Tensor
    ln2: Optional[NormCache] = None
    ffn: Optional[FfnCache] = None


def layer_fwd(lp: LayerParams, cfg: ModelConfig, policy, layer: int, x: torch.Tensor, offset: int,
              kv_fwd: Optional[Callable] = None, counters=None):
    """model.layer_fwd (model.py:424-456): norm -> kv_fwd -> q -> scores ->
    out-projection -> residual, then (when lp has the FFN half) LN2 -> FFN -> residual."""
    _check_dropout(cfg, policy)
    kv_fwd = kv_fwd or (lambda xh, lp_: local_kv_fwd(xh, lp_, cfg))
    xh, ln1 = norm3(x, lp.ln1_gain, lp.ln1_bias, cfg, out_dtype=cfg.act_dtype)
    k, v, kv_ctx = kv_fwd(xh, lp)
    q = linear3(xh, lp.attn_q, cfg, cfg.act_dtype)
    ctx, sc = scores_fwd(q, k, v, offset, cfg, policy, layer, counters)
    x_mid = _dropout(linear3(ctx, lp.attn_out, cfg), policy, layer, "attn_out", offset,
                     residual=x.to(torch.float32).contiguous())  # model.py:447-448
    if not lp.has_ffn:
        return x_mid, LayerCache(offset, ln1, xh, kv_ctx, q, k, v, sc, ctx)
    yh, ln2 = norm3(x_mid, lp.ln2_gain, lp.ln2_bias, cfg, out_dtype=cfg.act_dtype)
    x_out, fc = ffn_fwd(yh, lp, cfg, policy, layer, residual=x_mid, offset=offset)
    return x_out, LayerCache(offset, ln1, xh, kv_ctx, q, k, v, sc, ctx, ln2, fc)


def layer_bwd(lp: LayerParams, cfg: ModelConfig, policy, layer: int, cache: LayerCache,
              grad_out: torch.Tensor, kv_bwd: Optional[Callable] = None):
    """model.layer_bwd (model.py:459-499) -> (grad_in, grads LayerParams)."""
    _check_dropout(cfg, policy)
    kv_bwd = kv_bwd or (lambda kv_ctx, lp_, gk, gv: local_kv_bwd(kv_ctx, lp_, gk, gv, cfg))
    grad_out = grad_out.to(torch.float32).contiguous()
    ffn_grads = None
    if lp.has_ffn:  # model.py:474-477
        grad_yh, ffn_grads = ffn_bwd(cache.ffn, lp, grad_out, cfg, policy)
        grad_mid, ln2_gg, ln2_bg = norm3_bwd(cache.ln2, lp.ln2_gain, grad_yh, grad_res=grad_out)
    else:
        grad_mid = grad_out
    g_att = _dropout(grad_mid, policy, layer, "attn_out", cache.offset)  # dropout3_bwd, model.py:479
    grad_ctx, out_wg, out_bg = linear3_bwd(cache.ctx, lp.attn_out, g_att, cfg)
    gq, gk, gv = scores_bwd(cache.scores, cache.q, cache.k, cache.v, grad_ctx, cfg, policy)
    gxq, q_wg, q_bg = linear3_bwd(cache.xh, lp.attn_q, gq, cfg)
    gxkv, k_wg, k_bg, v_wg, v_bg = kv_bwd(cache.kv_ctx, lp, gk, gv)
    grad_xh = gxq + gxkv
    g_in, g_gain, g_bias = norm3_bwd(cache.ln1, lp.ln1_gain, grad_xh, grad_res=grad_mid)
    grads = LayerParams(g_gain, g_bias, LinearParams(q_wg, q_bg), LinearParams(k_wg, k_bg),
                        LinearParams(v_wg, v_bg), LinearParams(out_wg, out_bg))
    if ffn_grads is not None:
        ff_in_wg, ff_in_bg, ff_out_wg, ff_out_bg = ffn_grads
        grads.ln2_gain, grads.ln2_bias = ln2_gg, ln2_bg
        grads.ff_in, grads.ff_out = LinearParams(ff_in_wg, ff_in_bg), LinearParams(ff_out_wg, ff_out_bg)
    return g_in, grads


# ------------------------------------------------------------------ whole model


@dataclass
class Parameters:
    """model.Parameters (model.py:97-137); on a distributed worker ``pos_table``
    holds only that worker's rows.  The same container carries gradients."""

    token_table: torch.Tensor
    pos_table: torch.Tensor
    layers: list
    final_gain: torch.Tensor
    final_bias: torch.Tensor
    head: LinearParams

    def named_arrays(self):
        yield "token_table", self.token_table
        yield "pos_table", self.pos_table
        for i, lp in enumerate(self.layers):
            for n, a in lp.named_arrays():
                yield f"layer{i}.{n}", a
        yield "final_gain", self.final_gain
        yield "final_bias", self.final_bias
        yield "head.weight", self.head.weight
        yield "head.bias", self.head.bias

    def arrays(self) -> list:
        return [a for _, a in self.named_arrays()]

    def replace_arrays(self, arrays) -> "Parameters":
        """model.Parameters.replace_arrays (model.py:142-166): same structure from a
        flat list in named order."""
        it = iter(arrays)
        lin = lambda: LinearParams(next(it), next(it))  # noqa: E731
        tok, pos = next(it), next(it)
        layers = []
        for lp in self.layers:
            g1, b1 = next(it), next(it)
            q, k, v, o = lin(), lin(), lin(), lin()
            nl = LayerParams(g1, b1, q, k, v, o)
            if lp.has_ffn:
                nl.ln2_gain, nl.ln2_bias = next(it), next(it)
                nl.ff_in, nl.ff_out = lin(), lin()
            layers.append(nl)
        fg, fb = next(it), next(it)
        return Parameters(tok, pos, layers, fg, fb, lin())

    def copy(self) -> "Parameters":
        return self.replace_arrays([a.clone() for a in self.arrays()])

    def zip_map(self, other: "Parameters", fn) -> "Parameters":
        return self.replace_arrays([fn(a, b) for a, b in zip(self.arrays(), other.arrays())])


def sgd_step(params: Parameters, grads: Parameters, lr: float) -> Parameters:
    """model.sgd_step (model.py:621-623): fresh parameters w - lr*g, inputs untouched."""
    return params.zip_map(grads, lambda w, g: w - lr * g)


def flatten_arrays(arrays) -> torch.Tensor:
    """model.flatten_arrays (model.py:629-630)."""
    return torch.cat([a.reshape(-1) for a in arrays]) if arrays else torch.zeros(0)


def unflatten_like(vec: torch.Tensor, arrays) -> list:
    """model.unflatten_like (model.py:633-642)."""
    needed = sum(a.numel() for a in arrays)
    if vec.numel() != needed:
        raise ShapeError(f"flat vector has {vec.numel()} elements, structure needs {needed}")
    out, pos = [], 0
    for a in arrays:
        out.append(vec[pos:pos + a.numel()].view(a.shape))
        pos += a.numel()
    return out


def grad_norm(grads: Parameters) -> float:
    """model.grad_norm (model.py:645-650): Euclidean norm folded in parameter order (fp64)."""
    total = torch.zeros((), dtype=torch.float64, device=grads.token_table.device)
    for _, g in grads.named_arrays():
        total += (g.to(torch.float64) ** 2).sum()
    return float(total.sqrt())


def _ids(t: torch.Tensor, vocab: int, what: str) -> torch.Tensor:
    """int32 device ids, range-checked like nnops.embed_tokens / cross_entropy."""
    ids = t.to(torch.int32).contiguous()
    lo, hi = torch.aminmax(ids)
    if int(lo) < 0 or int(hi) >= vocab:
        raise ValueError(f"{what} id out of range for vocab {vocab}")
    return ids


@dataclass
class EmbedCache:
    tokens: torch.Tensor
    policy: object = None
    offset: int = 0


def embed_fwd(params: Parameters, cfg: ModelConfig, tokens: torch.Tensor, offset: int = 0, policy=None):
    """model.embed_fwd (model.py:517-533): token + position embeddings of one block."""
    _check_dropout(cfg, policy)
    if tokens.dim() != 2:
        raise ShapeError(f"tokens must be (batch, seq_len), got shape {tuple(tokens.shape)}")
    m = tokens.shape[1]
    if params.pos_table.shape[0] != m:
        raise ShapeError(f"position table has {params.pos_table.shape[0]} rows, block has {m}")
    ids = _ids(tokens, params.token_table.shape[0], "token")
    x = K.embed_fwd(ids, params.token_table.contiguous(), params.pos_table.contiguous())
    pol = as_policy(policy)
    if pol.active:  # model.py:526 (layer 0, tag "embed")
        x = _dropout(x, pol, 0, "embed", offset, out=x)
    return x, EmbedCache(ids, pol, offset)


def embed_bwd(cache: EmbedCache, vocab: int, policy, grad_x: torch.Tensor):
    """model.embed_bwd (model.py:536-540) -> (grad_token_table, grad_pos_table)."""
    g = grad_x.to(torch.float32).contiguous()
    pol = as_policy(cache.policy)
    if pol.active:
        g = _dropout(g, pol, 0, "embed", cache.offset)
    return K.embed_bwd(cache.tokens, g, vocab)


@dataclass
class HeadCache:
    lnf: NormCache
    xf: torch.Tensor
    logits: torch.Tensor
    grad_logits: Optional[torch.Tensor]
    shape3: tuple
    vocab: int
    cfg: object = None


def _head_operand(params: Parameters, cfg: ModelConfig):
    """Head weight [E][V] and bias with V padded to a multiple of 32 for the tcgen05
    GEMM (padded columns have zero weights; the loss ignores them)."""
    w, b = params.head.weight, params.head.bias
    v = w.shape[1]
    vp = (v + 31) // 32 * 32 if cfg.precision == "bf16" else v
    if vp != v:
        w = torch.nn.functional.pad(w, (0, vp - v))
        b = torch.nn.functional.pad(b, (0, vp - v))
    return _as_act(w, cfg).contiguous(), b.contiguous(), vp


def head_fwd(x: torch.Tensor, params: Parameters, targets: Optional[torch.Tensor],
             cfg: Optional[ModelConfig] = None):
    """model.head_fwd (model.py:552-562): final LN, vocabulary projection and the
    mean cross-entropy.  Returns (loss or None, HeadCache).  Without ``cfg`` the
    bf16 tcgen05 path runs (the residual stream x is fp32 in both precisions)."""
    cfg = cfg if cfg is not None else _Precision(torch.empty(0, dtype=torch.bfloat16))
    bsz, m, e = x.shape
    v = params.head.weight.shape[1]
    xf, lnf = norm3(x.reshape(bsz * m, e), params.final_gain, params.final_bias, cfg, out_dtype=cfg.act_dtype)
    w, b, vp = _head_operand(params, cfg)
    logits = torch.empty(bsz * m, vp, dtype=torch.float32, device=x.device)
    K.gemm(xf, w, b_mn_major=True, bias=b, out=logits, M=bsz * m, N=vp, K=e)
    if targets is None:
        return None, HeadCache(lnf, xf, logits, None, (bsz, m, e), v, cfg)
    ids = _ids(targets.reshape(-1), v, "target")
    n = bsz * m
    loss_rows, grad = K.cross_entropy(logits, ids, v, scale=1.0 / n)
    loss = loss_rows.sum() / n
    if not bool(torch.isfinite(loss)):
        raise ValueError("cross_entropy produced a non-finite loss")
    return float(loss), HeadCache(lnf, xf, logits, grad, (bsz, m, e), v, cfg)


def head_bwd(cache: HeadCache, params: Parameters, cfg: Optional[ModelConfig] = None):
    """model.head_bwd (model.py:565-570) -> (grad_x, final_gain_g, final_bias_g, head_wg, head_bg)."""
    cfg = cfg if cfg is not None else cache.cfg
    if cache.grad_logits is None:
        raise ValueError("head_bwd requires a forward pass that computed the loss")
    n, vp = cache.grad_logits.shape
    e = cache.xf.shape[1]
    v = cache.vocab
    w, _, _ = _head_operand(params, cfg)
    ga = _as_act(cache.grad_logits, cfg).contiguous()
    grad_xf = torch.empty(n, e, dtype=torch.float32, device=ga.device)
    K.gemm(ga, w, out=grad_xf, M=n, N=e, K=vp)  # g . W^T  (W [E][Vp] = [N][K])
    head_wg = torch.empty(e, vp, dtype=torch.float32, device=ga.device)
    K.gemm(cache.xf, ga, a_mn_major=True, b_mn_major=True, out=head_wg, M=e, N=vp, K=n)
    head_bg = torch.zeros(vp, dtype=torch.float32, device=ga.device)
    K.cat_cast_colsum([(cache.grad_logits, vp, vp)], n, dst=None, colsum=head_bg)
    grad_x, g_gain, g_bias = norm3_bwd(cache.lnf, params.final_gain, grad_xf)
    return grad_x.view(cache.shape3), g_gain, g_bias, head_wg[:, :v].contiguous(), head_bg[:v].contiguous()


@dataclass
class SequentialCache:
    embed: EmbedCache
    layers: list
    head: HeadCache
    policy: object = None


def forward(params: Parameters, cfg: ModelConfig, tokens: torch.Tensor, targets=None, policy=None,
            counters=None):
    """model.forward (model.py:583-600): whole-sequence forward on one worker."""
    _check_dropout(cfg, policy)
    x, ec = embed_fwd(params, cfg, tokens, 0, policy)
    caches = []
    for li, lp in enumerate(params.layers):
        x, c = layer_fwd(lp, cfg, policy, li, x, 0, None, counters)
        caches.append(c)
    loss, hc = head_fwd(x, params, targets, cfg)
    return loss, SequentialCache(ec, caches, hc, policy)


def backward(params: Parameters, cfg: ModelConfig, cache: SequentialCache) -> Parameters:
    """model.backward (model.py:603-618): gradients of the mean-over-tokens loss."""
    grad_x, fg, fb, hw, hb = head_bwd(cache.head, params, cfg)
    layer_grads = [None] * len(params.layers)
    for li in range(len(params.layers) - 1, -1, -1):
        grad_x, layer_grads[li] = layer_bwd(params.layers[li], cfg, cache.policy, li, cache.layers[li], grad_x)
    gt, gp = embed_bwd(cache.embed, cfg.vocab, cache.policy, grad_x)
    return Parameters(gt, gp, layer_grads, fg, fb, LinearParams(hw, hb))
