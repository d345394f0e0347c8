"""Tensor-level wrappers over the C ABI (torch is used for device memory and
streams only; every op here runs a liblss.so kernel on the current stream).

Precision names follow the reference's ``ModelConfig.precision``
(model.py:50, tensor.py:24-32): ``"bf16"`` runs the tcgen05 path (bf16
operands, fp32 accumulation); ``"single"`` is the fp32 check mode (FFMA
kernels).  ``"double"`` has no GPU path (fp64 tensor throughput is not a
B200 target) and raises.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native
from ._native import LSS_BF16, LSS_F32, BwdSource, GemmEpilogue, call
from .errors import ShapeError, UnsupportedError

LAYERNORM_EPS = 1e-5  # nnops.py:28

_DT = {"bf16": LSS_BF16, "single": LSS_F32}
_TORCH = {LSS_BF16: torch.bfloat16, LSS_F32: torch.float32}


def code(precision: str) -> int:
    try:
        return _DT[precision]
    except KeyError:
        raise UnsupportedError(f"precision {precision!r} has no B200 path (use 'bf16' or 'single')")


def act_dtype(precision: str) -> torch.dtype:
    return _TORCH[code(precision)]


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need(t: torch.Tensor, name: str, dtype=None):
    if not t.is_cuda:
        raise ShapeError(f"{name} must be a CUDA tensor (no CPU path)")
    if not t.is_contiguous():
        raise ShapeError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ShapeError(f"{name} has dtype {t.dtype}, expected {dtype}")


# ----------------------------------------------------------------- LayerNorm


def layernorm_fwd(x, gain, bias, out=None, out_dtype=torch.bfloat16, eps=LAYERNORM_EPS, mean=None,
                  rstd=None):
    """nnops.layernorm_fwd (nnops.py:199-208) over the last dim.  Returns (y, mean, rstd)."""
    _need(x, "x", torch.float32)
    e = x.shape[-1]
    rows = x.numel() // e
    if gain.shape != (e,) or bias.shape != (e,):
        raise ShapeError(f"layernorm gain/bias {tuple(gain.shape)} do not match embed {e}")
    y = out if out is not None else torch.empty(x.shape, dtype=out_dtype, device=x.device)
    mean = mean if mean is not None else torch.empty(rows, dtype=torch.float32, device=x.device)
    rstd = rstd if rstd is not None else torch.empty(rows, dtype=torch.float32, device=x.device)
    dt = LSS_BF16 if y.dtype == torch.bfloat16 else LSS_F32
    call("lss_layernorm_fwd", _ptr(x), _ptr(gain), _ptr(bias), _ptr(y), dt, _ptr(mean), _ptr(rstd),
         rows, e, eps, _stream())
    return y, mean, rstd


def layernorm_bwd(grad_xh, x, mean, rstd, gain, grad_res=None, grad_x=None, grad_gain=None,
                  grad_bias=None, alpha=1.0):
    """nnops.layernorm_bwd (nnops.py:211-227) + residual (model.py:486).  grad_gain /
    grad_bias are accumulated (+= alpha * sums); pass zeroed buffers for a plain result."""
    _need(grad_xh, "grad_xh", torch.float32)
    _need(x, "x", torch.float32)
    e = x.shape[-1]
    rows = x.numel() // e
    gx = grad_x if grad_x is not None else torch.empty_like(x)
    gg = grad_gain if grad_gain is not None else torch.zeros(e, dtype=torch.float32, device=x.device)
    gb = grad_bias if grad_bias is not None else torch.zeros(e, dtype=torch.float32, device=x.device)
    call("lss_layernorm_bwd", _ptr(grad_xh), _ptr(x), _ptr(mean), _ptr(rstd), _ptr(gain),
         _ptr(grad_res), _ptr(gx), _ptr(gg), _ptr(gb), alpha, rows, e, _stream())
    return gx, gg, gb


# ----------------------------------------------------------------- GEMM


def gemm(a, b, *, a_mn_major=False, b_mn_major=False, out=None, out_dtype=torch.float32, alpha=1.0,
         bias=None, residual=None, seg_width=0, M=None, N=None, K=None, lda=None, ldb=None,
         act=None, pre=None, aux=None):
    """C = act(alpha * A.B^T (+bias) (+residual)) with A [M,K] or (a_mn_major) [K,M],
    B [N,K] or (b_mn_major) [K,N].  ``out`` may be a tensor or a list of up to 3
    (tensor, ld) column segments of ``seg_width`` columns.  ``act``: None,
    "gelu" (tanh GeLU; ``pre`` receives the pre-activation) or "gelu_bwd"
    (multiply by GeLU' of ``aux``, the stored pre-activation)."""
    dt = LSS_BF16 if a.dtype == torch.bfloat16 else LSS_F32
    if b.dtype != a.dtype:
        raise ShapeError("gemm operands must share a dtype")
    if M is None:
        M = a.shape[-1] if a_mn_major else a.numel() // a.shape[-1]
        K = a.numel() // a.shape[-1] if a_mn_major else a.shape[-1]
    if N is None:
        N = b.shape[-1] if b_mn_major else b.numel() // b.shape[-1]
    lda = lda if lda is not None else a.shape[-1]
    ldb = ldb if ldb is not None else b.shape[-1]
    ep = GemmEpilogue()
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype, device=a.device)
    segs = out if isinstance(out, (list, tuple)) else [(out, out.shape[-1])]
    for i, (t, ld) in enumerate(segs):
        ep.out[i] = t.data_ptr()
        ep.ldo[i] = ld
    ep.seg_width = seg_width if seg_width else N
    ep.out_dtype = LSS_BF16 if segs[0][0].dtype == torch.bfloat16 else LSS_F32
    ep.alpha = alpha
    ep.bias = bias.data_ptr() if bias is not None else None
    ep.residual = residual.data_ptr() if residual is not None else None
    ep.ld_res = residual.shape[-1] if residual is not None else 0
    if act is not None:
        codes = {"gelu": _native.ACT_GELU, "gelu_bwd": _native.ACT_GELU_BWD}
        if act not in codes:
            raise ValueError(f"unknown activation {act!r}")
        ep.act = codes[act]
        if pre is not None:
            if pre.dtype != segs[0][0].dtype:
                raise ShapeError("pre-activation buffer must have the output dtype")
            ep.pre, ep.ld_pre = pre.data_ptr(), pre.shape[-1]
        if aux is not None:
            ep.aux, ep.ld_aux = aux.data_ptr(), aux.shape[-1]
            ep.aux_dtype = LSS_BF16 if aux.dtype == torch.bfloat16 else LSS_F32
    call("lss_gemm", dt, _ptr(a), lda, int(a_mn_major), _ptr(b), ldb, int(b_mn_major), M, N, K,
         ctypes.byref(ep), _stream())
    return out


# ----------------------------------------------------------------- weights / casts


def stage_weights(wq, wk, wv, wo, bq, bk, bv, precision="bf16", bufs=None):
    """Stage reference-layout weights ([d_in, d_out]) into the GEMM operand layouts."""
    e = wq.shape[0]
    dt = code(precision)
    tdt = _TORCH[dt]
    dev = wq.device
    if bufs is None:
        bufs = dict(wqkv_t=torch.empty(3 * e, e, dtype=tdt, device=dev),
                    wqkv=torch.empty(e, 3 * e, dtype=tdt, device=dev),
                    wo_t=torch.empty(e, e, dtype=tdt, device=dev),
                    wo=torch.empty(e, e, dtype=tdt, device=dev),
                    bqkv=torch.empty(3 * e, dtype=torch.float32, device=dev))
    call("lss_stage_weights", dt, _ptr(wq), _ptr(wk), _ptr(wv), _ptr(wo), _ptr(bq), _ptr(bk), _ptr(bv),
         _ptr(bufs["wqkv_t"]), _ptr(bufs["wqkv"]), _ptr(bufs["wo_t"]), _ptr(bufs["wo"]),
         _ptr(bufs["bqkv"]), e, _stream())
    return bufs


def cat_cast_colsum(srcs, rows, dst=None, colsum=None, alpha=1.0, out_dtype=torch.bfloat16):
    """srcs: list of (fp32 tensor, ld, cols) or (fp32 tensor, ld, cols, nslots, mask,
    slot_stride): the latter is the ascending sum of the masked slots (slot k at
    tensor + k * slot_stride elements).  Writes the column concatenation into
    ``dst`` (ld = total cols) and accumulates alpha * column sums into ``colsum``."""
    n = len(srcs)
    ptrs = (ctypes.c_void_p * n)(*[s[0].data_ptr() for s in srcs])
    lds = (ctypes.c_long * n)(*[s[1] for s in srcs])
    cols = (ctypes.c_int * n)(*[s[2] for s in srcs])
    total = sum(s[2] for s in srcs)
    dt = LSS_BF16 if (dst is not None and dst.dtype == torch.bfloat16) or (
        dst is None and out_dtype == torch.bfloat16) else LSS_F32
    if all(len(s) == 3 for s in srcs):
        call("lss_cat_cast_colsum", dt, ptrs, lds, cols, n, _ptr(dst), total, _ptr(colsum), alpha, rows,
             _stream())
        return dst, colsum
    ext = [s if len(s) == 6 else (*s, 1, 1, 0) for s in srcs]
    nsl = (ctypes.c_int * n)(*[s[3] for s in ext])
    msk = (ctypes.c_uint * n)(*[s[4] & 0xFFFFFFFF for s in ext])
    sst = (ctypes.c_long * n)(*[s[5] for s in ext])
    call("lss_cat_cast_colsum_ex", dt, ptrs, lds, cols, nsl, msk, sst, n, _ptr(dst), total, _ptr(colsum), alpha,
         rows, _stream())
    return dst, colsum


# ----------------------------------------------------------------- attention


def rows_pad(rows: int) -> int:
    return _native.rows_pad(rows)


def _rows_view(t: torch.Tensor, name: str, workers: int, bsz: int, seg_len: int, e: int) -> int:
    """Validate a [G][B][seg][ld] (or [B][t][ld] when G == 1) row layout with `e`
    visible columns; return the row stride ld in elements."""
    if not t.is_cuda:
        raise ShapeError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dim() == 4:
        if tuple(t.shape) != (workers, bsz, seg_len, e):
            raise ShapeError(f"{name} shape {tuple(t.shape)} != {(workers, bsz, seg_len, e)}")
    elif t.dim() == 3 and workers == 1:
        if tuple(t.shape) != (bsz, seg_len, e):
            raise ShapeError(f"{name} shape {tuple(t.shape)} != {(bsz, seg_len, e)}")
    else:
        raise ShapeError(f"{name} must be [workers, batch, seg, E] (or [batch, t, E] for one segment)")
    ld = t.stride(-2)
    if t.stride(-1) != 1 or ld < e:
        raise ShapeError(f"{name} rows must be contiguous")
    st = t.stride()
    bad_b = bsz > 1 and st[-3] != seg_len * ld
    bad_g = t.dim() == 4 and workers > 1 and st[0] != bsz * seg_len * ld
    if bad_b or bad_g:
        raise ShapeError(f"{name} must be a row-strided view of a [G][B][seg][ld] buffer")
    return ld


def attn_fwd(q, k, v, *, workers, seg_len, heads, offset, causal, out=None, lse2=None):
    """model.scores_fwd core.  q [B,m,E]; k, v [G,B,seg,E] views (same row stride,
    e.g. the two halves of the packed all-gather buffer) or [B,t,E] when G == 1.
    Returns (ctx [B,m,E], lse2 [B,H,m_pad] base-2 log-sum-exp)."""
    _need(q, "q")
    bsz, m, e = q.shape
    if e % heads:
        raise ShapeError(f"embed {e} not divisible by heads {heads}")
    ldk = _rows_view(k, "k", workers, bsz, seg_len, e)
    ldv = _rows_view(v, "v", workers, bsz, seg_len, e)
    if ldk != ldv or k.dtype != q.dtype or v.dtype != q.dtype:
        raise ShapeError("k and v must share dtype and row stride with q's dtype")
    dt = LSS_BF16 if q.dtype == torch.bfloat16 else LSS_F32
    o = out if out is not None else torch.empty_like(q)
    lse = lse2 if lse2 is not None else torch.empty(bsz, heads, rows_pad(m), dtype=torch.float32,
                                                   device=q.device)
    call("lss_attn_fwd", dt, _ptr(q), _ptr(k), _ptr(v), ldk, _ptr(o), _ptr(lse), bsz, m, workers,
         seg_len, heads, e // heads, offset, int(causal), _stream())
    return o, lse


def attn_bwd(q, k, v, o, grad_o, lse2, *, workers, seg_len, heads, offset, causal, grad_q=None,
             grad_k=None, grad_v=None, delta=None):
    """model.scores_bwd core.  Returns (grad_q fp32 [B,m,E], grad_k, grad_v fp32 in the
    [G,B,seg,E] row layout of the given buffers -- allocated packed [G,B,seg,2E]
    (dK | dV halves) when not supplied)."""
    for t, n in ((q, "q"), (o, "o"), (grad_o, "grad_o")):
        _need(t, n, q.dtype)
    bsz, m, e = q.shape
    ldk = _rows_view(k, "k", workers, bsz, seg_len, e)
    if _rows_view(v, "v", workers, bsz, seg_len, e) != ldk:
        raise ShapeError("k and v must share a row stride")
    dt = LSS_BF16 if q.dtype == torch.bfloat16 else LSS_F32
    dev = q.device
    gq = grad_q if grad_q is not None else torch.empty(bsz, m, e, dtype=torch.float32, device=dev)
    if grad_k is None:
        packed = torch.empty(workers, bsz, seg_len, 2 * e, dtype=torch.float32, device=dev)
        grad_k, grad_v = packed[..., :e], packed[..., e:]
    lddkv = grad_k.stride(-2)
    if grad_v.stride(-2) != lddkv or grad_k.dtype != torch.float32:
        raise ShapeError("grad_k / grad_v must be fp32 with a shared row stride")
    dl = delta if delta is not None else torch.empty(bsz, heads, rows_pad(m), dtype=torch.float32,
                                                     device=dev)
    if deterministic() and dt == LSS_BF16:  # fixed-point dQ: bitwise repeatable
        attn_delta(o, grad_o, dl, heads=heads, scaled=True)
        dq64 = torch.zeros(bsz, m, e, dtype=torch.int64, device=dev)
        src = dict(q=q, grad_o=grad_o, grad_q=gq, grad_q_fixed=dq64, row0=0, rows=m, pos0=offset, g_begin=0,
                   g_end=workers, lse2=lse2, delta=dl)
        attn_bwd_sources(k, v, [src], grad_k=grad_k, grad_v=grad_v, workers=workers, seg_len=seg_len, heads=heads,
                         causal=causal)
        fixed_to_f32(gq, dq64)
        return gq, grad_k, grad_v
    call("lss_attn_bwd", dt, _ptr(q), _ptr(k), _ptr(v), ldk, _ptr(o), _ptr(grad_o), _ptr(lse2),
         _ptr(dl), _ptr(gq), _ptr(grad_k), _ptr(grad_v), lddkv, bsz, m, workers, seg_len, heads,
         e // heads, offset, int(causal), _stream())
    return gq, grad_k, grad_v


# ----------------------------------------------------------------- balanced-schedule pieces


def _drop(dropout):
    return ctypes.byref(dropout) if dropout is not None else None


def attn_fwd_partial(q, k, v, *, rows, row0, workers, seg_len, heads, offset, causal, g_begin, g_end, out,
                     lse2, dropout=None, splits=1, scratch=None, ready=None):
    """Partial attention of q rows [row0, row0+rows) (global position offset + row0 for
    the first) over key segments [g_begin, g_end) into out[:, row0:row0+rows] and
    lse2[..., row0:row0+rows] (full-size [B,m,E] / [B,H,m_pad] buffers).

    ``splits`` > 1 splits every CTA's key range inside the launch (lss_attn_fwd_split);
    ``scratch`` = (o_part [S-1, B, m, E] bf16, lse_part [S-1, B, H, m_pad] fp32)
    holds the partials of splits 1..S-1, shaped like out / lse2.  ``ready`` =
    (flags int32 [G] tensor, seq, own segment): fused gather, segment g read after
    flags[g] >= seq (see comm.TorchDistComm.gather_pull)."""
    bsz, m, e = q.shape
    ldk = _rows_view(k, "k", workers, bsz, seg_len, e)
    if _rows_view(v, "v", workers, bsz, seg_len, e) != ldk:
        raise ShapeError("k and v must share a row stride")
    qv = q[:, row0:row0 + rows]
    ov = out[:, row0:row0 + rows]
    lv = lse2[:, :, row0:]
    args = (LSS_BF16, _ptr(qv), rows, m * e, _ptr(k), _ptr(v), ldk, _ptr(ov), m * e, _ptr(lv), lse2.shape[-1], bsz,
            workers, seg_len, heads, e // heads, offset + row0, int(causal), g_begin, g_end, _drop(dropout))
    if splits <= 1 and ready is None:
        call("lss_attn_fwd_ex", *args, _stream())
        return
    rflags, rseq, own = ready if ready is not None else (None, 0, -1)
    if splits > 1:
        op, lp = scratch
        if op.shape[0] < splits - 1 or op.shape[1:] != out.shape or lp.shape[1:] != lse2.shape:
            raise ShapeError(f"attn_fwd_partial: scratch for {splits - 1} partials shaped like out / lse2 required")
        parts = (_ptr(op[0][:, row0:]), op[0].numel(), _ptr(lp[0][:, :, row0:]), lp[0].numel())
    else:
        parts = (None, 0, None, 0)
    if rflags is not None and (rflags.dtype != torch.int32 or rflags.numel() < workers):
        raise ShapeError("attn_fwd_partial: ready flags must be int32 [workers]")
    call("lss_attn_fwd_split", *args, splits, *parts, _ptr(rflags) if rflags is not None else None,
         rseq & 0xFFFFFFFF, own, _stream())


def attn_merge(o_a, lse_a, o_b, lse_b, *, row0, rows, heads, o_out=None, lse_out=None):
    """Combine two partial attentions of rows [row0, row0+rows) (in place into a by default)."""
    bsz, m, e = o_a.shape
    o_out = o_a if o_out is None else o_out
    lse_out = lse_a if lse_out is None else lse_out
    sl = lambda t: t[:, row0:]  # noqa: E731
    call("lss_attn_merge", _ptr(sl(o_a)), _ptr(lse_a[:, :, row0:]), _ptr(sl(o_b)), _ptr(lse_b[:, :, row0:]),
         _ptr(sl(o_out)), _ptr(lse_out[:, :, row0:]), bsz, rows, heads, m * e, lse_a.shape[-1], _stream())


def attn_delta(o, grad_o, delta, *, heads, scaled=True):
    bsz, m, e = o.shape
    dt = LSS_BF16 if o.dtype == torch.bfloat16 else LSS_F32
    call("lss_attn_delta", dt, _ptr(o), _ptr(grad_o), _ptr(delta), bsz, m, heads, e // heads, int(scaled),
         _stream())


def _bwd_source_array(sources):
    arr = (BwdSource * len(sources))()
    for i, src in enumerate(sources):
        q = src["q"]
        arr[i].q = q.data_ptr()
        arr[i].grad_o = src["grad_o"].data_ptr()
        arr[i].grad_q = src["grad_q"].data_ptr()
        arr[i].m_src = q.shape[1]
        arr[i].row0 = src["row0"]
        arr[i].rows = src["rows"]
        arr[i].pos0 = src["pos0"]
        arr[i].g_begin = src["g_begin"]
        arr[i].g_end = src["g_end"]
        arr[i].lse2 = src["lse2"].data_ptr()
        arr[i].delta = src["delta"].data_ptr()
        arr[i].pitch = src["lse2"].shape[-1]
        fx = src.get("grad_q_fixed")  # deterministic mode: int64 fixed-point dQ accumulator
        if fx is not None:
            if fx.dtype != torch.int64 or tuple(fx.shape) != tuple(src["grad_q"].shape):
                raise ShapeError("grad_q_fixed must be int64 shaped like grad_q")
            arr[i].grad_q_fixed = fx.data_ptr()
        ready = src.get("ready")  # (flag address, seq): inputs pushed by a partner
        if ready is not None:
            arr[i].ready = int(ready[0])
            arr[i].ready_seq = ready[1] & 0xFFFFFFFF
    return arr


def attn_bwd_sources(k, v, sources, *, grad_k=None, grad_v=None, seg_dst=None, peer=False, ld_dkv=None,
                     workers, seg_len, heads, causal, dropout=None):
    """Multi-source backward.  sources: dicts with q, grad_o, grad_q (fp32, pre-zeroed),
    row0, rows, pos0 (global position of tensor row 0), g_begin, g_end, lse2, delta.

    dK|dV go either to grad_k / grad_v ([G][B][seg][ld] local, the reduce-scatter
    input) or, with ``seg_dst`` (G device addresses of [B][seg][ld_dkv] fp32 blocks,
    dV at +E; ``peer`` when they are NVLink peer memory), straight to each key
    segment's owner: the fused reduce-scatter (lss_attn_bwd_p2p)."""
    q0 = sources[0]["q"]
    bsz, _, e = q0.shape
    ldk = _rows_view(k, "k", workers, bsz, seg_len, e)
    arr = _bwd_source_array(sources)
    if seg_dst is not None:
        if len(seg_dst) != workers:
            raise ShapeError(f"seg_dst has {len(seg_dst)} entries for {workers} workers")
        tab = (ctypes.c_void_p * workers)(*[int(a) for a in seg_dst])
        call("lss_attn_bwd_p2p", LSS_BF16, _ptr(k), _ptr(v), ldk, arr, len(sources), tab, int(peer),
             int(ld_dkv if ld_dkv is not None else 2 * e), bsz, workers, seg_len, heads, e // heads, int(causal),
             _drop(dropout), _stream())
        return
    call("lss_attn_bwd_ex", LSS_BF16, _ptr(k), _ptr(v), ldk, arr, len(sources), _ptr(grad_k), _ptr(grad_v),
         grad_k.stride(-2), bsz, workers, seg_len, heads, e // heads, int(causal), _drop(dropout), _stream())


def dropout_rows(x, out, *, rows_per_sample, offset, site_key, thresh, scale, residual=None):
    """nnops.dropout_fwd / dropout_bwd on a (rows, cols) activation (row r = sample
    r // rows_per_sample at position offset + r % rows_per_sample): out = x * keep *
    scale (+ residual).  x / out same dtype (bf16 or fp32), may alias."""
    cols = x.shape[-1]
    rows = x.numel() // cols
    if out.dtype != x.dtype or out.numel() != x.numel():
        raise ShapeError("dropout_rows: out must match x")
    dt = LSS_BF16 if x.dtype == torch.bfloat16 else LSS_F32
    call("lss_dropout_rows", dt, _ptr(x), cols, _ptr(out), cols, _ptr(residual),
         residual.shape[-1] if residual is not None else 0, rows, cols, rows_per_sample, offset, site_key, thresh,
         scale, _stream())
    return out


def stream_signal(flag_addr: int, value: int, stream=None) -> None:
    """Stream-ordered write of value to the (possibly peer-mapped) flag word."""
    s = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    call("lss_stream_signal", ctypes.c_void_p(int(flag_addr)), value & 0xFFFFFFFF, s)


def stream_wait(flag_addr: int, value: int, stream=None) -> None:
    """Block the stream until the flag word reaches value (wrap-safe >=)."""
    s = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    call("lss_stream_wait", ctypes.c_void_p(int(flag_addr)), value & 0xFFFFFFFF, s)


def stream_wait_bounded(flags_addr: int, count: int, skip: int, value: int, stream=None) -> None:
    """Block the stream until every one of ``count`` consecutive flag words (except index
    ``skip``) reaches value -- a one-warp spin kernel with the runtime deadline and the
    host abort word (the front-end stream_wait cannot time out)."""
    s = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    call("lss_stream_wait_bounded", ctypes.c_void_p(int(flags_addr)), int(count), int(skip), value & 0xFFFFFFFF, s)


def stream_wait_guarded(flags_addr: int, count: int, skip: int, value: int, stream=None) -> None:
    """Front-end waits (no SM, released as soon as the flags land) plus a one-warp guard
    kernel on a private high-priority stream that, past the deadline or on a host abort,
    raises the status word and writes the flags itself so the stream drains."""
    s = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    call("lss_stream_wait_guarded", ctypes.c_void_p(int(flags_addr)), int(count), int(skip), value & 0xFFFFFFFF, s)


def abort_waits(on: bool = True) -> None:
    """Host-side abort: every bounded wait (stream or in-kernel) returns at once while set."""
    call("lss_abort_waits", int(bool(on)))


def timestamp(dst):
    """Diagnostic: write the GPU global timer (ns) into the int64 scalar view dst."""
    call("lss_timestamp", _ptr(dst), _stream())


def sum_slots(dst, src, mask=None):
    """dst = src.sum(0) for src [S, ...] fp32 contiguous (the owner's half of the fused
    reduce-scatter); with ``mask`` only the slots whose bit is set (ascending)."""
    if not src.is_contiguous() or not dst.is_contiguous() or src[0].numel() != dst.numel():
        raise ShapeError("sum_slots: contiguous src [S, *dst.shape] required")
    if mask is None:
        call("lss_sum_slots", _ptr(dst), _ptr(src), src.shape[0], src[0].numel(), dst.numel(), _stream())
    else:
        call("lss_sum_slots_mask", _ptr(dst), _ptr(src), src.shape[0], int(mask) & 0xFFFFFFFF, src[0].numel(),
             dst.numel(), _stream())
    return dst


def embed_fwd(tokens, token_table, pos_table, out=None):
    """model.embed_fwd (model.py:517-533), dropout 0: token rows + this block's positions."""
    _need(tokens, "tokens", torch.int32)
    _need(token_table, "token_table", torch.float32)
    _need(pos_table, "pos_table", torch.float32)
    b, m = tokens.shape
    e = token_table.shape[1]
    if pos_table.shape != (m, e):
        raise ShapeError(f"position table has {pos_table.shape[0]} rows, block has {m}")
    x = out if out is not None else torch.empty(b, m, e, dtype=torch.float32, device=tokens.device)
    call("lss_embed_fwd", _ptr(tokens), _ptr(token_table), _ptr(pos_table), _ptr(x), b, m, e, _stream())
    return x


def embed_bwd(tokens, grad_x, vocab, *, grad_token=None, grad_pos=None, alpha_token=1.0, alpha_pos=1.0):
    """model.embed_bwd (model.py:536-540) -> (grad_token_table (accumulated), grad_pos_table)."""
    _need(tokens, "tokens", torch.int32)
    _need(grad_x, "grad_x", torch.float32)
    b, m, e = grad_x.shape
    gt = grad_token if grad_token is not None else torch.zeros(vocab, e, dtype=torch.float32, device=grad_x.device)
    gp = grad_pos if grad_pos is not None else torch.empty(m, e, dtype=torch.float32, device=grad_x.device)
    call("lss_embed_bwd", _ptr(tokens), _ptr(grad_x), _ptr(gt), _ptr(gp), b, m, e, alpha_token, alpha_pos,
         _stream())
    return gt, gp


def cross_entropy(logits, targets, vocab, *, scale, grad=True):
    """nnops.cross_entropy (nnops.py:274-299) on logits [n][ld >= vocab]: per-row
    losses and (optionally) grad = (softmax - onehot) * scale, padded columns zero."""
    _need(logits, "logits", torch.float32)
    _need(targets, "targets", torch.int32)
    n, ld = logits.shape
    loss_rows = torch.empty(n, dtype=torch.float32, device=logits.device)
    g = torch.empty(n, ld, dtype=torch.float32, device=logits.device) if grad else None
    call("lss_cross_entropy", _ptr(logits), ld, _ptr(targets), n, vocab, scale, _ptr(loss_rows), _ptr(g),
         ld, _stream())
    return loss_rows, g


def sgd_update(params, grads, lr):
    """params -= lr * grads (flat fp32, in place): model.sgd_step (model.py:621-623)."""
    _need(params, "params", torch.float32)
    _need(grads, "grads", torch.float32)
    if params.numel() != grads.numel():
        raise ShapeError("sgd_update: params / grads sizes differ")
    call("lss_sgd_update", _ptr(params), _ptr(grads), params.numel(), lr, _stream())


def adam_update(params, grads, m, v, *, lr, step, beta1=0.9, beta2=0.999, eps=1e-8):
    """Bias-corrected Adam in place (optim.adam_step, optim.py:35-53); step is 1-based."""
    for t, n in ((params, "params"), (grads, "grads"), (m, "m"), (v, "v")):
        _need(t, n, torch.float32)
        if t.numel() != params.numel():
            raise ShapeError(f"adam_update: {n} size differs")
    call("lss_adam_update", _ptr(params), _ptr(grads), _ptr(m), _ptr(v), params.numel(), lr, beta1, beta2, eps,
         step, _stream())


def ipc_export(t):
    """(64-byte handle, offset) of a device tensor's memory for another process."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_long(0)
    call("lss_ipc_export", _ptr(t), h, ctypes.byref(off))
    return h.raw, off.value


def ipc_import(handle: bytes, offset: int) -> int:
    """Device address (int) of a peer process's exported memory."""
    p = ctypes.c_void_p(0)
    call("lss_ipc_import", handle, offset, ctypes.byref(p))
    return p.value


def ipc_close(addr: int, offset: int) -> None:
    call("lss_ipc_close", ctypes.c_void_p(addr), offset)


def copy_d2d(dst_addr: int, src_addr: int, nbytes: int, stream=None) -> None:
    """Copy-engine D2D copy (src may be IPC-mapped peer memory), stream-ordered."""
    s = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    call("lss_copy_d2d", ctypes.c_void_p(int(dst_addr)), ctypes.c_void_p(int(src_addr)), int(nbytes), s)


def peer_access(device: int, peer: int) -> bool:
    return bool(_native.load().lss_peer_access(device, peer))


def add_(y, x):
    """y += x (fp32, device)."""
    call("lss_add_f32", _ptr(y), _ptr(x), y.numel(), _stream())
    return y


# ----------------------------------------------------------------- failure semantics (ABI v9)

_RUNTIME = {"wait_timeout_s": 60.0, "numerics": False, "deterministic": False}
_CONFIGURED: set = set()


def runtime_config(*, wait_timeout_s: float | None = None, numerics: bool | None = None,
                   deterministic: bool | None = None, device=None) -> None:
    """Deadline of every in-kernel cross-GPU wait (seconds, 0 = unbounded; the
    reference Communicator's default timeout is 60 s, collectives.py:159), the
    opt-in NaN / Inf check in the GEMM / attention epilogues (tensor.py:79-95) and
    the deterministic mode (fixed-point dQ, column sums without atomics: bitwise
    repeatable runs, collectives.py:5-7).  Applies to ``device`` (default: current)
    now and to every device configured later."""
    if wait_timeout_s is not None:
        _RUNTIME["wait_timeout_s"] = float(wait_timeout_s)
    if numerics is not None:
        _RUNTIME["numerics"] = bool(numerics)
    if deterministic is not None:
        _RUNTIME["deterministic"] = bool(deterministic)
    _CONFIGURED.clear()
    ensure_runtime(device)


def ensure_runtime(device=None) -> None:
    """Push the runtime configuration to ``device`` once (device globals are per GPU)."""
    d = torch.cuda.current_device() if device is None else torch.device(device).index
    if d is None:
        d = torch.cuda.current_device()
    if d in _CONFIGURED:
        return
    flags = (1 if _RUNTIME["numerics"] else 0) | (2 if _RUNTIME["deterministic"] else 0)
    with torch.cuda.device(d):
        call("lss_runtime_config", int(_RUNTIME["wait_timeout_s"] * 1e9), flags)
    _CONFIGURED.add(d)


def numerics_enabled() -> bool:
    return _RUNTIME["numerics"]


def deterministic() -> bool:
    return _RUNTIME["deterministic"]


def fixed_to_f32(dst: torch.Tensor, src: torch.Tensor, accumulate: bool = False) -> torch.Tensor:
    """dst (=, or += ) src * 2^-32: the int64 fixed-point dQ of the deterministic backward."""
    _need(dst, "dst", torch.float32)
    _need(src, "src", torch.int64)
    if dst.numel() != src.numel():
        raise ShapeError("fixed_to_f32: sizes differ")
    call("lss_fixed_to_f32", _ptr(dst), _ptr(src), dst.numel(), int(accumulate), _stream())
    return dst


def status(clear: bool = False) -> tuple:
    """(comm_timeout, nonfinite) reported by the kernels since the last clear (mapped
    host memory: no device synchronisation; meaningful once the work completed)."""
    out = (ctypes.c_uint * 2)()
    call("lss_status", out, int(clear))
    return bool(out[0]), bool(out[1])


def raise_status(clear: bool = True) -> None:
    """Raise CommTimeout / NumericsError for what the kernels reported."""
    from .errors import CommTimeout, NumericsError

    timed_out, nonfinite = status(clear)
    if timed_out:
        raise CommTimeout("a cross-GPU wait ran past its deadline (a peer is dead or out of step); "
                          "the results of that step are void")
    if nonfinite:
        raise NumericsError("a kernel produced NaN or Inf")


def check_finite(t: torch.Tensor) -> None:
    """Report (status word 1) NaN / Inf anywhere in a contiguous fp32 / bf16 tensor."""
    _need(t, "tensor")
    dt = LSS_BF16 if t.dtype == torch.bfloat16 else LSS_F32
    if t.dtype not in (torch.bfloat16, torch.float32):
        raise ShapeError(f"check_finite: dtype {t.dtype}")
    call("lss_check_finite", _ptr(t), t.numel(), dt, _stream())


def checked(*tensors):
    """With the numerics check on: every kernel output checked for NaN / Inf before it
    is returned (the reference checks every matmul / softmax output, tensor.py:79-95)
    -- synchronises, so it is a debugging mode.  Returns the first tensor."""
    if _RUNTIME["numerics"]:
        ensure_runtime()
        for t in tensors:
            if t is not None and t.is_contiguous() and t.dtype in (torch.float32, torch.bfloat16) and \
                    t.numel() % (8 if t.dtype == torch.bfloat16 else 4) == 0:
                check_finite(t)
        torch.cuda.current_stream().synchronize()
        raise_status()
    return tensors[0] if tensors else None


def flag_release(addr: int, count: int, value: int) -> None:
    """Write ``value`` to ``count`` flag words from a private non-blocking stream."""
    call("lss_flag_release", ctypes.c_void_p(int(addr)), int(count), value & 0xFFFFFFFF)
