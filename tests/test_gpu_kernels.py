"""Kernel-level parity on the B200: every liblss.so entry point against the CPU
oracle (oracle/lss_oracle.py, pinned to the reference) or, for plain GEMMs,
against an fp32 matmul of the same (bf16-rounded) operands.

Tolerances (normalized max|a-b|/max|b|): bf16 operands with
fp32 accumulation <= 1e-2 (north star); fp32 check mode <= 1e-4.
"""

import numpy as np
import pytest

from conftest import nerr
from oracle import lss_oracle as O

pytestmark = pytest.mark.gpu

BF16_TOL = 1e-2
F32_TOL = 1e-4


def _t(a, dev, dtype):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32, device=dev).to(dtype)


def _np(t):
    import torch

    return t.detach().to(torch.float32).cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("prec", ["bf16", "single"])
def test_gemm_layouts_and_epilogue(cuda, rng, a_mn, b_mn, prec):
    import torch
    from paper_2311_02382_b200 import kernels as K

    M, N, Kd = 296, 512, 200
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    a = rng.standard_normal((M, Kd))
    b = rng.standard_normal((N, Kd))
    ta = _t(a.T if a_mn else a, cuda, dt).contiguous()
    tb = _t(b.T if b_mn else b, cuda, dt).contiguous()
    an = _np(ta).T if a_mn else _np(ta)
    bn = _np(tb).T if b_mn else _np(tb)
    bias = rng.standard_normal(N)
    res = rng.standard_normal((M, N))
    want = 0.5 * an @ bn.T + bias + res
    out = K.gemm(ta, tb, a_mn_major=a_mn, b_mn_major=b_mn, alpha=0.5,
                 bias=_t(bias, cuda, torch.float32), residual=_t(res, cuda, torch.float32),
                 M=M, N=N, K=Kd)
    torch.cuda.synchronize()
    assert nerr(_np(out), want) < 1e-5


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", [(1024, 768, 4096), (1000, 544, 2056)])
def test_gemm_cta_pair(cuda, rng, a_mn, b_mn, shape):
    """The CTA-pair (cta_group::2, 256 x 256) kernel that long-K products use
    (M >= 512, K >= 2048), incl. ragged M / N / K and both operand layouts,
    against the fp64 product of the same bf16 operands."""
    import torch
    from paper_2311_02382_b200 import kernels as K

    M, N, Kd = shape
    a = rng.standard_normal((M, Kd))
    b = rng.standard_normal((N, Kd))
    ta = _t(a.T if a_mn else a, cuda, torch.bfloat16).contiguous()
    tb = _t(b.T if b_mn else b, cuda, torch.bfloat16).contiguous()
    an = _np(ta).T if a_mn else _np(ta)
    bn = _np(tb).T if b_mn else _np(tb)
    bias = rng.standard_normal(N)
    res = rng.standard_normal((M, N))
    want = 0.25 * an @ bn.T + bias + res
    out = K.gemm(ta, tb, a_mn_major=a_mn, b_mn_major=b_mn, alpha=0.25,
                 bias=_t(bias, cuda, torch.float32), residual=_t(res, cuda, torch.float32),
                 M=M, N=N, K=Kd)
    torch.cuda.synchronize()
    assert nerr(_np(out), want) < 1e-5


def test_gemm_split_bf16_segments(cuda, rng):
    """QKV projection epilogue: one GEMM writes Q to one buffer and K|V to another."""
    import torch
    from paper_2311_02382_b200 import kernels as K

    M, E = 200, 128
    x = _t(rng.standard_normal((M, E)), cuda, torch.bfloat16)
    w = _t(rng.standard_normal((3 * E, E)) / np.sqrt(E), cuda, torch.bfloat16)
    q = torch.empty(M, E, dtype=torch.bfloat16, device=cuda)
    kv = torch.empty(M, 2 * E, dtype=torch.bfloat16, device=cuda)
    K.gemm(x, w, out=[(q, E), (kv[:, :E], 2 * E), (kv[:, E:], 2 * E)], seg_width=E)
    torch.cuda.synchronize()
    want = _np(x) @ _np(w).T
    assert nerr(_np(q), want[:, :E]) < 1e-2
    assert nerr(_np(kv), want[:, E:]) < 1e-2


def test_layernorm_fwd_bwd(cuda, rng):
    import torch
    from paper_2311_02382_b200 import kernels as K

    rows, E = 77, 256
    x = rng.standard_normal((rows, E)) * 3 + 1
    g = 1 + 0.1 * rng.standard_normal(E)
    bb = 0.1 * rng.standard_normal(E)
    gy = rng.standard_normal((rows, E))
    res = rng.standard_normal((rows, E))
    tx = _t(x, cuda, torch.float32)
    y, mu, rs = K.layernorm_fwd(tx, _t(g, cuda, torch.float32), _t(bb, cuda, torch.float32),
                                out_dtype=torch.float32)
    gx, gg, gb = K.layernorm_bwd(_t(gy, cuda, torch.float32), tx, mu, rs, _t(g, cuda, torch.float32),
                                 grad_res=_t(res, cuda, torch.float32))
    torch.cuda.synchronize()
    y_ref, cache = O.layernorm_fwd(x, g, bb)
    gx_ref, gg_ref, gb_ref = O.layernorm_bwd(cache, g, gy)
    assert nerr(_np(y), y_ref) < 1e-5
    assert nerr(_np(gx), gx_ref + res) < 1e-5
    assert nerr(_np(gg), gg_ref) < 1e-5
    assert nerr(_np(gb), gb_ref) < 1e-5


ATTN_CASES = [
    # (batch, rows m, workers G, heads, rank, causal)
    (1, 300, 2, 2, 1, True),
    (1, 300, 2, 2, 0, True),
    (1, 256, 2, 2, 1, False),
    (2, 136, 3, 1, 2, True),
    (1, 520, 1, 2, 0, True),
]


def _attn_inputs(rng, bsz, m, G, H, rank, dev, dt, scale=1.0):
    E = 64 * H
    seq = m * G
    q = rng.standard_normal((bsz, m, E)) * scale
    k = rng.standard_normal((bsz, seq, E)) * scale
    v = rng.standard_normal((bsz, seq, E))
    tq = _t(q, dev, dt)
    kv = np.concatenate([k.reshape(bsz, G, m, E), v.reshape(bsz, G, m, E)], axis=-1).transpose(1, 0, 2, 3)
    tkv = _t(kv, dev, dt).contiguous()
    qn = _np(tq)
    kvn = _np(tkv)  # [G,B,m,2E]
    kn = kvn[..., :E].transpose(1, 0, 2, 3).reshape(bsz, seq, E)
    vn = kvn[..., E:].transpose(1, 0, 2, 3).reshape(bsz, seq, E)
    return tq, tkv, qn, kn, vn


@pytest.mark.parametrize("case", ATTN_CASES)
@pytest.mark.parametrize("prec", ["bf16", "single"])
def test_attention_fwd_bwd_vs_oracle(cuda, rng, case, prec):
    import torch
    from paper_2311_02382_b200 import kernels as K

    bsz, m, G, H, rank, causal = case
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    tol = BF16_TOL if prec == "bf16" else F32_TOL
    E = 64 * H
    tq, tkv, qn, kn, vn = _attn_inputs(rng, bsz, m, G, H, rank, cuda, dt)
    offset = rank * m
    o, lse = K.attn_fwd(tq, tkv[..., :E], tkv[..., E:], workers=G, seg_len=m, heads=H, offset=offset,
                        causal=causal)
    torch.cuda.synchronize()
    ctx_ref, p_ref = O.scores_fwd(qn, kn, vn, offset, H, causal)
    assert nerr(_np(o), ctx_ref) < tol
    # lse (base 2) of the scaled scores
    s = np.einsum("bhid,bhjd->bhij", qn.reshape(bsz, m, H, 64).transpose(0, 2, 1, 3),
                  kn.reshape(bsz, -1, H, 64).transpose(0, 2, 1, 3)) / 8.0
    if causal:
        s = np.where(O.causal_keep(m, G * m, offset), s, -np.inf)
    mx = s.max(-1, keepdims=True)
    lse_ref = (np.log(np.exp(s - mx).sum(-1)) + mx[..., 0]) / np.log(2)
    assert np.abs(_np(lse)[:, :, :m] - lse_ref).max() < (2e-2 if prec == "bf16" else 1e-4)
    # backward
    go = rng.standard_normal((bsz, m, E))
    tgo = _t(go, cuda, dt)
    gq, gk, gv = K.attn_bwd(tq, tkv[..., :E], tkv[..., E:], o, tgo, lse, workers=G, seg_len=m, heads=H,
                            offset=offset, causal=causal)
    torch.cuda.synchronize()
    dq_ref, dk_ref, dv_ref = O.scores_bwd(p_ref, qn, kn, vn, _np(tgo), H)
    dk = _np(gk).transpose(1, 0, 2, 3).reshape(bsz, -1, E)
    dv = _np(gv).transpose(1, 0, 2, 3).reshape(bsz, -1, E)
    btol = 2 * tol
    assert nerr(_np(gq), dq_ref) < btol
    assert nerr(dk, dk_ref) < btol
    assert nerr(dv, dv_ref) < btol


SPLIT_CASES = [
    # (batch, rows m, workers G, heads, rank, row0, rows, g_begin, g_end, splits)
    (1, 700, 4, 2, 3, 0, 700, 0, 3, 3),    # dense remote segments (the N>=4 case)
    (1, 700, 4, 2, 3, 0, 700, 1, 4, 5),    # ends in the diagonal segment
    (2, 300, 3, 2, 2, 128, 172, 0, 3, 4),  # row window, batch 2, ragged tiles
    (1, 520, 2, 1, 0, 0, 520, 0, 1, 6),    # causal diagonal: short CTAs, empty splits
]


@pytest.mark.parametrize("case", SPLIT_CASES)
@pytest.mark.parametrize("drop", [False, True])
def test_attention_fwd_key_split(cuda, rng, case, drop):
    """lss_attn_fwd_split (key range split inside one launch + N-way lse merge) ==
    the unsplit partial launch, and == the oracle over the same key range."""
    import torch
    from paper_2311_02382_b200 import kernels as K
    from paper_2311_02382_b200.dropout import DropoutPolicy

    bsz, m, G, H, rank, row0, rows, g0, g1, S = case
    E = 64 * H
    tq, tkv, qn, kn, vn = _attn_inputs(rng, bsz, m, G, H, rank, cuda, torch.bfloat16)
    mp = K.rows_pad(m)
    dd = DropoutPolicy(0.2, seed=5).desc(0) if drop else None
    outs = []
    for splits in (1, S):
        o = torch.zeros(bsz, m, E, dtype=torch.bfloat16, device=cuda)
        lse = torch.zeros(bsz, H, mp, device=cuda)
        scratch = (torch.full((S - 1, bsz, m, E), float("nan"), dtype=torch.bfloat16, device=cuda),
                   torch.full((S - 1, bsz, H, mp), float("nan"), device=cuda))
        K.attn_fwd_partial(tq, tkv[..., :E], tkv[..., E:], rows=rows, row0=row0, workers=G, seg_len=m, heads=H,
                           offset=rank * m, causal=True, g_begin=g0, g_end=g1, out=o, lse2=lse, dropout=dd,
                           splits=splits, scratch=scratch)
        torch.cuda.synchronize()
        outs.append((_np(o)[:, row0:row0 + rows], _np(lse)[:, :, row0:row0 + rows]))
    (o1, l1), (os_, ls) = outs
    assert np.isfinite(os_).all()
    assert nerr(os_, o1) < BF16_TOL
    assert np.abs(ls - l1).max() < 1e-3
    if not drop:  # oracle over keys [g0*m, g1*m): causal offset relative to the first key
        ctx_ref, _ = O.scores_fwd(qn[:, row0:row0 + rows], kn[:, g0 * m:g1 * m], vn[:, g0 * m:g1 * m],
                                  rank * m + row0 - g0 * m, H, True)
        assert nerr(os_, ctx_ref) < BF16_TOL


def test_attention_peaked_softmax_bf16(cuda, rng):
    """Stress variant of SURVEY.md §8(d): scores scaled up so the online max moves a lot."""
    import torch
    from paper_2311_02382_b200 import kernels as K

    bsz, m, G, H = 1, 384, 2, 1
    tq, tkv, qn, kn, vn = _attn_inputs(rng, bsz, m, G, H, 1, cuda, torch.bfloat16, scale=3.0)
    o, lse = K.attn_fwd(tq, tkv[..., :64], tkv[..., 64:], workers=G, seg_len=m, heads=H, offset=m,
                        causal=True)
    torch.cuda.synchronize()
    ctx_ref, _ = O.scores_fwd(qn, kn, vn, m, H, True)
    assert nerr(_np(o), ctx_ref) < BF16_TOL


def test_attention_rejects_unsupported_head_dim(cuda):
    import torch
    from paper_2311_02382_b200 import kernels as K
    from paper_2311_02382_b200.errors import UnsupportedError

    q = torch.zeros(1, 16, 96, dtype=torch.bfloat16, device=cuda)  # d = 32 with 3 heads
    kv = torch.zeros(1, 1, 16, 192, dtype=torch.bfloat16, device=cuda)
    with pytest.raises(UnsupportedError):
        K.attn_fwd(q, kv[..., :96], kv[..., 96:], workers=1, seg_len=16, heads=3, offset=0, causal=True)
