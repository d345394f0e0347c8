"""The reference-side binding of INTEGRATION.md §1, as code.

``patch_reference(seqpar.model)`` routes the reference's attention core --
``model.scores_fwd`` / ``model.scores_bwd`` (model.py:280-359), the functions its
``layer_fwd`` / ``layer_bwd`` call through module globals (model.py:445, 481) --
to the B200 kernels, while every other reference function (LayerNorm, the
projections, the sharded engines, the communicator) keeps running in numpy.  It
is the one-line swap a maintainer of the reference would make to put the hot
loop of its layer on the GPU; ``tests/test_gpu_integration.py`` runs the
reference's own layer and engines through it.

Arrays cross the boundary as host numpy <-> torch CUDA copies (the reference is a
host program); the ScoreCache the reference threads from forward to backward
holds the B200 cache (ctx + log-sum-exp, not the full probability matrix).
"""

from __future__ import annotations

import numpy as np
import torch

from . import model as M


def patch_reference(ref_model, precision: str = "bf16", device="cuda"):
    """Replace ``ref_model.scores_fwd / scores_bwd`` (a ``seqpar.model`` module) with
    the B200 path in ``precision`` ("bf16" tcgen05 or "single" fp32 check mode).
    Returns a function that restores the originals."""
    orig_fwd, orig_bwd = ref_model.scores_fwd, ref_model.scores_bwd
    dev = torch.device(device)

    def t(a):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32, device=dev)

    def b200_cfg(cfg):
        return M.ModelConfig(**{**cfg.to_dict(), "precision": precision})

    def scores_fwd(q, k, v, offset, cfg, policy, layer, counters=None):
        bcfg = b200_cfg(cfg)
        ctx, cache = M.scores_fwd(t(q), t(k), t(v), offset, bcfg, policy, layer, counters)
        return ctx.float().cpu().numpy().astype(q.dtype), (cache, bcfg)

    def scores_bwd(cache, q, k, v, grad_ctx, cfg, policy):
        sc, bcfg = cache
        dq, dk, dv = M.scores_bwd(sc, t(q), t(k), t(v), t(grad_ctx), bcfg, policy)
        return tuple(a.float().cpu().numpy().astype(q.dtype) for a in (dq, dk, dv))

    ref_model.scores_fwd, ref_model.scores_bwd = scores_fwd, scores_bwd

    def restore():
        ref_model.scores_fwd, ref_model.scores_bwd = orig_fwd, orig_bwd

    return restore
