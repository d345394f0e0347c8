"""Sequence-parallel LSS engine on B200 (reference: seqpar/sharded.py).

Two layers of API:

* **The reference's own functions, same signatures** (sharded.py:63-348):
  ``ShardSpec``, ``slice_batch``, ``DistParameters``, ``shard_params``,
  ``forward(comm, group, dist, cfg, tokens_seg, targets_seg, *, policy, step,
  counters, fused)``, ``backward(comm, group, dist, cfg, cache, *, step)``,
  ``sync(comm, group, rank, grads, *, step, extra)``, ``train_step`` and
  ``run_steps``.  ``comm`` is a :mod:`collectives` communicator (worker threads
  on one GPU, or torch.distributed / NCCL, one process per GPU) and every
  array is a torch CUDA tensor; the layer math runs through ``model.layer_fwd``
  / ``layer_bwd`` on the sm_100a kernels.  With ``fused=True`` (the default)
  the kv hooks exchange the packed [K_r | V_r] segments in ONE all-gather per
  layer and the packed fp32 [dK | dV] partials in ONE reduce-scatter (the
  reference's ``fused=False`` arithmetic in one collective per direction,
  SURVEY §0.3); ``fused=False`` is the reference's two-collective ablation.
* **The resident engine** (:mod:`engine`, re-exported here): ``LSSAttention``
  / ``lss_step`` keep every buffer in HBM, fuse the gather into the forward
  attention and the reduce-scatter into the backward kernel's epilogue over
  NVLink, and fold the double gradient averaging into one all-reduce.  This
  is the path bench.py measures.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import model
from ._spec import ShardSpec, slice_batch
from .balance import BalancePlan, block_pairs, choose_fwd_splits, fwd_cta_tiles, make_plan  # noqa: F401
from .comm import Ledger, SimComm, TorchDistComm  # noqa: F401
from .dropout import DropoutPolicy, as_policy
from .engine import (GRAD_NAMES, EngineOptions, LSSAttention, layer_grad_size, lss_backward,  # noqa: F401
                     lss_forward, lss_step, make_sim_group)
from .errors import ShapeError
from .model import ModelConfig, Parameters
from .tensor import StepCounters


@dataclass
class DistParameters:
    """sharded.py:63-70: a worker's parameters -- full replica of everything except
    the position table, of which only the owned rows are present."""

    spec: ShardSpec
    params: Parameters


def shard_params(full: Parameters, spec: ShardSpec) -> DistParameters:
    """sharded.py:73-81: deep copy for one worker with its position rows sliced out."""
    if full.pos_table.shape[0] != spec.seq_len:
        raise ShapeError(f"position table has {full.pos_table.shape[0]} rows, expected {spec.seq_len}")
    p = full.copy()
    p.pos_table = full.pos_table[spec.offset:spec.offset + spec.block].clone()
    return DistParameters(spec=spec, params=p)


@dataclass
class ShardedCache:
    embed: object
    layers: list
    head: object
    policy: DropoutPolicy
    fused: bool


def _kv_hooks(comm, group, wrank, cfg: ModelConfig, step: int, li: int, fused: bool):
    """The kv_fwd / kv_bwd closures of sharded.forward / backward (sharded.py:137-154,
    184-202) for layer ``li``."""
    if fused:
        def kv_fwd(xh, lp):
            # this block's [K_r | V_r], ONE all-gather along the segment dim -> (G, B, m, 2E);
            # model.scores_fwd reads K and V as (G, B, m, E) views of it
            e = xh.shape[-1]
            kv = torch.cat([model.linear3(xh, lp.attn_k, cfg, cfg.act_dtype),
                            model.linear3(xh, lp.attn_v, cfg, cfg.act_dtype)], dim=-1).unsqueeze(0)
            full = comm.all_gather(group, wrank, kv, dim=0, step=step, phase="forward", layer=li)
            return full[..., :e], full[..., e:], xh

        def kv_bwd(kv_ctx, lp, grad_k, grad_v):
            # the packed fp32 [dK | dV] partials over the whole sequence: ONE reduce-scatter
            e = grad_k.shape[-1]
            dkv = torch.cat([grad_k.reshape(-1, *grad_k.shape[-3:]), grad_v.reshape(-1, *grad_v.shape[-3:])], -1)
            own = comm.reduce_scatter(group, wrank, dkv, dim=0, step=step, phase="backward", layer=li)[0]
            gkx, k_wg, k_bg = model.linear3_bwd(kv_ctx, lp.attn_k, own[..., :e].contiguous(), cfg)
            gvx, v_wg, v_bg = model.linear3_bwd(kv_ctx, lp.attn_v, own[..., e:].contiguous(), cfg)
            return gkx + gvx, k_wg, k_bg, v_wg, v_bg
    else:  # the reference's ablation: K and V gathered / reduce-scattered separately
        def kv_fwd(xh, lp):
            k = comm.all_gather(group, wrank, model.linear3(xh, lp.attn_k, cfg, cfg.act_dtype), dim=1, step=step,
                                phase="forward", layer=li)
            v = comm.all_gather(group, wrank, model.linear3(xh, lp.attn_v, cfg, cfg.act_dtype), dim=1, step=step,
                                phase="forward", layer=li)
            return k, v, xh

        def kv_bwd(kv_ctx, lp, grad_k, grad_v):
            gk = comm.reduce_scatter(group, wrank, grad_k.contiguous(), dim=1, step=step, phase="backward", layer=li)
            gv = comm.reduce_scatter(group, wrank, grad_v.contiguous(), dim=1, step=step, phase="backward", layer=li)
            gkx, k_wg, k_bg = model.linear3_bwd(kv_ctx, lp.attn_k, gk, cfg)
            gvx, v_wg, v_bg = model.linear3_bwd(kv_ctx, lp.attn_v, gv, cfg)
            return gkx + gvx, k_wg, k_bg, v_wg, v_bg
    return kv_fwd, kv_bwd


def forward(comm, group, dist: DistParameters, cfg: ModelConfig, tokens_seg, targets_seg, *, policy=None,
            step: int = 0, counters: StepCounters | None = None, fused: bool = True):
    """sharded.forward (sharded.py:113-158): forward over this worker's block;
    returns (partial loss over its own tokens, ShardedCache)."""
    spec, params = dist.spec, dist.params
    wrank = group.members[spec.rank]
    policy = as_policy(policy)
    if tokens_seg.shape[1] != spec.block:
        raise ShapeError(f"token block has {tokens_seg.shape[1]} columns, expected {spec.block}")
    x, e_cache = model.embed_fwd(params, cfg, tokens_seg, spec.offset, policy)
    caches = []
    for li, lp in enumerate(params.layers):
        kv_fwd, _ = _kv_hooks(comm, group, wrank, cfg, step, li, fused)
        x, c = model.layer_fwd(lp, cfg, policy, li, x, spec.offset, kv_fwd, counters)
        caches.append(c)
    partial_loss, h_cache = model.head_fwd(x, params, targets_seg, cfg)
    return partial_loss, ShardedCache(e_cache, caches, h_cache, policy, fused)


def backward(comm, group, dist: DistParameters, cfg: ModelConfig, cache: ShardedCache, *, step: int = 0) -> Parameters:
    """sharded.backward (sharded.py:161-216): gradients of this worker's partial loss,
    one reduce-scatter per layer; position-row gradient divided by the group size."""
    spec, params = dist.spec, dist.params
    wrank = group.members[spec.rank]
    policy = cache.policy
    grad_x, fg, fb, hw, hb = model.head_bwd(cache.head, params, cfg)
    layer_grads = [None] * len(params.layers)
    for li in range(len(params.layers) - 1, -1, -1):
        _, kv_bwd = _kv_hooks(comm, group, wrank, cfg, step, li, cache.fused)
        grad_x, layer_grads[li] = model.layer_bwd(params.layers[li], cfg, policy, li, cache.layers[li], grad_x,
                                                  kv_bwd)
    grad_tok, grad_pe = model.embed_bwd(cache.embed, cfg.vocab, policy, grad_x)
    if group.size > 1:
        grad_pe = grad_pe / group.size
    return Parameters(grad_tok, grad_pe, layer_grads, fg, fb, model.LinearParams(hw, hb))


def sync(comm, group, rank: int, grads: Parameters, *, step: int = 0, extra: float | None = None):
    """sharded.sync (sharded.py:219-244): ONE flat all-reduce-mean of every gradient
    except the position rows, with ``extra`` (the partial loss) riding along."""
    shared = [(n, a) for n, a in grads.named_arrays() if n != "pos_table"]
    vec = model.flatten_arrays([a for _, a in shared])
    if extra is not None:
        vec = torch.cat([vec, torch.tensor([float(extra)], dtype=vec.dtype, device=vec.device)])
    out = comm.all_reduce_mean(group, rank, vec, step=step, phase="sync")
    extra_mean = float(out[-1]) if extra is not None else None
    if extra is not None:
        out = out[:vec.numel() - 1]
    averaged = iter(model.unflatten_like(out, [a for _, a in shared]))
    merged = [a if n == "pos_table" else next(averaged) for n, a in grads.named_arrays()]
    return grads.replace_arrays(merged), extra_mean


def train_step(comm, group, dist: DistParameters, cfg: ModelConfig, tokens_seg, targets_seg, *, lr: float,
               policy=None, step: int = 0, fused: bool = True):
    """sharded.train_step (sharded.py:247-275): forward -> backward -> sync -> SGD;
    returns (group-mean loss, this worker's counters)."""
    counters = StepCounters()
    partial, cache = forward(comm, group, dist, cfg, tokens_seg, targets_seg, policy=policy, step=step,
                             counters=counters, fused=fused)
    grads = backward(comm, group, dist, cfg, cache, step=step)
    grads, mean_loss = sync(comm, group, group.members[dist.spec.rank], grads, step=step, extra=partial)
    dist.params = model.sgd_step(dist.params, grads, lr)
    return mean_loss, counters


@dataclass
class ShardedRun:
    """sharded.ShardedRun (sharded.py:278-287)."""

    comm: object
    workers: list
    step_losses: list
    partial_losses: list
    counters: list
    grad_norms: list
    last_grads: list | None


def run_steps(cfg: ModelConfig, params_full: Parameters, n_workers: int, batches, *, lr: float, policy=None,
              fused: bool = True, keep_last_grads: bool = False, timeout: float = 60.0) -> ShardedRun:
    """sharded.run_steps (sharded.py:289-348) with SGD: ``n_workers`` worker threads
    on the current GPU (collectives.Communicator), each step's dropout policy
    derived as ``policy.at_step(step)``."""
    from .collectives import Communicator, run_workers

    comm = Communicator(n_workers, timeout=timeout)
    group = comm.group("sequence", tuple(range(n_workers)))
    base = as_policy(policy)

    def worker(rank: int):
        spec = ShardSpec(rank, n_workers, cfg.seq_len)
        dist = shard_params(params_full, spec)
        losses, partials, counts, norms, grads_out = [], [], [], [], None
        for s, (tokens, targets) in enumerate(batches):
            pol = base.at_step(s) if base.active else base
            tok, tgt = slice_batch(tokens, spec), slice_batch(targets, spec)
            counters = StepCounters()
            partial, cache = forward(comm, group, dist, cfg, tok, tgt, policy=pol, step=s, counters=counters,
                                     fused=fused)
            grads = backward(comm, group, dist, cfg, cache, step=s)
            grads, mean_loss = sync(comm, group, rank, grads, step=s, extra=partial)
            dist.params = model.sgd_step(dist.params, grads, lr)
            if keep_last_grads and s == len(batches) - 1:
                grads_out = grads
            losses.append(mean_loss)
            partials.append(partial)
            counts.append(counters)
            norms.append(model.grad_norm(grads))
        return dist, losses, partials, counts, norms, grads_out

    res = run_workers(n_workers, worker, comm=comm)
    return ShardedRun(comm, [r[0] for r in res], res[0][1], [r[2] for r in res], [r[3] for r in res],
                      [r[4] for r in res], [r[5] for r in res] if keep_last_grads else None)


__all__ = ["ShardSpec", "slice_batch", "DistParameters", "shard_params", "forward", "backward", "sync", "train_step",
           "run_steps", "ShardedCache", "ShardedRun", "EngineOptions", "LSSAttention", "lss_step", "lss_forward",
           "lss_backward", "make_sim_group", "TorchDistComm", "SimComm", "Ledger", "GRAD_NAMES", "BalancePlan",
           "make_plan"]
