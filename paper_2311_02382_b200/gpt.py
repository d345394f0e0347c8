"""Sequence-distributed decoder: the reference's whole-model path on B200 engines.

Reference: sharded.forward / sharded.backward / sharded.sync (sharded.py:90-244)
and hybrid.train_step (hybrid.py:95-126) for the GPT of model.py:497-618
(SURVEY §8(f) rows f2 and f4).  One :class:`GPTRank` per GPU holds

  * the token-embedding table (replica) and THIS rank's rows of the position
    table (model.embed_fwd, model.py:517-533);
  * ``cfg.n_layers`` complete-layer LSS engines (attention half with the packed
    K/V all-gather and the fused dK|dV reduce-scatter, plus the LN2 / FFN half);
  * the final LayerNorm, the vocabulary head (padded to 32 columns for the
    tcgen05 GEMM) and the fused cross-entropy over this rank's tokens.

Gradient sync keeps the reference's arithmetic with ONE world all-reduce: every
gradient except the position rows lives in one flat buffer, pre-scaled by
1/(D*N) in the kernels that write it (the layer engines' alpha, the head and
embedding alphas), and this rank's partial loss rides along as the trailing
element (sharded.sync's ``extra``).  The position rows stay local with the
reference's /N (sharded.py:207-208) and are averaged over the data group when
D > 1 (hybrid.vertical_sync, hybrid.py:76-92).
"""

from __future__ import annotations

import torch

from . import kernels as K
from .comm import SimComm
from .errors import ShapeError
from .model import LinearParams, ModelConfig, Parameters
from .sharded import LSSAttention, ShardSpec, layer_grad_size, lss_backward, lss_forward


def _pad16(n: int) -> int:
    return (n + 15) // 16 * 16


class GPTRank:
    """One rank of the sequence-distributed decoder (replicas x seq_workers grid)."""

    def __init__(self, cfg: ModelConfig, spec: ShardSpec, *, replicas: int = 1, device=None,
                 balanced: bool | None = None, fused_rs: bool | None = None):
        if spec.seq_len != cfg.seq_len:
            raise ShapeError(f"shard spec length {spec.seq_len} != config seq_len {cfg.seq_len}")
        self.cfg, self.spec, self.replicas = cfg, spec, replicas
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        dev, f32 = self.device, torch.float32
        L, E, V, B, m = cfg.n_layers, cfg.embed_dim, cfg.vocab, cfg.batch, spec.block
        self.B, self.m, self.E, self.V = B, m, E, V
        self.Vp = (V + 31) // 32 * 32 if cfg.precision == "bf16" else V
        self.grad_scale = 1.0 / (replicas * spec.workers)
        nl = _pad16(layer_grad_size(cfg, True))
        # flat layout: [token V*E | layer 0 .. L-1 | final gain | final bias | head E*Vp | head bias Vp | loss]
        o = 0
        self._off = {}
        for name, n in [("tok", V * E)] + [(f"layer{i}", nl) for i in range(L)] + \
                       [("fg", E), ("fb", E), ("hw", E * self.Vp), ("hb", self.Vp), ("loss", 1)]:
            self._off[name] = (o, n)
            o += _pad16(n)
        self.grads = torch.zeros(o, dtype=f32, device=dev)
        self.params = torch.zeros(o, dtype=f32, device=dev)
        nle = layer_grad_size(cfg, True)
        self.engines = [LSSAttention(cfg, spec, grad_scale=self.grad_scale, device=dev, balanced=balanced,
                                     fused_rs=fused_rs, with_ffn=True, grads=self._slot(self.grads, f"layer{i}")[:nle])
                        for i in range(L)]
        self.g_pos = torch.zeros(m, E, dtype=f32, device=dev)   # local position rows
        self.pos = torch.zeros(m, E, dtype=f32, device=dev)
        ad = cfg.act_dtype
        M = B * m
        self.x0 = torch.empty(B, m, E, dtype=f32, device=dev)
        self.xf = torch.empty(M, E, dtype=ad, device=dev)
        self.mean_f, self.rstd_f = torch.empty(M, dtype=f32, device=dev), torch.empty(M, dtype=f32, device=dev)
        self.logits = torch.empty(M, self.Vp, dtype=f32, device=dev)
        self.g_logits = torch.empty(M, self.Vp, dtype=ad, device=dev)
        self.g_xf = torch.empty(M, E, dtype=f32, device=dev)
        self.g_x = torch.empty(B, m, E, dtype=f32, device=dev)
        self.head_w = None
        self.tokens = None
        self.loss_sum = None

    def _slot(self, buf, name):
        o, n = self._off[name]
        return buf[o:o + n]

    def _views(self, buf):
        E, V, Vp = self.E, self.V, self.Vp
        return dict(tok=self._slot(buf, "tok").view(V, E), fg=self._slot(buf, "fg"), fb=self._slot(buf, "fb"),
                    hw=self._slot(buf, "hw").view(E, Vp), hb=self._slot(buf, "hb"), loss=self._slot(buf, "loss"))

    # ------------------------------------------------------------ parameters
    def bind_params(self, P: Parameters) -> None:
        """Load the full-model Parameters (pos_table = the FULL table or exactly this
        rank's rows) into the flat fp32 buffers and stage the operands."""
        pv = self._views(self.params)
        pv["tok"].copy_(P.token_table)
        pt = P.pos_table
        o, m = self.spec.offset, self.m
        self.pos.copy_(pt[o:o + m] if pt.shape[0] == self.cfg.seq_len and pt.shape[0] != m else pt)
        for i, (eng, lp) in enumerate(zip(self.engines, P.layers)):
            eng.bind_params(lp, self._slot(self.params, f"layer{i}")[:eng.grads.numel()])
        pv["fg"].copy_(P.final_gain)
        pv["fb"].copy_(P.final_bias)
        pv["hw"].zero_()
        pv["hb"].zero_()
        pv["hw"][:, :self.V].copy_(P.head.weight)
        pv["hb"][:self.V].copy_(P.head.bias)
        self._stage_head()

    def _stage_head(self):
        pv = self._views(self.params)
        self.head_w = pv["hw"].to(self.cfg.act_dtype).contiguous()  # [E][Vp]: B operand N-major

    def parameters(self) -> Parameters:
        """Views of the bound parameters (pos_table = this rank's rows)."""
        pv = self._views(self.params)
        return Parameters(pv["tok"], self.pos, [e.param_lp for e in self.engines], pv["fg"], pv["fb"],
                          LinearParams(pv["hw"][:, :self.V], pv["hb"][:self.V]))

    def gradients(self) -> Parameters:
        gv = self._views(self.grads)
        return Parameters(gv["tok"], self.g_pos, [e.grad_params() for e in self.engines], gv["fg"], gv["fb"],
                          LinearParams(gv["hw"][:, :self.V], gv["hb"][:self.V]))

    def optimizer_step(self, opt, opt_pos) -> None:
        """hybrid.train_step's update (hybrid.py:125): one fused update of every
        replicated parameter, one of the local position rows, then restage."""
        opt.step(self.params, self.grads)
        opt_pos.step(self.pos, self.g_pos)
        for e in self.engines:
            e.load_params(e.param_lp)
        self._stage_head()

    # ------------------------------------------------------------ step pieces
    def embed(self, tokens_seg: torch.Tensor, policy=None) -> torch.Tensor:
        """Token + position rows (model.embed_fwd, model.py:517-533), dropout at the
        ``embed`` site of layer 0 when ``policy`` is active."""
        ids = tokens_seg.to(torch.int32).contiguous()
        if ids.shape != (self.B, self.m):
            raise ShapeError(f"tokens must be {(self.B, self.m)}, got {tuple(ids.shape)}")
        self.tokens = ids
        self.grads.zero_()
        for li, e in enumerate(self.engines):
            e.set_dropout(policy, li)
        x = K.embed_fwd(ids, self._views(self.params)["tok"], self.pos, out=self.x0)
        e0 = self.engines[0]
        if e0._dd is not None:
            e0._drop_rows(x.view(-1, self.E), x.view(-1, self.E), "embed")
        return x

    def head(self, x: torch.Tensor, targets_seg: torch.Tensor) -> torch.Tensor:
        """Final LN, head, cross-entropy of this rank's tokens and its backward to the
        last layer's output; the partial loss goes into the flat buffer's last slot."""
        B, m, E, V, Vp = self.B, self.m, self.E, self.V, self.Vp
        M = B * m
        a = self.grad_scale
        pv, gv = self._views(self.params), self._views(self.grads)
        K.layernorm_fwd(x.view(M, E), pv["fg"], pv["fb"], out=self.xf, mean=self.mean_f, rstd=self.rstd_f)
        K.gemm(self.xf, self.head_w, b_mn_major=True, bias=pv["hb"], out=self.logits, M=M, N=Vp, K=E)
        tg = targets_seg.to(torch.int32).contiguous().view(-1)
        loss_rows, g32 = K.cross_entropy(self.logits, tg, V, scale=1.0 / M)
        self.loss_sum = loss_rows.sum()
        gv["loss"].copy_(self.loss_sum.view(1) * (a / M))  # partial (mean) loss, pre-scaled for the all-reduce
        K.cat_cast_colsum([(g32, Vp, Vp)], M, dst=self.g_logits, colsum=gv["hb"], alpha=a)
        K.gemm(self.g_logits, self.head_w, out=self.g_xf, M=M, N=E, K=Vp)  # g . W^T
        K.gemm(self.xf, self.g_logits, a_mn_major=True, b_mn_major=True, alpha=a, out=gv["hw"], M=E, N=Vp, K=M)
        K.layernorm_bwd(self.g_xf, x.view(M, E), self.mean_f, self.rstd_f, pv["fg"], grad_x=self.g_x.view(M, E),
                        grad_gain=gv["fg"], grad_bias=gv["fb"], alpha=a)
        return self.g_x

    def embed_backward(self, g: torch.Tensor) -> None:
        e0 = self.engines[0]
        if e0._dd is not None:  # dropout_bwd(embed), in place on the incoming gradient
            e0._drop_rows(g.view(-1, self.E), g.view(-1, self.E), "embed")
        K.embed_bwd(self.tokens, g, self.V, grad_token=self._views(self.grads)["tok"], grad_pos=self.g_pos,
                    alpha_token=self.grad_scale, alpha_pos=self.grad_scale)

    def loss(self) -> torch.Tensor:
        """The synced (grid-mean) loss after :func:`gpt_step` with sync (device scalar)."""
        return self._views(self.grads)["loss"][0]


def gpt_step(ranks, comm, tokens, targets, *, step: int = 0, sync: bool = True, data_comm=None, policy=None):
    """One training-step forward + backward (+ sync) of the decoder on every rank
    (sharded.forward / backward / sync, hybrid.vertical_sync).  ``ranks`` is this
    process's [GPTRank] (or G of them with a SimComm); tokens / targets are the
    ranks' (B, m) blocks.  Returns the ranks' loss device scalars (grid mean
    after sync).  ``policy``: dropout (dropout.DropoutPolicy / rate / None), the
    same masks as the sequential model.forward.  Like sharded.forward it is used
    as given: a multi-step driver derives ``policy.at_step(step)`` (and
    ``.fork(replica)`` on a D x N grid) per step, as sharded.run_steps /
    hybrid.run_steps (sharded.py:320, hybrid.py:172-174) and
    hybrid.run_engine_steps do."""
    L = len(ranks[0].engines)
    xs = [r.embed(t, policy) for r, t in zip(ranks, tokens)]
    for li in range(L):
        xs = lss_forward([r.engines[li] for r in ranks], comm, xs, step=step, layer=li)
    gs = [r.head(x, t) for r, x, t in zip(ranks, xs, targets)]
    for li in range(L - 1, -1, -1):
        gs = lss_backward([r.engines[li] for r in ranks], comm, gs, step=step, layer=li, sync=False)
    for r, g in zip(ranks, gs):
        r.embed_backward(g)
    if sync:
        if isinstance(comm, SimComm):
            comm.all_reduce_sum([r.grads for r in ranks], step)
        else:
            comm.all_reduce_sum(ranks[0].grads, step)
            if ranks[0].replicas > 1:  # position rows: data-group mean only (hybrid.py:76-92)
                if data_comm is None:
                    raise ValueError("replicas > 1 needs data_comm (the data-parallel group)")
                data_comm.all_reduce_sum(ranks[0].g_pos, step)
        # the position rows were scaled by 1/(D*N): the data-group sum leaves /N (sharded.py:207-208)
    return [r.loss() for r in ranks]
