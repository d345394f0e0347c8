"""Generate golden fixtures by running the REAL reference (seqpar) on seeded inputs.

Run in the dev container (needs /root/reference):  python tests/golden/make_golden.py

For each case the reference's own layer code runs on G simulated workers
(threads + its Communicator), exactly as sharded.forward/backward wire it
(sharded.py:138-143 fused kv_fwd, 186-190 fused kv_bwd, 219-244 sync):
model.layer_fwd / model.layer_bwd (model.py:424-499) with the FFN half's
weights set to zero so the layer reduces to its attention half (the FFN then
adds exactly 0 and its backward passes grad_out through unchanged).

Inputs are rounded to float32 and then computed in float64 ("double"
precision, the reference's default).  Stored: inputs, per-rank outputs
concatenated (y, dx), and the group-averaged attention-parameter grads.

FULL_CASES (files full_*.npz) run the complete pre-norm layer with live FFN
weights (LN2 -> ff_in -> tanh-GeLU -> ff_out -> residual, model.py:362-390,
449-452, 475-478) and additionally store the LN2 / FFN parameters and their
group-averaged grads.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from seqpar import model  # noqa: E402
from seqpar.collectives import Communicator, run_workers  # noqa: E402
from seqpar.model import ModelConfig  # noqa: E402
from seqpar.nnops import DropoutPolicy, LinearParams  # noqa: E402
from seqpar.sharded import ShardSpec  # noqa: E402

OUT = Path(__file__).resolve().parent

CASES = {
    # name: (seq_len, embed, heads, workers, batch, causal, out dtype)
    "small_causal": (256, 128, 2, 2, 1, True, np.float64),
    "small_noncausal": (256, 128, 2, 2, 1, False, np.float64),
    "batch2_g3": (192, 128, 2, 3, 2, True, np.float64),
    "configA": (1024, 256, 4, 2, 1, True, np.float32),
}

GRAD_NAMES = ("ln1_gain", "ln1_bias", "wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo")
FFN_NAMES = ("ln2_gain", "ln2_bias", "w_in", "b_in", "w_out", "b_out")

FULL_CASES = {
    # name: (seq_len, embed, heads, workers, batch, causal, ff_dim, out dtype)
    "full_g2_causal": (256, 128, 2, 2, 1, True, 512, np.float64),
    "full_g1_b2": (128, 128, 2, 1, 2, True, 256, np.float64),
}


def run_case(seq, e, h, g, b, causal, seed=0, ff_dim=0, policy=None):
    cfg = ModelConfig(embed_dim=e, n_layers=1, n_heads=h, ff_dim=ff_dim or 8, vocab=16, seq_len=seq,
                      batch=b, causal=causal, precision="double")
    rng = np.random.default_rng(seed)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    lp = model.init_params(cfg, seed).layers[0]
    # non-trivial LN affine and biases so every gradient is exercised
    lp.ln1_gain = f32(1.0 + 0.1 * rng.standard_normal(e))
    lp.ln1_bias = f32(0.1 * rng.standard_normal(e))
    lin = lambda p: LinearParams(f32(p.weight), f32(0.05 * rng.standard_normal(e)))  # noqa: E731
    lp.attn_q, lp.attn_k, lp.attn_v, lp.attn_out = (lin(lp.attn_q), lin(lp.attn_k),
                                                    lin(lp.attn_v), lin(lp.attn_out))
    if ff_dim:  # live FFN half with non-trivial LN2 affine and biases
        lp.ln2_gain = f32(1.0 + 0.1 * rng.standard_normal(e))
        lp.ln2_bias = f32(0.1 * rng.standard_normal(e))
        lp.ff_in = LinearParams(f32(lp.ff_in.weight), f32(0.05 * rng.standard_normal(ff_dim)))
        lp.ff_out = LinearParams(f32(lp.ff_out.weight), f32(0.05 * rng.standard_normal(e)))
    else:
        lp.ff_in = LinearParams(np.zeros_like(lp.ff_in.weight), np.zeros_like(lp.ff_in.bias))
        lp.ff_out = LinearParams(np.zeros_like(lp.ff_out.weight), np.zeros_like(lp.ff_out.bias))
    x = f32(rng.standard_normal((b, seq, e)))
    gy = f32(rng.standard_normal((b, seq, e)))
    off = policy if policy is not None else DropoutPolicy.off()
    comm = Communicator(g, timeout=120.0)
    group = comm.group("sequence", tuple(range(g)))

    def worker(rank):
        spec = ShardSpec(rank, g, seq)
        xs = np.ascontiguousarray(x[:, spec.offset:spec.offset + spec.block])
        gys = np.ascontiguousarray(gy[:, spec.offset:spec.offset + spec.block])

        def kv_fwd(xh, lp_):  # sharded.py:139-143
            xh_full = comm.all_gather(group, rank, xh, dim=1, step=0, phase="forward", layer=0)
            return model.linear3(xh_full, lp_.attn_k), model.linear3(xh_full, lp_.attn_v), xh_full

        def kv_bwd(kv_ctx, lp_, gk, gv):  # sharded.py:186-191
            grad_full, k_wg, k_bg, v_wg, v_bg = model.local_kv_bwd(kv_ctx, lp_, gk, gv)
            seg = comm.reduce_scatter(group, rank, grad_full, dim=1, step=0, phase="backward",
                                      layer=0)
            return seg, k_wg, k_bg, v_wg, v_bg

        y, cache = model.layer_fwd(lp, cfg, off, 0, xs, spec.offset, kv_fwd)
        dx, grads = model.layer_bwd(lp, cfg, off, 0, cache, gys, kv_bwd)
        flat = [grads.ln1_gain, grads.ln1_bias, grads.attn_q.weight, grads.attn_q.bias,
                grads.attn_k.weight, grads.attn_k.bias, grads.attn_v.weight, grads.attn_v.bias,
                grads.attn_out.weight, grads.attn_out.bias]
        if ff_dim:
            flat += [grads.ln2_gain, grads.ln2_bias, grads.ff_in.weight, grads.ff_in.bias,
                     grads.ff_out.weight, grads.ff_out.bias]
        vec = np.concatenate([a.ravel() for a in flat])
        vec = comm.all_reduce_mean(group, rank, vec, step=0, phase="sync")  # sharded.py:238
        return y, dx, vec, [a.shape for a in flat]

    res = run_workers(g, worker, comm=comm)
    y = np.concatenate([r[0] for r in res], axis=1)
    dx = np.concatenate([r[1] for r in res], axis=1)
    vec, shapes = res[0][2], res[0][3]
    grads, pos = {}, 0
    for name, shp in zip(GRAD_NAMES + (FFN_NAMES if ff_dim else ()), shapes):
        n = int(np.prod(shp))
        grads["g_" + name] = vec[pos:pos + n].reshape(shp)
        pos += n
    params = dict(ln1_gain=lp.ln1_gain, ln1_bias=lp.ln1_bias, wq=lp.attn_q.weight,
                  bq=lp.attn_q.bias, wk=lp.attn_k.weight, bk=lp.attn_k.bias,
                  wv=lp.attn_v.weight, bv=lp.attn_v.bias, wo=lp.attn_out.weight,
                  bo=lp.attn_out.bias)
    if ff_dim:
        params.update(ln2_gain=lp.ln2_gain, ln2_bias=lp.ln2_bias, w_in=lp.ff_in.weight, b_in=lp.ff_in.bias,
                      w_out=lp.ff_out.weight, b_out=lp.ff_out.bias)
    return x, gy, params, y, dx, grads


DROP_CASES = {
    # name: (seq_len, embed, heads, workers, batch, causal, ff_dim, rate, seed) -- position-keyed dropout
    # at every site; G=2 must equal G=1 on the same masks
    "drop_layer_g1": (128, 128, 2, 1, 2, True, 256, 0.1, 1234),
    "drop_layer_g2": (256, 128, 2, 2, 1, True, 256, 0.1, 1234),
    # m = 512 per rank at world 2: the balanced causal schedule is active (NCCL test)
    "drop_layer_g2_big": (1024, 128, 2, 2, 1, True, 256, 0.1, 4321),
}


def gpt_case(seed=5, policy=None, name="gpt_small"):
    """Whole decoder: model.forward / model.backward sequentially,
    2 layers, vocab 40 (not a multiple of 32: exercises the padded head)."""
    cfg = ModelConfig(embed_dim=128, n_layers=2, n_heads=2, ff_dim=256, vocab=40, seq_len=128, batch=2,
                      causal=True, precision="double")
    rng = np.random.default_rng(seed)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    params = model.init_params(cfg, seed)
    params.token_table = f32(params.token_table)
    params.pos_table = f32(params.pos_table)
    for lp in params.layers:
        lp.ln1_gain = f32(1.0 + 0.1 * rng.standard_normal(128))
        lp.ln1_bias = f32(0.1 * rng.standard_normal(128))
        lp.ln2_gain = f32(1.0 + 0.1 * rng.standard_normal(128))
        lp.ln2_bias = f32(0.1 * rng.standard_normal(128))
        for n in ("attn_q", "attn_k", "attn_v", "attn_out", "ff_in", "ff_out"):
            lin = getattr(lp, n)
            setattr(lp, n, LinearParams(f32(lin.weight), f32(0.05 * rng.standard_normal(lin.bias.shape))))
    params.final_gain = f32(1.0 + 0.1 * rng.standard_normal(128))
    params.final_bias = f32(0.1 * rng.standard_normal(128))
    params.head = LinearParams(f32(params.head.weight), f32(0.05 * rng.standard_normal(40)))
    tokens = rng.integers(0, 40, (2, 128))
    targets = rng.integers(0, 40, (2, 128))
    loss, cache = model.forward(params, cfg, tokens, targets, policy)
    grads = model.backward(params, cfg, cache)
    arrays = dict(tokens=tokens.astype(np.int32), targets=targets.astype(np.int32),
                  loss=np.array(loss, dtype=np.float64),
                  meta=np.array([128, 128, 2, 1, 2, 1], dtype=np.int64), ff_dim=np.array(256), n_layers=np.array(2),
                  vocab=np.array(40))
    for n, a in params.named_arrays():
        arrays["p." + n] = np.asarray(a, np.float32)
    for n, a in grads.named_arrays():
        arrays["g." + n] = np.asarray(a, np.float64)
    if policy is not None:
        arrays["drop"] = np.array([policy.rate, policy.seed], dtype=np.float64)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(name, "written, loss", loss)


NS_CASES = {
    # north-star shape (BASELINE.json: E_m=1024, 16 heads) through the real reference,
    # name: (seq_len, workers, causal); inputs from ns_inputs.ns_inputs(seq, 1024, seed=0)
    "ns_l2048_g2": (2048, 2, True),
    "ns_l2048_g8": (2048, 8, True),
    "ns_l2048_g4_noncausal": (2048, 4, False),
}


def ns_case(name, seq, g, causal):
    """The reference's layer_fwd / layer_bwd at E=1024, 16 heads on G simulated workers
    (fused kv hooks, sharded.py:138-143 / 186-190; sync sharded.py:238), fp64.  The
    inputs are rebuilt from the seed by the tests, so only outputs are stored: every
    row sum of y / dx and of each weight gradient (checksums covering every element),
    every ROW_STRIDE-th row of y / dx, every WROW_STRIDE-th row of each weight
    gradient, the LN / bias gradients in full."""
    from ns_inputs import ATTN_NAMES, ROW_STRIDE, WROW_STRIDE, ns_inputs

    e, h = 1024, 16
    x32, gy32, p32 = ns_inputs(seq, e, seed=0)
    cfg = ModelConfig(embed_dim=e, n_layers=1, n_heads=h, ff_dim=8, vocab=16, seq_len=seq, batch=1,
                      causal=causal, precision="double")
    lp = model.init_params(cfg, 0).layers[0]
    d = {k: v.astype(np.float64) for k, v in p32.items()}
    lp.ln1_gain, lp.ln1_bias = d["ln1_gain"], d["ln1_bias"]
    lp.attn_q, lp.attn_k = LinearParams(d["wq"], d["bq"]), LinearParams(d["wk"], d["bk"])
    lp.attn_v, lp.attn_out = LinearParams(d["wv"], d["bv"]), LinearParams(d["wo"], d["bo"])
    lp.ff_in = LinearParams(np.zeros_like(lp.ff_in.weight), np.zeros_like(lp.ff_in.bias))
    lp.ff_out = LinearParams(np.zeros_like(lp.ff_out.weight), np.zeros_like(lp.ff_out.bias))
    x, gy = x32.astype(np.float64), gy32.astype(np.float64)
    comm = Communicator(g, timeout=600.0)
    group = comm.group("sequence", tuple(range(g)))
    off = DropoutPolicy.off()

    def worker(rank):
        spec = ShardSpec(rank, g, seq)
        xs = np.ascontiguousarray(x[:, spec.offset:spec.offset + spec.block])
        gys = np.ascontiguousarray(gy[:, spec.offset:spec.offset + spec.block])

        def kv_fwd(xh, lp_):  # sharded.py:139-143
            xh_full = comm.all_gather(group, rank, xh, dim=1, step=0, phase="forward", layer=0)
            return model.linear3(xh_full, lp_.attn_k), model.linear3(xh_full, lp_.attn_v), xh_full

        def kv_bwd(kv_ctx, lp_, gk, gv):  # sharded.py:186-191
            grad_full, k_wg, k_bg, v_wg, v_bg = model.local_kv_bwd(kv_ctx, lp_, gk, gv)
            seg = comm.reduce_scatter(group, rank, grad_full, dim=1, step=0, phase="backward", layer=0)
            return seg, k_wg, k_bg, v_wg, v_bg

        y, cache = model.layer_fwd(lp, cfg, off, 0, xs, spec.offset, kv_fwd)
        dx, grads = model.layer_bwd(lp, cfg, off, 0, cache, gys, kv_bwd)
        flat = [grads.ln1_gain, grads.ln1_bias, grads.attn_q.weight, grads.attn_q.bias,
                grads.attn_k.weight, grads.attn_k.bias, grads.attn_v.weight, grads.attn_v.bias,
                grads.attn_out.weight, grads.attn_out.bias]
        vec = comm.all_reduce_mean(group, rank, np.concatenate([a.ravel() for a in flat]), step=0,
                                   phase="sync")  # sharded.py:238
        return y, dx, vec, [a.shape for a in flat]

    res = run_workers(g, worker, comm=comm)
    y = np.concatenate([r[0] for r in res], axis=1)
    dx = np.concatenate([r[1] for r in res], axis=1)
    vec, shapes = res[0][2], res[0][3]
    arrays = dict(meta=np.array([seq, e, h, g, 1, int(causal)], dtype=np.int64),
                  y_rows=y[:, ::ROW_STRIDE].astype(np.float32), dx_rows=dx[:, ::ROW_STRIDE].astype(np.float32),
                  y_rowsum=y.sum(-1), dx_rowsum=dx.sum(-1))
    pos = 0
    for nm, shp in zip(ATTN_NAMES, shapes):
        n = int(np.prod(shp))
        gr = vec[pos:pos + n].reshape(shp)
        pos += n
        if gr.ndim == 2:
            arrays["g_" + nm + "_rows"] = gr[::WROW_STRIDE].astype(np.float32)
            arrays["g_" + nm + "_rowsum"] = gr.sum(1)
            arrays["g_" + nm + "_colsum"] = gr.sum(0)
        else:
            arrays["g_" + nm] = gr
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(name, "written", {k: v.shape for k, v in arrays.items() if k in ("y_rows", "g_wq_rows")})


def main(only=None):
    keep = (lambda n: True) if not only else (lambda n: n in only)  # noqa: E731
    sys.path.insert(0, str(OUT))
    for name, (seq, g, causal) in NS_CASES.items():
        if keep(name):
            ns_case(name, seq, g, causal)
    for name, (seq, e, h, g, b, causal, odt) in CASES.items():
        if not keep(name):
            continue
        x, gy, params, y, dx, grads = run_case(seq, e, h, g, b, causal)
        arrays = dict(x=x.astype(np.float32), grad_y=gy.astype(np.float32),
                      meta=np.array([seq, e, h, g, b, int(causal)], dtype=np.int64),
                      y=y.astype(odt), dx=dx.astype(odt))
        arrays.update({k: v.astype(np.float32) for k, v in params.items()})
        arrays.update({k: v.astype(odt) for k, v in grads.items()})
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
        print(name, "written", {k: v.shape for k, v in arrays.items() if k in ("x", "y")})
    for name, (seq, e, h, g, b, causal, ff, odt) in FULL_CASES.items():
        if not keep(name):
            continue
        x, gy, params, y, dx, grads = run_case(seq, e, h, g, b, causal, ff_dim=ff)
        arrays = dict(x=x.astype(np.float32), grad_y=gy.astype(np.float32),
                      meta=np.array([seq, e, h, g, b, int(causal)], dtype=np.int64),
                      ff_dim=np.array(ff, dtype=np.int64), y=y.astype(odt), dx=dx.astype(odt))
        arrays.update({k: v.astype(np.float32) for k, v in params.items()})
        arrays.update({k: v.astype(odt) for k, v in grads.items()})
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
        print(name, "written", {k: v.shape for k, v in arrays.items() if k in ("x", "y", "w_in")})
    if keep("gpt_small"):
        gpt_case()
    if keep("gpt_drop"):
        gpt_case(policy=DropoutPolicy(0.1, seed=99), name="gpt_drop")
    for name, (seq, e, h, g, b, causal, ff, rate, dseed) in DROP_CASES.items():
        if not keep(name):
            continue
        pol = DropoutPolicy(rate, seed=dseed)
        x, gy, params, y, dx, grads = run_case(seq, e, h, g, b, causal, ff_dim=ff, policy=pol)
        arrays = dict(x=x.astype(np.float32), grad_y=gy.astype(np.float32),
                      meta=np.array([seq, e, h, g, b, int(causal)], dtype=np.int64),
                      ff_dim=np.array(ff, dtype=np.int64), drop=np.array([rate, dseed], dtype=np.float64),
                      y=y.astype(np.float64), dx=dx.astype(np.float64))
        arrays.update({k: v.astype(np.float32) for k, v in params.items()})
        arrays.update({k: v.astype(np.float64) for k, v in grads.items()})
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
        print(name, "written")


if __name__ == "__main__":
    import sys

    main(sys.argv[1:] or None)  # optional case names: regenerate only those
