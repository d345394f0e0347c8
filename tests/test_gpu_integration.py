"""The reference-signature boundary on the B200, end to end.

1. ``sharded.forward / backward / sync`` and ``hybrid.vertical_sync /
   train_step / run_steps`` with the reference's own signatures
   (sharded.py:113-348, hybrid.py:76-190), worker threads on one GPU through
   ``collectives.Communicator`` (the reference's model of a job): the whole
   decoder on G=2 sequence workers == the real reference's sequential
   ``model.forward / backward`` golden; the 2x2 grid == the sequential model on
   the combined batch.
2. INTEGRATION.md §1 run for real: the REFERENCE's own ``model.layer_fwd /
   layer_bwd`` and its threaded ``sharded.run_steps``, with only its attention
   core (``scores_fwd / scores_bwd``) routed to the B200 kernels by
   ``integration.patch_reference`` == the unpatched reference.  Needs the
   reference installed under baseline/_ref (``pip install --target
   baseline/_ref``); skipped when absent.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import assert_close_ref

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
REF_INSTALL = ROOT / "baseline" / "_ref"


def _gpt(cuda):
    from test_gpu_layer import _gpt_from_golden

    z = np.load(GOLDEN / "gpt_small.npz")
    return z, _gpt_from_golden(z, cuda)


@pytest.mark.parametrize("fused", [True, False])
def test_sharded_reference_api_matches_sequential_golden(cuda, fused):
    """sharded.run_steps (threads) -> forward / backward / sync on 2 workers: the
    synced gradients equal the reference's sequential gradients, PE rows concatenate
    (test_sharded.py:82-113), partial losses average to the full loss (116-123), and
    the ledger holds L gathers + L reduce-scatters + 1 all-reduce (140-179)."""
    import torch
    from paper_2311_02382_b200 import model as M
    from paper_2311_02382_b200 import sharded

    z, P = _gpt(cuda)
    L, h, v, seq = int(z["n_layers"]), int(z["meta"][2]), int(z["vocab"]), 128
    cfg = M.ModelConfig(embed_dim=128, n_layers=L, n_heads=h, ff_dim=int(z["ff_dim"]), vocab=v, seq_len=seq,
                        batch=2, precision="single")
    tok, tgt = torch.as_tensor(z["tokens"], device=cuda), torch.as_tensor(z["targets"], device=cuda)
    run = sharded.run_steps(cfg, P, 2, [(tok, tgt)], lr=0.0, fused=fused, keep_last_grads=True)
    tol = 1e-4
    assert abs(run.step_losses[0] - float(z["loss"])) / float(z["loss"]) < tol
    assert abs(np.mean([p[0] for p in run.partial_losses]) - float(z["loss"])) / float(z["loss"]) < tol
    g0 = dict(run.last_grads[0].named_arrays())
    g0["pos_table"] = torch.cat([run.last_grads[r].pos_table for r in range(2)], 0)
    for name in [n for n in z.files if n.startswith("g.")]:
        key = name[2:]
        if key.endswith("attn_k.bias"):
            continue
        assert_close_ref(g0[key].cpu().numpy(), z[name], tol, key)
    for key in g0:  # replicated gradients identical on every worker after sync
        if key != "pos_table":
            assert torch.equal(dict(run.last_grads[1].named_arrays())[key], g0[key])
    led = run.comm.ledger
    per = 1 if fused else 2
    assert led.count("all-gather") == per * L and led.count("reduce-scatter") == per * L
    assert led.count("all-reduce") == 1
    if fused:  # ONE packed [K_r|V_r] gather: 2*B*l*E elements per record
        assert all(r.elements == 2 * 2 * seq * 128 for r in led.records if r.kind == "all-gather")


def test_hybrid_reference_api_grid_matches_combined_batch(cuda):
    """hybrid.run_steps on a 2x2 grid (worker threads, seq groups + data groups,
    sharded.sync then vertical_sync, test_hybrid.py:100-110) == the sequential model
    on the two replicas' batches combined; one SGD step applied identically."""
    import torch
    from paper_2311_02382_b200 import hybrid
    from paper_2311_02382_b200 import model as M

    z, P = _gpt(cuda)
    L, h, v, seq = int(z["n_layers"]), int(z["meta"][2]), int(z["vocab"]), 128
    cfg = M.ModelConfig(embed_dim=128, n_layers=L, n_heads=h, ff_dim=int(z["ff_dim"]), vocab=v, seq_len=seq,
                        batch=2, precision="single")
    g = torch.Generator(device=cuda).manual_seed(3)
    batches = [[(torch.randint(0, v, (2, seq), generator=g, device=cuda),
                 torch.randint(0, v, (2, seq), generator=g, device=cuda)) for _ in range(2)]]
    run = hybrid.run_steps(cfg, P, hybrid.GridLayout(2, 2), batches, lr=0.0, keep_last_grads=True)
    tok = torch.cat([batches[0][0][0], batches[0][1][0]], 0)
    tgt = torch.cat([batches[0][0][1], batches[0][1][1]], 0)
    cfg4 = M.ModelConfig(**{**cfg.__dict__, "batch": 4})
    loss, cache = M.forward(P, cfg4, tok, tgt)
    want = dict(M.backward(P, cfg4, cache).named_arrays())
    assert abs(run.step_losses[0] - loss) / loss < 1e-4
    got = dict(run.last_grads[0].named_arrays())
    lay = run.layout
    got["pos_table"] = torch.cat([run.last_grads[r].pos_table for r in lay.seq_members(0)], 0)
    for key, w in want.items():
        if key.endswith("attn_k.bias"):
            continue
        assert_close_ref(got[key].cpu().numpy(), w.cpu().numpy(), 1e-4, key)
    # traffic: per-layer collectives stay in the sequence groups, syncs in both (test_hybrid.py:130-147)
    kinds = {(r.kind, r.group[:3]) for r in run.comm.ledger.records}
    assert ("all-gather", "seq") in kinds and ("all-reduce", "dat") in kinds
    assert not any(r.group.startswith("data") for r in run.comm.ledger.records if r.kind != "all-reduce")


# ---------------------------------------------------------------- INTEGRATION.md §1 (reference + B200 core)


@pytest.fixture(scope="module")
def seqpar():
    if not (REF_INSTALL / "seqpar").exists():
        pytest.skip("reference not installed under baseline/_ref")
    sys.path.insert(0, str(REF_INSTALL))
    import seqpar  # noqa: F401
    from seqpar import model, nnops, sharded

    return model, nnops, sharded


@pytest.mark.parametrize("precision", ["bf16", "single"])
def test_reference_layer_with_b200_attention_core(cuda, seqpar, precision):
    from paper_2311_02382_b200.integration import patch_reference

    model, nnops, _ = seqpar
    cfg = model.ModelConfig(embed_dim=128, n_layers=1, n_heads=2, ff_dim=256, vocab=16, seq_len=256, batch=2,
                            precision="single")
    lp = model.init_params(cfg, 0).layers[0]
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 256, 128)).astype(np.float32)
    gy = rng.standard_normal((2, 256, 128)).astype(np.float32)
    off = nnops.DropoutPolicy.off()

    def run():
        y, cache = model.layer_fwd(lp, cfg, off, 0, x, 0, model.local_kv_fwd)
        dx, grads = model.layer_bwd(lp, cfg, off, 0, cache, gy, model.local_kv_bwd)
        return y, dx, grads

    y0, dx0, g0 = run()
    restore = patch_reference(model, precision)
    try:
        y1, dx1, g1 = run()
    finally:
        restore()
    tol = 1e-2 if precision == "bf16" else 1e-4
    assert_close_ref(y1, y0, tol, "y")
    assert_close_ref(dx1, dx0, tol, "dx")
    for n in ("ln1_gain", "ln1_bias", "attn_q", "attn_k", "attn_v", "attn_out", "ln2_gain", "ln2_bias", "ff_in",
              "ff_out"):
        a, b = getattr(g1, n), getattr(g0, n)
        pairs = [(n, a, b)] if isinstance(a, np.ndarray) else [(n + ".weight", a.weight, b.weight),
                                                                 (n + ".bias", a.bias, b.bias)]
        for name, ga, gb in pairs:
            if name == "attn_k.bias":  # mathematically zero (softmax shift invariance)
                continue
            assert_close_ref(ga, gb, tol, name)


def test_reference_sharded_engine_with_b200_attention_core(cuda, seqpar):
    """The reference's own threaded sharded.run_steps (its Communicator, fused kv
    hooks, sync, SGD) for 2 steps on 2 workers with the B200 attention core."""
    from paper_2311_02382_b200.integration import patch_reference

    model, _, sharded = seqpar
    cfg = model.ModelConfig(embed_dim=128, n_layers=2, n_heads=2, ff_dim=256, vocab=40, seq_len=128, batch=2,
                            precision="single")
    params = model.init_params(cfg, 1)
    rng = np.random.default_rng(1)
    batches = [(rng.integers(0, 40, (2, 128)), rng.integers(0, 40, (2, 128))) for _ in range(2)]
    ref = sharded.run_steps(cfg, params, 2, batches, lr=0.05)
    restore = patch_reference(model, "single")
    try:
        got = sharded.run_steps(cfg, params, 2, batches, lr=0.05)
    finally:
        restore()
    assert np.allclose(got.step_losses, ref.step_losses, rtol=1e-4)
    for (n, a), (_, b) in zip(got.workers[0].params.named_arrays(), ref.workers[0].params.named_arrays()):
        if n.endswith("attn_k.bias"):  # its gradient is mathematically zero: both sides are rounding noise
            assert np.abs(a - b).max() < 1e-6
            continue
        assert_close_ref(a, b, 1e-4, n)
