"""CPU: host-side logic of the B200 path (no kernels): shard geometry, config
validation, grid layout, ledger semantics."""

import pytest


def test_shard_spec_geometry_and_partition_error():
    from paper_2311_02382_b200.errors import PartitionError
    from paper_2311_02382_b200.sharded import ShardSpec

    spec = ShardSpec(7, 8, 50112)
    assert spec.block == 6264 and spec.offset == 7 * 6264
    with pytest.raises(PartitionError):
        ShardSpec(0, 3, 10)
    with pytest.raises(ValueError):
        ShardSpec(3, 3, 9)


def test_slice_batch_rows_are_bit_exact():
    import torch
    from paper_2311_02382_b200.errors import ShapeError
    from paper_2311_02382_b200.sharded import ShardSpec, slice_batch

    x = torch.arange(2 * 12 * 3, dtype=torch.float32).view(2, 12, 3)
    parts = [slice_batch(x, ShardSpec(r, 4, 12)) for r in range(4)]
    assert torch.equal(torch.cat(parts, dim=1), x)
    assert torch.equal(parts[2], x[:, 6:9])
    with pytest.raises(ShapeError):
        slice_batch(x, ShardSpec(0, 2, 10))


def test_model_config_validation_mirrors_reference():
    from paper_2311_02382_b200.errors import ShapeError, UnsupportedError
    from paper_2311_02382_b200.model import ModelConfig

    with pytest.raises(ShapeError):
        ModelConfig(embed_dim=10, n_layers=1, n_heads=3, ff_dim=4, vocab=7, seq_len=4)
    with pytest.raises(ValueError):
        ModelConfig(embed_dim=8, n_layers=-1, n_heads=2, ff_dim=4, vocab=7, seq_len=4)
    with pytest.raises(ValueError):
        ModelConfig(embed_dim=8, n_layers=1, n_heads=2, ff_dim=4, vocab=7, seq_len=4, dropout=1.0)
    with pytest.raises(UnsupportedError):
        ModelConfig(embed_dim=8, n_layers=1, n_heads=2, ff_dim=4, vocab=7, seq_len=4, precision="double")
    cfg = ModelConfig(embed_dim=1024, n_layers=1, n_heads=16, ff_dim=4096, vocab=256, seq_len=50112)
    assert cfg.head_dim == 64 and cfg.causal and cfg.precision == "bf16"


def test_grid_layout_matches_reference_geometry():
    """hybrid.py:36-61 / test_hybrid.py:25-46."""
    from paper_2311_02382_b200.hybrid import GridLayout

    lay = GridLayout(2, 4)
    assert lay.world == 8
    assert lay.seq_members(1) == (4, 5, 6, 7)
    assert lay.data_members(2) == (2, 6)
    assert lay.coords(5) == (1, 1)
    assert lay.grad_scale == 1 / 8
    with pytest.raises(ValueError):
        GridLayout(0, 2)


def test_ledger_counts():
    from paper_2311_02382_b200.comm import Ledger

    led = Ledger()
    led.record("all-gather", "sequence", 10, 0, "forward", 0)
    led.record("reduce-scatter", "sequence", 10, 0, "backward", 0)
    led.record("all-reduce", "world", 5, 0, "sync")
    assert led.count() == 3 and led.count("all-gather") == 1 and led.count(phase="sync") == 1


def test_folded_gradient_scale_equals_double_average():
    """(1/D) sum_d (1/N) sum_n g == sum_{d,n} g / (D*N)  (hybrid.py:76-92 + sharded.py:238)."""
    import numpy as np

    r = np.random.default_rng(0)
    D, N = 2, 4
    g = r.standard_normal((D, N, 5))
    two_step = np.mean([np.mean(g[d], axis=0) for d in range(D)], axis=0)
    folded = (g / (D * N)).sum(axis=(0, 1))
    np.testing.assert_allclose(folded, two_step, rtol=1e-14)


@pytest.mark.parametrize("G", [2, 3, 4, 5, 8])
def test_balance_plan_equalises_causal_work(G):
    """Every rank of a balanced causal group ends with G/2 block-units of work
    (block = m x m query-key pairs; the diagonal block counts 1/2)."""
    from paper_2311_02382_b200.sharded import make_plan

    m = 6264
    plans = [make_plan(r, G, m, True) for r in range(G)]
    split = (m // 2) // 128 * 128
    work = [r + 0.5 for r in range(G)]
    for r, pl in enumerate(plans):
        if pl.role == "heavy":
            moved = pl.a * split / m + pl.b * (m - split) / m
            work[r] -= moved
            work[pl.partner] += moved
            assert plans[pl.partner].role == "light" and plans[pl.partner].partner == r
            assert (pl.a, pl.b) == (plans[pl.partner].a, plans[pl.partner].b)
            assert pl.a + pl.b == 2 * r - G + 1 and pl.a <= r and pl.b <= r
    assert max(work) - min(work) < 0.05 * G / 2, work
    assert not any(p.active for p in (make_plan(r, G, m, False) for r in range(G)))
