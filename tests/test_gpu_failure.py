"""Failure and numerics semantics on the B200 (ABI v9, include/lss.h).

* A cross-GPU wait whose peer never signals does not hang the GPU: in-kernel
  waits (fused-gather segment flags) give up at their deadline and the host
  raises CommTimeout (the reference's rendezvous timeout, collectives.py:242-252);
  front-end stream waits are released by the communicator's watchdog.
* With the numerics check on, a NaN / Inf produced by a GEMM or attention kernel
  raises NumericsError (tensor.py:79-95); off, nothing is reported.
"""

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture
def runtime(cuda):
    from paper_2311_02382_b200 import kernels as K

    K.status(clear=True)
    yield K
    K.runtime_config(wait_timeout_s=60.0, numerics=False)
    K.status(clear=True)


def test_in_kernel_wait_deadline_raises_comm_timeout(runtime):
    import torch
    from paper_2311_02382_b200.errors import CommTimeout

    K = runtime
    K.runtime_config(wait_timeout_s=0.3)
    G, m, H, E = 2, 256, 2, 128
    dev = torch.device("cuda")
    q = torch.randn(1, m, E, device=dev).to(torch.bfloat16)
    kv = torch.randn(G, 1, m, 2 * E, device=dev).to(torch.bfloat16)
    out = torch.empty(1, m, E, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(1, H, K.rows_pad(m), device=dev)
    flags = torch.zeros(G, dtype=torch.int32, device=dev)  # segment 0 never arrives
    t0 = time.monotonic()
    K.attn_fwd_partial(q, kv[..., :E], kv[..., E:], rows=m, row0=0, workers=G, seg_len=m, heads=H, offset=m,
                       causal=True, g_begin=0, g_end=G, out=out, lse2=lse, ready=(flags, 1, 1))
    torch.cuda.synchronize()  # returns: the producer gave up at the deadline
    assert time.monotonic() - t0 < 30
    with pytest.raises(CommTimeout):
        K.raise_status()
    K.raise_status()  # cleared


def test_watchdog_releases_stream_wait(runtime):
    import torch
    from paper_2311_02382_b200.comm import WaitWatchdog
    from paper_2311_02382_b200.errors import CommTimeout

    K = runtime
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    wd = WaitWatchdog(0.3, lambda: K.flag_release(flags.data_ptr(), flags.numel(), 1 << 30))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        K.stream_wait(flags.data_ptr() + 4, 7, s)  # a peer that never signals
        wd.track(s, "test wait")
        y = torch.ones(8, device="cuda") * 2
    t0 = time.monotonic()
    s.synchronize()  # drains once the watchdog released the flag words
    assert time.monotonic() - t0 < 30
    assert float(y.sum()) == 16.0
    with pytest.raises(CommTimeout):
        wd.check()


def test_numerics_check_raises_on_nonfinite(runtime):
    import torch
    from paper_2311_02382_b200 import model as M
    from paper_2311_02382_b200.errors import NumericsError

    K = runtime
    dev = torch.device("cuda")
    x = torch.randn(1, 64, 128, device=dev)
    w = M.LinearParams(torch.randn(128, 128, device=dev) / 11, torch.zeros(128, device=dev))
    M.linear3(x, w)  # check off: fine
    x_bad = x.clone()
    x_bad[0, 3, 5] = float("inf")
    M.linear3(x_bad, w)  # check off: not reported
    torch.cuda.synchronize()
    assert K.status(clear=True) == (False, False)
    K.runtime_config(numerics=True)
    M.linear3(x, w)  # finite: passes
    with pytest.raises(NumericsError):  # GEMM epilogue report
        M.linear3(x_bad.to(torch.bfloat16), w)
    cfg = M.ModelConfig(embed_dim=128, n_layers=1, n_heads=2, ff_dim=8, vocab=8, seq_len=64)
    q = torch.randn(1, 64, 128, device=dev).to(torch.bfloat16)
    kv = torch.randn(1, 64, 128, device=dev).to(torch.bfloat16)
    M.scores_fwd(q, kv, kv, 0, cfg)
    q[0, 7, 9] = float("nan")
    with pytest.raises(NumericsError):  # attention epilogue report
        M.scores_fwd(q, kv, kv, 0, cfg)


def test_engine_step_numerics_and_timeout_status(runtime):
    """lss_step with the check on: a finite step passes; a NaN in the input raises
    NumericsError at the end of the step."""
    import torch
    from paper_2311_02382_b200.errors import NumericsError
    from paper_2311_02382_b200.model import LayerParams, LinearParams, ModelConfig
    from paper_2311_02382_b200.sharded import ShardSpec, lss_step, make_sim_group, slice_batch

    K = runtime
    dev = torch.device("cuda")
    E, l, G = 128, 512, 2
    cfg = ModelConfig(embed_dim=E, n_layers=1, n_heads=2, ff_dim=8, vocab=8, seq_len=l)
    u = lambda: torch.randn(E, E, device=dev) / np.sqrt(E)  # noqa: E731
    zb = lambda: torch.zeros(E, device=dev)  # noqa: E731
    lp = LayerParams(torch.ones(E, device=dev), zb(), LinearParams(u(), zb()), LinearParams(u(), zb()),
                     LinearParams(u(), zb()), LinearParams(u(), zb()))
    engines, comm = make_sim_group(cfg, lp, G, device=dev)
    x = torch.randn(1, l, E, device=dev)
    gy = torch.randn(1, l, E, device=dev)
    K.runtime_config(numerics=True)
    lss_step(engines, comm, [slice_batch(x, ShardSpec(r, G, l)) for r in range(G)],
             [slice_batch(gy, ShardSpec(r, G, l)) for r in range(G)])
    x[0, 300, 1] = float("nan")
    with pytest.raises(NumericsError):
        lss_step(engines, comm, [slice_batch(x, ShardSpec(r, G, l)) for r in range(G)],
                 [slice_batch(gy, ShardSpec(r, G, l)) for r in range(G)])
