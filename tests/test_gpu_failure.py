"""Failure and numerics semantics on the B200 (ABI v9, include/lss.h).

* A cross-GPU wait whose peer never signals does not hang the GPU: every wait
  on a flag -- the attention kernels' in-kernel waits and the bounded stream
  waits (one-warp spin kernels) -- gives up at its deadline and the host raises
  CommTimeout (the reference's rendezvous timeout, collectives.py:242-252); a
  host abort releases them at once (CommAborted, collectives.py:200-209).
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
    K.attn_fwd_partial(q, kv[..., :E], kv[..., E:], rows=m, row0=0, workers=G, seg_len=m, heads=H, offset=m,
                       causal=True, g_begin=0, g_end=G, out=out, lse2=lse, ready=(flags, 1, 1))
    assert _drain(torch.cuda.current_stream()) < 30  # the producer gave up at the deadline
    with pytest.raises(CommTimeout):
        K.raise_status()
    K.raise_status()  # cleared


def _drain(stream, limit=30.0):
    """Poll (no blocking synchronize) until the stream drained; seconds taken."""
    t0 = time.monotonic()
    while not stream.query():
        assert time.monotonic() - t0 < limit, "stream did not drain"
        time.sleep(0.01)
    return time.monotonic() - t0


def test_bounded_stream_wait_deadline(runtime):
    """A flag nobody signals: the bounded stream wait (one-warp spin kernel) gives up at
    the deadline, the stream drains, the host raises CommTimeout."""
    import torch
    from paper_2311_02382_b200.errors import CommTimeout

    K = runtime
    K.runtime_config(wait_timeout_s=0.3)
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    flags[2] = 9  # already satisfied; 0, 1 and 3 never are (index 1 is skipped)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        K.stream_wait_bounded(flags.data_ptr(), 4, 1, 7, s)
        y = torch.ones(8, device="cuda") * 2
    assert _drain(s) < 20
    assert float(y.sum()) == 16.0
    with pytest.raises(CommTimeout):
        K.raise_status()


def test_guarded_stream_wait_deadline(runtime):
    """The engine's default stream wait: front-end waits plus a guard kernel that, past
    the deadline, raises the status word and writes the flags so the stream drains."""
    import torch
    from paper_2311_02382_b200.errors import CommTimeout

    K = runtime
    K.runtime_config(wait_timeout_s=0.3)
    flags = torch.zeros(3, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        K.stream_wait_guarded(flags.data_ptr(), 3, 0, 7, s)  # words 1, 2 never signalled
        y = torch.ones(8, device="cuda") * 3
    assert _drain(s) < 20
    assert float(y.sum()) == 24.0
    assert int(flags[1]) >= 7 and int(flags[2]) >= 7 and int(flags[0]) == 0  # released by the guard
    with pytest.raises(CommTimeout):
        K.raise_status()


def test_guarded_wait_satisfied_by_signal(runtime):
    import torch

    K = runtime
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    s, t = torch.cuda.Stream(), torch.cuda.Stream()
    K.stream_wait_guarded(flags.data_ptr(), 2, -1, 5, s)
    K.stream_signal(flags.data_ptr(), 5, t)
    K.stream_signal(flags.data_ptr() + 4, 6, t)
    assert _drain(s) < 20
    torch.cuda.synchronize()  # the guard kernel exits once the flags landed
    assert K.status(clear=True) == (False, False)
    assert int(flags[0]) == 5 and int(flags[1]) == 6  # not touched by the guard


def test_host_abort_releases_waits(runtime):
    """Communicator.abort semantics: with a long deadline, the host abort word releases
    a parked wait at once (collectives.py:200-209)."""
    import torch

    K = runtime
    K.runtime_config(wait_timeout_s=120.0)
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    K.stream_wait_bounded(flags.data_ptr(), 1, -1, 5, s)
    time.sleep(0.3)
    assert not s.query()  # still parked
    K.abort_waits(True)
    try:
        assert _drain(s) < 20
    finally:
        K.abort_waits(False)
    assert K.status(clear=True) == (False, False)  # an abort is not a timeout


def test_bounded_wait_satisfied_by_signal(runtime):
    """The normal path: a stream signal on another stream satisfies the bounded wait."""
    import torch

    K = runtime
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    s, t = torch.cuda.Stream(), torch.cuda.Stream()
    K.stream_wait_bounded(flags.data_ptr(), 2, -1, 3, s)
    K.stream_signal(flags.data_ptr(), 3, t)
    K.stream_signal(flags.data_ptr() + 4, 4, t)
    assert _drain(s) < 20
    assert K.status(clear=True) == (False, False)


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
