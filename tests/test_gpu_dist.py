"""Multi-process parity of the LSS layer against the real reference's goldens.
Runs tests/dist_check.py / hybrid_check.py under torchrun, 3 consecutive steps
each (golden, fresh inputs vs the oracle, golden again).  NCCL cases need one GPU
per rank; the oversubscribed cases run 8 ranks (the 8-GPU protocol: 8-slot
fused reduce-scatter, 4 balanced pairs, flag hand-offs, the 2 x 4 hybrid fold)
on whatever GPUs are visible, several ranks per GPU, with gloo as the process
group (NCCL refuses two ranks on one device) and the same IPC / flag data plane.
The CPU gloo tests in test_dist_gloo.py cover the host logic everywhere."""

import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _gpus():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("case,world,fused", [("configA", 2, 1), ("batch2_g3", 3, 1), ("small_causal", 2, 1),
                                              ("small_noncausal", 4, 1), ("configA", 2, 0), ("small_causal", 4, 0),
                                              ("full_g2_causal", 2, 1), ("drop_layer_g2", 2, 1),
                                              ("drop_layer_g2_big", 2, 1), ("configA", 4, 1),
                                              ("drop_layer_g2_big", 4, 1)])
def test_nccl_lss_layer_matches_reference(case, world, fused):
    """fused=1: dK|dV reduce-scatter fused into the backward over NVLink peer memory
    (lss_attn_bwd_p2p + barrier + slot sum); fused=0: the NCCL reduce-scatter."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    import os

    from conftest import free_port

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(ROOT / "tests" / "dist_check.py"),
           "--case", case, "--expect-fused", str(fused), "--fused-rs", str(fused), "--steps", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=dict(os.environ))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout


def test_nccl_hybrid_grid_training_step():
    """2 x 2 hybrid grid (two replicas of a 2-rank sequence group) over NCCL:
    one step of run_steps == the oracle's doubly averaged SGD update."""
    if _gpus() < 4:
        pytest.skip("needs 4 GPUs")
    from conftest import free_port

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(ROOT / "tests" / "hybrid_check.py"),
           "--steps", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout


def _oversubscribed(script, args, world=8):
    if _gpus() < 1:
        pytest.skip("needs a GPU")
    from conftest import free_port

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(ROOT / "tests" / script),
           "--backend", "gloo", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout
    return r.stdout


@pytest.mark.parametrize("case", ["ns_l2048_g8", "drop_layer_g2_big"])
def test_eight_rank_protocol_oversubscribed(case):
    """World 8 (BASELINE config 3's G=8): at E=1024 / 16 heads against the real
    reference's ns_l2048_g8 golden (m=256: every rank in a balanced pair), and with
    dropout at every site; 3 steps each."""
    out = _oversubscribed("dist_check.py", ["--case", case, "--steps", "3", "--expect-fused", "1"])
    if case.startswith("ns_"):
        assert "balanced=True" in out


def test_hybrid_two_by_four_oversubscribed():
    """BASELINE config 5's 2 x 4 grid layout (replica-major, seq groups of 4 with the
    balanced schedule, data groups of 2), 2 SGD steps vs the doubly averaged oracle."""
    out = _oversubscribed("hybrid_check.py", ["--case", "configA", "--steps", "2"])
    assert "2x4" in out
