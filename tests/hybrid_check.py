"""D x N hybrid training-step check under torchrun (2 x world/2 grid):

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tests/hybrid_check.py [--case configA --steps 2]

A 2 x N grid (GridLayout, replica-major): two replicas, each an N-worker LSS
sequence group with its own data (at world 8: BASELINE config 5's 2 x 4
layout).  Every rank runs hybrid.run_engine_steps (layer fwd + bwd, the folded
world all-reduce with 1/(D*N), SGD update of the bound parameters) for
``--steps`` steps; after each step rank 0 checks the parameter update against
the oracle's (1/D) sum_d (group-averaged grads of replica d) at the parameters
that step started from, and all ranks must hold identical parameters
(hybrid.train_step, hybrid.py:95-126).  One GPU per rank.
Invoked by tests/test_gpu_dist.py.
"""

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import torch
    import torch.distributed as dist

    from conftest import nerr
    from oracle import lss_oracle as O
    from paper_2311_02382_b200 import optim
    from paper_2311_02382_b200.comm import Ledger, TorchDistComm
    from paper_2311_02382_b200.hybrid import GridLayout, make_groups, run_engine_steps
    from paper_2311_02382_b200.model import ModelConfig, layer_params_from_arrays
    from paper_2311_02382_b200.sharded import LSSAttention, ShardSpec, slice_batch

    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="small_causal")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    args = ap.parse_args()
    if int(os.environ["LOCAL_WORLD_SIZE"]) > torch.cuda.device_count():
        # kernels that spin on flags other ranks write must not share a GPU across processes
        # (Xid 109 context-switch timeouts on this driver, B200_PROFILING.md)
        raise SystemExit("one GPU per rank required")
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    lay = GridLayout(2, world // 2)
    replica, seq_index = lay.coords(rank)
    seq_g, _data_g, world_g = make_groups(lay)
    z = np.load(ROOT / "tests" / "golden" / f"{args.case}.npz")
    seq, e, h, _g, b, causal = (int(v) for v in z["meta"])
    names = ("ln1_gain", "ln1_bias", "wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo")
    cfg = ModelConfig(embed_dim=e, n_layers=1, n_heads=h, ff_dim=8, vocab=16, seq_len=seq, batch=b,
                      causal=bool(causal))
    lp = layer_params_from_arrays(*[z[k] for k in names], device=dev)
    datas = [(z["x"], z["grad_y"])]
    r = np.random.default_rng(11)
    datas.append((r.standard_normal(z["x"].shape).astype(np.float32),
                  r.standard_normal(z["x"].shape).astype(np.float32)))
    spec = ShardSpec(seq_index, lay.seq_workers, seq)
    eng = LSSAttention(cfg, spec, grad_scale=lay.grad_scale, device=dev)
    eng.bind_params(lp)
    x = torch.as_tensor(datas[replica][0], device=dev)
    gy = torch.as_tensor(datas[replica][1], device=dev)
    comm = TorchDistComm(seq_g, world_g, Ledger())
    lr = 1e-2
    ok = True
    order = dict(zip(["ln1_gain", "ln1_bias", "attn_q.weight", "attn_q.bias", "attn_k.weight", "attn_k.bias",
                      "attn_v.weight", "attn_v.bias", "attn_out.weight", "attn_out.bias"], names))
    for step in range(args.steps):
        p0 = eng.params.clone()
        comm.ledger.clear()
        norms = run_engine_steps(eng, comm, [(slice_batch(x, spec), slice_batch(gy, spec))], optim.SGD(lr))
        torch.cuda.synchronize()
        comm.check()
        allp = [torch.empty_like(eng.params) for _ in range(world)]
        if args.backend == "nccl":
            dist.all_gather(allp, eng.params)
        else:
            cpu = [torch.empty(eng.params.numel()) for _ in range(world)]
            dist.all_gather(cpu, eng.params.cpu())
            allp = cpu
        ok = ok and all(torch.equal(a, allp[0]) for a in allp)
        if rank == 0:
            start = {n: t.double().cpu().numpy() for n, t in eng._flat_views(p0).items()}
            p = O.AttnParams(*[start[ours] for ours in order])
            gs = [O.lss_attention(xd.astype(np.float64), gd.astype(np.float64), p, h, lay.seq_workers,
                                  bool(causal))["grads"] for xd, gd in datas]
            upd = (eng.params - p0).double().cpu().numpy()
            got = {n: t for n, t in eng._flat_views(torch.as_tensor(upd)).items()}
            for ours, gold in order.items():
                if gold == "bk":
                    continue
                want = -lr * (getattr(gs[0], gold) + getattr(gs[1], gold)) / 2.0  # (1/D) sum_d
                err = nerr(got[ours].numpy(), want)
                if err > 2e-2:
                    print(f"hybrid_check step {step}: {ours} update error {err:.3e}", flush=True)
                    ok = False
            ok = ok and comm.ledger.count("all-reduce") == 1 and len(norms) == 1 and np.isfinite(norms[0])
    if rank == 0:
        print(f"hybrid_check 2x{lay.seq_workers} {args.case} backend={args.backend} steps={args.steps}: "
              f"{'OK' if ok else 'FAIL'} (fused_rs={eng.seg_dst is not None}, balanced={eng.plan.active})", flush=True)
    flag = torch.tensor([0 if ok else 1], device=dev if args.backend == "nccl" else "cpu")
    dist.all_reduce(flag)
    dist.destroy_process_group()
    sys.exit(int(flag.item() != 0))


if __name__ == "__main__":
    main()
