"""Interleaved same-process A/B of the multi-GPU step: modes toggled every few steps,
CUDA-event time per block, max over ranks.  torchrun --nproc-per-node N tools/ab_dist.py"""
import math, os, sys, torch, torch.distributed as dist
sys.path.insert(0, ".")
import dataclasses
from paper_2311_02382_b200.comm import Ledger, TorchDistComm
from paper_2311_02382_b200.model import LayerParams, LinearParams, ModelConfig
from paper_2311_02382_b200.sharded import LSSAttention, ShardSpec

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
comm = TorchDistComm(None, None, Ledger())
l, E = 50112, 1024
cfg = ModelConfig(embed_dim=E, n_layers=1, n_heads=16, ff_dim=4 * E, vocab=256, seq_len=l)
g = torch.Generator(device=dev).manual_seed(1)
u = lambda: (torch.rand(E, E, generator=g, device=dev) * 2 - 1) / math.sqrt(E)
z = lambda: torch.zeros(E, device=dev)
lp = LayerParams(torch.ones(E, device=dev), z(), LinearParams(u(), z()), LinearParams(u(), z()),
                 LinearParams(u(), z()), LinearParams(u(), z()))
spec = ShardSpec(rank, world, l)
x = torch.randn(1, spec.block, E, device=dev)
gy = torch.randn(1, spec.block, E, device=dev)
eng = LSSAttention(cfg, spec, grad_scale=1.0 / world, device=dev)
eng.load_params(lp)

MODES = {
    "fused+b1k": dict(ce=True, flags=True, split=True, fused=True, b1k=True),
    "fused": dict(ce=True, flags=True, split=True, fused=True, b1k=False),
    "ce+flags": dict(ce=True, flags=True, split=True, fused=False),
    "nccl-p2p": dict(ce=False, flags=False, split=True, fused=False),
}
sel = sys.argv[1:] or list(MODES)

def setmode(m):
    comm.use_flags = m["flags"]
    eng.options = dataclasses.replace(eng.options, ce_p2p=m["ce"], fwd_split=m["split"], fused_gather=m["fused"],
                                      b1_in_kernel=m.get("b1k", False))

for name in sel:  # warm every mode (maps buffers once, collectively)
    setmode(MODES[name])
    for _ in range(3):
        eng.step(x, gy, comm)
torch.cuda.synchronize()
res = {n: [] for n in sel}
for rep in range(8):
    for name in sel[rep % len(sel):] + sel[:rep % len(sel)]:  # rotate: no position bias
        setmode(MODES[name])
        eng.step(x, gy, comm)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):
            eng.step(x, gy, comm)
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / 4], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name].append(t.item())
if rank == 0:
    for n, v in res.items():
        v = sorted(v)
        print(f"N={world} {n:12s} median {v[len(v)//2]:.3f} ms  min {v[0]:.3f}  all {[round(a,2) for a in res[n]]}", flush=True)
dist.destroy_process_group()
