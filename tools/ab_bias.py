"""Interleaved A/B of the balanced schedule's split bias (one engine per bias)."""
import math, os, sys, torch, torch.distributed as dist
sys.path.insert(0, ".")
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
biases = [int(a) for a in sys.argv[1:]] or [0, 2, 4, 6]
engs = {}
for bval in biases:
    e = LSSAttention(cfg, spec, grad_scale=1.0 / world, device=dev, split_bias=bval)
    e.load_params(lp)
    for _ in range(3):
        e.step(x, gy, comm)
    engs[bval] = e
torch.cuda.synchronize()
res = {b_: [] for b_ in biases}
for rep in range(8):
    for bval in biases[rep % len(biases):] + biases[:rep % len(biases)]:  # rotate: no position bias
        e = engs[bval]
        e.step(x, gy, comm)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):
            e.step(x, gy, comm)
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / 4], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[bval].append(t.item())
if rank == 0:
    for bval, v in res.items():
        v = sorted(v)
        print(f"N={world} bias {bval:2d} split {engs[bval].plan.split:5d} median {v[len(v)//2]:.3f} ms  min {v[0]:.3f}",
              flush=True)
dist.destroy_process_group()
