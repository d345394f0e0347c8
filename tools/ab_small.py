"""Same-process A/B of the small HBM-bound kernels of one N=1 step (LayerNorm fwd/bwd,
cast + column sums) across two builds: python tools/ab_small.py libA.so libB.so"""
import os, statistics, sys, torch
sys.path.insert(0, ".")
from paper_2311_02382_b200 import _native
from paper_2311_02382_b200 import kernels as K

libs = []
for p in sys.argv[1:3]:
    _native._lib = None
    os.environ["LSS_LIB"] = p
    libs.append(_native.load())
dev = torch.device("cuda:0")
M, E = 50112, 1024
g = torch.Generator(device=dev).manual_seed(0)
r = lambda *s: torch.randn(*s, generator=g, device=dev)  # noqa: E731
x, gxh, gres = r(M, E), r(M, E), r(M, E)
gain, bias = r(E), r(E)
xh = torch.empty(M, E, dtype=torch.bfloat16, device=dev)
mean, rstd = torch.empty(M, device=dev), torch.empty(M, device=dev)
gx, gg, gb = torch.empty(M, E, device=dev), torch.zeros(E, device=dev), torch.zeros(E, device=dev)
dq, dkv = r(M, E), r(M, 2 * E)
dqkv, cs = torch.empty(M, 3 * E, dtype=torch.bfloat16, device=dev), torch.zeros(3 * E, device=dev)
cases = {
    "layernorm_fwd": lambda: K.layernorm_fwd(x, gain, bias, out=xh, mean=mean, rstd=rstd),
    "layernorm_bwd": lambda: K.layernorm_bwd(gxh, x, mean, rstd, gain, grad_res=gres, grad_x=gx, grad_gain=gg,
                                             grad_bias=gb, alpha=1.0),
    "cat_cast_colsum": lambda: K.cat_cast_colsum([(dq, E, E), (dkv, 2 * E, 2 * E)], M, dst=dqkv, colsum=cs),
}
res = {(i, n): [] for i in range(2) for n in cases}
for rep in range(12):
    for i in ((0, 1) if rep % 2 == 0 else (1, 0)):
        _native._lib = libs[i]
        for n, f in cases.items():
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record(); f(); b.record(); torch.cuda.synchronize()
            if rep >= 2:
                res[(i, n)].append(a.elapsed_time(b) * 1e3)
for n in cases:
    print(f"{n:18s} A {statistics.median(res[(0, n)]):7.1f} us   B {statistics.median(res[(1, n)]):7.1f} us")
