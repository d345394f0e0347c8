"""Same-process A/B of the GEMM shapes of one LSS step (N=1, l=50112, E=1024) across
two builds of liblss.so (same ABI): python tools/ab_gemm.py libA.so libB.so"""
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
bf = torch.bfloat16
g = torch.Generator(device=dev).manual_seed(0)
r = lambda *s, dt=bf: torch.randn(*s, generator=g, device=dev).to(dt)  # noqa: E731
xh, w3t, b3 = r(M, E), r(3 * E, E), r(3 * E, dt=torch.float32)
q, kv = torch.empty(M, E, dtype=bf, device=dev), torch.empty(M, 2 * E, dtype=bf, device=dev)
ctx, wo_t, bo, x = r(M, E), r(E, E), r(E, dt=torch.float32), r(M, E, dt=torch.float32)
y = torch.empty(M, E, device=dev)
dqkv, w3 = r(M, 3 * E), r(E, 3 * E)
dxh, gw3 = torch.empty(M, E, device=dev), torch.empty(E, 3 * E, device=dev)
cases = {
    "qkv fwd (bf16 out, bias, split)": lambda: K.gemm(xh, w3t, bias=b3, seg_width=E, out=[(q, E), (kv[:, :E], 2 * E),
                                                                                          (kv[:, E:], 2 * E)],
                                                        M=M, N=3 * E, K=E),
    "out-proj (fp32 out, bias, residual)": lambda: K.gemm(ctx, wo_t, bias=bo, residual=x, out=y, M=M, N=E, K=E),
    "dx (fp32 out, K=3E)": lambda: K.gemm(dqkv, w3, out=dxh, M=M, N=E, K=3 * E),
    "dWqkv (fp32 out, MN-major, K=l)": lambda: K.gemm(xh, dqkv, a_mn_major=True, b_mn_major=True, out=gw3, M=E,
                                                      N=3 * E, K=M),
}
res = {(i, n): [] for i in range(2) for n in cases}
for rep in range(10):
    for i in ((0, 1) if rep % 2 == 0 else (1, 0)):
        _native._lib = libs[i]
        for n, f in cases.items():
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record(); f(); b.record(); torch.cuda.synchronize()
            if rep >= 2:
                res[(i, n)].append(a.elapsed_time(b) * 1e3)
for n in cases:
    print(f"{n:40s} A {statistics.median(res[(0, n)]):7.1f} us   B {statistics.median(res[(1, n)]):7.1f} us")
