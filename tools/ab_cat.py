"""Same-process A/B of the backward's cast + bias-gradient column sums ([dQ | dK|dV] fp32
-> bf16 [m, 3E], l=50112, E=1024) across two builds: python tools/ab_cat.py libA.so libB.so"""
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
dq, dkv = torch.randn(M, E, device=dev), torch.randn(M, 2 * E, device=dev)
dst = torch.empty(M, 3 * E, dtype=torch.bfloat16, device=dev)
res, times = [], {0: [], 1: []}
for rep in range(12):
    for i, lib in enumerate(libs):
        _native._lib = lib
        cs = torch.zeros(3 * E, device=dev)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        K.cat_cast_colsum([(dq, E, E), (dkv, 2 * E, 2 * E)], M, dst=dst, colsum=cs, alpha=0.5)
        e1.record()
        torch.cuda.synchronize()
        if rep == 0:
            res.append((dst.float().clone(), cs.clone()))
        elif rep >= 2:
            times[i].append(e0.elapsed_time(e1))
for i in range(2):
    print(sys.argv[1 + i], "cat_cast median %.1f us" % (1e3 * statistics.median(times[i])))
print("max |ddst|", (res[0][0] - res[1][0]).abs().max().item(),
      "rel dcolsum", ((res[0][1] - res[1][1]).abs().max() / res[0][1].abs().max()).item())
