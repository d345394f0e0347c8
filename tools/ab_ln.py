"""Same-process A/B of the LayerNorm forward and backward at l=50112, E=1024 across two
builds: python tools/ab_ln.py libA.so libB.so"""
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
x = torch.randn(50112, 1024, device=dev)
gxh, res = torch.randn(50112, 1024, device=dev), torch.randn(50112, 1024, device=dev)
g, b = torch.randn(1024, device=dev), torch.randn(1024, device=dev)
outs = []
for rep in range(12):
    for i, lib in enumerate(libs):
        _native._lib = lib
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        y, mu, rs = K.layernorm_fwd(x, g, b)
        e1.record()
        e2 = torch.cuda.Event(True)
        gx, ggain, gbias = K.layernorm_bwd(gxh, x, mu, rs, g, grad_res=res,
                                           grad_gain=torch.zeros(1024, device=dev), grad_bias=torch.zeros(1024, device=dev))
        e2.record()
        torch.cuda.synchronize()
        if rep == 0:
            outs.append((y.float().clone(), mu.clone(), gx.clone(), ggain.clone()))
        elif rep >= 2:
            outs.append((i, e0.elapsed_time(e1), e1.elapsed_time(e2)))
for i in range(2):
    t = [v for j, v, _ in outs[2:] if j == i]
    tb = [v for j, _, v in outs[2:] if j == i]
    print(sys.argv[1 + i], "ln fwd median %.1f us, bwd %.1f us" % (1e3 * statistics.median(t), 1e3 * statistics.median(tb)))
print("max |dy|", (outs[0][0] - outs[1][0]).abs().max().item(), "max |dmu|", (outs[0][1] - outs[1][1]).abs().max().item(),
      "max |dgx|", (outs[0][2] - outs[1][2]).abs().max().item(),
      "rel dgain", ((outs[0][3] - outs[1][3]).abs().max() / outs[0][3].abs().max()).item())
