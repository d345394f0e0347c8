"""Forward kernel: plain instance vs PART instance (always-ready flags), same lib, N=1 shape.
python tools/ab_part.py [lib.so ...]"""
import sys, ctypes, statistics, torch
sys.path.insert(0, '.')
from paper_2311_02382_b200 import _native
paths = [a for a in sys.argv[1:] if a.endswith(".so")] or ["paper_2311_02382_b200/liblss.so"]
dev = torch.device('cuda:0')
B, m, E, H = 1, 50112, 1024, 16
torch.manual_seed(0)
q = torch.randn(B, m, E, device=dev).bfloat16(); kv = torch.randn(1, B, m, 2 * E, device=dev).bfloat16()
mp = (m + 127) // 128 * 128
o = torch.empty(B, m, E, device=dev, dtype=torch.bfloat16); lse = torch.empty(B, H, mp, device=dev)
flags = torch.ones(4, dtype=torch.int32, device=dev)
P = lambda t: ctypes.c_void_p(t.data_ptr())
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
kp, vp = ctypes.c_void_p(kv.data_ptr()), ctypes.c_void_p(kv.data_ptr() + E * 2)
fns = []
for path in paths:
    lib = ctypes.CDLL(path)
    for name, argt in _native.SIGNATURES.items():
        if hasattr(lib, name):
            getattr(lib, name).argtypes = argt; getattr(lib, name).restype = ctypes.c_int
    fns.append((path + " plain", lambda lib=lib: lib.lss_attn_fwd(0, P(q), kp, vp, 2 * E, P(o), P(lse), B, m, 1, m, H, 64, 0, 1, s)))
    fns.append((path + " PART", lambda lib=lib: lib.lss_attn_fwd_split(0, P(q), m, m * E, kp, vp, 2 * E, P(o), m * E, P(lse), mp, B, 1, m, H, 64, 0, 1, 0, 1, None, 1, None, 0, None, 0, P(flags), 0, 0, s)))
times = {n: [] for n, _ in fns}
for rep in range(12):
    for n, f in (fns[rep % len(fns):] + fns[:rep % len(fns)]):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); rc = f(); e1.record(); torch.cuda.synchronize()
        assert rc == 0, n
        if rep >= 2: times[n].append(e0.elapsed_time(e1))
for n, _ in fns:
    print(n, 'median %.3f ms  min %.3f' % (statistics.median(times[n]), min(times[n])))
