"""A/B kernel timing: python tools/abn.py libA.so libB.so [fwd|bwd]"""
import sys, ctypes, statistics, numpy as np, torch
sys.path.insert(0, '.')
from paper_2311_02382_b200 import _native
libs = []
for path in [a for a in sys.argv[1:] if a.endswith(".so")]:
    lib = ctypes.CDLL(path)
    for name, argt in _native.SIGNATURES.items():
        if hasattr(lib, name):
            getattr(lib, name).argtypes = argt; getattr(lib, name).restype = ctypes.c_int
    libs.append(lib)
which = 'fwd' if 'fwd' in sys.argv else 'bwd'
NL = len(libs)
dev = torch.device('cuda:0')
B, m, E, H = 1, 50112, 1024, 16
torch.manual_seed(0)
q = torch.randn(B, m, E, device=dev).bfloat16(); kv = torch.randn(1, B, m, 2 * E, device=dev).bfloat16()
mp = (m + 127) // 128 * 128
o = torch.empty(B, m, E, device=dev, dtype=torch.bfloat16); lse = torch.empty(B, H, mp, device=dev)
go = torch.randn(B, m, E, device=dev).bfloat16()
dq = torch.empty(B, m, E, device=dev); dkv = torch.empty(1, B, m, 2 * E, device=dev); dl = torch.empty(B, H, mp, device=dev)
P = lambda t: ctypes.c_void_p(t.data_ptr())
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
kp, vp = ctypes.c_void_p(kv.data_ptr()), ctypes.c_void_p(kv.data_ptr() + E * 2)
def fwd(lib): return lib.lss_attn_fwd(0, P(q), kp, vp, 2 * E, P(o), P(lse), B, m, 1, m, H, 64, 0, 1, s)
def bwd(lib): return lib.lss_attn_bwd(0, P(q), kp, vp, 2 * E, P(o), P(go), P(lse), P(dl), P(dq), ctypes.c_void_p(dkv.data_ptr()), ctypes.c_void_p(dkv.data_ptr() + E * 4), 2 * E, B, m, 1, m, H, 64, 0, 1, s)
assert fwd(libs[0]) == 0
fn = bwd if which == 'bwd' else fwd
times = {i: [] for i in range(NL)}
for rep in range(12):
    for i in range(NL):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); rc = fn(libs[i]); e1.record(); torch.cuda.synchronize()
        assert rc == 0
        if rep >= 2: times[i].append(e0.elapsed_time(e1))
for i in range(NL):
    print([a for a in sys.argv[1:] if a.endswith('.so')][i], which, 'median %.3f ms  min %.3f' % (statistics.median(times[i]), min(times[i])))
