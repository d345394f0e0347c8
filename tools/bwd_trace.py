"""Per-tile event timeline of attn_bwd_tc_kernel / attn_fwd_tc_kernel (CTA 0, l=50112,
16 heads, causal).

    nvcc ... -DLSS_BWD_TRACE -DLSS_FWD_TRACE -o abvar/trace.so paper_2311_02382_b200/csrc/lss_capi.cu
    python tools/bwd_trace.py abvar/trace.so [fwd]

Prints, for the steady-state iterations, the median clock64 offset of each traced
event from the previous iteration's ds_full arrival (slot 4), i.e. where in the
tile period each warp role waits."""
import ctypes
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_02382_b200 import _native  # noqa: E402

SLOTS = {16: "MMA: issue_s start", 17: "MMA: S operands ready", 6: "MMA: p_full passed (dV)",
         14: "MMA: dV issued", 0: "MMA: ds_full passed (dK)", 15: "MMA: dP issued", 8: "MMA: dQ issued",
         1: "EW: s_full passed", 7: "EW: S loaded", 13: "EW: P computed", 2: "EW: p_full arrived",
         11: "EW: ds_free passed", 3: "EW: dp_full passed", 9: "EW: dS computed", 10: "EW: dS stored",
         12: "EW: dS^T in TMEM", 4: "EW: ds_full arrived", 5: "drain: dq_full passed", 18: "TMA: q_empty passed"}

FWD_SLOTS = {7: "MMA: kv_full passed", 5: "MMA: s_empty passed (S issue)", 6: "MMA: p_full passed (PV issue)",
             0: "softmax: s_full passed", 1: "softmax: S loaded, s_empty arrived", 2: "softmax: P computed",
             3: "softmax: o_full passed", 4: "softmax: p_full arrived"}
FWD = "fwd" in sys.argv[2:]
lib = ctypes.CDLL(sys.argv[1])
for name, argt in _native.SIGNATURES.items():
    if hasattr(lib, name):
        getattr(lib, name).argtypes = argt
        getattr(lib, name).restype = ctypes.c_int
dev = torch.device("cuda:0")
B, m, E, H = 1, 50112, 1024, 16
torch.manual_seed(0)
q = torch.randn(B, m, E, device=dev).bfloat16()
kv = torch.randn(1, B, m, 2 * E, device=dev).bfloat16()
mp = (m + 127) // 128 * 128
o = torch.empty(B, m, E, device=dev, dtype=torch.bfloat16)
lse = torch.empty(B, H, mp, device=dev)
go = torch.randn(B, m, E, device=dev).bfloat16()
dq = torch.empty(B, m, E, device=dev)
dkv = torch.empty(1, B, m, 2 * E, device=dev)
dl = torch.empty(B, H, mp, device=dev)
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
kp, vp = ctypes.c_void_p(kv.data_ptr()), ctypes.c_void_p(kv.data_ptr() + E * 2)
assert lib.lss_attn_fwd(0, P(q), kp, vp, 2 * E, P(o), P(lse), B, m, 1, m, H, 64, 0, 1, s) == 0
for _ in range(0 if FWD else 3):
    assert lib.lss_attn_bwd(0, P(q), kp, vp, 2 * E, P(o), P(go), P(lse), P(dl), P(dq),
                            ctypes.c_void_p(dkv.data_ptr()), ctypes.c_void_p(dkv.data_ptr() + E * 4), 2 * E,
                            B, m, 1, m, H, 64, 0, 1, s) == 0
torch.cuda.synchronize()
if FWD:
    tr = np.zeros((8, 1024), dtype=np.int64)
    assert lib.lss_debug_fwd_trace(tr.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong))) == 0
    SLOTS = FWD_SLOTS
    n = int((tr[4] != 0).sum())
    its = range(20, max(21, n - 5))
else:
    tr = np.zeros((20, 512), dtype=np.int64)
    assert lib.lss_debug_bwd_trace(tr.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong))) == 0
    its = range(40, 400)
period = statistics.median(tr[4][i] - tr[4][i - 1] for i in its)
print(f"tile period ({'p_full' if FWD else 'ds_full'} to next): {period:.0f} cycles over {len(its)} tiles")
rows = []
for slot, name in SLOTS.items():
    offs = [int(tr[slot][i] - tr[4][i - 1]) for i in its if tr[slot][i] and tr[4][i - 1]]
    if offs:
        rows.append((statistics.median(offs), name, slot))
for off, name, slot in sorted(rows):
    print(f"{off:8.0f}  {name} (slot {slot})")
