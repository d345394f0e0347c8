"""Per-rank compute cost of the sequence-sharded forward/backward attention phases,
one rank at a time on one GPU, no communication (buffers hold random data)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2311_02382_b200.model import LayerParams, LinearParams, ModelConfig
from paper_2311_02382_b200.sharded import LSSAttention, ShardSpec
from paper_2311_02382_b200 import kernels as K

l, E, H = 50112, 1024, 16
dev = torch.device("cuda", 0)
cfg = ModelConfig(embed_dim=E, n_layers=1, n_heads=H, ff_dim=4 * E, vocab=256, seq_len=l)
g = torch.Generator(device=dev).manual_seed(0)
u = lambda: (torch.rand(E, E, generator=g, device=dev) * 2 - 1) / E ** 0.5
zb = lambda: torch.zeros(E, device=dev)
lp = LayerParams(torch.ones(E, device=dev), zb(), LinearParams(u(), zb()), LinearParams(u(), zb()),
                 LinearParams(u(), zb()), LinearParams(u(), zb()))

def tm(f, n=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n

for G in [int(a) for a in sys.argv[1:]] or [4, 8]:
    for r in range(G):
        e = LSSAttention(cfg, ShardSpec(r, G, l), device=dev)
        e.load_params(lp)
        for t in (e.q, e.kv_full, e.dctx):
            t.normal_(generator=g)
        for nm in ("q_peer", "do_peer"):
            if hasattr(e, nm):
                getattr(e, nm).normal_(generator=g)
        def loc():
            e.fwd_attend_local(0); e.fwd_attend_local(1)
        def rem():
            e.fwd_attend_delegated(); e.fwd_attend_remote(1); e.fwd_attend_remote(0)
        t_loc = tm(loc)
        t_rem = tm(lambda: (loc(), rem())) - t_loc
        e.split_fwd = False
        t_unsplit = tm(e.fwd_attend)
        # valid lse for the bwd
        e.fwd_attend()
        if hasattr(e, "lsef_peer"):
            e.lsef_peer.copy_(e.lse_peer); e.delta_peer.zero_()
        e.seg_dst = None
        K.attn_delta(e.ctx, e.dctx, e.delta, heads=H, scaled=True)
        t_bwd = tm(e.bwd_attend)
        print(f"G={G} r={r} {e.plan.role:5s} pairs={e.computed_pairs()/ (l*l/2/G):.3f}  fwd local {t_loc:.3f} "
              f"remote {t_rem:.3f} sum {t_loc+t_rem:.3f} unsplit {t_unsplit:.3f}  bwd {t_bwd:.3f}", flush=True)
        del e
        torch.cuda.empty_cache()
