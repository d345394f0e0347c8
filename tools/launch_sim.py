"""Per-launch forward timing of a G-way rank (fused/unsplit structure), vs the wave model."""
import sys, torch, heapq
sys.path.insert(0, ".")
from paper_2311_02382_b200.model import LayerParams, LinearParams, ModelConfig
from paper_2311_02382_b200.sharded import LSSAttention, ShardSpec, fwd_cta_tiles, choose_fwd_splits
from paper_2311_02382_b200 import balance as BAL
from paper_2311_02382_b200 import engine as ENG
from paper_2311_02382_b200 import kernels as K

l, E, H = 50112, 1024, 16
dev = torch.device("cuda", 0)
cfg = ModelConfig(embed_dim=E, n_layers=1, n_heads=H, ff_dim=4 * E, vocab=256, seq_len=l)
g = torch.Generator(device=dev).manual_seed(0)
US = 1.447
def tm(f, n=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for r in [int(a) for a in sys.argv[2:]] or [0, G - 1]:
    e = LSSAttention(cfg, ShardSpec(r, G, l), device=dev)
    for t in (e.q, e.kv_full):
        t.normal_(generator=g)
    if hasattr(e, "q_peer"):
        e.q_peer.normal_(generator=g)
    m = e.m
    jobs = [(e.q, row0, rows, e.spec.offset, g0, g1, e.ctx, e.lse2) for row0, rows, g0, g1 in e.own_ranges()]
    pl = e.plan
    if pl.role == "light":
        jobs.append((e.q_peer, 0, pl.split, pl.partner * m, 0, pl.a, e.o_peer, e.lse_peer))
        if pl.b:
            jobs.append((e.q_peer, pl.split, m - pl.split, pl.partner * m, 0, pl.b, e.o_peer, e.lse_peer))
    tot = 0
    for q, row0, rows, off, g0, g1, out, lse in jobs:
        tiles = fwd_cta_tiles(rows, off + row0, g0, g1, m, True)
        ideal = sum(tiles) * 16 / 148 * US
        res = []
        for S in (1, 2, 3, 4, 6):
            BAL._SPLIT_CACHE.clear()
            old = ENG.choose_fwd_splits
            f = lambda: e._attn_part(q, rows=rows, row0=row0, offset=off, g_begin=g0, g_end=g1, out=out, lse2=lse)
            ENG.choose_fwd_splits = lambda *a, S=S: S  # the engine's split choice, forced
            res.append((S, round(tm(f), 1)))
            ENG.choose_fwd_splits = old
        BAL._SPLIT_CACHE.clear()
        pick = choose_fwd_splits(rows, off + row0, g0, g1, m, True, 16, 148, E)
        print(f"G={G} r={r} {pl.role:5s} rows={rows:5d} pos0={off+row0:6d} segs=[{g0},{g1}) ctas={len(tiles)*16:4d} "
              f"maxtiles={max(tiles)} ideal={ideal:6.1f}us pick S={pick} measured {res}", flush=True)
    del e
    torch.cuda.empty_cache()
