"""Causal load balancing of the LSS engine and the forward launch-split model.

With contiguous segments (ShardSpec, reference sharded.py:37-61 -- required for
bit-exact segment ownership) and the causal mask (model.py:301-304), rank r
attends to r full key segments plus its diagonal, so the slowest rank bounds
a G-way group at (G/2)/(G - 1/2) of ideal.  ``BalancePlan``
pairs rank r with G-1-r without changing ownership; ``choose_fwd_splits``
picks the in-launch key split of the partial forward launches by simulating
their dispatch onto the SMs.
"""

from __future__ import annotations

from dataclasses import dataclass

@dataclass(frozen=True)
class BalancePlan:
    """Balanced causal schedule for one rank (ownership unchanged).

    With contiguous segments (ShardSpec) and the causal mask, rank r attends to
    r full key segments plus its diagonal: work ~ (r + 1/2) m^2, so the slowest
    rank bounds the group at (G/2)/(G - 1/2) of ideal.  Pairing rank r with
    G-1-r gives every pair exactly G m^2 of work; the heavy rank delegates
    D2 = 2r - G + 1 half-blocks (query-row half x full key segment) to its light
    partner: its top rows [0, split) against key segments [0, a) and its bottom
    rows [split, m) against [0, b), a + b = D2.  The partner needs the heavy
    rank's Q rows (sent forward) and returns normalised partial contexts + lse,
    merged by log-sum-exp; backward it receives dO, lse, delta and returns dQ
    rows, while its dK/dV contributions land in its own packed buffer, so the
    reduce-scatter is unchanged.  Extra traffic per step: 2 (B m E) bf16 + 1
    (B m E) fp32 each way -- small next to the K/V gather.
    """

    role: str = "none"  # "none" | "heavy" | "light"
    partner: int = -1
    split: int = 0      # first bottom row (multiple of 128)
    a: int = 0          # delegated key segments for the top rows: [0, a)
    b: int = 0          # delegated key segments for the bottom rows: [0, b)

    @property
    def active(self) -> bool:
        return self.role != "none"


def make_plan(rank: int, workers: int, block: int, causal: bool, bias_tiles: int = 0) -> BalancePlan:
    """``bias_tiles``: move the split down by that many 128-row tiles, i.e. hand
    bias_tiles*128*block more (query, key) pairs per (batch, head) from every heavy
    rank to its light partner (a - b = 1 for every pair) -- balances measured time
    rather than pair counts (the heavy rank's mix runs slower per pair)."""
    if not causal or workers < 2:
        return BalancePlan()
    split = (block // 2) // 128 * 128
    if split == 0:
        return BalancePlan()
    split = max(128, min(split + 128 * bias_tiles, (block - 1) // 128 * 128))
    partner = workers - 1 - rank
    d2 = lambda r: 2 * r - workers + 1  # noqa: E731  half-blocks rank r must give away
    if d2(rank) > 0:
        n = d2(rank)
        return BalancePlan("heavy", partner, split, (n + 1) // 2, n // 2)
    if partner != rank and d2(partner) > 0:
        n = d2(partner)
        return BalancePlan("light", partner, split, (n + 1) // 2, n // 2)
    return BalancePlan()


_SPLIT_MAX = 8
# per-CTA fixed cost (launch, prologue, pipeline fill / drain, epilogue) in key-tile
# units (~1.45 us each): fitted to per-launch timings of the G=4 / G=8 partial
# launches (scratch/launch_sim.py; the model then picks the measured-best S for
# 11 of 12 launches, 3 us lost in total)
_TILE_OVH = 8.0
_SPLIT_CACHE: dict = {}


def fwd_cta_tiles(rows: int, pos0: int, g0: int, g1: int, seg_len: int, causal: bool) -> list:
    """Visible key tiles of each query-tile-pair CTA of a partial forward launch, in
    grid order (heaviest first for causal), as attn_fwd_tc_kernel counts them."""
    tps = -(-seg_len // 128)
    n_pairs = -(-rows // 256)
    out = []
    for unit in range(n_pairs):
        pair = n_pairs - 1 - unit if causal else unit
        if not causal:
            out.append((g1 - g0) * tps)
            continue
        max_key = pos0 + min(pair * 256 + 256, rows) - 1
        n = 0
        for g in range(g0, g1):
            seg0 = g * seg_len
            if seg0 > max_key:
                break
            n = (g - g0) * tps + min(seg_len - 1, max_key - seg0) // 128 + 1
        out.append(n)
    return out


def choose_fwd_splits(rows: int, pos0: int, g0: int, g1: int, seg_len: int, causal: bool, slices: int,
                      sms: int, embed: int) -> int:
    """Key-split count for one partial forward launch: the S minimising the simulated
    makespan of the grid (CTAs dispatched in grid order to the first free SM, each
    split a CTA of ceil(n/S) tiles + the fixed cost) plus the N-way merge."""
    key = (rows, pos0, g0, g1, seg_len, causal, slices, sms, embed)
    if key in _SPLIT_CACHE:
        return _SPLIT_CACHE[key]
    import heapq

    tiles = fwd_cta_tiles(rows, pos0, g0, g1, seg_len, causal)
    best, best_t = 1, None
    for S in range(1, _SPLIT_MAX + 1):
        if S > 1 and max(tiles) < 4 * S:
            break
        free = [0.0] * sms
        for g0s in range(0, slices, 4):  # grid: groups of 4 slices (ATT_FWD_HGROUP), heavy pairs first
            for n in tiles:
                for _ in range(min(4, slices - g0s)):
                    for s in range(S):
                        c = (s + 1) * n // S - s * n // S + _TILE_OVH
                        heapq.heappush(free, heapq.heappop(free) + c)
        t = max(free)
        if S > 1:  # merge: reads S partials + writes the result (~1.45 us per tile unit, ~6 TB/s)
            t += 1.5 + rows * embed * 2 * (S + 1) / 6e12 / 1.45e-6
        if best_t is None or t < best_t * 0.97:
            best, best_t = S, t
    _SPLIT_CACHE[key] = best
    return best


def block_pairs(rows: int, p0: int, lo: int, hi: int, causal: bool) -> int:
    """Unmasked pairs of query rows at positions p0..p0+rows-1 against keys [lo, hi):
    sum_i clamp(p0 + i + 1 - lo, 0, hi - lo) (causal) or rows * (hi - lo)."""
    w = hi - lo
    if not causal:
        return rows * w
    c0 = p0 + 1 - lo
    i_a = max(0, 1 - c0)            # first row with a visible key
    i_b = max(0, w - c0)            # first row seeing the whole range
    e1 = min(rows, i_b)
    part = 0
    if e1 > i_a:
        n = e1 - i_a
        part = n * c0 + (i_a + e1 - 1) * n // 2
    if rows > i_b:
        part += (rows - i_b) * w
    return part
