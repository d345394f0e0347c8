// Segment attention forward for the LSS layer on sm_100a (tcgen05 + TMEM + TMA).
//
// Semantics follow model.scores_fwd (reference model.py:280-326): for this
// rank's query rows (global positions offset..offset+m) against the keys and
// values of the WHOLE sequence, S = Q_h K_h^T / sqrt(d), causal keep-mask
// key <= global query position (model.py:301-304), row softmax
// (tensor.py:104-131), ctx[:, h*d:(h+1)*d] = P V_h.  Instead of caching P the
// kernel emits the row log-sum-exp (base 2) so the backward recomputes P.
//
// K/V rows are laid out [G][B][seg][ld] (two TMA maps, one per operand); for the
// packed all-gather buffer [G][B][seg][2E] K is columns [0,E) and V [E,2E),
// i.e. the rank-ordered concatenation of every rank's [K_r|V_r]
// (sharded.py:144-154 math, one collective).  The kernel walks the
// key tiles segment by segment, so a segment length that is not a multiple of
// 128 costs one partial tile per segment (masked), never a straddling TMA box.
//
// CTA = 2 query tiles (256 rows) of one (batch, head); 12 warps:
//   warp 0      TMA producer (Q once; K/V ring of KV_STAGES)
//   warp 1      MMA issuer (single thread): S_w = Q_w K^T (SS), O_w += P_w V (TS)
//   warp 2      TMEM allocator
//   warps 4-7   softmax for query tile 0 (thread <-> row <-> TMEM lane)
//   warps 8-11  softmax for query tile 1
// TMEM (512 cols): S0 | S1 | O0 | O1 | P0 | P1  (128,128,64,64,64,64).
// S is released as soon as the softmax warps have loaded it, so S_{j+1} runs
// on the tensor core while the exponentials of tile j are computed; P lives in
// its own TMEM columns and feeds the P.V MMA directly (A operand from TMEM).
// O rescaling is lazy (only when a row max grows by > 2^8).
#pragma once
#include "common.cuh"

#ifndef LSS_FWD_SOFTMAX_REGS
#define LSS_FWD_SOFTMAX_REGS 232  // setmaxnreg budget: 128 x CTRL + 256 x SOFTMAX <= 64K
#define LSS_FWD_CTRL_REGS 40
#endif
#ifndef LSS_FWD_MAXTREE
#define LSS_FWD_MAXTREE 1  // row max as independent chains (A/B builds: 0 = one serial chain)
#endif
#ifndef LSS_FWD_SUMCHAINS
#define LSS_FWD_SUMCHAINS 1  // independent accumulators of the row sum (A/B builds)
#endif
#ifndef LSS_FWD_EXP2_DEG
#define LSS_FWD_EXP2_DEG 2  // degree of the FMA-pipe exp2 (A/B on B200: 5.79 ms vs 6.22 ms at degree 3)
#endif
#ifndef LSS_FWD_POLY8
#define LSS_FWD_POLY8 3  // exponent pairs (of every 8) on the FMA-pipe polynomial; the rest on MUFU ex2
#endif                   // (l=50112, 232-register softmax: 0 -> 7.15 ms, 2 -> 6.3, 3 -> 6.1-6.2, 4 -> 6.2)

namespace lss {

#ifdef LSS_FWD_TRACE
__device__ long long g_fwd_trace[8][1024];
#define FWD_TRACE(slot, it)                                                           \
  do {                                                                                \
    if (blockIdx.x == 0 && (it) < 1024) g_fwd_trace[slot][it] = clock64();            \
  } while (0)
#else
#define FWD_TRACE(slot, it) \
  do {                      \
  } while (0)
#endif

#ifndef LSS_FWD_HGROUP
#define LSS_FWD_HGROUP 4
#endif
constexpr int ATT_FWD_HGROUP = LSS_FWD_HGROUP;  // (batch, head) slices interleaved by the forward grid

constexpr int ATT_BM = 128;
constexpr int ATT_BN = 128;
constexpr int ATT_D = 64;
#ifndef LSS_FWD_KV_STAGES
#define LSS_FWD_KV_STAGES 3
#endif
constexpr int ATT_KV_STAGES = LSS_FWD_KV_STAGES;  // K/V TMA ring depth
constexpr int ATT_TILE_BYTES = ATT_BM * ATT_D * 2;  // 16 KB (Q, K or V tile)
constexpr int ATT_FWD_THREADS = 384;
constexpr int ATT_FWD_SMEM = (2 + 2 * ATT_KV_STAGES) * ATT_TILE_BYTES + 1024 + 256;

struct AttnFwdParams {
  int B, m, m_pad, G, seg_len, H;  // q: m rows per batch; kv: [G][B][seg_len][ld]
  int g_begin, g_end;              // key segments [g_begin, g_end) attended (partial attention)
  long offset;                     // global position of q row 0
  int causal;
  float scale_log2;                // log2(e)/sqrt(d)
  __nv_bfloat16* o;                // row r of batch b at o + b*o_bstride + r*E
  long o_bstride;
  float* lse2;                     // [B][H][lse_pitch] (+ row), base 2: m + log2(l); pad rows = +inf
  int lse_pitch;                   // rows with no visible key (partial ranges) get O = 0, lse = -inf
  // attention-probability dropout (model.scores_fwd, model.py:313-317; used when DROP):
  // site = mix(mix(seed, tag 2), layer + 1); row key = mix(mix(mix(site, b + 1), h + 1), q_pos);
  // keep (q_pos, k_pos) iff (mix(row key, k_pos) >> 11) >= drop_thresh; kept P scaled by drop_scale
  uint64_t drop_site;
  uint64_t drop_thresh;
  float drop_scale;
  // key split (few query tiles over a long key range, e.g. a rank's remote segments):
  // split s of `splits` attends key tiles [s*n/S, (s+1)*n/S) of its CTA's n visible
  // tiles; split 0 writes o / lse2, split s > 0 the partial slot s-1 (same row layout),
  // merged afterwards by attn_merge_n_kernel
  int splits;
  __nv_bfloat16* o_part;
  long o_part_stride;
  float* lse_part;
  long lse_part_stride;
  // fused all-gather: key segment g != own_seg is read only after seg_ready[g] reaches
  // ready_seq (the copy stream signals each segment as it lands); null = all resident
  const uint32_t* seg_ready;
  uint32_t ready_seq;
  int own_seg;
};

// PART: key-split grid / fused-gather flags / top-down segment order; the plain
// instance (ascending tiles, no split) is kept for A/B builds (-DLSS_FWD_PLAIN).  The
// tile walk is incremental: a runtime division per tile in the softmax loop cost 4-8%.
template <bool DROP, bool PART>
__global__ void __launch_bounds__(ATT_FWD_THREADS, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, AttnFwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                                   // 2 tiles
  uint8_t* sK = smem + 2 * ATT_TILE_BYTES;              // KV_STAGES tiles
  uint8_t* sV = sK + ATT_KV_STAGES * ATT_TILE_BYTES;    // KV_STAGES tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + ATT_KV_STAGES * ATT_TILE_BYTES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + ATT_KV_STAGES;
  uint64_t* s_full = kv_empty + ATT_KV_STAGES;  // [2]
  uint64_t* s_empty = s_full + 2;               // [2]
  uint64_t* p_full = s_empty + 2;               // [2]
  uint64_t* o_full = p_full + 2;                // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int E = p.H * ATT_D;
  // 1-D grid in groups of ATT_FWD_HGROUP (batch, head) slices: inside a group the
  // heaviest (late, causal) query-tile pairs of every slice go first
  // (longest-processing-time order, so no slice leaves its heavy tiles for the
  // tail), while only a group's K/V streams are live at once (L2-resident).
  const int n_pairs = (p.m + 2 * ATT_BM - 1) / (2 * ATT_BM);
  const int hb = p.H * p.B;
  const int nsplit = PART ? p.splits : 1;
  const int split = PART ? (int)blockIdx.x % nsplit : 0;  // innermost: a tile's splits run together
  const int cta = PART ? (int)blockIdx.x / nsplit : (int)blockIdx.x;
  const int grp_first = (cta / (ATT_FWD_HGROUP * n_pairs)) * ATT_FWD_HGROUP;
  const int grp_size = min(ATT_FWD_HGROUP, hb - grp_first);
  const int in_grp = cta - grp_first * n_pairs;
  const int slice = grp_first + in_grp % grp_size;
  const int h = slice % p.H;
  const int b = slice / p.H;
  const int unit = in_grp / grp_size;
  const int pair = p.causal ? (n_pairs - 1 - unit) : unit;
  const int q0 = pair * 2 * ATT_BM;
  const bool has1 = q0 + ATT_BM < p.m;
  const int q_last = min(q0 + 2 * ATT_BM, p.m) - 1;  // last valid local row in this CTA
  const int tps = (p.seg_len + ATT_BN - 1) / ATT_BN;  // key tiles per segment
  // Key tiles are visited from the highest visible segment down (the diagonal, then
  // the nearest remote segments: the order the fused gather delivers them); the top
  // segment g_top may be partly visible (n_top tiles), the ones below are full.
  int g_top = p.g_end - 1, n_top = tps;
  if (p.causal) {
    const long max_key = p.offset + q_last;  // keys > max_key are masked for every row
    g_top = p.g_begin - 1;
    n_top = 0;
    for (int g = p.g_begin; g < p.g_end; ++g) {
      const long seg0 = (long)g * p.seg_len;
      if (seg0 > max_key) break;
      g_top = g;
      n_top = (int)(min((long)p.seg_len - 1, max_key - seg0) / ATT_BN) + 1;
    }
  }
  int n_kv = g_top < p.g_begin ? 0 : (g_top - p.g_begin) * tps + n_top;
  const int j_base = PART ? (int)(((long)split * n_kv) / nsplit) : 0;  // this split's key tiles
  if (PART) n_kv = (int)(((long)(split + 1) * n_kv) / nsplit) - j_base;
  auto tile_of = [&](int jt, int& g, int& t) {  // visit index -> (segment, tile in segment)
    if (!PART) {  // ascending
      g = p.g_begin + jt / tps;
      t = jt % tps;
    } else if (jt < n_top) {
      g = g_top;
      t = jt;
    } else {
      g = g_top - 1 - (jt - n_top) / tps;
      t = (jt - n_top) % tps;
    }
  };
  auto next_tile = [&](int& g, int& t) {  // the visit after (g, t)
    if (!PART) {
      if (++t == tps) { t = 0; ++g; }
    } else if (++t == (g == g_top ? n_top : tps)) {
      t = 0;
      --g;
    }
  };
  __nv_bfloat16* const o_dst = (!PART || split == 0) ? p.o : p.o_part + (long)(split - 1) * p.o_part_stride;
  float* const lse_dst = (!PART || split == 0) ? p.lse2 : p.lse_part + (long)(split - 1) * p.lse_part_stride;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < ATT_KV_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], has1 ? 2 : 1);  // one PV commit per query tile
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(&s_full[w], 1);
      mbar_init(&s_empty[w], 128);
      mbar_init(&p_full[w], 128);
      mbar_init(&o_full[w], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM column bases of query tile w (arithmetic, not arrays: a runtime-indexed
  // array lands in local memory, an LDL on every softmax iteration)
  auto tS = [&](int w) { return tmem + 128u * w; };
  auto tO = [&](int w) { return tmem + 256u + 64u * w; };
  auto tP = [&](int w) { return tmem + 384u + 64u * w; };

  if (warp < 4) {
   reg_dealloc<LSS_FWD_CTRL_REGS>();  // control warpgroup: TMA, MMA, TMEM alloc
   if (warp == 0) {
    if (n_kv > 0) {
      // ------------------------------------------------ TMA producer (warp-uniform loop)
      if (elect_one()) {
        mbar_arrive_expect_tx(q_full, (has1 ? 2 : 1) * ATT_TILE_BYTES);
        tma_load_3d(&tmQ, q_full, sQ, h * ATT_D, q0, b);
        if (has1) tma_load_3d(&tmQ, q_full, sQ + ATT_TILE_BYTES, h * ATT_D, q0 + ATT_BM, b);
      }
      __syncwarp();
      int g_ready = p.own_seg;  // segments known to be resident
      int g, t;
      tile_of(j_base, g, t);
      for (int j = 0; j < n_kv; ++j, next_tile(g, t)) {
        const int st = j % ATT_KV_STAGES;
        const uint32_t ph = (j / ATT_KV_STAGES) & 1;
        if (PART && p.seg_ready != nullptr && g != g_ready && g != p.own_seg) {  // fused gather: wait for it
          if (lane == 0) wait_flag_geq(p.seg_ready + g, p.ready_seq);
          __syncwarp();
          g_ready = g;
        }
        mbar_wait(&kv_empty[st], ph ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&kv_full[st], 2 * ATT_TILE_BYTES);
          tma_load_4d(&tmK, &kv_full[st], sK + st * ATT_TILE_BYTES, h * ATT_D, t * ATT_BN, b, g);
          tma_load_4d(&tmV, &kv_full[st], sV + st * ATT_TILE_BYTES, h * ATT_D, t * ATT_BN, b, g);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1 || (warp == 3 && has1)) {
    if (n_kv > 0) {
      // ------------------------------------------------ MMA issuers: warp 1 for query
      // tile 0, warp 3 for tile 1 (warp-uniform loops, one elected lane issues).  Each
      // tile's S / PV stream follows only its own softmax warpgroup, so the two
      // warpgroups run a free ping-pong on the shared tensor pipe and MUFU.
      constexpr uint32_t idS = idesc_bf16_f32(ATT_BM, ATT_BN, 0, 0);
      constexpr uint32_t idO = idesc_bf16_f32(ATT_BM, ATT_D, 0, 1);
      const int w = warp == 1 ? 0 : 1;
      const uint32_t q_addr = smem_u32(sQ);
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int jj) {  // O_w += P_w(jj) V(jj)
        const int st = jj % ATT_KV_STAGES;
        const uint32_t v_addr = smem_u32(sV + st * ATT_TILE_BYTES);
        mbar_wait(&p_full[w], jj & 1);
        tc_fence_after();
        if (lane == 0 && w == 0) FWD_TRACE(6, jj);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < ATT_BN / 16; ++k) {
            mma_bf16_ts(tO(w), tP(w) + k * 8, smem_desc_sw128(v_addr + k * 2048, 8192, 1024), idO,
                        (jj > 0 || k > 0) ? 1u : 0u);
          }
          mma_commit(&o_full[w]);
          mma_commit(&kv_empty[st]);  // this tile's reads of the K/V stage are done
        }
        __syncwarp();
      };
      for (int j = 0; j < n_kv; ++j) {
        const int st = j % ATT_KV_STAGES;
        mbar_wait(&kv_full[st], (j / ATT_KV_STAGES) & 1);
        tc_fence_after();
        if (lane == 0 && w == 0) FWD_TRACE(7, j);
        const uint32_t k_addr = smem_u32(sK + st * ATT_TILE_BYTES);
        if (j > 0) mbar_wait(&s_empty[w], (j - 1) & 1);  // S_w(j) = Q_w K(j)^T
        tc_fence_after();
        if (lane == 0 && w == 0) FWD_TRACE(5, j);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < ATT_D / 16; ++k) {
            mma_bf16_ss(tS(w), smem_desc_sw128(q_addr + w * ATT_TILE_BYTES + k * 32, 16, 1024),
                        smem_desc_sw128(k_addr + k * 32, 16, 1024), idS, k > 0 ? 1u : 0u);
          }
          mma_commit(&s_full[w]);
        }
        __syncwarp();
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(n_kv - 1);
    }
   }
  } else {
    reg_alloc<LSS_FWD_SOFTMAX_REGS>();  // softmax warpgroups get the register file
    // ------------------------------------------------ softmax (one row per thread)
    const int w = (warp - 4) / 4;  // query tile of this warpgroup
    const int quad = warp % 4;
    const int r = quad * 32 + lane;                    // row within tile == TMEM lane
    const int lrow = q0 + w * ATT_BM + r;              // local query row
    const long qpos = p.offset + lrow;                 // global query position
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const bool active = (w == 0) || has1;
    if (active && n_kv > 0) {
      float m_run = -INFINITY, l_run = 0.f;
      const int tile_first_row = q0 + w * ATT_BM;  // for the mask decision (warp-uniform)
      int g, t;
      tile_of(j_base, g, t);
      for (int j = 0; j < n_kv; ++j, next_tile(g, t)) {
        const int valid_cols = min(ATT_BN, p.seg_len - t * ATT_BN);
        const long key0 = (long)g * p.seg_len + (long)t * ATT_BN;
        const bool need_mask = valid_cols < ATT_BN ||
                               (p.causal && key0 + ATT_BN - 1 > p.offset + tile_first_row);
        mbar_wait(&s_full[w], j & 1);
        tc_fence_after();
        if (w == 0 && r == 0) FWD_TRACE(0, j);
        float s[ATT_BN];
        {
          uint32_t rr[64];
          tmem_ld64(tS(w) + lane_off, rr);
#pragma unroll
          for (int i = 0; i < 64; ++i) s[i] = __uint_as_float(rr[i]);
          tmem_ld64(tS(w) + lane_off + 64, rr);
#pragma unroll
          for (int i = 0; i < 64; ++i) s[64 + i] = __uint_as_float(rr[i]);
        }
        tc_fence_before();
        mbar_arrive(&s_empty[w]);
        if (w == 0 && r == 0) FWD_TRACE(1, j);
        if (need_mask) {
          const long lim = p.causal ? (qpos - key0) : (long)(ATT_BN - 1);
#pragma unroll
          for (int c = 0; c < ATT_BN; ++c)
            if (c >= valid_cols || (long)c > lim) s[c] = -INFINITY;
        }
#if LSS_FWD_MAXTREE
        // row max as 4 independent FMNMX3 chains (one serial chain was 64 dependent
        // ALU ops per tile with only two softmax warps per SM sub-partition to hide them)
        float mq[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          constexpr int Q = ATT_BN / 4;
          mq[i] = fmaxf(s[Q * i], s[Q * i + 1]);
#pragma unroll
          for (int k = 2; k < Q; k += 2) mq[i] = fmaxf(mq[i], fmaxf(s[Q * i + k], s[Q * i + k + 1]));
        }
        const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
#else
        float mx = s[0];
#pragma unroll
        for (int c = 1; c < ATT_BN; ++c) mx = fmaxf(mx, s[c]);
#endif
        const float m_tile = mx * p.scale_log2;
        float alpha = 1.f;
        bool rescale = false;
        if (m_tile > m_run + 8.f) {  // also true on the first tile (m_run = -inf)
          alpha = ex2(m_run - m_tile);
          rescale = (j > 0);
          m_run = m_tile;
        }
        const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
        uint32_t pk[ATT_BN / 2];
        float2 sum2[LSS_FWD_SUMCHAINS];
#pragma unroll
        for (int i = 0; i < LSS_FWD_SUMCHAINS; ++i) sum2[i] = make_float2(0.f, 0.f);
        uint64_t drop_row = 0;
        if (DROP) drop_row = drop_mix(drop_mix(drop_mix(p.drop_site, (uint64_t)b + 1), (uint64_t)h + 1), (uint64_t)qpos);
        {
          const float2 slv = make_float2(p.scale_log2, p.scale_log2), nm = make_float2(-m_use, -m_use);
#pragma unroll
          for (int c = 0; c < ATT_BN; c += 2) {
            const float2 x = ffma2(make_float2(s[c], s[c + 1]), slv, nm);  // packed FFMA2
            float2 e;
            if (((c / 2) & 7) < LSS_FWD_POLY8) {  // FMA-pipe share (MUFU relief)
              e = exp2_poly2<LSS_FWD_EXP2_DEG>(x);
            } else {
              e = make_float2(ex2(x.x), ex2(x.y));
            }
            sum2[(c / 2) % LSS_FWD_SUMCHAINS] = fadd2(sum2[(c / 2) % LSS_FWD_SUMCHAINS], e);  // undropped
            if (DROP) {
              e.x = drop_keep(drop_row, (uint64_t)(key0 + c), p.drop_thresh) ? e.x * p.drop_scale : 0.f;
              e.y = drop_keep(drop_row, (uint64_t)(key0 + c + 1), p.drop_thresh) ? e.y * p.drop_scale : 0.f;
            }
            pk[c / 2] = pack_bf16(e.x, e.y);
          }
        }
#pragma unroll
        for (int i = 1; i < LSS_FWD_SUMCHAINS; ++i) sum2[0] = fadd2(sum2[0], sum2[i]);
        const float sum = sum2[0].x + sum2[0].y;
        l_run = l_run * alpha + sum;
        if (w == 0 && r == 0) FWD_TRACE(2, j);
        if (j > 0) {
          mbar_wait(&o_full[w], (j - 1) & 1);  // PV_{j-1} done: P buffer free, O stable
          tc_fence_after();
        }
        if (w == 0 && r == 0) FWD_TRACE(3, j);
        // tcgen05.ld/st are warp-collective: rescale the whole warp's rows if any row needs it
        if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
          for (int c = 0; c < ATT_D / 32; ++c) {
            uint32_t oo[32];
            tmem_ld32(tO(w) + lane_off + c * 32, oo);
#pragma unroll
            for (int i = 0; i < 32; ++i) oo[i] = __float_as_uint(__uint_as_float(oo[i]) * alpha);
            tmem_st32(tO(w) + lane_off + c * 32, oo);
          }
        }
        {
          uint32_t p0[32], p1[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            p0[i] = pk[i];
            p1[i] = pk[32 + i];
          }
          tmem_st32(tP(w) + lane_off + 0, p0);
          tmem_st32(tP(w) + lane_off + 32, p1);
        }
        tc_fence_before();
        mbar_arrive(&p_full[w]);
        if (w == 0 && r == 0) FWD_TRACE(4, j);
      }
      // ---------------------------------------------- epilogue
      mbar_wait(&o_full[w], (n_kv - 1) & 1);
      tc_fence_after();
      uint32_t oo[ATT_D];
      tmem_ld64(tO(w) + lane_off, oo);
      {
        // stage the warp's 32 rows x 128 B in this query tile's (now idle) Q buffer,
        // 16-byte chunks XOR-swizzled by row, then store whole 128-byte rows: 4 rows
        // per instruction instead of 32 half-filled sectors
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        const uint32_t stg = smem_u32(sQ + w * ATT_TILE_BYTES) + quad * 32 * 128;
#pragma unroll
        for (int i = 0; i < ATT_D / 8; ++i)
          st_shared_v4(stg + lane * 128 + ((i ^ (lane & 7)) << 4),
                       pack_bf16(__uint_as_float(oo[8 * i + 0]) * inv, __uint_as_float(oo[8 * i + 1]) * inv),
                       pack_bf16(__uint_as_float(oo[8 * i + 2]) * inv, __uint_as_float(oo[8 * i + 3]) * inv),
                       pack_bf16(__uint_as_float(oo[8 * i + 4]) * inv, __uint_as_float(oo[8 * i + 5]) * inv),
                       pack_bf16(__uint_as_float(oo[8 * i + 6]) * inv, __uint_as_float(oo[8 * i + 7]) * inv));
        if (g_numerics_check) {  // NaN / Inf in O or the row statistics (tensor.py:79-95, 131)
          bool bad = l_run > 0.f && (nonfinite(m_run) || nonfinite(l_run));
#pragma unroll
          for (int i = 0; i < ATT_D; ++i) bad |= nonfinite(__uint_as_float(oo[i]) * inv);
          report_nonfinite(bad);
        }
        __syncwarp();
        const int row_w0 = q0 + w * ATT_BM + quad * 32;  // local row of the warp's first row
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int rr = j * 4 + (int)lane / 8, q = (int)lane % 8;
          const float4 val = ld_shared_f4(stg + rr * 128 + ((q ^ (rr & 7)) << 4));
          if (row_w0 + rr < p.m)
            *reinterpret_cast<float4*>(o_dst + (long)b * p.o_bstride + (long)(row_w0 + rr) * E + h * ATT_D + q * 8) =
                val;
        }
      }
      if (lrow < p.m) {
        lse_dst[((long)b * p.H + h) * p.lse_pitch + lrow] = l_run > 0.f ? m_run + __log2f(l_run) : -INFINITY;
      } else if (lrow < p.m_pad) {
        lse_dst[((long)b * p.H + h) * p.lse_pitch + lrow] = INFINITY;
      }
    } else if (active) {
      // no key tile of [g_begin, g_end) is visible to this CTA: empty partial
      if (lrow < p.m) {
        uint4* dst = reinterpret_cast<uint4*>(o_dst + (long)b * p.o_bstride + (long)lrow * E + h * ATT_D);
#pragma unroll
        for (int i = 0; i < ATT_D / 8; ++i) dst[i] = make_uint4(0u, 0u, 0u, 0u);
        lse_dst[((long)b * p.H + h) * p.lse_pitch + lrow] = -INFINITY;
      } else if (lrow < p.m_pad) {
        lse_dst[((long)b * p.H + h) * p.lse_pitch + lrow] = INFINITY;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

}  // namespace lss
