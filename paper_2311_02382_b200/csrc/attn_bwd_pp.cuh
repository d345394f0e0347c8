// Segment attention backward, ping-pong variant (same semantics, parameters and
// outputs as attn_bwd_tc_kernel in attn_bwd.cuh: model.scores_bwd, model.py:329-359).
//
// The single-tile kernel keeps ONE 128-query tile in flight: its two elementwise
// warpgroups split the tile's columns and move in lockstep, so the tensor pipe
// waits for the elementwise work and the elementwise work waits for the tensor pipe
// (ncu: 28% of the elementwise warps' samples are barrier waits on MMA results, the
// tensor pipe is busy 46% of the time).  Here every 128-query tile is split into
// two 64-query sub-tiles and the two elementwise warpgroups take alternate
// sub-tiles -- warpgroup w owns sub-tiles j = w, w+2, ... -- each with its own
// TMEM S^T / dP^T buffers, so two sub-tiles are in flight and the MMA warp serves
// whichever warpgroup is ready (an event loop over non-blocking barrier probes).
//
// TMEM (512 cols): S^T/P^T buffers [0,64) [64,128), dP^T/dS^T [128,192) [192,256),
//   dV [256,320), dK [320,384), dQ x2 [384,512) (dQ of a 128-query PAIR of sub-tiles,
//   M = 128, computed once both halves of dS are in SMEM).
// MMA shapes: S^T, dP^T M128 N64 K64; dV, dK M128 N64 K64 (A = P^T / dS^T from TMEM);
//   dQ M128 N64 K128 (A = dS from SMEM, MN-major).  Same tensor-pipe cycles per
//   128x128 tile as the single-tile kernel (floor = M*N/256 per K16 step).
// SMEM: K, V; 4 Q/dO sub-tile stages (8 KB each operand, 64-row TMA boxes) + their
//   lse / delta; 2 dS buffers [2 sub-tiles][128 kv][64 q]; dQ staging.
#pragma once
#include "attn_bwd.cuh"

namespace lss {

constexpr int ATP_SUB = 64;                                 // query rows per sub-tile
constexpr int ATP_QSTAGES = 4;
constexpr int ATP_SUB_BYTES = ATP_SUB * ATT_D * 2;          // 8 KB (Q or dO sub-tile)
constexpr int ATP_QSTAGE_BYTES = 2 * ATP_SUB_BYTES;         // Q | dO
constexpr int ATP_LD_BYTES = 2 * ATP_SUB * 4;               // lse2[64] | delta[64]
constexpr int ATP_SMEM = 2 * ATT_TILE_BYTES + ATP_QSTAGES * ATP_QSTAGE_BYTES + ATP_QSTAGES * ATP_LD_BYTES +
                         2 * ATB_DS_BYTES + ATB_STG_BYTES + 1024 + 256;

// warp-uniform non-blocking probe of an mbarrier phase (lane 0 decides for the warp,
// so an elected issue inside the branch never runs divergent; a completed phase stays
// completed until its consumer moves on)
LSS_DEV bool mbar_probe(uint64_t* bar, uint32_t parity) {
  return __shfl_sync(0xffffffffu, (int)mbar_try_wait(bar, parity), 0) != 0;
}

template <bool DROP>
__global__ void __launch_bounds__(ATB_THREADS, 1)
    attn_bwd_pp_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       const __grid_constant__ BwdMaps maps, const __grid_constant__ AttnBwdParams p) {
  static_assert(ATB_EW == 2, "the ping-pong kernel pairs two elementwise warpgroups");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + ATT_TILE_BYTES;
  uint8_t* sQst = sV + ATT_TILE_BYTES;                     // 4 stages: Q sub-tile | dO sub-tile
  uint8_t* sLD = sQst + ATP_QSTAGES * ATP_QSTAGE_BYTES;    // 4 stages: lse2[64] | delta[64]
  uint8_t* sdS = sLD + ATP_QSTAGES * ATP_LD_BYTES;         // 2 buffers x 2 sub-tiles [128 kv][64 q] bf16
  uint8_t* sStage = sdS + 2 * ATB_DS_BYTES;                // dQ staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + ATB_STG_BYTES);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;     // [4]
  uint64_t* q_empty = bars + 5;    // [4]
  uint64_t* s_full = bars + 9;     // [2] per warpgroup buffer
  uint64_t* p_full = bars + 11;    // [2]
  uint64_t* dp_full = bars + 13;   // [2]
  uint64_t* ds_full = bars + 15;   // [2]
  uint64_t* mma_done = bars + 17;
  uint64_t* dq_full = bars + 18;   // [2] per TMEM dQ buffer (pair parity)
  uint64_t* dq_empty = bars + 20;  // [2]
  uint64_t* ds_free = bars + 22;   // [2] per SMEM dS buffer (pair parity)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int h = blockIdx.y;
  const int b = blockIdx.z;
  const int tps = (p.seg_len + ATT_BN - 1) / ATT_BN;
  const int g = p.g_lo + (int)blockIdx.x / tps;
  const int kt = blockIdx.x % tps;
  const int kv_row0 = kt * ATT_BN;
  const int kv_valid = min(ATT_BN, p.seg_len - kv_row0);
  const long kpos0 = (long)g * p.seg_len + kv_row0;
  int src_first[ATB_MAX_SRC], src_n[ATB_MAX_SRC];
  int n_iter = 0;  // 128-query tiles (pairs of sub-tiles)
#pragma unroll
  for (int s = 0; s < ATB_MAX_SRC; ++s) {
    src_first[s] = 0;
    src_n[s] = 0;
    if (s < p.nsrc && g >= p.src[s].g_begin && g < p.src[s].g_end) {
      const int n_qt = (p.src[s].rows + ATT_BM - 1) / ATT_BM;
      int first = 0;
      if (p.causal) {
        const long d0 = kpos0 - (p.src[s].pos0 + p.src[s].row0);
        first = d0 <= 0 ? 0 : (int)min((long)n_qt, d0 / ATT_BM);
      }
      src_first[s] = first;
      src_n[s] = n_qt - first;
      n_iter += n_qt - first;
    }
  }
  const int n_sub = 2 * n_iter;
  auto locate = [&](int it, int& s_out, int& qrow_out) {
    int s = 0;
#pragma unroll
    for (int k = 0; k < ATB_MAX_SRC - 1; ++k)
      if (s == k && it >= src_n[k]) {
        it -= src_n[k];
        s = k + 1;
      }
    s_out = s;
    qrow_out = p.src[s].row0 + (src_first[s] + it) * ATT_BM;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(kv_full, 1);
    for (int s = 0; s < ATP_QSTAGES; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(&s_full[w], 1);
      mbar_init(&p_full[w], 128);
      mbar_init(&dp_full[w], 1);
      mbar_init(&ds_full[w], 128);
      mbar_init(&dq_full[w], 1);
      mbar_init(&dq_empty[w], 128);
      mbar_init(&ds_free[w], 1);
    }
    mbar_init(mma_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem + 0, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 320, tdQ = tmem + 384;

  if (warp < 4) {
    reg_dealloc<ATB_REG_CTRL>();
    if (warp == 0) {
      if (n_sub > 0) {
        // ------------------------------------------------ TMA producer
        if (elect_one()) {
          mbar_arrive_expect_tx(kv_full, 2 * ATT_TILE_BYTES);
          tma_load_4d(&tmK, kv_full, sK, h * ATT_D, kv_row0, b, g);
          tma_load_4d(&tmV, kv_full, sV, h * ATT_D, kv_row0, b, g);
        }
        __syncwarp();
        int src_ready = -1;
        for (int j = 0; j < n_sub; ++j) {
          const int s = j % ATP_QSTAGES;
          mbar_wait(&q_empty[s], ((j / ATP_QSTAGES) & 1) ^ 1);
          int src, qrow;
          locate(j >> 1, src, qrow);
          const int q0 = qrow + ATP_SUB * (j & 1);
          if (p.src[src].ready != nullptr && src != src_ready) {  // fused hand-off: wait for the push
            if (lane == 0) wait_flag_geq(p.src[src].ready, p.src[src].ready_seq);
            __syncwarp();
            src_ready = src;
          }
          uint8_t* st = sQst + s * ATP_QSTAGE_BYTES;
          uint8_t* ld = sLD + s * ATP_LD_BYTES;
          const long lo = ((long)b * p.H + h) * p.src[src].pitch + q0;
          if (elect_one()) {
            mbar_arrive_expect_tx(&q_full[s], ATP_QSTAGE_BYTES + ATP_LD_BYTES);
            tma_load_3d(&maps.q[src], &q_full[s], st, h * ATT_D, q0, b);
            tma_load_3d(&maps.dO[src], &q_full[s], st + ATP_SUB_BYTES, h * ATT_D, q0, b);
            bulk_load_1d(ld, p.src[src].lse2 + lo, ATP_SUB * 4, &q_full[s]);
            bulk_load_1d(ld + ATP_SUB * 4, p.src[src].delta + lo, ATP_SUB * 4, &q_full[s]);
          }
          __syncwarp();
        }
      }
    } else if (warp == 1) {
      if (n_sub > 0) {
        // ------------------------------------------------ MMA issuer: event loop over the two
        // warpgroups' pipelines; a tcgen05.mma is issued only once its inputs are ready,
        // so the in-order tensor pipe never stalls behind one warpgroup while the other waits
        constexpr uint32_t idS = idesc_bf16_f32(128, ATP_SUB, 0, 0);  // S^T, dP^T
        constexpr uint32_t idKN = idesc_bf16_f32(128, 64, 0, 1);      // dV, dK (B MN-major)
        constexpr uint32_t idQ = idesc_bf16_f32(128, 64, 1, 1);       // dQ (A and B MN-major)
        const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV);
        auto stage_addr = [&](int j) { return smem_u32(sQst + (j % ATP_QSTAGES) * ATP_QSTAGE_BYTES); };
        auto mma_ss4 = [&](uint32_t d, uint32_t a_addr, uint32_t b_addr) {  // M128 N64 K64, K-major
#pragma unroll
          for (int k = 0; k < ATT_D / 16; ++k)
            mma_bf16_ss(d, smem_desc_sw128(a_addr + k * 32, 16, 1024), smem_desc_sw128(b_addr + k * 32, 16, 1024),
                        idS, k > 0);
        };
        // per warpgroup: next S to issue, next dV (after P), next dP, next dK (after dS)
        int sj[2] = {0, 1}, pj[2] = {0, 1}, qj[2] = {0, 1}, dj[2] = {0, 1};
        int dq_next = 0;  // next pair whose dQ is issued
        mbar_wait(kv_full, 0);
        tc_fence_after();
        while (dj[0] < n_sub || dj[1] < n_sub || dq_next < n_iter) {
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            // S_j = K Q_j^T into buffer w: needs its Q/dO stage and dV_{j-2} issued (buffer reuse,
            // in-order pipe)
            int j = sj[w];
            if (j < n_sub && j - 2 < pj[w] && mbar_probe(&q_full[j % ATP_QSTAGES], (j / ATP_QSTAGES) & 1)) {
              tc_fence_after();
              if (elect_one()) {
                mma_ss4(tS + ATP_SUB * w, k_addr, stage_addr(j));
                mma_commit(&s_full[w]);
              }
              __syncwarp();
              sj[w] = j + 2;
            }
            // dP_j = V dO_j^T into buffer w: needs S_j issued (stage resident) and dK_{j-2} issued
            j = qj[w];
            if (j < n_sub && j < sj[w] && j - 2 < dj[w]) {
              if (elect_one()) {
                mma_ss4(tdP + ATP_SUB * w, v_addr, stage_addr(j) + ATP_SUB_BYTES);
                mma_commit(&dp_full[w]);
              }
              __syncwarp();
              qj[w] = j + 2;
            }
            // dV += P_j^T dO_j once the warpgroup published P_j
            j = pj[w];
            if (j < n_sub && j < sj[w] && mbar_probe(&p_full[w], (j >> 1) & 1)) {
              tc_fence_after();
              const uint32_t do_addr = stage_addr(j) + ATP_SUB_BYTES;
              if (elect_one()) {
#pragma unroll
                for (int k = 0; k < ATP_SUB / 16; ++k)
                  mma_bf16_ts(tdV, tS + ATP_SUB * w + 8 * k, smem_desc_sw128(do_addr + k * 2048, 8192, 1024), idKN,
                              (j > 0 || k > 0));
              }
              __syncwarp();
              pj[w] = j + 2;
            }
            // dK += dS_j^T Q_j once the warpgroup published dS_j (then the stage is free)
            j = dj[w];
            if (j < n_sub && j < qj[w] && j < pj[w] && mbar_probe(&ds_full[w], (j >> 1) & 1)) {
              tc_fence_after();
              const uint32_t q_addr = stage_addr(j);
              if (elect_one()) {
#pragma unroll
                for (int k = 0; k < ATP_SUB / 16; ++k)
                  mma_bf16_ts(tdK, tdP + ATP_SUB * w + 8 * k, smem_desc_sw128(q_addr + k * 2048, 8192, 1024), idKN,
                              (j > 0 || k > 0));
                mma_commit(&q_empty[j % ATP_QSTAGES]);
              }
              __syncwarp();
              dj[w] = j + 2;
            }
          }
          // dQ of pair pr = dS_pr K once both halves of dS_pr are in SMEM (both dK issued)
          if (dq_next < n_iter && dj[0] > 2 * dq_next && dj[1] > 2 * dq_next + 1) {
            const int pr = dq_next;
            if (pr > 1) {
              mbar_wait(&dq_empty[pr & 1], ((pr >> 1) - 1) & 1);
              tc_fence_after();
            }
            const uint32_t ds_addr = smem_u32(sdS + (pr & 1) * ATB_DS_BYTES);
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < ATT_BN / 16; ++k)
                mma_bf16_ss(tdQ + (pr & 1) * 64, smem_desc_sw128(ds_addr + k * 2048, ATT_TILE_BYTES, 1024),
                            smem_desc_sw128(k_addr + k * 2048, 8192, 1024), idQ, k > 0);
              mma_commit(&dq_full[pr & 1]);
              mma_commit(&ds_free[pr & 1]);
            }
            __syncwarp();
            dq_next = pr + 1;
          }
        }
        if (elect_one()) mma_commit(mma_done);
        __syncwarp();
      }
    }
  } else if (warp < 4 + 4 * ATB_EW) {
    reg_alloc<ATB_REG_EW>();
    // ------------------------------------------------ elementwise: warpgroup w, sub-tiles j = w, w+2, ...
    const int w = (warp - 4) / 4;
    const int quad = warp % 4;
    const int t = quad * 32 + lane;  // key row within tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const long kpos = kpos0 + t;
    const uint64_t drop_head = DROP ? drop_mix(drop_mix(p.drop_site, (uint64_t)b + 1), (uint64_t)h + 1) : 0;
    const bool row_ok = t < kv_valid;
    constexpr int NC = ATP_SUB;
    const uint32_t tSw = tS + ATP_SUB * w, tdPw = tdP + ATP_SUB * w;
    for (int j = w; j < n_sub; j += 2) {
      int src, qrow;
      locate(j >> 1, src, qrow);
      const long q0 = p.src[src].pos0 + qrow + ATP_SUB * (j & 1);  // global position of the sub-tile's first query
      const int s = j % ATP_QSTAGES;
      const uint32_t s_lse = smem_u32(sLD + s * ATP_LD_BYTES), s_dsc = s_lse + ATP_SUB * 4;
      float lse[NC];
      mbar_wait(&q_full[s], (j / ATP_QSTAGES) & 1);
      bwd_ld_vec<NC>(s_lse, lse);
      mbar_wait(&s_full[w], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sv[NC];
      tmem_ld_n<NC>(tSw + lane_off, sv);
      const bool need_mask = !row_ok || (p.causal && kpos0 + ATT_BN - 1 > q0);
      const uint64_t keep = DROP ? bwd_drop_bits<NC>(drop_head, q0, kpos, p.drop_thresh) : 0;
      {
        uint32_t pk[NC / 2];
        if (need_mask) {
          const long first_vis = kpos - q0;
          const int fv = !row_ok ? NC : (p.causal ? (int)max(0L, min((long)NC, first_vis)) : 0);
          bwd_p<true, DROP, NC>(sv, lse, p.scale_log2, fv, pk, keep, p.drop_scale);
        } else {
          bwd_p<false, DROP, NC>(sv, lse, p.scale_log2, 0, pk, keep, p.drop_scale);
        }
        tmem_st_n<NC / 2>(tSw + lane_off, pk);
      }
      tc_fence_before();
      mbar_arrive(&p_full[w]);
      float dsc[NC];
      bwd_ld_vec<NC>(s_dsc, dsc);
      mbar_wait(&dp_full[w], (j >> 1) & 1);
      tc_fence_after();
      {
        uint32_t dk[NC / 2];
        {
          uint32_t dp[NC / 2];
          tmem_ld_n<NC / 2>(tdPw + lane_off, dp);
          bwd_ds<0, NC / 2, NC, DROP>(sv, dp, dsc, p.scale, dk, keep, p.drop_scale);
        }
        {
          uint32_t dp[NC / 2];
          tmem_ld_n<NC / 2>(tdPw + lane_off + NC / 2, dp);
          bwd_ds<NC / 2, NC / 2, NC, DROP>(sv, dp, dsc, p.scale, dk, keep, p.drop_scale);
        }
        const int pr = j >> 1;
        if (pr > 1) mbar_wait(&ds_free[pr & 1], ((pr >> 1) - 1) & 1);
        // dS^T row t of this sub-tile -> its half of the pair's SW128 K-major dS buffer
        const uint32_t row = smem_u32(sdS + (pr & 1) * ATB_DS_BYTES + w * ATT_TILE_BYTES + t * 128);
#pragma unroll
        for (int c = 0; c < NC / 8; ++c)
          st_shared_v4(row + ((c ^ (t & 7)) << 4), dk[4 * c], dk[4 * c + 1], dk[4 * c + 2], dk[4 * c + 3]);
        tmem_st_n<NC / 2>(tdPw + lane_off, dk);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&ds_full[w]);
    }
    // dK / dV epilogue (as attn_bwd_tc_kernel): warpgroup 0 stages dK, warpgroup 1 dV
    constexpr int EC = 64;
    const bool is_v = w == 1;
    const uint32_t stage = smem_u32(sdS);
    if (n_sub > 0) {
      mbar_wait(mma_done, 0);
      tc_fence_after();
      uint32_t v[32];
#pragma unroll
      for (int c = 0; c < EC / 32; ++c) {
        tmem_ld32((is_v ? tdV : tdK) + lane_off + c * 32, v);
        if (g_numerics_check) {
          bool bad = false;
#pragma unroll
          for (int i = 0; i < 32; ++i) bad |= nonfinite(__uint_as_float(v[i]));
          report_nonfinite(bad);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int chunk = (is_v ? 16 : 0) + (c * 32) / 4 + i;
          st_shared_v4(stage + t * 512 + ((chunk ^ (t & 7)) << 4), v[4 * i], v[4 * i + 1], v[4 * i + 2],
                       v[4 * i + 3]);
        }
      }
    }
    named_bar_sync(2, 128 * ATB_EW);
    {
      float* seg = p.seg_tab[0] ? p.seg_tab[g] : p.dkv + g * p.seg_stride;
      const int ew_warp = warp - 4;
      const long col = (lane < 16 ? 0 : p.dv_off) + h * ATT_D + (lane & 15) * 4;
      for (int r = ew_warp; r < kv_valid; r += 4 * ATB_EW) {
        float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
        if (n_sub > 0) val = ld_shared_f4(stage + r * 512 + ((lane ^ (r & 7)) << 4));
        *reinterpret_cast<float4*>(seg + ((long)b * p.seg_len + kv_row0 + r) * p.ld_dkv + col) = val;
      }
    }
  } else {
    reg_dealloc<ATB_REG_DRAIN>();
    // ------------------------------------------------ dQ drain (per 128-query pair, as attn_bwd_tc_kernel)
    const int quad = warp % 4;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const bool issuer = (r == 0);
    const uint32_t row0 = smem_u32(sStage + r * 128);
    const uint32_t row1 = smem_u32(sStage + ATB_STG_BYTES / 2 + r * 128);
    for (int it = 0; it < n_iter; ++it) {
      mbar_wait(&dq_full[it & 1], (it >> 1) & 1);
      tc_fence_after();
      {
        int src, q0;
        locate(it, src, q0);
        long long* fx = p.src[src].dq_fixed;
        if (fx != nullptr) {  // deterministic mode: int64 fixed point, integer bulk adds (attn_bwd.cuh)
          const bool row_ok = q0 + r < p.src[src].m_src;
          long long* grow = fx + ((long)b * p.src[src].m_src + q0 + r) * ((long)p.H * ATT_D) + h * ATT_D;
          const uint32_t srow = smem_u32(sStage + r * 256);
#pragma unroll 1
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t v[32];
            tmem_ld32(tdQ + (it & 1) * 64 + lane_off + hh * 32, v);
            if (hh == 1) {
              tc_fence_before();
              mbar_arrive(&dq_empty[it & 1]);
            }
            bulk_wait_read0();
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              const long long e0 = __float2ll_rn(__uint_as_float(v[2 * c]) * 4294967296.f);
              const long long e1 = __float2ll_rn(__uint_as_float(v[2 * c + 1]) * 4294967296.f);
              asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(srow + c * 16), "l"(e0), "l"(e1) : "memory");
            }
            fence_proxy_async_smem();
            if (row_ok) bulk_reduce_add_u64(grow + hh * 32, sStage + r * 256, 256);
            bulk_commit();
          }
          continue;
        }
      }
      if (issuer) bulk_wait_read0();
      named_bar_sync(1, 128);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t v[32];
        tmem_ld32(tdQ + (it & 1) * 64 + lane_off + hh * 32, v);
        if (g_numerics_check) {
          bool bad = false;
#pragma unroll
          for (int i = 0; i < 32; ++i) bad |= nonfinite(__uint_as_float(v[i]));
          report_nonfinite(bad);
        }
        const uint32_t rowh = hh ? row1 : row0;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          st_shared_v4(rowh + ((c ^ (r & 7)) << 4), v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
      }
      tc_fence_before();
      mbar_arrive(&dq_empty[it & 1]);
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (issuer) {
        int src, q0;
        locate(it, src, q0);
        tma_reduce_add_3d(&maps.dq[src], sStage, h * ATT_D, q0, b);
        tma_reduce_add_3d(&maps.dq[src], sStage + ATB_STG_BYTES / 2, h * ATT_D + 32, q0, b);
        bulk_commit();
      }
    }
    bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

}  // namespace lss
