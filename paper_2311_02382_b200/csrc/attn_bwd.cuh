// Segment attention backward for the LSS layer on sm_100a (tcgen05 + TMEM + TMA).
//
// Semantics follow model.scores_bwd (reference model.py:329-359):
//   dP = dO V^T, dV = P^T dO, dS = P (dP - rowsum(dP P)) / sqrt(d),
//   dQ = dS K, dK = dS^T Q,
// with P recomputed from the forward's base-2 log-sum-exp and
// rowsum(dP P) = rowsum(dO O) = delta precomputed per query row.  dK/dV span
// the FULL key length (this rank's partial contribution for every rank's key
// rows) and are written in the [G][B][seg][ld] fp32 layout; with dv = dk + E and
// ld = 2E that is the packed [dK|dV] buffer the reduce-scatter consumes
// directly (sharded.py:192-199 math, one collective).
//
// CTA = one 128-row key tile of one (batch, head); it walks the query tiles of
// this rank that can see the keys (causal: q_pos >= k_pos).  Transposed
// formulation so the key rows are TMEM lanes:
//   S^T  = K Q_i^T   (TMEM, 128 cols)          dP^T = V dO_i^T   (TMEM, 128 cols)
//   P^T, dS^T computed by 256 threads (2 warpgroups, 64 query columns each)
//   dV  += P^T dO_i  (A = P^T from TMEM)
//   dK  += dS^T Q_i  (A = dS^T from SMEM, K-major)
//   dQ_i = dS K      (A = dS^T from SMEM read MN-major) -> drained by a 4th
//                    warpgroup into fp32 dQ with TMA tensor reduce-add
// TMEM: S^T[0,128) dP^T[128,256) dV[256,320) dK[320,384) dQ[384,448) P^T[448,512)
// 16 warps: 0 TMA, 1 MMA, 2 TMEM alloc, 4-11 elementwise, 12-15 dQ drain;
// setmaxnreg gives the elementwise warps the register file.
// Pipelining: S/dP of tile i+1 are issued as soon as tile i's values are in
// registers; dS^T is double-buffered in SMEM so the elementwise warps only wait
// for dV_i (P^T buffer) before publishing tile i+1, and the dQ drain runs on
// its own warps, decoupled from the elementwise critical path.
#pragma once
#include "attn_fwd.cuh"
#include "common.cuh"

namespace lss {

constexpr int ATB_QSTAGE_BYTES = 2 * ATT_TILE_BYTES + 2 * 512;  // Q, dO, lse2[128], delta[128]
constexpr int ATB_DS_BYTES = 2 * ATT_TILE_BYTES;                 // dS^T tile: 2 sub-tiles [128 kv][64 q]
constexpr int ATB_STG_BYTES = 128 * 64 * 4;                      // dQ staging [128 q][64] fp32 (2 SW128 halves)
constexpr int ATB_SMEM = 2 * ATT_TILE_BYTES /*K,V*/ + 2 * ATB_QSTAGE_BYTES + 2 * ATB_DS_BYTES + ATB_STG_BYTES +
                         1024 + 256;
constexpr int ATB_THREADS = 512;

// A query-row source of the backward: rows [row0, row0+rows) of a [B][m_src][E]
// (Q, dO, dQ) tensor triple whose row 0 sits at global position pos0, attending
// key segments [g_begin, g_end).  A launch processes up to ATB_MAX_SRC sources
// (this rank's own rows, and rows delegated by a partner in the balanced causal
// schedule); every key tile accumulates dK/dV from all of them in TMEM, so each
// dK/dV row has exactly one writer.
constexpr int ATB_MAX_SRC = 3;
struct BwdSource {
  int row0, rows;
  long pos0;
  int g_begin, g_end;
  const float* lse2;   // [B][H][pitch] (+inf beyond the tensor's last row)
  const float* delta;  // [B][H][pitch] rowsum(dO*O)/sqrt(d)
  int pitch;
};
struct BwdMaps {
  CUtensorMap q[ATB_MAX_SRC];
  CUtensorMap dO[ATB_MAX_SRC];
  CUtensorMap dq[ATB_MAX_SRC];  // fp32 [B][m_src][E], box 32 x 128, reduce-add target
};
struct AttnBwdParams {
  int B, G, seg_len, H, nsrc;
  int causal;
  float scale_log2;  // log2(e)/sqrt(d)
  float scale;       // 1/sqrt(d)
  BwdSource src[ATB_MAX_SRC];
  float* dk;         // [G][B][seg_len][ld_dkv] fp32, fully written
  float* dv;         // same layout
  long ld_dkv;
};

LSS_DEV void bulk_load_1d(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

#ifdef LSS_BWD_TRACE
__device__ long long g_bwd_trace[8][512];
#define BWD_TRACE(slot, it)                                                          \
  do {                                                                               \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (it) < 512)         \
      g_bwd_trace[slot][it] = clock64();                                             \
  } while (0)
#else
#define BWD_TRACE(slot, it) \
  do {                      \
  } while (0)
#endif

// P^T and dS^T for one key row and 64 query columns:
//   p = 2^(s*log2e/sqrt(d) - lse2[q]),  ds = p * (dp/sqrt(d) - delta[q]/sqrt(d))
// lse2 / scaled delta come from shared memory as 128-bit broadcast loads; the
// causal / tail mask (column c visible iff c >= fv) is compiled only into the
// MASK instance so full tiles carry no per-element predicate work.
template <bool MASK>
LSS_DEV void bwd_pds(const uint32_t (&sv)[64], const uint32_t (&dp)[64], uint32_t s_lse, uint32_t s_dsc,
                     float sl2, float scale, int fv, uint32_t (&pk)[32], uint32_t (&dk)[32]) {
  const float2 sl2v = make_float2(sl2, sl2), scv = make_float2(scale, scale);
#pragma unroll
  for (int c4 = 0; c4 < 16; ++c4) {
    const float4 l = ld_shared_f4(s_lse + c4 * 16);
    const float4 d = ld_shared_f4(s_dsc + c4 * 16);
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int c = 4 * c4 + 2 * h2;
      const float2 nl = h2 ? make_float2(-l.z, -l.w) : make_float2(-l.x, -l.y);
      const float2 nd = h2 ? make_float2(-d.z, -d.w) : make_float2(-d.x, -d.y);
      const float2 x = ffma2(make_float2(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), sl2v, nl);
      float2 e;
      if (!MASK && (c4 & 3) == 0 && h2 == 0) {  // 1 pair in 8 on the FMA pipe (x <= ~0 here)
        e = exp2_poly2(x);
      } else {
        e = make_float2(ex2(x.x), ex2(x.y));
      }
      if (MASK) {
        e.x = (c >= fv) ? e.x : 0.f;
        e.y = (c + 1 >= fv) ? e.y : 0.f;
      }
      const float2 t = ffma2(make_float2(__uint_as_float(dp[c]), __uint_as_float(dp[c + 1])), scv, nd);
      const float2 ds = fmul2(e, t);
      pk[c / 2] = pack_bf16(e.x, e.y);
      dk[c / 2] = pack_bf16(ds.x, ds.y);
    }
  }
}

__global__ void __launch_bounds__(ATB_THREADS, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       const __grid_constant__ BwdMaps maps, const __grid_constant__ AttnBwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + ATT_TILE_BYTES;
  uint8_t* sQst = sV + ATT_TILE_BYTES;              // 2 stages: Q, dO, lse2, delta
  uint8_t* sdS = sQst + 2 * ATB_QSTAGE_BYTES;       // 2 buffers x 2 sub-tiles [128 kv][64 q] bf16
  uint8_t* sStage = sdS + 2 * ATB_DS_BYTES;         // dQ staging, 2 x [128 q][32] fp32 (SW128)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + ATB_STG_BYTES);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;   // [2]
  uint64_t* q_empty = bars + 3;  // [2]
  uint64_t* sdp_full = bars + 5;
  uint64_t* sdp_free = bars + 6;
  uint64_t* pds_full = bars + 7;
  uint64_t* pv_free = bars + 8;   // dV_i (and everything before it) complete
  uint64_t* dq_full = bars + 9;
  uint64_t* dq_empty = bars + 10;
  uint64_t* mma_done = bars + 11;  // one-shot: every MMA of the CTA complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int E = p.H * ATT_D;
  const int h = blockIdx.y;
  const int b = blockIdx.z;
  const int tps = (p.seg_len + ATT_BN - 1) / ATT_BN;
  const int g = blockIdx.x / tps;
  const int kt = blockIdx.x % tps;
  const int kv_row0 = kt * ATT_BN;                         // row within segment
  const int kv_valid = min(ATT_BN, p.seg_len - kv_row0);
  const long kpos0 = (long)g * p.seg_len + kv_row0;        // global key position of row 0
  // per-source query-tile ranges visible to this key tile (causal: q_pos >= k_pos)
  int src_first[ATB_MAX_SRC], src_n[ATB_MAX_SRC];
  int n_iter = 0;
#pragma unroll
  for (int s = 0; s < ATB_MAX_SRC; ++s) {
    src_first[s] = 0;
    src_n[s] = 0;
    if (s < p.nsrc && g >= p.src[s].g_begin && g < p.src[s].g_end) {
      const int n_qt = (p.src[s].rows + ATT_BM - 1) / ATT_BM;
      int first = 0;
      if (p.causal) {
        const long d0 = kpos0 - (p.src[s].pos0 + p.src[s].row0);  // first source row seeing key row 0
        first = d0 <= 0 ? 0 : (int)min((long)n_qt, d0 / ATT_BM);
      }
      src_first[s] = first;
      src_n[s] = n_qt - first;
      n_iter += n_qt - first;
    }
  }
  // iteration -> (source, tensor row of the query tile)
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
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    mbar_init(sdp_full, 1);
    mbar_init(sdp_free, 256);
    mbar_init(pds_full, 256);
    mbar_init(pv_free, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 128);
    mbar_init(mma_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem + 0, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 320,
                 tdQ = tmem + 384, tP = tmem + 448;

  if (warp < 4) {
    reg_dealloc<56>();
    if (warp == 0) {
      if (n_iter > 0) {
        // ------------------------------------------------ TMA producer (warp-uniform loop)
        if (elect_one()) {
          mbar_arrive_expect_tx(kv_full, 2 * ATT_TILE_BYTES);
          tma_load_4d(&tmK, kv_full, sK, h * ATT_D, kv_row0, b, g);
          tma_load_4d(&tmV, kv_full, sV, h * ATT_D, kv_row0, b, g);
        }
        __syncwarp();
        for (int it = 0; it < n_iter; ++it) {
          const int s = it & 1;
          mbar_wait(&q_empty[s], ((it >> 1) & 1) ^ 1);
          if (elect_one()) {
            int src, q0;
            locate(it, src, q0);
            uint8_t* st = sQst + s * ATB_QSTAGE_BYTES;
            mbar_arrive_expect_tx(&q_full[s], ATB_QSTAGE_BYTES);
            tma_load_3d(&maps.q[src], &q_full[s], st, h * ATT_D, q0, b);
            tma_load_3d(&maps.dO[src], &q_full[s], st + ATT_TILE_BYTES, h * ATT_D, q0, b);
            const long lo = ((long)b * p.H + h) * p.src[src].pitch + q0;
            bulk_load_1d(st + 2 * ATT_TILE_BYTES, p.src[src].lse2 + lo, 512, &q_full[s]);
            bulk_load_1d(st + 2 * ATT_TILE_BYTES + 512, p.src[src].delta + lo, 512, &q_full[s]);
          }
          __syncwarp();
        }
      }
    } else if (warp == 1) {
      if (n_iter > 0) {
        // ------------------------------------------------ MMA issuer (warp-uniform loop,
        // one elected lane issues: descriptors stay in the uniform datapath)
        constexpr uint32_t idSS = idesc_bf16_f32(128, 128, 0, 0);  // S^T, dP^T
        constexpr uint32_t idKN = idesc_bf16_f32(128, 64, 0, 1);   // dV, dK (B MN-major)
        constexpr uint32_t idQ = idesc_bf16_f32(128, 64, 1, 1);    // dQ (A and B MN-major)
        const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV);
        auto issue_sdp = [&](int it) {
          const int s = it & 1;
          mbar_wait(&q_full[s], (it >> 1) & 1);
          tc_fence_after();
          const uint32_t q_addr = smem_u32(sQst + s * ATB_QSTAGE_BYTES);
          const uint32_t do_addr = q_addr + ATT_TILE_BYTES;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < ATT_D / 16; ++k)
              mma_bf16_ss(tS, smem_desc_sw128(k_addr + k * 32, 16, 1024),
                          smem_desc_sw128(q_addr + k * 32, 16, 1024), idSS, k > 0);
#pragma unroll
            for (int k = 0; k < ATT_D / 16; ++k)
              mma_bf16_ss(tdP, smem_desc_sw128(v_addr + k * 32, 16, 1024),
                          smem_desc_sw128(do_addr + k * 32, 16, 1024), idSS, k > 0);
            mma_commit(sdp_full);
          }
          __syncwarp();
        };
        mbar_wait(kv_full, 0);
        tc_fence_after();
        issue_sdp(0);
        for (int it = 0; it < n_iter; ++it) {
          if (it + 1 < n_iter) {
            mbar_wait(sdp_free, it & 1);
            if (lane == 0) BWD_TRACE(6, it);
            issue_sdp(it + 1);
          }
          const int s = it & 1;
          const uint32_t q_addr = smem_u32(sQst + s * ATB_QSTAGE_BYTES);
          const uint32_t do_addr = q_addr + ATT_TILE_BYTES;
          const uint32_t ds_addr = smem_u32(sdS + s * ATB_DS_BYTES);
          mbar_wait(pds_full, it & 1);
          tc_fence_after();
          if (lane == 0) BWD_TRACE(0, it);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < ATT_BM / 16; ++k)  // dV += P^T dO
              mma_bf16_ts(tdV, tP + k * 8, smem_desc_sw128(do_addr + k * 2048, 8192, 1024), idKN,
                          (it > 0 || k > 0));
            mma_commit(pv_free);
#pragma unroll
            for (int k = 0; k < ATT_BM / 16; ++k)  // dK += dS^T Q
              mma_bf16_ss(tdK, smem_desc_sw128(ds_addr + (k >> 2) * ATT_TILE_BYTES + (k & 3) * 32, 16, 1024),
                          smem_desc_sw128(q_addr + k * 2048, 8192, 1024), idKN, (it > 0 || k > 0));
            mma_commit(&q_empty[s]);
          }
          __syncwarp();
          if (it > 0) {
            mbar_wait(dq_empty, (it - 1) & 1);  // drain has read dQ_{it-1} out of TMEM
            tc_fence_after();
          }
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < ATT_BN / 16; ++k)  // dQ = dS K
              mma_bf16_ss(tdQ, smem_desc_sw128(ds_addr + k * 2048, ATT_TILE_BYTES, 1024),
                          smem_desc_sw128(k_addr + k * 2048, 8192, 1024), idQ, k > 0);
            mma_commit(dq_full);
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit(mma_done);
        __syncwarp();
      }
    }
  } else if (warp < 12) {
    reg_alloc<184>();
    // ------------------------------------------------ elementwise P^T / dS^T (+ dK/dV epilogue)
    const int half = (warp - 4) / 4;  // query columns [64*half, 64*half+64) of each tile
    const int quad = warp % 4;
    const int t = quad * 32 + lane;   // key row within tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const long kpos = kpos0 + t;
    const bool row_ok = t < kv_valid;
    for (int it = 0; it < n_iter; ++it) {
      const int s = it & 1;
      int src, qrow;
      locate(it, src, qrow);
      const long q0 = p.src[src].pos0 + qrow;  // global position of the tile's first query
      const uint32_t st = smem_u32(sQst + s * ATB_QSTAGE_BYTES);
      const uint32_t s_lse = st + 2 * ATT_TILE_BYTES + half * 256;        // lse2[q], 64 floats
      const uint32_t s_dsc = st + 2 * ATT_TILE_BYTES + 512 + half * 256;  // delta[q]/sqrt(d)
      mbar_wait(sdp_full, it & 1);
      tc_fence_after();
      if (t == 0 && half == 0) BWD_TRACE(1, it);
      uint32_t sv[64], dp[64];
      tmem_ld64(tS + lane_off + half * 64, sv);
      tmem_ld64(tdP + lane_off + half * 64, dp);
      tc_fence_before();
      mbar_arrive(sdp_free);
      if (t == 0 && half == 0) BWD_TRACE(7, it);
      // query column c of this half is visible to key row t iff c >= fv
      const bool need_mask = !row_ok || (p.causal && kpos0 + ATT_BN - 1 > q0 + half * 64);
      uint32_t pk[32], dk[32];
      if (need_mask) {
        const long first_vis = kpos - q0 - half * 64;
        const int fv = !row_ok ? 64 : (p.causal ? (int)max(0L, min(64L, first_vis)) : 0);
        bwd_pds<true>(sv, dp, s_lse, s_dsc, p.scale_log2, p.scale, fv, pk, dk);
      } else {
        bwd_pds<false>(sv, dp, s_lse, s_dsc, p.scale_log2, p.scale, 0, pk, dk);
      }
      if (t == 0 && half == 0) BWD_TRACE(2, it);
      if (it > 0) {
        mbar_wait(pv_free, (it - 1) & 1);  // dV_{it-1} (and dK/dQ_{it-2}) complete
        tc_fence_after();
      }
      if (t == 0 && half == 0) BWD_TRACE(3, it);
      tmem_st32(tP + lane_off + half * 32, pk);
      // dS^T row t, query columns [64*half, +64) -> buffer s, sub-tile `half`, SW128 K-major
      {
        const uint32_t row = smem_u32(sdS + s * ATB_DS_BYTES + half * ATT_TILE_BYTES + t * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          st_shared_v4(row + ((c ^ (t & 7)) << 4), dk[4 * c], dk[4 * c + 1], dk[4 * c + 2], dk[4 * c + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(pds_full);
      if (t == 0 && half == 0) BWD_TRACE(4, it);
    }
    // dK (half 0) / dV (half 1) epilogue after the one-shot mma_done commit
    float* dst = (half ? p.dv : p.dk) + (((long)g * p.B + b) * p.seg_len + kv_row0 + t) * p.ld_dkv +
                 h * ATT_D;
    if (n_iter > 0) {
      mbar_wait(mma_done, 0);
      tc_fence_after();
      uint32_t v[64];
      tmem_ld64((half ? tdV : tdK) + lane_off, v);
      if (row_ok) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          reinterpret_cast<float4*>(dst)[i] =
              make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                          __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
      }
    } else if (row_ok) {
#pragma unroll
      for (int i = 0; i < 16; ++i) reinterpret_cast<float4*>(dst)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else {
    reg_dealloc<80>();
    // ------------------------------------------------ dQ drain: TMEM -> swizzled SMEM -> TMA reduce-add
    const int quad = warp % 4;
    const int r = quad * 32 + lane;  // query row within tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const bool issuer = (r == 0);
    const uint32_t row0 = smem_u32(sStage + r * 128);                      // cols [0,32)
    const uint32_t row1 = smem_u32(sStage + ATB_STG_BYTES / 2 + r * 128);  // cols [32,64)
    for (int it = 0; it < n_iter; ++it) {
      mbar_wait(dq_full, it & 1);
      tc_fence_after();
      if (r == 0) BWD_TRACE(5, it);
      uint32_t v[64];
      tmem_ld64(tdQ + lane_off, v);
      tc_fence_before();
      mbar_arrive(dq_empty);
      if (issuer) bulk_wait_read0();  // previous reduce has finished reading the staging tile
      named_bar_sync(1, 128);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        st_shared_v4(row0 + ((c ^ (r & 7)) << 4), v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
        st_shared_v4(row1 + ((c ^ (r & 7)) << 4), v[32 + 4 * c], v[33 + 4 * c], v[34 + 4 * c], v[35 + 4 * c]);
      }
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
    if (issuer) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

}  // namespace lss
