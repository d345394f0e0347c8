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
//   S^T  = K Q_i^T - lse2/c  (TMEM, 128 cols)    dP^T = V dO_i^T - delta  (TMEM, 128 cols)
//        (the row statistics enter as one extra K16 MMA step: ones x aux operand)
//   P^T  computed by 256 threads (2 warpgroups, 64 query columns each) into its own
//        TMEM columns; dS^T written back as bf16 over dP^T and into SMEM
//   dV  += P^T dO_i  (A = P^T from TMEM)
//   dK  += dS^T Q_i  (A = dS^T from TMEM)
//   dQ_i = dS K      (A = dS^T from SMEM read MN-major) -> drained by a 4th
//                    warpgroup into fp32 dQ with TMA tensor reduce-add
// TMEM: S^T[0,128) dP^T/dS^T[128,256) dV[256,320) dK[320,384) dQ[384,448) P^T[448,512)
// 16 warps: 0 TMA, 1 MMA, 2 TMEM alloc + aux builder, 3 aux builder, 4-11
// elementwise, 12-15 dQ drain; setmaxnreg gives the elementwise warps the registers.
// Pipelining: S_{i+1} is issued as soon as the elementwise warps hold S^T_i in
// registers, dV_i as soon as P^T_i is in TMEM, and dK_i dP_{i+1} dQ_i after dS_i,
// so the only tensor work the elementwise warps can wait on is dP_{i+1}; a 3-stage
// Q / dO ring keeps S_{i+1}'s operands resident a phase early.
#pragma once
#include "attn_fwd.cuh"
#include "common.cuh"

#ifndef LSS_BWD_POLY8
#define LSS_BWD_POLY8 2  // exponent pairs (of every 8) on the FMA-pipe polynomial (A/B ms, current kernel: 0/8 14.8, 1/8 13.46, 2/8 13.40, 3/8 13.70, 4/8 13.67)
#endif

namespace lss {

#ifndef LSS_BWD_FOLD
#define LSS_BWD_FOLD 1  // lse2 / delta folded into the S^T / dP^T MMAs (no-dropout instance)
#endif
// Folding: S^T - lse2/c and dP^T - delta are produced by the tensor core with one
// extra K16 step each, A = a constant all-ones tile and B = a per-query-tile
// operand holding -lse2/c (resp. -delta) split into two bf16 terms (hi + lo, ~2^-17
// relative): the elementwise warps then need no per-column broadcast loads
// (512 shared-memory wavefronts per tile, ~19% of the kernel's SMEM traffic, and
// 2 x 64 registers).  The operands are K16 slices (128 rows x 32 bytes) of two
// 128-byte-swizzled K-major tiles (the 32-byte swizzle reads 3x slower on the
// tensor core): tile 0 = [ones | L_0 | L_1 | L_2], tile 1 = [D_0 | D_1 | D_2 | -].
// Without FOLD (dropout instance) the region holds the per-stage lse2 / delta.
constexpr int ATB_AUX_STAGES = 3;                    // aux ring: built up to 3 query tiles ahead
constexpr int ATB_AUX_BYTES = 2 * ATT_TILE_BYTES;    // the two aux tiles
constexpr int ATB_QSTAGE_BYTES = 2 * ATT_TILE_BYTES;  // Q, dO
constexpr int ATB_QSTAGES = 3;                        // Q / dO ring: S_{i+1} is issued one phase earlier
constexpr int ATB_DS_BYTES = 2 * ATT_TILE_BYTES;      // dS^T tile: 2 sub-tiles [128 kv][64 q]
constexpr int ATB_STG_BYTES = 128 * 64 * 4;                      // dQ staging [128 q][64] fp32 (2 SW128 halves)
constexpr int ATB_SMEM = 2 * ATT_TILE_BYTES /*K,V*/ + ATB_QSTAGES * ATB_QSTAGE_BYTES + ATB_DS_BYTES + ATB_STG_BYTES +
                         ATB_AUX_BYTES + 1024 + 256;
static_assert(ATB_SMEM <= 232448, "backward shared memory");
#ifndef LSS_BWD_EW
#define LSS_BWD_EW 2  // elementwise warpgroups (A/B builds: 4 = 32 query columns per thread)
#endif
constexpr int ATB_EW = LSS_BWD_EW;

// setmaxnreg budgets (control WG, elementwise WGs, dQ-drain WG): sum <= 64K registers
// setmaxnreg.inc draws only on what the CTA's .dec warps released: with the launch
// allocation A = 65536 / threads rounded down to 8 (128 at EW=2, 80 at EW=4),
// 128*(A-CTRL) + 128*(A-DRAIN) >= 128*EW*(EW_REGS - A), or the .inc waits forever
#ifndef LSS_BWD_REG_CTRL
#define LSS_BWD_REG_CTRL (LSS_BWD_EW == 2 ? 56 : 40)
#endif
#ifndef LSS_BWD_REG_DRAIN
#define LSS_BWD_REG_DRAIN (LSS_BWD_EW == 2 ? 80 : 56)
#endif
#ifndef LSS_BWD_REG_EW
#define LSS_BWD_REG_EW (LSS_BWD_EW == 2 ? 184 : 96)
#endif
constexpr int ATB_REG_CTRL = LSS_BWD_REG_CTRL;
constexpr int ATB_REG_EW = LSS_BWD_REG_EW;
constexpr int ATB_REG_DRAIN = LSS_BWD_REG_DRAIN;
constexpr int ATB_REG_LAUNCH = (65536 / (128 * (2 + ATB_EW))) / 8 * 8;
static_assert((ATB_REG_LAUNCH - ATB_REG_CTRL) + (ATB_REG_LAUNCH - ATB_REG_DRAIN) >=
                  ATB_EW * (ATB_REG_EW - ATB_REG_LAUNCH), "setmaxnreg: the elementwise warps would wait forever");
constexpr int ATB_NC = 128 / ATB_EW;                // query columns per elementwise thread
constexpr int ATB_THREADS = 128 * (2 + ATB_EW);     // control WG + EW WGs + dQ-drain WG

// A query-row source of the backward: rows [row0, row0+rows) of a [B][m_src][E]
// (Q, dO, dQ) tensor triple whose row 0 sits at global position pos0, attending
// key segments [g_begin, g_end).  A launch processes up to ATB_MAX_SRC sources
// (this rank's own rows, and rows delegated by a partner in the balanced causal
// schedule); every key tile accumulates dK/dV from all of them in TMEM, so each
// dK/dV row has exactly one writer.
constexpr int ATB_MAX_SRC = 3;
constexpr int ATB_MAX_SEG = 16;  // workers reachable through the segment table (one NVLink domain)
struct BwdSource {
  int row0, rows;
  long pos0;
  int g_begin, g_end;
  const float* lse2;   // [B][H][pitch] (+inf beyond the tensor's last row)
  const float* delta;  // [B][H][pitch] rowsum(dO*O)/sqrt(d)
  int pitch;
  int m_src;           // rows of the [B][m_src][E] tensors
  float* dq;           // fp32 [B][m_src][E], accumulated with vector reductions
  long long* dq_fixed; // deterministic mode: int64 [B][m_src][E], round(dQ * 2^32), integer adds
  const uint32_t* ready;  // non-null: inputs pushed by a partner, usable once *ready >= ready_seq
  uint32_t ready_seq;
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
  // dK|dV destination of key segment g: a [B][seg_len][ld_dkv] fp32 block, dK at
  // column h*d and dV at dv_off + h*d, fully written.  Either one local buffer
  // (seg_tab null: block g at dkv + g*seg_stride, the reduce-scatter input) or a
  // table of per-segment blocks that may live in PEER memory (the owner's receive
  // slot for this rank): the reduce-scatter then happens inside this epilogue.
  float* dkv;
  long seg_stride;
  long dv_off;
  long ld_dkv;
  int peer;                     // seg_tab entries are peer (NVLink) memory (informational)
  // attention-probability dropout (DROP instances; model.scores_bwd, model.py:350-352)
  uint64_t drop_site;
  uint64_t drop_thresh;
  float drop_scale;
  float* seg_tab[ATB_MAX_SEG];  // used when seg_tab[0] != nullptr
  int g_lo;                     // first key segment of the grid (the fused path skips segments no source reads)
};

LSS_DEV void bulk_load_1d(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

#ifdef LSS_BWD_TRACE
__device__ long long g_bwd_trace[20][512];
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

template <int N>
LSS_DEV void tmem_ld_n(uint32_t taddr, uint32_t (&r)[N]);
template <>
LSS_DEV void tmem_ld_n<32>(uint32_t taddr, uint32_t (&r)[32]) { tmem_ld32(taddr, r); }
template <>
LSS_DEV void tmem_ld_n<64>(uint32_t taddr, uint32_t (&r)[64]) { tmem_ld64(taddr, r); }
template <>
LSS_DEV void tmem_ld_n<16>(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : LSS_R8(0), LSS_R8(8)
      : "r"(taddr)
      : "memory");
}
template <int N>
LSS_DEV void tmem_st_n(uint32_t taddr, const uint32_t (&r)[N]);
template <>
LSS_DEV void tmem_st_n<32>(uint32_t taddr, const uint32_t (&r)[32]) { tmem_st32(taddr, r); }
template <>
LSS_DEV void tmem_st_n<16>(uint32_t taddr, const uint32_t (&r)[16]) { tmem_st16(taddr, r); }

template <int NC>
LSS_DEV void bwd_ld_vec(uint32_t saddr, float (&v)[NC]) {
#pragma unroll
  for (int c4 = 0; c4 < NC / 4; ++c4) {
    const float4 l = ld_shared_f4(saddr + c4 * 16);
    v[4 * c4] = l.x;
    v[4 * c4 + 1] = l.y;
    v[4 * c4 + 2] = l.z;
    v[4 * c4 + 3] = l.w;
  }
}

// keep bits of the thread's key row (global position kpos) against query columns
// q_first .. q_first+NC-1 of head (b, h): the forward's mask, recomputed
template <int NC>
LSS_DEV uint64_t bwd_drop_bits(uint64_t head_key, long q_first, long kpos, uint64_t thresh) {
  uint64_t bits = 0;
#pragma unroll 4
  for (int c = 0; c < NC; ++c)
    bits |= (uint64_t)drop_keep(drop_mix(head_key, (uint64_t)(q_first + c)), (uint64_t)kpos, thresh) << c;
  return bits;
}

template <bool MASK, bool DROP, int NC>
LSS_DEV void bwd_p(uint32_t (&sv)[NC], const float (&lse)[NC], float sl2, int fv, uint32_t (&pk)[NC / 2],
                   uint64_t keep = 0, float dscale = 1.f) {
  const float2 sl2v = make_float2(sl2, sl2);
#pragma unroll
  for (int c = 0; c < NC; c += 2) {
    const float2 x = ffma2(make_float2(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), sl2v,
                           make_float2(-lse[c], -lse[c + 1]));
    float2 e;
    if (!MASK && ((c / 2) & 7) < LSS_BWD_POLY8) {  // MUFU/FMA balance
      e = exp2_poly2(x);
    } else {
      e = make_float2(ex2(x.x), ex2(x.y));
    }
    if (MASK) {
      e.x = (c >= fv) ? e.x : 0.f;
      e.y = (c + 1 >= fv) ? e.y : 0.f;
    }
    sv[c] = __float_as_uint(e.x);  // dS needs the undropped probabilities
    sv[c + 1] = __float_as_uint(e.y);
    if (DROP) {  // dV uses the dropped ones (aw_d)
      e.x = ((keep >> c) & 1) ? e.x * dscale : 0.f;
      e.y = ((keep >> (c + 1)) & 1) ? e.y * dscale : 0.f;
    }
    pk[c / 2] = pack_bf16(e.x, e.y);
  }
}

// Folded variants: the accumulator already holds S^T - lse2/c (resp. dP^T - delta)
template <bool MASK, int NC>
LSS_DEV void bwd_p_f(uint32_t (&sv)[NC], float sl2, int fv, uint32_t (&pk)[NC / 2]) {
  const float2 sl2v = make_float2(sl2, sl2);
#pragma unroll
  for (int c = 0; c < NC; c += 2) {
    const float2 x = fmul2(make_float2(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), sl2v);
    float2 e;
    if (!MASK && ((c / 2) & 7) < LSS_BWD_POLY8) {
      e = exp2_poly2(x);
    } else {
      e = make_float2(ex2(x.x), ex2(x.y));
    }
    if (MASK) {
      e.x = (c >= fv) ? e.x : 0.f;
      e.y = (c + 1 >= fv) ? e.y : 0.f;
    }
    sv[c] = __float_as_uint(e.x);
    sv[c + 1] = __float_as_uint(e.y);
    pk[c / 2] = pack_bf16(e.x, e.y);
  }
}
template <int C0, int NH, int NC>
LSS_DEV void bwd_ds_f(const uint32_t (&pv)[NC], const uint32_t (&dp)[NH], float scale, uint32_t (&dk)[NC / 2]) {
  const float2 scv = make_float2(scale, scale);
#pragma unroll
  for (int c = 0; c < NH; c += 2) {
    const float2 pp = fmul2(make_float2(__uint_as_float(pv[C0 + c]), __uint_as_float(pv[C0 + c + 1])), scv);
    const float2 ds = fmul2(pp, make_float2(__uint_as_float(dp[c]), __uint_as_float(dp[c + 1])));
    dk[(C0 + c) / 2] = pack_bf16(ds.x, ds.y);
  }
}

// hi + lo bf16 split of v (lo = 0 when v is infinite: padded query rows carry lse2 = +inf)
LSS_DEV uint32_t bf16_hilo(float v) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(v);
  float r = v - __bfloat162float(hi);
  if (!(fabsf(r) < INFINITY)) r = 0.f;
  const __nv_bfloat16 lo = __float2bfloat16_rn(r);
  return (uint32_t)__bfloat16_as_ushort(hi) | ((uint32_t)__bfloat16_as_ushort(lo) << 16);
}

// Register-lean variants for 32-column slices (4 elementwise warpgroups): lse2 and
// the scaled delta are read from shared memory 4 columns at a time (128-bit
// broadcast loads) instead of being held in 2 x NC registers.
template <bool MASK, bool DROP, int NC>
LSS_DEV void bwd_p_s(uint32_t (&sv)[NC], uint32_t s_lse, float sl2, int fv, uint32_t (&pk)[NC / 2],
                     uint64_t keep = 0, float dscale = 1.f) {
  const float2 sl2v = make_float2(sl2, sl2);
#pragma unroll
  for (int c4 = 0; c4 < NC; c4 += 4) {
    const float4 l = ld_shared_f4(s_lse + c4 * 4);
    const float lse[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
    for (int c = c4; c < c4 + 4; c += 2) {
      const float2 x = ffma2(make_float2(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), sl2v,
                             make_float2(-lse[c - c4], -lse[c - c4 + 1]));
      float2 e;
      if (!MASK && ((c / 2) & 7) < LSS_BWD_POLY8) {
        e = exp2_poly2(x);
      } else {
        e = make_float2(ex2(x.x), ex2(x.y));
      }
      if (MASK) {
        e.x = (c >= fv) ? e.x : 0.f;
        e.y = (c + 1 >= fv) ? e.y : 0.f;
      }
      sv[c] = __float_as_uint(e.x);
      sv[c + 1] = __float_as_uint(e.y);
      if (DROP) {
        e.x = ((keep >> c) & 1) ? e.x * dscale : 0.f;
        e.y = ((keep >> (c + 1)) & 1) ? e.y * dscale : 0.f;
      }
      pk[c / 2] = pack_bf16(e.x, e.y);
    }
  }
}

template <int C0, int NH, int NC, bool DROP>
LSS_DEV void bwd_ds_s(const uint32_t (&pv)[NC], const uint32_t (&dp)[NH], uint32_t s_dsc, float scale,
                      uint32_t (&dk)[NC / 2], uint64_t keep = 0, float dscale = 1.f) {
  const float2 scv = make_float2(scale, scale);
#pragma unroll
  for (int c4 = 0; c4 < NH; c4 += 4) {
    const float4 d = ld_shared_f4(s_dsc + (C0 + c4) * 4);
    const float dsc[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
    for (int c = c4; c < c4 + 4; c += 2) {
      float2 sc = scv;
      if (DROP) {
        sc.x = ((keep >> (C0 + c)) & 1) ? scale * dscale : 0.f;
        sc.y = ((keep >> (C0 + c + 1)) & 1) ? scale * dscale : 0.f;
      }
      const float2 t = ffma2(make_float2(__uint_as_float(dp[c]), __uint_as_float(dp[c + 1])), sc,
                             make_float2(-dsc[c - c4], -dsc[c - c4 + 1]));
      const float2 ds = fmul2(make_float2(__uint_as_float(pv[C0 + c]), __uint_as_float(pv[C0 + c + 1])), t);
      dk[(C0 + c) / 2] = pack_bf16(ds.x, ds.y);
    }
  }
}

// dS^T for columns [C0, C0+NH) of the thread's slice: ds = p (dp/sqrt(d) - delta/sqrt(d));
// with dropout dp is the gradient of the dropped probabilities and is masked first
// (grad_aw = grad_aw_d * keep * 1/(1-rate))
template <int C0, int NH, int NC, bool DROP>
LSS_DEV void bwd_ds(const uint32_t (&pv)[NC], const uint32_t (&dp)[NH], const float (&dsc)[NC], float scale,
                    uint32_t (&dk)[NC / 2], uint64_t keep = 0, float dscale = 1.f) {
  const float2 scv = make_float2(scale, scale);
#pragma unroll
  for (int c = 0; c < NH; c += 2) {
    float2 sc = scv;
    if (DROP) {
      sc.x = ((keep >> (C0 + c)) & 1) ? scale * dscale : 0.f;
      sc.y = ((keep >> (C0 + c + 1)) & 1) ? scale * dscale : 0.f;
    }
    const float2 t = ffma2(make_float2(__uint_as_float(dp[c]), __uint_as_float(dp[c + 1])), sc,
                           make_float2(-dsc[C0 + c], -dsc[C0 + c + 1]));
    const float2 ds =
        fmul2(make_float2(__uint_as_float(pv[C0 + c]), __uint_as_float(pv[C0 + c + 1])), t);
    dk[(C0 + c) / 2] = pack_bf16(ds.x, ds.y);
  }
}

template <bool DROP>
__global__ void __launch_bounds__(ATB_THREADS, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       const __grid_constant__ BwdMaps maps, const __grid_constant__ AttnBwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + ATT_TILE_BYTES;
  uint8_t* sQst = sV + ATT_TILE_BYTES;                   // ATB_QSTAGES stages: Q, dO
  uint8_t* sdS = sQst + ATB_QSTAGES * ATB_QSTAGE_BYTES;  // 2 sub-tiles [128 kv][64 q] bf16
  uint8_t* sStage = sdS + ATB_DS_BYTES;                  // dQ staging, 2 x [128 q][32] fp32 (SW128)
  uint8_t* sAux = sStage + ATB_STG_BYTES;  // FOLD: aux tiles; otherwise lse2 / delta per Q stage
  uint64_t* bars = reinterpret_cast<uint64_t*>(sAux + ATB_AUX_BYTES);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;   // [ATB_QSTAGES]
  uint64_t* q_empty = bars + 4;  // [ATB_QSTAGES]
  uint64_t* s_full = bars + 7;   // S^T_i in TMEM
  uint64_t* s_empty = bars + 8;  // S^T_i loaded into registers (S_{i+1} may overwrite it)
  uint64_t* p_full = bars + 9;   // P^T_i in TMEM
  uint64_t* dv_done = bars + 10; // dV_i complete (the P^T columns are free)
  uint64_t* dp_full = bars + 11; // dP^T_i in TMEM (and every earlier MMA complete)
  uint64_t* ds_full = bars + 12; // dS^T_i in TMEM + SMEM (dP^T_i consumed)
  uint64_t* mma_done = bars + 13;  // one-shot: every MMA of the CTA complete
  uint64_t* dq_full = bars + 14;   // dQ_i in TMEM
  uint64_t* dq_empty = bars + 15;  // dQ_i read out by the drain
  uint64_t* ds_free = bars + 16;   // dQ_i has read the SMEM dS tile
  uint64_t* aux_full = bars + 17;  // [ATB_AUX_STAGES] FOLD: aux L / D operands built
  uint64_t* aux_empty = bars + 17 + ATB_AUX_STAGES;  // [ATB_AUX_STAGES] S_it and dP_it complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17 + 2 * ATB_AUX_STAGES);
  // K16 slice addresses inside the aux tiles
  auto aux_l = [&](int s) { return smem_u32(sAux) + (1 + s) * 32; };
  auto aux_d = [&](int s) { return smem_u32(sAux + ATT_TILE_BYTES) + s * 32; };
  auto stats = [&](int s) { return sAux + s * 1024; };  // !FOLD: lse2[128] | delta[128] of Q stage s
  constexpr bool FOLD = LSS_BWD_FOLD && !DROP;

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  // head-major dispatch (key tiles fastest): the ~148 resident CTAs share one or
  // two heads' Q/dO stream in L2 (head-fastest order measured 2% slower)
  const int h = blockIdx.y;
  const int b = blockIdx.z;
  const int tps = (p.seg_len + ATT_BN - 1) / ATT_BN;
  const int g = p.g_lo + (int)blockIdx.x / tps;
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
  auto locate = [&](int it, int& s_out, int& qrow_out) {  // (register selects: no local-memory indexing)
    int s = 0;
#pragma unroll
    for (int k = 0; k < ATB_MAX_SRC - 1; ++k)
      if (s == k && it >= src_n[k]) {
        it -= src_n[k];
        s = k + 1;
      }
    int first = src_first[0];
#pragma unroll
    for (int k = 1; k < ATB_MAX_SRC; ++k)
      if (s == k) first = src_first[k];
    s_out = s;
    qrow_out = p.src[s].row0 + (first + it) * ATT_BM;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(kv_full, 1);
    for (int s = 0; s < ATB_QSTAGES; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < ATB_AUX_STAGES; ++s) {
      mbar_init(&aux_full[s], 64);
      mbar_init(&aux_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, 128 * ATB_EW);
    mbar_init(p_full, 128 * ATB_EW);
    mbar_init(dv_done, 1);
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 128 * ATB_EW);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 128);
    mbar_init(ds_free, 1);
    mbar_init(mma_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  if (FOLD && warp == 3) {  // the ones operand
    const uint32_t one2 = 0x3F803F80u;  // slice 0 of aux tile 0: chunks 0, 1 of every row
    for (int r = lane; r < 128; r += 32) {
      const uint32_t row = smem_u32(sAux) + r * 128;
      st_shared_v4(row + ((0 ^ (r & 7)) << 4), one2, one2, one2, one2);
      st_shared_v4(row + ((1 ^ (r & 7)) << 4), one2, one2, one2, one2);
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // P^T (bf16) overwrites S^T and dS^T overwrites dP^T: elementwise warpgroup qd
  // reads fp32 columns [qd*NC, +NC) and writes its packed bf16 result to the first
  // half of those same columns, so no warpgroup overwrites data another still reads.
  const uint32_t tS = tmem + 0, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 320, tdQ = tmem + 384,
                 tP = tmem + 448;

  if (warp < 4) {
    reg_dealloc<ATB_REG_CTRL>();
    if (warp == 0) {
      if (n_iter > 0) {
        // ------------------------------------------------ TMA producer (warp-uniform loop)
        if (elect_one()) {
          mbar_arrive_expect_tx(kv_full, 2 * ATT_TILE_BYTES);
          tma_load_4d(&tmK, kv_full, sK, h * ATT_D, kv_row0, b, g);
          tma_load_4d(&tmV, kv_full, sV, h * ATT_D, kv_row0, b, g);
        }
        __syncwarp();
        int src_ready = -1;  // last source whose pushed inputs were waited for
        for (int it = 0; it < n_iter; ++it) {
          const int s = it % ATB_QSTAGES;
          mbar_wait(&q_empty[s], ((it / ATB_QSTAGES) & 1) ^ 1);
          if (lane == 0) BWD_TRACE(18, it);
          int src, q0;
          locate(it, src, q0);
          if (p.src[src].ready != nullptr && src != src_ready) {  // fused hand-off: wait for the push
            if (lane == 0) wait_flag_geq(p.src[src].ready, p.src[src].ready_seq);
            __syncwarp();
            src_ready = src;
          }
          uint8_t* st = sQst + s * ATB_QSTAGE_BYTES;
          const long lo = ((long)b * p.H + h) * p.src[src].pitch + q0;
          if (elect_one()) {
            mbar_arrive_expect_tx(&q_full[s], 2 * ATT_TILE_BYTES + (FOLD ? 0 : 1024));
            tma_load_3d(&maps.q[src], &q_full[s], st, h * ATT_D, q0, b);
            tma_load_3d(&maps.dO[src], &q_full[s], st + ATT_TILE_BYTES, h * ATT_D, q0, b);
            if (!FOLD) {  // FOLD: the aux builders read the row statistics themselves
              bulk_load_1d(stats(s), p.src[src].lse2 + lo, 512, &q_full[s]);
              bulk_load_1d(stats(s) + 512, p.src[src].delta + lo, 512, &q_full[s]);
            }
          }
          __syncwarp();
        }
      }
    } else if (FOLD && warp >= 2) {
      // ------------------------------------------------ aux operand builders (warps 2-3):
      // row r of aux L = (-lse2[r]/c) as hi|lo bf16, aux D = (-delta_raw[r]) likewise,
      // K columns 2..15 of the slice zero.
      // Their own ring (aux_empty is committed after dP_it) lets them run up to
      // ATB_AUX_STAGES tiles ahead of the tensor core, reading lse2 / delta from global
      // memory directly, so the build latency stays off the S / dP issue path.
      const float inv_c = -1.f / p.scale_log2, inv_s = -1.f / p.scale;
      const int j = (int)(warp - 2) * 32 + (int)lane;  // rows j and j + 64
      int src_ready = -1;  // last source whose pushed inputs were waited for
      for (int it = 0; it < n_iter; ++it) {
        const int s = it % ATB_AUX_STAGES;
        int src, q0;
        locate(it, src, q0);
        if (p.src[src].ready != nullptr && src != src_ready) {  // fused hand-off: lse2 / delta pushed too
          if (lane == 0) wait_flag_geq(p.src[src].ready, p.src[src].ready_seq);
          __syncwarp();
          src_ready = src;
        }
        const long lo = ((long)b * p.H + h) * p.src[src].pitch + q0;
        float l2v[2], dsv[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {  // coherent loads: a partner may have pushed them during this launch
          asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(l2v[k]) : "l"(p.src[src].lse2 + lo + j + 64 * k)
                       : "memory");
          asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(dsv[k]) : "l"(p.src[src].delta + lo + j + 64 * k)
                       : "memory");
        }
        if (it >= ATB_AUX_STAGES) mbar_wait(&aux_empty[s], (it / ATB_AUX_STAGES - 1) & 1);
        const uint32_t al = aux_l(s), ad = aux_d(s);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int r = j + 64 * k;
          const uint32_t hl = bf16_hilo(l2v[k] * inv_c), hd = bf16_hilo(dsv[k] * inv_s);
          // slice base + row r: logical chunks 0 / 1 of the slice, SW128 XOR by (r & 7)
          const uint32_t x = (uint32_t)(r & 7) << 4, rl = (al & ~127u) + r * 128, rd = (ad & ~127u) + r * 128;
          const uint32_t cl = al & 127u, cd = ad & 127u;  // slice byte offset in the row
          st_shared_v4(rl + (cl ^ x), hl, 0u, 0u, 0u);
          st_shared_v4(rl + ((cl + 16) ^ x), 0u, 0u, 0u, 0u);
          st_shared_v4(rd + (cd ^ x), hd, 0u, 0u, 0u);
          st_shared_v4(rd + ((cd + 16) ^ x), 0u, 0u, 0u, 0u);
        }
        fence_proxy_async_smem();
        mbar_arrive(&aux_full[s]);
      }
    } else if (warp == 1) {
      if (n_iter > 0) {
        // ------------------------------------------------ MMA issuer (warp-uniform loop,
        // one elected lane issues: descriptors stay in the uniform datapath)
        constexpr uint32_t idSS = idesc_bf16_f32(128, 128, 0, 0);  // S^T, dP^T
        constexpr uint32_t idKN = idesc_bf16_f32(128, 64, 0, 1);   // dV, dK (B MN-major)
        constexpr uint32_t idQ = idesc_bf16_f32(128, 64, 1, 1);    // dQ (A and B MN-major)
        const uint32_t k_addr = smem_u32(sK), v_addr = smem_u32(sV), ones_addr = smem_u32(sAux);
        // K16 step k of a bf16 TMEM operand written by the elementwise warpgroups
        auto ew_col = [](int k) { return (uint32_t)((16 * k / ATB_NC) * ATB_NC + (16 * k % ATB_NC) / 2); };
        auto q_stage = [&](int it) { return smem_u32(sQst + (it % ATB_QSTAGES) * ATB_QSTAGE_BYTES); };
        auto issue_s = [&](int it) {  // S^T_it = K Q_it^T
          if (lane == 0) BWD_TRACE(16, it);
          mbar_wait(&q_full[it % ATB_QSTAGES], (it / ATB_QSTAGES) & 1);
          if (FOLD) mbar_wait(&aux_full[it % ATB_AUX_STAGES], (it / ATB_AUX_STAGES) & 1);
          tc_fence_after();
          if (lane == 0) BWD_TRACE(17, it);
          const uint32_t q_addr = q_stage(it);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < ATT_D / 16; ++k)
              mma_bf16_ss(tS, smem_desc_sw128(k_addr + k * 32, 16, 1024),
                          smem_desc_sw128(q_addr + k * 32, 16, 1024), idSS, k > 0);
            if (FOLD)  // += 1 * (-lse2/c)
              mma_bf16_ss(tS, smem_desc_sw128(ones_addr, 16, 1024), smem_desc_sw128(aux_l(it % ATB_AUX_STAGES), 16, 1024),
                          idSS, 1u);
            mma_commit(s_full);
          }
          __syncwarp();
        };
        auto issue_dp = [&](int it) {  // dP^T_it = V dO_it^T (stage already resident)
          const uint32_t do_addr = q_stage(it) + ATT_TILE_BYTES;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < ATT_D / 16; ++k)
              mma_bf16_ss(tdP, smem_desc_sw128(v_addr + k * 32, 16, 1024),
                          smem_desc_sw128(do_addr + k * 32, 16, 1024), idSS, k > 0);
            if (FOLD)  // += 1 * (-delta)
              mma_bf16_ss(tdP, smem_desc_sw128(ones_addr, 16, 1024),
                          smem_desc_sw128(aux_d(it % ATB_AUX_STAGES), 16, 1024), idSS, 1u);
            mma_commit(dp_full);
            if (FOLD) mma_commit(&aux_empty[it % ATB_AUX_STAGES]);
          }
          __syncwarp();
        };
        auto issue_dv = [&](int it) {  // dV += P^T_it dO_it once P^T_it is in TMEM
          mbar_wait(p_full, it & 1);
          tc_fence_after();
          if (lane == 0) BWD_TRACE(6, it);
          const uint32_t do_addr = q_stage(it) + ATT_TILE_BYTES;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < ATT_BM / 16; ++k)
              mma_bf16_ts(tdV, tP + 8 * k, smem_desc_sw128(do_addr + k * 2048, 8192, 1024), idKN,
                          (it > 0 || k > 0));
            mma_commit(dv_done);
          }
          __syncwarp();
        };
        auto issue_dq = [&](int it) {  // dQ_it = dS_it K into TMEM once the drain read dQ_{it-1}
          if (it > 0) {
            mbar_wait(dq_empty, (it - 1) & 1);
            tc_fence_after();
          }
          const uint32_t ds_addr = smem_u32(sdS);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < ATT_BN / 16; ++k)
              mma_bf16_ss(tdQ, smem_desc_sw128(ds_addr + k * 2048, ATT_TILE_BYTES, 1024),
                          smem_desc_sw128(k_addr + k * 2048, 8192, 1024), idQ, k > 0);
            mma_commit(dq_full);
            mma_commit(ds_free);
          }
          __syncwarp();
        };
        mbar_wait(kv_full, 0);
        tc_fence_after();
        issue_s(0);
        issue_dp(0);
        // Tensor-pipe order (in-order execution):
        //   S_{i+1} dV_i | dK_i dP_{i+1} dQ_i | S_{i+2} dV_{i+1} | ...
        // P^T has its own TMEM columns, so S_{i+1} is issued as soon as the elementwise
        // warps have S^T_i in registers (s_empty) and is long complete when they come
        // back from dS_i; dP_{i+1} follows dK_i (it overwrites dS^T_i); dQ_i reads the
        // single SMEM dS tile and lands in TMEM for the drain warps.
        for (int it = 0; it < n_iter; ++it) {
          const bool more = it + 1 < n_iter;
          if (more) {
            mbar_wait(s_empty, it & 1);
            tc_fence_after();
            issue_s(it + 1);
          }
          issue_dv(it);
          if (lane == 0) BWD_TRACE(14, it);
          mbar_wait(ds_full, it & 1);
          tc_fence_after();
          if (lane == 0) BWD_TRACE(0, it);
          const uint32_t q_addr = q_stage(it);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < ATT_BM / 16; ++k)  // dK += dS^T Q  (A = dS^T from TMEM)
              mma_bf16_ts(tdK, tdP + ew_col(k), smem_desc_sw128(q_addr + k * 2048, 8192, 1024), idKN,
                          (it > 0 || k > 0));
            mma_commit(&q_empty[it % ATB_QSTAGES]);
          }
          __syncwarp();
          if (more) issue_dp(it + 1);
          if (lane == 0) BWD_TRACE(15, it);
          issue_dq(it);
          if (lane == 0) BWD_TRACE(8, it);
        }
        if (elect_one()) mma_commit(mma_done);
        __syncwarp();
      }
    }
  } else if (warp < 4 + 4 * ATB_EW) {
    reg_alloc<ATB_REG_EW>();
    // ------------------------------------------------ elementwise P^T / dS^T (+ dK/dV epilogue)
    const int qd = (warp - 4) / 4;    // query columns [NC*qd, NC*qd + NC) of each tile
    const int quad = warp % 4;
    const int t = quad * 32 + lane;   // key row within tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const long kpos = kpos0 + t;
    const uint64_t drop_head = DROP ? drop_mix(drop_mix(p.drop_site, (uint64_t)b + 1), (uint64_t)h + 1) : 0;
    const bool row_ok = t < kv_valid;
    constexpr int NC = ATB_NC;
    for (int it = 0; it < n_iter; ++it) {
      int src, qrow;
      locate(it, src, qrow);
      const long q0 = p.src[src].pos0 + qrow;  // global position of the tile's first query
      const uint32_t s_lse = smem_u32(stats(it % ATB_QSTAGES)) + qd * NC * 4;        // lse2[q]
      const uint32_t s_dsc = smem_u32(stats(it % ATB_QSTAGES)) + 512 + qd * NC * 4;  // delta[q]/sqrt(d)
      // ---- P^T = 2^(S^T log2e/sqrt(d) - lse2) into the P^T columns once dV_{it-1} has read them
      constexpr bool LEAN = NC < 64;  // 4 warpgroups: lse / delta streamed from SMEM
      float lse[FOLD ? 1 : NC];  // issued ahead of the S wait: the loads queue behind the tensor
      if constexpr (!FOLD) {      // core's SMEM operand traffic
        mbar_wait(&q_full[it % ATB_QSTAGES], (it / ATB_QSTAGES) & 1);
        if constexpr (!LEAN) bwd_ld_vec<NC>(s_lse, lse);
      }
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      if (t == 0 && qd == 0) BWD_TRACE(1, it);
      uint32_t sv[NC];
      tmem_ld_n<NC>(tS + lane_off + qd * NC, sv);
      tc_fence_before();
      mbar_arrive(s_empty);  // S_{it+1} may overwrite S^T
      if (t == 0 && qd == 0) BWD_TRACE(7, it);
      // query column c of this slice is visible to key row t iff c >= fv
      const bool need_mask = !row_ok || (p.causal && kpos0 + ATT_BN - 1 > q0 + qd * NC);
      const uint64_t keep = DROP ? bwd_drop_bits<NC>(drop_head, q0 + qd * NC, kpos, p.drop_thresh) : 0;
      {
        uint32_t pk[NC / 2];
        if (need_mask) {
          const long first_vis = kpos - q0 - qd * NC;
          const int fv = !row_ok ? NC : (p.causal ? (int)max(0L, min((long)NC, first_vis)) : 0);
          if constexpr (FOLD)
            bwd_p_f<true, NC>(sv, p.scale_log2, fv, pk);
          else if constexpr (LEAN)
            bwd_p_s<true, DROP, NC>(sv, s_lse, p.scale_log2, fv, pk, keep, p.drop_scale);
          else
            bwd_p<true, DROP, NC>(sv, lse, p.scale_log2, fv, pk, keep, p.drop_scale);
        } else {
          if constexpr (FOLD)
            bwd_p_f<false, NC>(sv, p.scale_log2, 0, pk);
          else if constexpr (LEAN)
            bwd_p_s<false, DROP, NC>(sv, s_lse, p.scale_log2, 0, pk, keep, p.drop_scale);
          else
            bwd_p<false, DROP, NC>(sv, lse, p.scale_log2, 0, pk, keep, p.drop_scale);
        }
        if (t == 0 && qd == 0) BWD_TRACE(13, it);
        if (it > 0) {
          mbar_wait(dv_done, (it - 1) & 1);
          tc_fence_after();
        }
        tmem_st_n<NC / 2>(tP + lane_off + qd * (NC / 2), pk);
      }
      tc_fence_before();
      mbar_arrive(p_full);
      if (t == 0 && qd == 0) BWD_TRACE(2, it);
      // ---- dS^T = P^T (dP^T/sqrt(d) - delta/sqrt(d)): dP_it completing implies dK_{it-1}
      // (TMEM dS^T reader) completed; dQ_{it-1} (the SMEM dS reader) signals ds_free.
      float dsc[FOLD ? 1 : NC];  // delta loads issued before the dP wait (same reason as lse)
      if constexpr (!LEAN && !FOLD) bwd_ld_vec<NC>(s_dsc, dsc);
      // the SMEM dS tile is free once dQ_{it-1} completed (long before dP_it, in practice)
      if (it > 0) mbar_wait(ds_free, (it - 1) & 1);
      if (t == 0 && qd == 0) BWD_TRACE(11, it);
      mbar_wait(dp_full, it & 1);
      tc_fence_after();
      if (t == 0 && qd == 0) BWD_TRACE(3, it);
      {
        // dS^T row t, query columns [NC*qd, +NC) -> SW128 K-major sub-tile (64 q per
        // sub-tile); each half is stored as soon as it is computed, so the proxy fence
        // below waits only for the second half's stores
        const int sub = (qd * NC) / 64, c0 = ((qd * NC) % 64) / 8;  // 16-byte chunk index in the 128B row
        const uint32_t row = smem_u32(sdS + sub * ATT_TILE_BYTES + t * 128);
        uint32_t dk[NC / 2];
        {  // dP^T in two halves keeps p, delta and dP within the register budget
          uint32_t dp[NC / 2];
          tmem_ld_n<NC / 2>(tdP + lane_off + qd * NC, dp);
          if constexpr (FOLD)
            bwd_ds_f<0, NC / 2, NC>(sv, dp, p.scale, dk);
          else if constexpr (LEAN)
            bwd_ds_s<0, NC / 2, NC, DROP>(sv, dp, s_dsc, p.scale, dk, keep, p.drop_scale);
          else
            bwd_ds<0, NC / 2, NC, DROP>(sv, dp, dsc, p.scale, dk, keep, p.drop_scale);
        }
#pragma unroll
        for (int c = 0; c < NC / 16; ++c)
          st_shared_v4(row + (((c0 + c) ^ (t & 7)) << 4), dk[4 * c], dk[4 * c + 1], dk[4 * c + 2], dk[4 * c + 3]);
        {
          uint32_t dp[NC / 2];
          tmem_ld_n<NC / 2>(tdP + lane_off + qd * NC + NC / 2, dp);
          if constexpr (FOLD)
            bwd_ds_f<NC / 2, NC / 2, NC>(sv, dp, p.scale, dk);
          else if constexpr (LEAN)
            bwd_ds_s<NC / 2, NC / 2, NC, DROP>(sv, dp, s_dsc, p.scale, dk, keep, p.drop_scale);
          else
            bwd_ds<NC / 2, NC / 2, NC, DROP>(sv, dp, dsc, p.scale, dk, keep, p.drop_scale);
        }
        if (t == 0 && qd == 0) BWD_TRACE(9, it);
#pragma unroll
        for (int c = NC / 16; c < NC / 8; ++c)
          st_shared_v4(row + (((c0 + c) ^ (t & 7)) << 4), dk[4 * c], dk[4 * c + 1], dk[4 * c + 2], dk[4 * c + 3]);
        if (t == 0 && qd == 0) BWD_TRACE(10, it);
        tmem_st_n<NC / 2>(tdP + lane_off + qd * NC, dk);
      }
      if (t == 0 && qd == 0) BWD_TRACE(12, it);
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(ds_full);
      if (t == 0 && qd == 0) BWD_TRACE(4, it);
    }
    // dK / dV epilogue after the one-shot mma_done commit.  The tile is staged in
    // the (now idle) Q / dO ring as [128 rows][dK 64 | dV 64] fp32 with 16-byte
    // chunks XOR-swizzled by row, then each warp stores whole 256-byte row
    // segments: full-line writes whether the destination is local HBM or the
    // owner's receive slot across NVLink (fused reduce-scatter).
    constexpr int EC = 128 / ATB_EW;  // accumulator columns per thread
    const bool is_v = qd * EC >= 64;
    const int col0 = (qd * EC) % 64;
    const uint32_t stage = smem_u32(sQst);
    static_assert(ATB_QSTAGES * ATB_QSTAGE_BYTES >= 128 * 512, "dK|dV staging");
    if (n_iter > 0) {
      mbar_wait(mma_done, 0);
      tc_fence_after();
      uint32_t v[32];
#pragma unroll
      for (int c = 0; c < EC / 32; ++c) {
        tmem_ld32((is_v ? tdV : tdK) + lane_off + col0 + c * 32, v);
        if (g_numerics_check) {  // NaN / Inf in dK / dV (tensor.py:79-95)
          bool bad = false;
#pragma unroll
          for (int i = 0; i < 32; ++i) bad |= nonfinite(__uint_as_float(v[i]));
          report_nonfinite(bad);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int chunk = (is_v ? 16 : 0) + (col0 + c * 32) / 4 + i;
          st_shared_v4(stage + t * 512 + ((chunk ^ (t & 7)) << 4), v[4 * i], v[4 * i + 1], v[4 * i + 2],
                       v[4 * i + 3]);
        }
      }
    }
    named_bar_sync(2, 128 * ATB_EW);
    {
      float* seg = p.seg_tab[0] ? p.seg_tab[g] : p.dkv + g * p.seg_stride;
      const int ew_warp = warp - 4;  // 0 .. 4*ATB_EW-1
      const long col = (lane < 16 ? 0 : p.dv_off) + h * ATT_D + (lane & 15) * 4;
      for (int r = ew_warp; r < kv_valid; r += 4 * ATB_EW) {
        float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
        if (n_iter > 0) val = ld_shared_f4(stage + r * 512 + ((lane ^ (r & 7)) << 4));
        *reinterpret_cast<float4*>(seg + ((long)b * p.seg_len + kv_row0 + r) * p.ld_dkv + col) = val;
      }
    }
  } else {
    reg_dealloc<ATB_REG_DRAIN>();
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
      {
        int src, q0;
        locate(it, src, q0);
        long long* fx = p.src[src].dq_fixed;
        if (fx != nullptr) {
          // Deterministic mode: this key tile's dQ contribution as int64 fixed point
          // (scale 2^32), added with integer bulk reductions -- associative, so the
          // sum over key tiles is bitwise identical whatever order the CTAs finish in.
          // Thread r owns row r of the staging buffer (128 rows x 32 int64 per half).
          const bool row_ok = q0 + r < p.src[src].m_src;
          long long* grow = fx + ((long)b * p.src[src].m_src + q0 + r) * ((long)p.H * ATT_D) + h * ATT_D;
          const uint32_t srow = smem_u32(sStage + r * 256);
#pragma unroll 1
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t v[32];
            tmem_ld32(tdQ + lane_off + hh * 32, v);
            if (hh == 1) {
              tc_fence_before();
              mbar_arrive(dq_empty);
            }
            bulk_wait_read0();  // this thread's previous reduce has read its staging row
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
      if (issuer) bulk_wait_read0();  // previous reduce has finished reading the staging tile
      named_bar_sync(1, 128);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {  // 32 columns at a time keeps the drain at 56 registers
        uint32_t v[32];
        tmem_ld32(tdQ + lane_off + hh * 32, v);
        if (g_numerics_check) {  // NaN / Inf in this key tile's dQ contribution
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
      mbar_arrive(dq_empty);
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
#ifndef LSS_BWD_NODQ
      if (issuer) {
#else
      if (issuer && it < 0) {
#endif
        int src, q0;
        locate(it, src, q0);
        tma_reduce_add_3d(&maps.dq[src], sStage, h * ATT_D, q0, b);
        tma_reduce_add_3d(&maps.dq[src], sStage + ATB_STG_BYTES / 2, h * ATT_D + 32, q0, b);
        bulk_commit();
      }
    }
    bulk_wait0();  // the issuer's tensor reduces / every thread's fixed-point row reduces
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

}  // namespace lss
