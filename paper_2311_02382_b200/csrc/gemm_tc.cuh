// tcgen05/TMEM/TMA GEMM for the LSS projections (sm_100a).
//
//   C[M, N] = alpha * (A[M, K] . B[N, K]^T) (+ bias[N]) (+ residual[M, N])
//
// A and B are bf16 and may each be K-major (row-major with K contiguous) or
// MN-major (row-major with M resp. N contiguous), which covers every product
// the attention half of model.layer_fwd / layer_bwd needs without transposing
// activations:
//   fwd  [Q|K|V] = xh . [Wq|Wk|Wv]          (A K-major, B = W^T cached K-major)
//        y       = x + ctx . Wo + bo         (residual epilogue)
//   bwd  dctx    = dy . Wo^T                 (B = Wo as stored, K-major)
//        dW      = xh^T . dy                 (A M-major, B N-major; fp32 out, alpha = 1/(D*N))
// (reference: nnops.linear_fwd/linear_bwd, nnops.py:180-193; model.linear3, model.py:237-245)
//
// Persistent warp-specialised kernel: warp 0 = TMA producer, warp 1 = MMA
// issuer (one thread), warp 2 = TMEM allocator, warps 4..7 = epilogue
// (TMEM -> registers -> global).  Tile 128 x 256 x 64, 4-stage smem ring,
// double-buffered TMEM accumulator (2 x 256 columns) so the epilogue of tile i
// overlaps the mainloop of tile i+1.
#pragma once
#include "common.cuh"

namespace lss {

struct GemmEpilogue {
  void* out[3];          // up to three column segments (e.g. Q / K|V destinations)
  long ldo[3];           // leading dimension (elements) of each segment
  int seg_width;         // columns per segment (multiple of 32); segment s covers [s*w, (s+1)*w)
  int out_bf16;          // 1: bf16 output, 0: fp32 output
  float alpha;
  const float* bias;     // [N] or null
  const float* residual; // [M, ld_res] fp32 or null
  long ld_res;
  // activation (applied after alpha / bias / residual), nnops.gelu_fwd / gelu_bwd
  // (nnops.py:235-245): 1 = tanh-GeLU, pre-activation also written to pre (same
  // dtype as out, leading dim ld_pre); 2 = multiply by GeLU'(aux[row][col])
  int act;
  void* pre;
  long ld_pre;
  const void* aux;
  long ld_aux;
  int aux_bf16;
};

constexpr float GELU_C = 0.7978845608028654f;  // sqrt(2/pi), nnops._GELU_C
constexpr float GELU_K = 0.044715f;
template <bool FAST>
LSS_DEV float lss_tanh(float x) {
  if (FAST) {
    float r;
    asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
  }
  return tanhf(x);
}
template <bool FAST>
LSS_DEV float gelu_f(float x) {
  return 0.5f * x * (1.f + lss_tanh<FAST>(GELU_C * (x + GELU_K * x * x * x)));
}
template <bool FAST>
LSS_DEV float gelu_grad(float x) {
  const float t = lss_tanh<FAST>(GELU_C * (x + GELU_K * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * GELU_C * (1.f + 3.f * GELU_K * x * x);
}

#ifndef LSS_GEMM_2CTA
#define LSS_GEMM_2CTA 1  // CTA-pair (cta_group::2) kernel for M >= 512
#endif
#ifndef LSS_GEMM_EPI_WG
#define LSS_GEMM_EPI_WG 2  // epilogue warpgroups (each takes 256 / WG accumulator columns of every tile)
#endif
constexpr int GEMM_BM = 128;
constexpr int GEMM_BN = 256;
constexpr int GEMM_BK = 64;
constexpr int GEMM_STAGES = LSS_GEMM_EPI_WG > 2 ? 3 : 4;
constexpr int GEMM_A_BYTES = GEMM_BM * GEMM_BK * 2;  // 16 KB
constexpr int GEMM_B_BYTES = GEMM_BN * GEMM_BK * 2;  // 32 KB
constexpr int GEMM_STAGE_BYTES = GEMM_A_BYTES + GEMM_B_BYTES;
constexpr int GEMM_EPI_WG = LSS_GEMM_EPI_WG;
constexpr int GEMM_EPI_BYTES = GEMM_EPI_WG * 4 * 32 * 32 * 4;  // per epilogue warp: a 32 x 32 fp32 staging tile
constexpr int GEMM_SMEM_BYTES = GEMM_STAGES * GEMM_STAGE_BYTES + GEMM_EPI_BYTES + 1024 /*align*/ + 256 /*bars*/;

// Epilogue store of a warp's 32 rows x 32 columns through shared memory: every lane
// holds one row (32 fp32 values); the tile is staged with 16-byte chunks XOR-swizzled
// by row, then written back with the lanes spread across columns, so each store
// instruction covers whole 64-byte (bf16) / 128-byte (fp32) row segments instead of
// 32 half-filled sectors.  row_base: first row of the warp's 32; rows >= M skipped.
template <bool BF16>
LSS_DEV void epi_store_rows(uint32_t stage, const float (&v)[32], void* out, long ld, long col, int row_base,
                            int M, uint32_t lane, const float* res = nullptr, long ld_res = 0) {
  constexpr int CH = BF16 ? 4 : 8;  // 16-byte chunks per row
  constexpr int RPI = 32 / CH;      // rows per store instruction
  float4 rv[32 / RPI];              // residual row segments, loaded ahead of the staging round trip
  if (!BF16 && res) {
#pragma unroll
    for (int i = 0; i < 32 / RPI; ++i) {
      const int r = i * RPI + (int)lane / CH, q = (int)lane % CH;
      rv[i] = row_base + r < M ? *reinterpret_cast<const float4*>(res + (long)(row_base + r) * ld_res + col + q * 4)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (BF16) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      st_shared_v4(stage + lane * 64 + ((q ^ (lane & 3)) << 4), pack_bf16(v[8 * q], v[8 * q + 1]),
                   pack_bf16(v[8 * q + 2], v[8 * q + 3]), pack_bf16(v[8 * q + 4], v[8 * q + 5]),
                   pack_bf16(v[8 * q + 6], v[8 * q + 7]));
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      st_shared_v4(stage + lane * 128 + ((q ^ (lane & 7)) << 4), __float_as_uint(v[4 * q]),
                   __float_as_uint(v[4 * q + 1]), __float_as_uint(v[4 * q + 2]), __float_as_uint(v[4 * q + 3]));
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 32 / RPI; ++i) {
    const int r = i * RPI + (int)lane / CH, q = (int)lane % CH;
    float4 val = ld_shared_f4(stage + r * (CH * 16) + ((q ^ (r & (CH - 1))) << 4));
    if (row_base + r < M) {
      if (!BF16 && res) {  // residual added here: whole 128-byte row segments per load
        val.x += rv[i].x;
        val.y += rv[i].y;
        val.z += rv[i].z;
        val.w += rv[i].w;
      }
      char* dst = reinterpret_cast<char*>(out) + ((long)(row_base + r) * ld + col) * (BF16 ? 2 : 4) + q * 16;
      *reinterpret_cast<float4*>(dst) = val;
    }
  }
  __syncwarp();  // the staging tile is reused by the next chunk
}
// Epilogue of one 128 x 256 accumulator tile held in this CTA's TMEM columns
// [acc, acc + 256): warp `quad` of the epilogue warpgroup owns rows quad*32.. (TMEM
// lanes), 32 columns at a time: alpha, bias, residual, activation, store.
LSS_DEV void gemm_epilogue_tile(uint32_t acc, int m0, int n0, int M, int N, const GemmEpilogue& ep, int quad,
                                uint32_t lane, uint32_t epi, bool check, int c_begin = 0, int c_end = GEMM_BN) {
  const int row_in_tile = quad * 32 + (int)lane;
  const int row = m0 + row_in_tile;
  const bool row_ok = row < M;
#pragma unroll 1
  for (int c = c_begin; c < c_end; c += 32) {
    uint32_t r[32];
    tmem_ld32(acc + ((uint32_t)(quad * 32) << 16) + c, r);
    const int n = n0 + c;
    if (n >= N) continue;  // warp-uniform
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * ep.alpha;
    if (!row_ok) {  // rows past M: staged but never stored (no operand loads)
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    } else {
    if (ep.bias) {  // the same 32 values in every lane: 8 broadcast float4 loads
      const float4* bp = reinterpret_cast<const float4*>(ep.bias + n);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 t = __ldg(bp + i);
        v[4 * i] += t.x;
        v[4 * i + 1] += t.y;
        v[4 * i + 2] += t.z;
        v[4 * i + 3] += t.w;
      }
    }
    if (ep.residual && (ep.act != 0 || ep.out_bf16)) {  // else added in the coalesced store phase
      const float4* rp = reinterpret_cast<const float4*>(ep.residual + (long)row * ep.ld_res + n);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 t = rp[i];
        v[4 * i] += t.x;
        v[4 * i + 1] += t.y;
        v[4 * i + 2] += t.z;
        v[4 * i + 3] += t.w;
      }
    }
    if (ep.act == 1) {  // tanh-GeLU; the pre-activation is kept for the backward
      if (ep.pre) {
        if (ep.out_bf16) {
          uint4* pp = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(ep.pre) + (long)row * ep.ld_pre + n);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            pp[i] = make_uint4(pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                               pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
        } else {
          float4* pp = reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.pre) + (long)row * ep.ld_pre + n);
#pragma unroll
          for (int i = 0; i < 8; ++i) pp[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = gelu_f<true>(v[i]);
    } else if (ep.act == 2) {  // chain rule through GeLU at the stored pre-activation
      if (ep.aux_bf16) {
        const uint4* ap = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(ep.aux) +
                                                         (long)row * ep.ld_aux + n);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 t = ap[i];
          const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            v[8 * i + 2 * j] *= gelu_grad<true>(__uint_as_float(w[j] << 16));
            v[8 * i + 2 * j + 1] *= gelu_grad<true>(__uint_as_float(w[j] & 0xFFFF0000u));
          }
        }
      } else {
        const float4* ap = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(ep.aux) +
                                                           (long)row * ep.ld_aux + n);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 t = ap[i];
          v[4 * i] *= gelu_grad<true>(t.x);
          v[4 * i + 1] *= gelu_grad<true>(t.y);
          v[4 * i + 2] *= gelu_grad<true>(t.z);
          v[4 * i + 3] *= gelu_grad<true>(t.w);
        }
      }
    }
    }  // row_ok
    if (check) {
      bool bad = false;
#pragma unroll
      for (int i = 0; i < 32; ++i) bad |= nonfinite(v[i]);
      report_nonfinite(bad);
    }
    const int seg = n / ep.seg_width;
    const long col = n - (long)seg * ep.seg_width;
    if (ep.out_bf16)
      epi_store_rows<true>(epi, v, ep.out[seg], ep.ldo[seg], col, m0 + quad * 32, M, lane);
    else
      epi_store_rows<false>(epi, v, ep.out[seg], ep.ldo[seg], col, m0 + quad * 32, M, lane,
                            ep.act == 0 && ep.residual ? ep.residual + (n - col) : nullptr, ep.ld_res);
  }
}

constexpr int GEMM_THREADS = 128 * (1 + GEMM_EPI_WG);  // control warpgroup + epilogue warpgroups

template <int A_MN, int B_MN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
                        GemmEpilogue ep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + GEMM_STAGES * GEMM_STAGE_BYTES);
  uint64_t* empty_bar = full_bar + GEMM_STAGES;
  uint64_t* tfull_bar = empty_bar + GEMM_STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int m_tiles = (M + GEMM_BM - 1) / GEMM_BM;
  const int n_tiles = (N + GEMM_BN - 1) / GEMM_BN;
  const int num_tiles = m_tiles * n_tiles;
  const int num_kb = (K + GEMM_BK - 1) / GEMM_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < GEMM_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 128 * GEMM_EPI_WG);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    {
      // ---------------- TMA producer (warp-uniform loop, elected lane issues)
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile / n_tiles) * GEMM_BM;
        const int n0 = (tile % n_tiles) * GEMM_BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (elect_one()) {
            uint8_t* sa = smem + stage * GEMM_STAGE_BYTES;
            uint8_t* sb = sa + GEMM_A_BYTES;
            mbar_arrive_expect_tx(&full_bar[stage], GEMM_STAGE_BYTES);
            const int k0 = kb * GEMM_BK;
            if (A_MN) {
              tma_load_2d(&tmA, &full_bar[stage], sa, m0, k0);
              tma_load_2d(&tmA, &full_bar[stage], sa + 8192, m0 + 64, k0);
            } else {
              tma_load_2d(&tmA, &full_bar[stage], sa, k0, m0);
            }
            if (B_MN) {
#pragma unroll
              for (int i = 0; i < 4; ++i) tma_load_2d(&tmB, &full_bar[stage], sb + i * 8192, n0 + 64 * i, k0);
            } else {
              tma_load_2d(&tmB, &full_bar[stage], sb, k0, n0);
            }
          }
          __syncwarp();
          if (++stage == GEMM_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    {
      // ---------------- MMA issuer (warp-uniform loop, elected lane issues)
      constexpr uint32_t idesc = idesc_bf16_f32(GEMM_BM, GEMM_BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
        const int buf = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty_bar[buf], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * GEMM_BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * GEMM_STAGE_BYTES);
          const uint32_t sb = sa + GEMM_A_BYTES;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k) {
              const uint64_t ad = A_MN ? smem_desc_sw128(sa + k * 2048, 8192, 1024)
                                       : smem_desc_sw128(sa + k * 32, 16, 1024);
              const uint64_t bd = B_MN ? smem_desc_sw128(sb + k * 2048, 8192, 1024)
                                       : smem_desc_sw128(sb + k * 32, 16, 1024);
              mma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
            }
            mma_commit(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == GEMM_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) mma_commit(&tfull_bar[buf]);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: thread <-> accumulator row
    // epilogue warpgroup eg takes accumulator columns [eg, eg+1) * 256 / GEMM_EPI_WG of every
    // tile (the epilogue, not the mainloop, bounded the K=E projections with one warpgroup)
    const int quad = warp % 4, eg = (warp - 4) / 4;
    const int c_begin = eg * (GEMM_BN / GEMM_EPI_WG), c_end = c_begin + GEMM_BN / GEMM_EPI_WG;
    const bool check = g_numerics_check != 0;  // NaN / Inf report (tensor.py:79-95), off by default
    const uint32_t epi = smem_u32(smem + GEMM_STAGES * GEMM_STAGE_BYTES + 256) + (warp - 4) * (32 * 32 * 4);
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int buf = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int m0 = (tile / n_tiles) * GEMM_BM;
      const int n0 = (tile % n_tiles) * GEMM_BN;
      mbar_wait(&tfull_bar[buf], acc_phase);
      tc_fence_after();
      gemm_epilogue_tile(tmem_base + buf * GEMM_BN, m0, n0, M, N, ep, quad, lane, epi, check, c_begin, c_end);
      tc_fence_before();
      mbar_arrive(&tempty_bar[buf]);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}


// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs on one TPC computes a
// 256 x 256 tile; each CTA loads its own 128 rows of A and 128 of the 256 rows of
// B, the leader issues M=256 MMAs that read both CTAs' shared memory, and each
// CTA's TMEM receives its own 128 rows of the accumulator.  Per SM that is 32 KB
// of operands per 64-deep K step instead of 48 KB (the 1-CTA kernel's TMA ingest
// did not keep the tensor pipe busy: 55% under ncu), and 6 pipeline stages fit.
//   full_bar (leader): both CTAs' TMA bytes (the peer's loads signal the leader)
//   empty_bar (each) : the leader's MMA commit, multicast to both CTAs
//   tfull_bar (each) : the leader's accumulator commit, multicast
//   tempty_bar (leader): both CTAs' epilogue warps (256 arrivals, remote for the peer)
constexpr int GEMM2_STAGES = LSS_GEMM_EPI_WG > 2 ? 4 : 6;
constexpr int GEMM2_STAGE_BYTES = GEMM_A_BYTES + GEMM_B_BYTES / 2;  // 32 KB per CTA
constexpr int GEMM2_SMEM_BYTES = GEMM2_STAGES * GEMM2_STAGE_BYTES + GEMM_EPI_BYTES + 1024 + 256;

LSS_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
LSS_DEV uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
LSS_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-SM TMA load: the data lands in this CTA's shared memory, the completion is
// signalled on the mbarrier at shared::cluster address bar_cl (the leader's)
LSS_DEV void tma_load_2d_2sm(const CUtensorMap* m, uint32_t bar_cl, void* smem, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cl), "r"(c0), "r"(c1)
      : "memory");
}
LSS_DEV void mma_bf16_ss_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
LSS_DEV void mma_commit_2sm(uint64_t* bar) {  // arrive on the same barrier in both CTAs of the pair
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <int A_MN, int B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                         int N, int K, GemmEpilogue ep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + GEMM2_STAGES * GEMM2_STAGE_BYTES);
  uint64_t* empty_bar = full_bar + GEMM2_STAGES;
  uint64_t* tfull_bar = empty_bar + GEMM2_STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int m_pairs = (M + 2 * GEMM_BM - 1) / (2 * GEMM_BM);
  const int n_tiles = (N + GEMM_BN - 1) / GEMM_BN;
  const int num_tiles = m_pairs * n_tiles;
  const int num_kb = (K + GEMM_BK - 1) / GEMM_BK;
  const int cluster = (int)blockIdx.x / 2, n_clusters = (int)gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < GEMM2_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 2 * 128 * GEMM_EPI_WG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs: own A rows, own half of B)
    const uint32_t full_leader = mapa_shared(smem_u32(full_bar), 0);
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = cluster; tile < num_tiles; tile += n_clusters) {
      const int m0 = (tile / n_tiles) * (2 * GEMM_BM) + (int)rank * GEMM_BM;
      const int n0 = (tile % n_tiles) * GEMM_BN + (int)rank * (GEMM_BN / 2);
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (elect_one()) {
          uint8_t* sa = smem + stage * GEMM2_STAGE_BYTES;
          uint8_t* sb = sa + GEMM_A_BYTES;
          const uint32_t fb = full_leader + stage * 8;
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * GEMM2_STAGE_BYTES);
          const int k0 = kb * GEMM_BK;
          if (A_MN) {
            tma_load_2d_2sm(&tmA, fb, sa, m0, k0);
            tma_load_2d_2sm(&tmA, fb, sa + 8192, m0 + 64, k0);
          } else {
            tma_load_2d_2sm(&tmA, fb, sa, k0, m0);
          }
          if (B_MN) {
            tma_load_2d_2sm(&tmB, fb, sb, n0, k0);
            tma_load_2d_2sm(&tmB, fb, sb + 8192, n0 + 64, k0);
          } else {
            tma_load_2d_2sm(&tmB, fb, sb, k0, n0);
          }
        }
        __syncwarp();
        if (++stage == GEMM2_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer (leader CTA only; M = 256 over the pair)
    constexpr uint32_t idesc = idesc_bf16_f32(2 * GEMM_BM, GEMM_BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int tile = cluster; tile < num_tiles; tile += n_clusters, ++local) {
      const int buf = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tempty_bar[buf], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + buf * GEMM_BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * GEMM2_STAGE_BYTES);
        const uint32_t sb = sa + GEMM_A_BYTES;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t ad = A_MN ? smem_desc_sw128(sa + k * 2048, 8192, 1024)
                                     : smem_desc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc_sw128(sb + k * 2048, 8192, 1024)
                                     : smem_desc_sw128(sb + k * 32, 16, 1024);
            mma_bf16_ss_2sm(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          mma_commit_2sm(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == GEMM2_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) mma_commit_2sm(&tfull_bar[buf]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs: own 128 rows of the 256 x 256 tile)
    const int quad = warp % 4, eg = (warp - 4) / 4;
    const int c_begin = eg * (GEMM_BN / GEMM_EPI_WG), c_end = c_begin + GEMM_BN / GEMM_EPI_WG;
    const bool check = g_numerics_check != 0;
    const uint32_t epi = smem_u32(smem + GEMM2_STAGES * GEMM2_STAGE_BYTES + 256) + (warp - 4) * (32 * 32 * 4);
    const uint32_t tempty_leader = mapa_shared(smem_u32(tempty_bar), 0);
    int local = 0;
    for (int tile = cluster; tile < num_tiles; tile += n_clusters, ++local) {
      const int buf = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int m0 = (tile / n_tiles) * (2 * GEMM_BM) + (int)rank * GEMM_BM;
      const int n0 = (tile % n_tiles) * GEMM_BN;
      mbar_wait(&tfull_bar[buf], acc_phase);
      tc_fence_after();
      gemm_epilogue_tile(tmem_base + buf * GEMM_BN, m0, n0, M, N, ep, quad, lane, epi, check, c_begin, c_end);
      tc_fence_before();
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_leader + buf * 8)
                   : "memory");
    }
  }

  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while its partner may still signal it
  tc_fence_after();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

}  // namespace lss
