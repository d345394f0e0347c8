// HBM-bound kernels around the attention core: LayerNorm fwd/bwd (nnops.py:199-227),
// weight staging, casts fused with bias-gradient column sums, the attention
// backward's per-row delta = rowsum(dO * O), and rank-local helpers.
#pragma once
#include "common.cuh"

namespace lss {

template <typename T>
LSS_DEV void store4(T* dst, float a, float b, float c, float d);
template <>
LSS_DEV void store4<float>(float* dst, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(dst) = make_float4(a, b, c, d);
}
template <>
LSS_DEV void store4<__nv_bfloat16>(__nv_bfloat16* dst, float a, float b, float c, float d) {
  uint2 v;
  v.x = pack_bf16(a, b);
  v.y = pack_bf16(c, d);
  *reinterpret_cast<uint2*>(dst) = v;
}

LSS_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum for blockDim.x <= 1024; `red` has >= 32 floats
LSS_DEV float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) / 32;
  float t = (l < nw) ? red[l] : 0.f;
  return warp_sum(t);
}

// two block-wide sums with one pair of barriers
LSS_DEV float2 block_sum2(float a, float b, float2* red) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = make_float2(a, b);
  __syncthreads();
  const int nw = (blockDim.x + 31) / 32;
  const float2 t = (l < nw) ? red[l] : make_float2(0.f, 0.f);
  return make_float2(warp_sum(t.x), warp_sum(t.y));
}

// One block per row; each thread owns 4 consecutive features (E % 4 == 0, E <= 4*blockDim).
template <typename TOut>
__global__ void layernorm_fwd_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                                     const float* __restrict__ bias, TOut* __restrict__ y,
                                     float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                     int E, float eps) {
  __shared__ float red[32];
  const long row = blockIdx.x;
  const int c = threadIdx.x * 4;
  const bool ok = c < E;
  float4 v = ok ? *reinterpret_cast<const float4*>(x + row * E + c) : make_float4(0.f, 0.f, 0.f, 0.f);
  const float mu = block_sum(v.x + v.y + v.z + v.w, red) / E;
  const float a = v.x - mu, b_ = v.y - mu, cc = v.z - mu, d = v.w - mu;
  const float var = block_sum(ok ? a * a + b_ * b_ + cc * cc + d * d : 0.f, red) / E;
  const float rs = rsqrtf(var + eps);
  if (ok) {
    const float4 g = *reinterpret_cast<const float4*>(gain + c);
    const float4 bb = *reinterpret_cast<const float4*>(bias + c);
    store4<TOut>(y + row * E + c, a * rs * g.x + bb.x, b_ * rs * g.y + bb.y, cc * rs * g.z + bb.z,
                 d * rs * g.w + bb.w);
  }
  if (threadIdx.x == 0) {
    mean_out[row] = mu;
    rstd_out[row] = rs;
  }
}

// Warp per row for E a multiple of 128 (E <= 2048): every lane holds E/128 float4
// of its row in registers, both reductions are warp shuffles (no block barriers), and a
// 256-thread block keeps 8 rows in flight -- the one-block-per-row kernel above left
// its SMs waiting on two __syncthreads round trips per 4 KB row.
template <typename TOut, int NV>
__global__ void __launch_bounds__(256) layernorm_fwd_warp_kernel(const float* __restrict__ x,
                                                               const float* __restrict__ gain,
                                                               const float* __restrict__ bias, TOut* __restrict__ y,
                                                               float* __restrict__ mean_out,
                                                               float* __restrict__ rstd_out, long rows, float eps) {
  constexpr int E = NV * 128;
  const long row = (long)blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  float4 v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = *reinterpret_cast<const float4*>(x + row * E + k * 128 + lane * 4);
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) sum += (v[k].x + v[k].y) + (v[k].z + v[k].w);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mu = sum / E;
  float sq = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    v[k].x -= mu; v[k].y -= mu; v[k].z -= mu; v[k].w -= mu;
    sq += (v[k].x * v[k].x + v[k].y * v[k].y) + (v[k].z * v[k].z + v[k].w * v[k].w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  const float rs = rsqrtf(sq / E + eps);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int c = k * 128 + lane * 4;
    const float4 g = __ldg(reinterpret_cast<const float4*>(gain + c));
    const float4 bb = __ldg(reinterpret_cast<const float4*>(bias + c));
    store4<TOut>(y + row * E + c, v[k].x * rs * g.x + bb.x, v[k].y * rs * g.y + bb.y, v[k].z * rs * g.z + bb.z,
                 v[k].w * rs * g.w + bb.w);
  }
  if (lane == 0) {
    mean_out[row] = mu;
    rstd_out[row] = rs;
  }
}

// gx = grad_res + rstd*(g - mean(g) - xhat*mean(g*xhat)), g = gxh*gain (nnops.py:211-227).
// Each block handles ROWS rows; column partial sums of gxh*xhat and gxh are
// accumulated in registers and added (scaled by alpha) to g_gain / g_bias once.
constexpr int LN_BWD_ROWS = 16;
__global__ void layernorm_bwd_kernel(const float* __restrict__ gxh, const float* __restrict__ x,
                                     const float* __restrict__ mean, const float* __restrict__ rstd,
                                     const float* __restrict__ gain, const float* __restrict__ grad_res,
                                     float* __restrict__ gx, float* __restrict__ g_gain,
                                     float* __restrict__ g_bias, float alpha, long rows, int E) {
  __shared__ float2 red[32];
  const int c = threadIdx.x * 4;
  const bool ok = c < E;
  float4 gg = make_float4(0.f, 0.f, 0.f, 0.f), gb = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 w = ok ? *reinterpret_cast<const float4*>(gain + c) : make_float4(0.f, 0.f, 0.f, 0.f);
  const long r0 = (long)blockIdx.x * LN_BWD_ROWS;
  // software pipeline: the next row's operands are loaded before this row's reduction
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 gy_n = z4, xv_n = z4;
  float mu_n = 0.f, rs_n = 0.f;
  if (r0 < rows) {
    mu_n = mean[r0];
    rs_n = rstd[r0];
    if (ok) {
      gy_n = *reinterpret_cast<const float4*>(gxh + r0 * E + c);
      xv_n = *reinterpret_cast<const float4*>(x + r0 * E + c);
    }
  }
  for (int i = 0; i < LN_BWD_ROWS; ++i) {
    const long row = r0 + i;
    if (row >= rows) break;
    const float mu = mu_n, rs = rs_n;
    const float4 gy = gy_n, xv = xv_n;
    if (i + 1 < LN_BWD_ROWS && row + 1 < rows) {
      mu_n = mean[row + 1];
      rs_n = rstd[row + 1];
      if (ok) {
        gy_n = *reinterpret_cast<const float4*>(gxh + (row + 1) * E + c);
        xv_n = *reinterpret_cast<const float4*>(x + (row + 1) * E + c);
      }
    }
    const float xh0 = (xv.x - mu) * rs, xh1 = (xv.y - mu) * rs, xh2 = (xv.z - mu) * rs,
                xh3 = (xv.w - mu) * rs;
    gg.x += gy.x * xh0; gg.y += gy.y * xh1; gg.z += gy.z * xh2; gg.w += gy.w * xh3;
    gb.x += gy.x; gb.y += gy.y; gb.z += gy.z; gb.w += gy.w;
    const float g0 = gy.x * w.x, g1 = gy.y * w.y, g2 = gy.z * w.z, g3 = gy.w * w.w;
    // the residual load is issued before the reduction's barriers so it overlaps them
    const float4 res = (ok && grad_res) ? *reinterpret_cast<const float4*>(grad_res + row * E + c)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
    const float2 sums = block_sum2(ok ? g0 + g1 + g2 + g3 : 0.f,
                                   ok ? g0 * xh0 + g1 * xh1 + g2 * xh2 + g3 * xh3 : 0.f, red);
    const float mg = sums.x / E, mgx = sums.y / E;
    if (ok) {
      *reinterpret_cast<float4*>(gx + row * E + c) =
          make_float4(res.x + rs * (g0 - mg - xh0 * mgx), res.y + rs * (g1 - mg - xh1 * mgx),
                      res.z + rs * (g2 - mg - xh2 * mgx), res.w + rs * (g3 - mg - xh3 * mgx));
    }
  }
  if (ok && g_gain) {  // null in the deterministic mode: ln_colsum_det_kernel sums instead
    atomicAdd(g_gain + c + 0, alpha * gg.x); atomicAdd(g_gain + c + 1, alpha * gg.y);
    atomicAdd(g_gain + c + 2, alpha * gg.z); atomicAdd(g_gain + c + 3, alpha * gg.w);
    atomicAdd(g_bias + c + 0, alpha * gb.x); atomicAdd(g_bias + c + 1, alpha * gb.y);
    atomicAdd(g_bias + c + 2, alpha * gb.z); atomicAdd(g_bias + c + 3, alpha * gb.w);
  }
}

// Concatenate up to 3 fp32 column blocks of `rows` rows into one row-major
// destination (bf16 or fp32), and add alpha * column sums into colsum (optional).
// Used for: grad_y -> bf16 (+ d bias_out), [dQ | dK dV] -> bf16 dQKV (+ d b_qkv).
struct CatSrc {
  const float* ptr[3];
  long ld[3];
  int cols[3];
  int n;
  // optional per source: the value is the ascending sum of the slots set in mask
  // (slot k at ptr + k * slot_stride) -- the fused reduce-scatter's owner sum folded
  // into the cast that feeds the projection backward (no dK|dV round trip)
  int nslot[3];
  uint32_t mask[3];
  long slot_stride[3];
};
constexpr int CAT_ROWS = 32;
template <typename TOut>
__global__ void cat_cast_colsum_kernel(CatSrc src, TOut* __restrict__ dst, long ld_dst,
                                       float* __restrict__ colsum, float alpha, long rows) {
  // grid.x over 4-column groups (blockDim.x threads each), grid.y over row blocks
  const int col4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  int s = 0, base = 0;
  while (s < src.n && col4 >= base + src.cols[s]) base += src.cols[s++];
  if (s >= src.n) return;
  const int lc = col4 - base;
  const float* sp = src.ptr[s];
  const long ld = src.ld[s];
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const long r0 = (long)blockIdx.y * CAT_ROWS;
  const bool full = r0 + CAT_ROWS <= rows && src.nslot[s] <= 1;
  if (full) {  // common case: all row loads in flight together
    float4 vv[CAT_ROWS];
#pragma unroll
    for (int i = 0; i < CAT_ROWS; ++i) vv[i] = *reinterpret_cast<const float4*>(sp + (r0 + i) * ld + lc);
#pragma unroll
    for (int i = 0; i < CAT_ROWS; ++i) {
      const float4 v = vv[i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      if (dst) store4<TOut>(dst + (r0 + i) * ld_dst + col4, v.x, v.y, v.z, v.w);
    }
  }
  for (int i = 0; i < (full ? 0 : CAT_ROWS); ++i) {
    const long r = r0 + i;
    if (r >= rows) break;
    float4 v;
    if (src.nslot[s] <= 1) {
      v = *reinterpret_cast<const float4*>(sp + r * ld + lc);
    } else {
      v = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int k = 0; k < src.nslot[s]; ++k) {
        if (!((src.mask[s] >> k) & 1u)) continue;
        const float4 u = *reinterpret_cast<const float4*>(sp + k * src.slot_stride[s] + r * ld + lc);
        v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
      }
    }
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    if (dst) store4<TOut>(dst + r * ld_dst + col4, v.x, v.y, v.z, v.w);
  }
  if (colsum) {
    atomicAdd(colsum + col4 + 0, alpha * acc.x);
    atomicAdd(colsum + col4 + 1, alpha * acc.y);
    atomicAdd(colsum + col4 + 2, alpha * acc.z);
    atomicAdd(colsum + col4 + 3, alpha * acc.w);
  }
}

// Warp-per-row LayerNorm backward for E a multiple of 128 (E <= 1024): each warp runs
// LNW_RPW rows with warp-shuffle reductions and keeps its affine-gradient column
// partials in registers (2 x E/32 per lane); the block's 8 warps combine them in
// shared memory and issue one atomic per column per block (g_gain null: the
// deterministic mode's separate column-sum kernel, as above).
constexpr int LNW_RPW = 8;  // rows per warp -> 64 rows per 256-thread block
template <int NV>
__global__ void __launch_bounds__(256) layernorm_bwd_warp_kernel(
    const float* __restrict__ gxh, const float* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ gain, const float* __restrict__ grad_res,
    float* __restrict__ gx, float* __restrict__ g_gain, float* __restrict__ g_bias, float alpha, long rows) {
  constexpr int E = NV * 128;
  extern __shared__ float colred[];  // [8 warps][E] (gain partials, then bias partials)
  const int wi = threadIdx.x / 32, lane = threadIdx.x % 32;
  float4 w[NV], gg[NV], gb[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    w[k] = __ldg(reinterpret_cast<const float4*>(gain + k * 128 + lane * 4));
    gg[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    gb[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const long rbase = (long)blockIdx.x * (8 * LNW_RPW) + wi;
#pragma unroll 1
  for (int i = 0; i < LNW_RPW; ++i) {
    const long row = rbase + 8L * i;
    if (row >= rows) break;
    const float mu = mean[row], rs = rstd[row];
    float4 gy[NV], xh[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      gy[k] = *reinterpret_cast<const float4*>(gxh + row * E + k * 128 + lane * 4);
      xh[k] = *reinterpret_cast<const float4*>(x + row * E + k * 128 + lane * 4);
    }
    float sg = 0.f, sgx = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      xh[k] = make_float4((xh[k].x - mu) * rs, (xh[k].y - mu) * rs, (xh[k].z - mu) * rs, (xh[k].w - mu) * rs);
      gg[k].x += gy[k].x * xh[k].x; gg[k].y += gy[k].y * xh[k].y; gg[k].z += gy[k].z * xh[k].z; gg[k].w += gy[k].w * xh[k].w;
      gb[k].x += gy[k].x; gb[k].y += gy[k].y; gb[k].z += gy[k].z; gb[k].w += gy[k].w;
      gy[k] = make_float4(gy[k].x * w[k].x, gy[k].y * w[k].y, gy[k].z * w[k].z, gy[k].w * w[k].w);  // g
      sg += (gy[k].x + gy[k].y) + (gy[k].z + gy[k].w);
      sgx += (gy[k].x * xh[k].x + gy[k].y * xh[k].y) + (gy[k].z * xh[k].z + gy[k].w * xh[k].w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sg += __shfl_xor_sync(0xffffffffu, sg, o);
      sgx += __shfl_xor_sync(0xffffffffu, sgx, o);
    }
    const float mg = sg / E, mgx = sgx / E;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int c = k * 128 + lane * 4;
      float4 r = grad_res ? *reinterpret_cast<const float4*>(grad_res + row * E + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      r.x += rs * (gy[k].x - mg - xh[k].x * mgx);
      r.y += rs * (gy[k].y - mg - xh[k].y * mgx);
      r.z += rs * (gy[k].z - mg - xh[k].z * mgx);
      r.w += rs * (gy[k].w - mg - xh[k].w * mgx);
      *reinterpret_cast<float4*>(gx + row * E + c) = r;
    }
  }
  if (!g_gain) return;  // deterministic mode: ln_colsum_det_kernel sums instead (block-uniform)
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
    for (int k = 0; k < NV; ++k)
      *reinterpret_cast<float4*>(colred + wi * E + k * 128 + lane * 4) = pass ? gb[k] : gg[k];
    __syncthreads();
    for (int c = threadIdx.x; c < E; c += 256) {
      float t = 0.f;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) t += colred[ww * E + c];
      atomicAdd((pass ? g_bias : g_gain) + c, alpha * t);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- deterministic column sums
// Bitwise-repeatable replacements for the atomicAdd column sums above, used in the
// deterministic mode (lss_runtime_config flag, the reference's run-to-run bitwise
// reproducibility, collectives.py:5-7): every column has ONE writer; its rows are
// dealt to DET_LANES row lanes x 4 accumulators in a fixed pattern and combined in
// a fixed order, so the result does not depend on scheduling.
constexpr int DET_COLS = 32, DET_LANES = 32;

__device__ __forceinline__ float cat_value(const CatSrc& src, int s, long r, int lc) {
  const float* sp = src.ptr[s];
  if (src.nslot[s] <= 1) return sp[r * src.ld[s] + lc];
  float v = 0.f;  // same ascending slot fold as cat_cast_colsum_kernel
  for (int k = 0; k < src.nslot[s]; ++k)
    if ((src.mask[s] >> k) & 1u) v += sp[k * src.slot_stride[s] + r * src.ld[s] + lc];
  return v;
}

__global__ void __launch_bounds__(DET_COLS * DET_LANES)
    colsum_det_kernel(CatSrc src, float* __restrict__ colsum, float alpha, long rows) {
  __shared__ float part[DET_LANES][DET_COLS + 1];
  const int cl = threadIdx.x % DET_COLS, rl = threadIdx.x / DET_COLS;
  const int col = blockIdx.x * DET_COLS + cl;
  int s = 0, base = 0;
  while (s < src.n && col >= base + src.cols[s]) base += src.cols[s++];
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  if (s < src.n) {
    const int lc = col - base;
    long r = rl;
    for (; r + 3 * DET_LANES < rows; r += 4 * DET_LANES) {
      a0 += cat_value(src, s, r, lc);
      a1 += cat_value(src, s, r + DET_LANES, lc);
      a2 += cat_value(src, s, r + 2 * DET_LANES, lc);
      a3 += cat_value(src, s, r + 3 * DET_LANES, lc);
    }
    for (; r < rows; r += DET_LANES) a0 += cat_value(src, s, r, lc);
  }
  part[rl][cl] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (rl == 0 && s < src.n) {
    float t = 0.f;
    for (int k = 0; k < DET_LANES; ++k) t += part[k][cl];
    colsum[col] += alpha * t;
  }
}

// LayerNorm affine gradients (nnops.py:217-218): g_gain += alpha * sum_r gxh * xhat,
// g_bias += alpha * sum_r gxh, one writer per column (deterministic mode).
__global__ void __launch_bounds__(DET_COLS * DET_LANES)
    ln_colsum_det_kernel(const float* __restrict__ gxh, const float* __restrict__ x,
                         const float* __restrict__ mean, const float* __restrict__ rstd,
                         float* __restrict__ g_gain, float* __restrict__ g_bias, float alpha, long rows, int E) {
  __shared__ float pg[DET_LANES][DET_COLS + 1], pb[DET_LANES][DET_COLS + 1];
  const int cl = threadIdx.x % DET_COLS, rl = threadIdx.x / DET_COLS;
  const int col = blockIdx.x * DET_COLS + cl;
  float g0 = 0.f, g1 = 0.f, b0 = 0.f, b1 = 0.f;
  if (col < E) {
    long r = rl;
    for (; r + DET_LANES < rows; r += 2 * DET_LANES) {
      const float u = gxh[r * E + col], w = gxh[(r + DET_LANES) * E + col];
      g0 += u * ((x[r * E + col] - mean[r]) * rstd[r]);
      g1 += w * ((x[(r + DET_LANES) * E + col] - mean[r + DET_LANES]) * rstd[r + DET_LANES]);
      b0 += u;
      b1 += w;
    }
    for (; r < rows; r += DET_LANES) {
      const float u = gxh[r * E + col];
      g0 += u * ((x[r * E + col] - mean[r]) * rstd[r]);
      b0 += u;
    }
  }
  pg[rl][cl] = g0 + g1;
  pb[rl][cl] = b0 + b1;
  __syncthreads();
  if (rl == 0 && col < E) {
    float tg = 0.f, tb = 0.f;
    for (int k = 0; k < DET_LANES; ++k) {
      tg += pg[k][cl];
      tb += pb[k][cl];
    }
    g_gain[col] += alpha * tg;
    g_bias[col] += alpha * tb;
  }
}

// dQ of the deterministic backward: int64 fixed point (scale 2^32) -> fp32
__global__ void fixed_to_f32_kernel(float* __restrict__ dst, const long long* __restrict__ src, long n,
                                    int accumulate) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const float v = (float)((double)src[i] * 2.3283064365386963e-10);  // 2^-32
    dst[i] = accumulate ? dst[i] + v : v;
  }
}

// Weight staging for the GEMMs (reference weights are [d_in, d_out], y = x W + b):
//   wqkv_t [3E][E] = [Wq | Wk | Wv]^T  (K-major B operand of the forward projection)
//   wqkv   [E][3E] = [Wq | Wk | Wv]    (K-major B operand of the input-gradient GEMM)
//   wo_t   [E][E]  = Wo^T, wo [E][E] = Wo
//   bqkv   [3E]    = [bq | bk | bv]
template <typename TW>
__global__ void weight_stage_kernel(const float* __restrict__ wq, const float* __restrict__ wk,
                                    const float* __restrict__ wv, const float* __restrict__ wo,
                                    const float* __restrict__ bq, const float* __restrict__ bk,
                                    const float* __restrict__ bv, TW* __restrict__ wqkv_t,
                                    TW* __restrict__ wqkv, TW* __restrict__ wo_t, TW* __restrict__ wo_n,
                                    float* __restrict__ bqkv, int E) {
  __shared__ float tile[32][33];
  const int which = blockIdx.z;  // 0..3 = q,k,v,o
  const float* w = which == 0 ? wq : which == 1 ? wk : which == 2 ? wv : wo;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;  // rows (in), cols (out)
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = i0 + r, j = j0 + threadIdx.x;
    float v = 0.f;
    if (i < E && j < E) {
      v = w[(long)i * E + j];
      if (which < 3) wqkv[(long)i * 3 * E + which * E + j] = TW(v);
      else wo_n[(long)i * E + j] = TW(v);
    }
    tile[r][threadIdx.x] = v;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = j0 + r, i = i0 + threadIdx.x;  // transposed: row j (out), col i (in)
    if (i < E && j < E) {
      const float v = tile[threadIdx.x][r];
      if (which < 3) wqkv_t[((long)which * E + j) * E + i] = TW(v);
      else wo_t[(long)j * E + i] = TW(v);
    }
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && which < 3) {
    const float* bsrc = which == 0 ? bq : which == 1 ? bk : bv;
    for (int j = threadIdx.y * blockDim.x + threadIdx.x; j < E; j += blockDim.x * blockDim.y)
      bqkv[which * E + j] = bsrc ? bsrc[j] : 0.f;
  }
}

// delta[b][h][row] = scale * sum_d dO[b,row,h*d+k] * O[b,row,h*d+k], padded rows set to 0.
template <typename T>
__global__ void attn_delta_kernel(const T* __restrict__ dO, const T* __restrict__ O,
                                  float* __restrict__ delta, int B, int m, int m_pad, int H, int d,
                                  float scale) {
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;  // over B*m_pad*H
  const long total = (long)B * m_pad * H;
  if (idx >= total) return;
  const int h = idx % H;
  const long br = idx / H;
  const int row = br % m_pad;
  const int b = br / m_pad;
  float acc = 0.f;
  if (row < m) {
    const T* a = dO + ((long)b * m + row) * (long)H * d + (long)h * d;
    const T* o = O + ((long)b * m + row) * (long)H * d + (long)h * d;
    for (int k = 0; k < d; ++k) acc += float(a[k]) * float(o[k]);
  }
  delta[((long)b * H + h) * m_pad + row] = acc * scale;
}

// bf16, head_dim 64, E % 256 == 0: one warp per row, 16-byte coalesced loads;
// lane l covers columns [8l + 256j, +8) so 8 consecutive lanes form one head.
__global__ void attn_delta_bf16_d64_kernel(const __nv_bfloat16* __restrict__ dO,
                                           const __nv_bfloat16* __restrict__ O, float* __restrict__ delta,
                                           int B, int m, int m_pad, int H, float scale) {
  const long wrow = ((long)blockIdx.x * blockDim.x + threadIdx.x) / 32;  // over B*m_pad
  const int lane = threadIdx.x % 32;
  if (wrow >= (long)B * m_pad) return;
  const int row = wrow % m_pad;
  const int b = wrow / m_pad;
  const int E = H * 64;
  for (int j = 0; j < E / 256; ++j) {
    float acc = 0.f;
    if (row < m) {
      const long off = ((long)b * m + row) * E + j * 256 + lane * 8;
      const uint4 av = *reinterpret_cast<const uint4*>(dO + off);
      const uint4 ov = *reinterpret_cast<const uint4*>(O + off);
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&av);
      const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 x = __bfloat1622float2(a2[i]), y = __bfloat1622float2(o2[i]);
        acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    if ((lane & 7) == 0) delta[((long)b * H + j * 4 + lane / 8) * m_pad + row] = acc * scale;
  }
}

// Merge two partial attentions over disjoint key ranges (log-sum-exp combine):
//   lse = log2(2^la + 2^lb),  O = 2^(la-lse) O_a + 2^(lb-lse) O_b
// One warp per (batch, row); lane l covers 8 columns per 256-column chunk.
// O_a/O_b/O_out are bf16 rows of E = H*64 (batch stride o_bstride elements),
// lse buffers are [B][H][pitch] (base 2).  O_out/lse_out may alias O_a/lse_a.
// N-way merge for the key-split forward: (o, lse) <- merge of (o, lse) and the
// nparts partials at op + i*o_pstride / lp + i*l_pstride (same row layout); one
// warp per row, 8 columns (one head) per lane and pass.
constexpr int ATT_MERGE_MAX = 15;
__global__ void attn_merge_n_kernel(__nv_bfloat16* o, float* lse, const __nv_bfloat16* op, const float* lp,
                                    int nparts, long o_pstride, long l_pstride, int B, int rows, int H,
                                    long o_bstride, int pitch) {
  const long w = ((long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (w >= (long)B * rows) return;
  const int row = w % rows, b = w / rows;
  const int E = H * 64;
  for (int c0 = 0; c0 < E; c0 += 256) {
    const int col = c0 + lane * 8;
    const bool on = col < E;
    const int h = col / 64;
    const long li = ((long)b * H + h) * pitch + row;
    float l = -INFINITY;
    if (on) {
      float ls[ATT_MERGE_MAX + 1];
      ls[0] = lse[li];
      float mx = ls[0];
      for (int i = 0; i < nparts; ++i) {
        ls[i + 1] = lp[i * l_pstride + li];
        mx = fmaxf(mx, ls[i + 1]);
      }
      const long off = (long)b * o_bstride + (long)row * E + col;
      float acc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = 0.f;
      float den = 0.f;
      if (mx != -INFINITY) {
        for (int i = 0; i <= nparts; ++i) {
          const float wi = exp2f(ls[i] - mx);
          if (wi == 0.f) continue;
          den += wi;
          const uint4 v = *reinterpret_cast<const uint4*>(i == 0 ? o + off : op + (i - 1) * o_pstride + off);
          const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 x = __bfloat1622float2(v2[k]);
            acc[2 * k] += wi * x.x;
            acc[2 * k + 1] += wi * x.y;
          }
        }
        l = mx + __log2f(den);
      }
      const float inv = den > 0.f ? 1.f / den : 0.f;
      uint4 r;
      uint32_t* r2 = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
      for (int k = 0; k < 4; ++k) r2[k] = pack_bf16(acc[2 * k] * inv, acc[2 * k + 1] * inv);
      *reinterpret_cast<uint4*>(o + off) = r;
    }
    __syncwarp();
    if (on && (lane & 7) == 0) lse[li] = l;
  }
}

__global__ void attn_merge_kernel(const __nv_bfloat16* oa, const float* la, const __nv_bfloat16* ob,
                                  const float* lb, __nv_bfloat16* oo, float* lo, int B, int rows, int H,
                                  long o_bstride, int pitch) {
  const long w = ((long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (w >= (long)B * rows) return;
  const int row = w % rows, b = w / rows;
  const int E = H * 64;
  for (int c0 = 0; c0 < E; c0 += 256) {
    const int col = c0 + lane * 8;
    const bool on = col < E;
    const int h = col / 64;
    const long li = ((long)b * H + h) * pitch + row;
    float wa = 0.f, wb = 0.f, l = -INFINITY;
    if (on) {
      const float a = la[li], c = lb[li];
      const float mx = fmaxf(a, c);
      if (mx != -INFINITY) {
        const float ea = exp2f(a - mx), eb = exp2f(c - mx);
        l = mx + __log2f(ea + eb);
        wa = ea / (ea + eb);
        wb = eb / (ea + eb);
      }
      const long off = (long)b * o_bstride + (long)row * E + col;
      const uint4 va = *reinterpret_cast<const uint4*>(oa + off);
      const uint4 vb = *reinterpret_cast<const uint4*>(ob + off);
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&va);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&vb);
      uint4 r;
      uint32_t* r2 = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 x = __bfloat1622float2(a2[i]), y = __bfloat1622float2(b2[i]);
        r2[i] = pack_bf16(wa * x.x + wb * y.x, wa * x.y + wb * y.y);
      }
      *reinterpret_cast<uint4*>(oo + off) = r;
    }
    __syncwarp();
    if (on && (lane & 7) == 0) lo[li] = l;
  }
}

__global__ void add_f32_kernel(float* __restrict__ y, const float* __restrict__ x, long n) {
  const long i = ((long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    float4 a = *reinterpret_cast<float4*>(y + i);
    const float4 b = *reinterpret_cast<const float4*>(x + i);
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    *reinterpret_cast<float4*>(y + i) = a;
  } else {
    for (long k = i; k < n; ++k) y[k] += x[k];
  }
}

// Write +inf into the padded tail of a [B*H][m_pad] log-sum-exp buffer.
__global__ void pad_fill_kernel(float* __restrict__ buf, long nrows, int m, int m_pad, float v) {
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int pad = m_pad - m;
  if (pad <= 0 || idx >= nrows * pad) return;
  buf[(idx / pad) * m_pad + m + (idx % pad)] = v;
}

// dst = sum over nslots of src[slot] (the owner's side of the fused dK|dV
// reduce-scatter: one slot per source rank, written by the peers' backward).
// dst = ascending-slot sum of the slots whose bit is set in mask (unset slots are
// never written by the fused reduce-scatter: their writers attend no key of this
// segment); mask 0 gives zeros.
__global__ void sum_slots_kernel(float4* __restrict__ dst, const float4* __restrict__ src, int nslots,
                                 uint32_t mask, long slot4, long n4) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    bool first = true;
    for (int s = 0; s < nslots; ++s) {
      if (!((mask >> s) & 1u)) continue;
      const float4 b = src[s * slot4 + i];
      if (first) {
        a = b;
        first = false;
      } else {
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
      }
    }
    dst[i] = a;
  }
}

// Optimizer updates over flat fp32 buffers, applied after the gradient
// all-reduce: model.sgd_step (model.py:621-623) and optim.adam_step (optim.py:35-53).
__global__ void sgd_update_kernel(float* __restrict__ p, const float* __restrict__ g, long n, float lr) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    p[i] -= lr * g[i];
}

__global__ void adam_update_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                                   float* __restrict__ v, long n, float lr, float beta1, float beta2, float eps,
                                   float inv_bc1, float inv_bc2) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = beta1 * m[i] + (1.f - beta1) * gi;
    const float vi = beta2 * v[i] + (1.f - beta2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi * inv_bc1) / (sqrtf(vi * inv_bc2) + eps);
  }
}

// ---------------------------------------------------------------- embeddings / loss
// model.embed_fwd (model.py:517-533): x[b][i] = token_table[tokens[b][i]] + pos_table[i]
// (pos_table holds exactly this block's rows).  One warp per (b, i) row, float4.
__global__ void embed_fwd_kernel(const int* __restrict__ tokens, const float* __restrict__ tok,
                                 const float* __restrict__ pos, float* __restrict__ x, long rows, int m, int e) {
  const long r = blockIdx.x * (long)(blockDim.x / 32) + threadIdx.x / 32;
  if (r >= rows) return;
  const int lane = threadIdx.x % 32;
  const float4* trow = reinterpret_cast<const float4*>(tok + (long)tokens[r] * e);
  const float4* prow = reinterpret_cast<const float4*>(pos + (long)(r % m) * e);
  float4* xrow = reinterpret_cast<float4*>(x + r * e);
  for (int c = lane; c < e / 4; c += 32) {
    const float4 a = trow[c], p = prow[c];
    xrow[c] = make_float4(a.x + p.x, a.y + p.y, a.z + p.z, a.w + p.w);
  }
}

// model.embed_bwd (model.py:536-540): grad_pe[i] = sum_b g[b][i] (written), grad_tok[id] +=
// g[b][i] (accumulated: nnops.embed_tokens_bwd scatter-add, nnops.py:258-262).
__global__ void embed_bwd_kernel(const int* __restrict__ tokens, const float* __restrict__ g,
                                 float* __restrict__ grad_tok, float* __restrict__ grad_pe, int batch, int m, int e,
                                 float alpha_tok, float alpha_pos) {
  const long i = blockIdx.x * (long)(blockDim.x / 32) + threadIdx.x / 32;  // position
  if (i >= m) return;
  const int lane = threadIdx.x % 32;
  for (int c = lane; c < e; c += 32) {
    float acc = 0.f;
    for (int b = 0; b < batch; ++b) {
      const long r = (long)b * m + i;
      const float v = g[r * e + c];
      acc += v;
      atomicAdd(grad_tok + (long)tokens[r] * e + c, alpha_tok * v);
    }
    grad_pe[i * e + c] = alpha_pos * acc;
  }
}

// nnops.cross_entropy (nnops.py:274-299): per row r of logits [n][ld] (first v
// columns): loss_r = logsumexp - logit[target], grad = (softmax - onehot) * scale.
// One 256-thread block per row.
__global__ void cross_entropy_kernel(const float* __restrict__ logits, long ld, const int* __restrict__ targets,
                                     int v, float scale, float* __restrict__ loss_rows, float* __restrict__ grad,
                                     long ld_grad) {
  const long r = blockIdx.x;
  const float* row = logits + r * ld;
  __shared__ float red[32];
  float mx = -INFINITY;
  for (int c = threadIdx.x; c < v; c += blockDim.x) mx = fmaxf(mx, row[c]);
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int w = 0; w < (int)(blockDim.x / 32); ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float se = 0.f;
  for (int c = threadIdx.x; c < v; c += blockDim.x) se += expf(row[c] - mx);
  for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = se;
  __syncthreads();
  se = 0.f;
  for (int w = 0; w < (int)(blockDim.x / 32); ++w) se += red[w];
  const int t = targets[r];
  const float lse = mx + logf(se);
  if (threadIdx.x == 0) loss_rows[r] = lse - row[t];
  if (grad) {
    const float inv = 1.f / se;
    float* grow = grad + r * ld_grad;
    for (int c = threadIdx.x; c < v; c += blockDim.x)
      grow[c] = (expf(row[c] - mx) * inv - (c == t ? 1.f : 0.f)) * scale;
    for (int c = v + threadIdx.x; c < ld_grad; c += blockDim.x) grow[c] = 0.f;  // padded head columns
  }
}

// nnops.dropout_fwd / dropout_bwd (nnops.py:143-166) over a (rows, cols) activation
// whose row r is (sample r / m, global position offset + r % m): out = x * keep *
// scale (+ residual).  site = mix(mix(seed, tag), layer + 1); row key =
// mix(mix(site, sample), position).  x / out fp32 or bf16 (same dtype).
LSS_DEV float to_f32(float v) { return v; }
LSS_DEV float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
LSS_DEV T from_f32(float v);
template <>
LSS_DEV float from_f32<float>(float v) { return v; }
template <>
LSS_DEV __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <typename T>
__global__ void dropout_rows_kernel(const T* __restrict__ x, long ldx, T* __restrict__ out, long ldo,
                                    const float* __restrict__ residual, long ld_res, long rows, int cols, int m,
                                    long offset, uint64_t site, uint64_t thresh, float scale) {
  for (long r = blockIdx.y; r < rows; r += gridDim.y) {
    const uint64_t key = drop_mix(drop_mix(site, (uint64_t)(r / m)), (uint64_t)(offset + r % m));
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x) {
      float v = to_f32(x[r * ldx + c]);
      v = drop_keep(key, (uint64_t)c, thresh) ? v * scale : 0.f;
      if (residual) v += residual[r * ld_res + c];
      out[r * ldo + c] = from_f32<T>(v);
    }
  }
}

}  // namespace lss
