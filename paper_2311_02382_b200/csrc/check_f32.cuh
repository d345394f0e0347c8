// fp32 "check mode" kernels: true-FFMA SIMT GEMM and attention, used when the
// caller asks for precision="single" (the north star's <= 1e-4 check mode; TF32
// tensor-core operands measurably miss that bound on dW).
// They follow the same reference semantics as the bf16 tcgen05 path
// (nnops.py:180-193, model.py:280-359) and the same memory layouts, so the
// host code drives both paths identically.  Not a performance path.
#pragma once
#include "common.cuh"
#include "gemm_tc.cuh"

namespace lss {

// C = alpha * A.B^T (+bias) (+residual); A(m,k) = A[m*sam + k*sak], B(n,k) = B[n*sbn + k*sbk]
constexpr int SG_T = 64;
__global__ void gemm_f32_simt_kernel(const float* __restrict__ A, long sam, long sak,
                                     const float* __restrict__ B, long sbn, long sbk, int M, int N,
                                     int K, GemmEpilogue ep) {
  __shared__ float As[16][SG_T + 1];
  __shared__ float Bs[16][SG_T + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // 256 threads, 4x4 outputs each
  const int m0 = blockIdx.y * SG_T, n0 = blockIdx.x * SG_T;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * SG_T; i += 256) {
      const int kk = i % 16, mm = i / 16;
      const int gm = m0 + mm, gn = n0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? A[gm * sam + gk * sak] : 0.f;
      Bs[kk][mm] = (gn < N && gk < K) ? B[gn * sbn + gk * sbk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + ty * 4 + i;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j] * ep.alpha;
      if (ep.bias) v += ep.bias[n];
      if (ep.residual) v += ep.residual[(long)row * ep.ld_res + n];
      if (ep.act == 1) {
        if (ep.pre) reinterpret_cast<float*>(ep.pre)[(long)row * ep.ld_pre + n] = v;
        v = gelu_f<false>(v);
      } else if (ep.act == 2) {
        v *= gelu_grad<false>(reinterpret_cast<const float*>(ep.aux)[(long)row * ep.ld_aux + n]);
      }
      const int seg = n / ep.seg_width;
      const long col = n - (long)seg * ep.seg_width;
      reinterpret_cast<float*>(ep.out[seg])[(long)row * ep.ldo[seg] + col] = v;
    }
  }
}

// Attention forward, fp32: one warp per (query row, head, batch); lanes own
// head dimensions (d <= 128), keys walked in order with an online softmax.
// q [B][m][E], kv [G][B][seg][2E]; o [B][m][E]; lse2 [B][H][m_pad] (base 2).
__global__ void attn_fwd_f32_kernel(const float* __restrict__ q, const float* __restrict__ kb,
                                    const float* __restrict__ vb, long ldkv, float* __restrict__ o, float* __restrict__ lse2, int B, int m,
                                    int m_pad, int G, int seg, int H, int d, long offset, int causal,
                                    float scale) {
  const int warps = blockDim.x / 32;
  const int row = blockIdx.x * warps + threadIdx.x / 32;
  const int h = blockIdx.y, b = blockIdx.z, lane = threadIdx.x % 32;
  if (row >= m) return;
  const int E = H * d;
  const long qpos = offset + row;
  float qv[4], acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = lane + 32 * i;
    qv[i] = k < d ? q[((long)b * m + row) * E + h * d + k] : 0.f;
  }
  float mrun = -INFINITY, l = 0.f;
  const long t = (long)G * seg;
  const long kend = causal ? min(t, qpos + 1) : t;
  for (long j = 0; j < kend; ++j) {
    const int g = j / seg;
    const long r = j % seg;
    const float* kr = kb + (((long)g * B + b) * seg + r) * ldkv + h * d;
    const float* vr = vb + (((long)g * B + b) * seg + r) * ldkv + h * d;
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = lane + 32 * i;
      if (k < d) s = fmaf(qv[i], kr[k], s);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    s *= scale;
    const float mnew = fmaxf(mrun, s);
    const float a = expf(mrun - mnew), pj = expf(s - mnew);
    l = l * a + pj;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = lane + 32 * i;
      acc[i] = acc[i] * a + (k < d ? pj * vr[k] : 0.f);
    }
    mrun = mnew;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = lane + 32 * i;
    if (k < d) o[((long)b * m + row) * E + h * d + k] = acc[i] / l;
  }
  if (lane == 0) lse2[((long)b * H + h) * m_pad + row] = (mrun + logf(l)) * 1.4426950408889634f;
}

// dQ rows: one warp per (query row, head, batch).
__global__ void attn_bwd_dq_f32_kernel(const float* __restrict__ q, const float* __restrict__ kb,
                                       const float* __restrict__ vb, long ldkv, const float* __restrict__ dO, const float* __restrict__ lse2,
                                       const float* __restrict__ delta, float* __restrict__ dq, int B,
                                       int m, int m_pad, int G, int seg, int H, int d, long offset,
                                       int causal, float scale) {
  const int warps = blockDim.x / 32;
  const int row = blockIdx.x * warps + threadIdx.x / 32;
  const int h = blockIdx.y, b = blockIdx.z, lane = threadIdx.x % 32;
  if (row >= m) return;
  const int E = H * d;
  const long qpos = offset + row;
  const float L = lse2[((long)b * H + h) * m_pad + row] * 0.6931471805599453f;
  const float D = delta[((long)b * H + h) * m_pad + row];
  float qv[4], gv[4], acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = lane + 32 * i;
    qv[i] = k < d ? q[((long)b * m + row) * E + h * d + k] : 0.f;
    gv[i] = k < d ? dO[((long)b * m + row) * E + h * d + k] : 0.f;
  }
  const long t = (long)G * seg;
  const long kend = causal ? min(t, qpos + 1) : t;
  for (long j = 0; j < kend; ++j) {
    const int g = j / seg;
    const long r = j % seg;
    const float* kr = kb + (((long)g * B + b) * seg + r) * ldkv + h * d;
    const float* vr = vb + (((long)g * B + b) * seg + r) * ldkv + h * d;
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = lane + 32 * i;
      if (k < d) {
        s = fmaf(qv[i], kr[k], s);
        dp = fmaf(gv[i], vr[k], dp);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, off);
      dp += __shfl_xor_sync(0xffffffffu, dp, off);
    }
    const float pj = expf(s * scale - L);
    const float ds = pj * (dp - D) * scale;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = lane + 32 * i;
      if (k < d) acc[i] = fmaf(ds, kr[k], acc[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = lane + 32 * i;
    if (k < d) dq[((long)b * m + row) * E + h * d + k] = acc[i];
  }
}

// dK/dV rows over the full key length: one warp per (key row, head, batch).
__global__ void attn_bwd_dkv_f32_kernel(const float* __restrict__ q, const float* __restrict__ kb,
                                        const float* __restrict__ vb, long ldkv,
                                        const float* __restrict__ dO, const float* __restrict__ lse2,
                                        const float* __restrict__ delta, float* __restrict__ dkb,
                                        float* __restrict__ dvb, long lddkv,
                                        int B, int m, int m_pad, int G, int seg, int H, int d,
                                        long offset, int causal, float scale) {
  const int warps = blockDim.x / 32;
  const long j = (long)blockIdx.x * warps + threadIdx.x / 32;  // global key row
  const int h = blockIdx.y, b = blockIdx.z, lane = threadIdx.x % 32;
  const long t = (long)G * seg;
  if (j >= t) return;
  const int E = H * d;
  const int g = j / seg;
  const long r = j % seg;
  const float* kr = kb + (((long)g * B + b) * seg + r) * ldkv + h * d;
  const float* vr = vb + (((long)g * B + b) * seg + r) * ldkv + h * d;
  float kvv[4], vv[4], dk[4] = {0.f, 0.f, 0.f, 0.f}, dv[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = lane + 32 * i;
    kvv[i] = k < d ? kr[k] : 0.f;
    vv[i] = k < d ? vr[k] : 0.f;
  }
  long i0 = causal ? max(0L, j - offset) : 0L;
  for (long i = i0; i < m; ++i) {
    const float* qr = q + ((long)b * m + i) * E + h * d;
    const float* gr = dO + ((long)b * m + i) * E + h * d;
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int k = lane + 32 * c;
      if (k < d) {
        s = fmaf(qr[k], kvv[c], s);
        dp = fmaf(gr[k], vv[c], dp);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, off);
      dp += __shfl_xor_sync(0xffffffffu, dp, off);
    }
    const float L = lse2[((long)b * H + h) * m_pad + i] * 0.6931471805599453f;
    const float D = delta[((long)b * H + h) * m_pad + i];
    const float pj = expf(s * scale - L);
    const float ds = pj * (dp - D) * scale;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int k = lane + 32 * c;
      if (k < d) {
        dv[c] = fmaf(pj, gr[k], dv[c]);
        dk[c] = fmaf(ds, qr[k], dk[c]);
      }
    }
  }
  float* dstk = dkb + (((long)g * B + b) * seg + r) * lddkv + h * d;
  float* dstv = dvb + (((long)g * B + b) * seg + r) * lddkv + h * d;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int k = lane + 32 * c;
    if (k < d) {
      dstk[k] = dk[c];
      dstv[k] = dv[c];
    }
  }
}

}  // namespace lss
