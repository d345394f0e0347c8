// extern "C" entry points of liblss.so (declared in include/lss.h).
// Host-side validation (mirroring the reference's ShapeError / PartitionError
// checks), TMA tensor-map construction and kernel launches.  No allocation,
// no host synchronisation: every call is ordered on the caller's stream.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "../../include/lss.h"
#include "attn_bwd.cuh"
#include "attn_fwd.cuh"
#include "check_f32.cuh"
#include "elementwise.cuh"
#include "gemm_tc.cuh"

using namespace lss;

namespace {

thread_local std::string g_last_error;
int g_deterministic = 0;  // LSS_RT_DETERMINISTIC: column sums without atomics (process-wide)

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LSS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return LSS_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// bf16 tensor map with 128B swizzle; dims[0] is the contiguous dimension.
int make_map(CUtensorMap* m, CUtensorMapDataType dt, int elem_bytes, int rank, const void* addr,
             const uint64_t* dims, const uint64_t* strides_elems, const uint32_t* box,
             CUtensorMapSwizzle sw) {
  auto fn = encode_fn();
  if (!fn) return fail(LSS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gdim[5], gstr[4];
  cuuint32_t bdim[5], estr[5];
  for (int i = 0; i < rank; ++i) {
    gdim[i] = dims[i];
    bdim[i] = box[i];
    estr[i] = 1;
  }
  for (int i = 0; i < rank - 1; ++i) gstr[i] = strides_elems[i] * elem_bytes;
  CUresult r = fn(m, dt, rank, const_cast<void*>(addr), gdim, gstr, bdim, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LSS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return LSS_OK;
}

// bf16 rows [outer][mid][rows][ld] viewed as a 4-D (or 3-D when outer == 1) map of
// `cols` visible columns; box 64 columns x 128 rows, 128B swizzle.
int map_rows(CUtensorMap* m, const void* base, int cols, long ld, long rows, long mid, long outer, int rank,
             int box_rows = 128) {
  uint64_t dims[4] = {(uint64_t)cols, (uint64_t)rows, (uint64_t)mid, (uint64_t)outer};
  uint64_t str[3] = {(uint64_t)ld, (uint64_t)(rows * ld), (uint64_t)(mid * rows * ld)};
  uint32_t box[4] = {64, (uint32_t)box_rows, 1, 1};
  return make_map(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rank, base, dims, str, box,
                  CU_TENSOR_MAP_SWIZZLE_128B);
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename K>
int set_smem(K kernel, int bytes) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return fail(LSS_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  return LSS_OK;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" {

int lss_abi_version(void) { return LSS_ABI_VERSION; }
const char* lss_last_error(void) { return g_last_error.c_str(); }
long lss_rows_pad(long rows) { return (rows + ATT_BM - 1) / ATT_BM * ATT_BM; }

int lss_layernorm_fwd(const float* x, const float* gain, const float* bias, void* y, int y_dtype,
                      float* mean, float* rstd, long rows, int embed, float eps, void* stream) {
  if (!x || !gain || !bias || !y || !mean || !rstd) return fail(LSS_ERR_ARG, "layernorm_fwd: null pointer");
  if (embed <= 0 || embed % 4 || embed > 4096) return fail(LSS_ERR_UNSUPPORTED, "layernorm_fwd: embed %d", embed);
  if (rows <= 0) return LSS_OK;
  if (embed % 128 == 0 && embed <= 2048 && (y_dtype == LSS_BF16 || y_dtype == LSS_F32)) {
    const long blocks = (rows + 7) / 8;  // warp per row, 8 rows per block
#define LSS_LN_WARP(NV)                                                                                        \
  do {                                                                                                          \
    if (y_dtype == LSS_BF16)                                                                                    \
      layernorm_fwd_warp_kernel<__nv_bfloat16, NV><<<blocks, 256, 0, S(stream)>>>(                              \
          x, gain, bias, reinterpret_cast<__nv_bfloat16*>(y), mean, rstd, rows, eps);                           \
    else                                                                                                        \
      layernorm_fwd_warp_kernel<float, NV><<<blocks, 256, 0, S(stream)>>>(x, gain, bias, reinterpret_cast<float*>(y), \
                                                                           mean, rstd, rows, eps);              \
  } while (0)
    switch (embed / 128) {
      case 1: LSS_LN_WARP(1); break;
      case 2: LSS_LN_WARP(2); break;
      case 4: LSS_LN_WARP(4); break;
      case 8: LSS_LN_WARP(8); break;
      case 16: LSS_LN_WARP(16); break;
      default: goto block_per_row;
    }
#undef LSS_LN_WARP
    return check_launch("layernorm_fwd");
  }
block_per_row:
  const int threads = ((embed / 4 + 31) / 32) * 32;
  if (y_dtype == LSS_BF16)
    layernorm_fwd_kernel<__nv_bfloat16><<<rows, threads, 0, S(stream)>>>(
        x, gain, bias, reinterpret_cast<__nv_bfloat16*>(y), mean, rstd, embed, eps);
  else if (y_dtype == LSS_F32)
    layernorm_fwd_kernel<float><<<rows, threads, 0, S(stream)>>>(x, gain, bias, reinterpret_cast<float*>(y),
                                                                 mean, rstd, embed, eps);
  else
    return fail(LSS_ERR_ARG, "layernorm_fwd: dtype %d", y_dtype);
  return check_launch("layernorm_fwd");
}

int lss_layernorm_bwd(const float* grad_xh, const float* x, const float* mean, const float* rstd,
                      const float* gain, const float* grad_res, float* grad_x, float* grad_gain,
                      float* grad_bias, float alpha, long rows, int embed, void* stream) {
  if (!grad_xh || !x || !mean || !rstd || !gain || !grad_x || !grad_gain || !grad_bias)
    return fail(LSS_ERR_ARG, "layernorm_bwd: null pointer");
  if (embed <= 0 || embed % 4 || embed > 4096) return fail(LSS_ERR_UNSUPPORTED, "layernorm_bwd: embed %d", embed);
  if (rows <= 0) return LSS_OK;
  const bool det = g_deterministic != 0;
  float* gg = det ? nullptr : grad_gain;
  bool warp_path = embed % 128 == 0 && embed <= 1024;  // (E=2048 would spill its register partials)
  if (warp_path) {  // warp per row (LNW_RPW rows per warp, 8 warps per block)
    const long wblocks = (rows + 8 * LNW_RPW - 1) / (8 * LNW_RPW);
    const size_t sm = 8 * (size_t)embed * sizeof(float);
#define LSS_LNB_WARP(NV)                                                                                      \
  do {                                                                                                        \
    if (sm > 48 * 1024) cudaFuncSetAttribute(layernorm_bwd_warp_kernel<NV>,                                   \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);            \
    layernorm_bwd_warp_kernel<NV><<<wblocks, 256, sm, S(stream)>>>(grad_xh, x, mean, rstd, gain, grad_res,     \
                                                                   grad_x, gg, grad_bias, alpha, rows);        \
  } while (0)
    switch (embed / 128) {
      case 1: LSS_LNB_WARP(1); break;
      case 2: LSS_LNB_WARP(2); break;
      case 4: LSS_LNB_WARP(4); break;
      case 8: LSS_LNB_WARP(8); break;
      default: warp_path = false;
    }
#undef LSS_LNB_WARP
  }
  if (!warp_path) {
    const int threads = ((embed / 4 + 31) / 32) * 32;
    const long blocks = (rows + LN_BWD_ROWS - 1) / LN_BWD_ROWS;
    layernorm_bwd_kernel<<<blocks, threads, 0, S(stream)>>>(grad_xh, x, mean, rstd, gain, grad_res, grad_x, gg,
                                                            grad_bias, alpha, rows, embed);
  }
  if (det)  // one writer per column, fixed order (bitwise repeatable)
    ln_colsum_det_kernel<<<(embed + DET_COLS - 1) / DET_COLS, DET_COLS * DET_LANES, 0, S(stream)>>>(
        grad_xh, x, mean, rstd, grad_gain, grad_bias, alpha, rows, embed);
  return check_launch("layernorm_bwd");
}

int lss_gemm(int dtype, const void* A, long lda, int a_mn_major, const void* B, long ldb, int b_mn_major,
             int M, int N, int K, const lss_gemm_epilogue* ep_in, void* stream) {
  if (!A || !B || !ep_in) return fail(LSS_ERR_ARG, "gemm: null pointer");
  if (M < 0 || N < 0 || K < 0) return fail(LSS_ERR_SHAPE, "gemm: negative extent");
  if (M == 0 || N == 0) return LSS_OK;
  GemmEpilogue ep;
  for (int i = 0; i < 3; ++i) {
    ep.out[i] = ep_in->out[i];
    ep.ldo[i] = ep_in->ldo[i];
  }
  ep.seg_width = ep_in->seg_width > 0 ? ep_in->seg_width : N;
  ep.out_bf16 = ep_in->out_dtype == LSS_BF16;
  ep.alpha = ep_in->alpha;
  ep.bias = ep_in->bias;
  ep.residual = ep_in->residual;
  ep.ld_res = ep_in->ld_res;
  ep.act = ep_in->act;
  ep.pre = ep_in->pre;
  ep.ld_pre = ep_in->ld_pre;
  ep.aux = ep_in->aux;
  ep.ld_aux = ep_in->ld_aux;
  ep.aux_bf16 = ep_in->aux_dtype == LSS_BF16;
  if (ep.act < LSS_ACT_NONE || ep.act > LSS_ACT_GELU_BWD) return fail(LSS_ERR_ARG, "gemm: activation %d", ep.act);
  if (ep.act == LSS_ACT_GELU_BWD && !ep.aux) return fail(LSS_ERR_ARG, "gemm: GeLU backward needs the pre-activation");
  if (ep.act == LSS_ACT_GELU && ep.pre && (ep.ld_pre < N || !aligned16(ep.pre) || ep.ld_pre % 8))
    return fail(LSS_ERR_SHAPE, "gemm: pre-activation buffer ld %ld / alignment", ep.ld_pre);
  if (ep.act == LSS_ACT_GELU_BWD && (ep.ld_aux < N || !aligned16(ep.aux) || ep.ld_aux % 8))
    return fail(LSS_ERR_SHAPE, "gemm: aux ld %ld / alignment", ep.ld_aux);
  if (ep.act != LSS_ACT_NONE && (ep.seg_width != N))
    return fail(LSS_ERR_UNSUPPORTED, "gemm: activation epilogue with split output segments");
  const int nseg = (N + ep.seg_width - 1) / ep.seg_width;
  if (nseg > 3) return fail(LSS_ERR_SHAPE, "gemm: %d output segments (max 3)", nseg);
  for (int s = 0; s < nseg; ++s)
    if (!ep.out[s]) return fail(LSS_ERR_ARG, "gemm: output segment %d is null", s);

  if (dtype == LSS_F32) {
    if (ep.out_bf16) return fail(LSS_ERR_UNSUPPORTED, "gemm f32: bf16 output");
    if (ep.act == LSS_ACT_GELU_BWD && ep.aux_bf16) return fail(LSS_ERR_UNSUPPORTED, "gemm f32: bf16 aux");
    const float* a = reinterpret_cast<const float*>(A);
    const float* b = reinterpret_cast<const float*>(B);
    const long sam = a_mn_major ? 1 : lda, sak = a_mn_major ? lda : 1;
    const long sbn = b_mn_major ? 1 : ldb, sbk = b_mn_major ? ldb : 1;
    dim3 grid((N + SG_T - 1) / SG_T, (M + SG_T - 1) / SG_T);
    gemm_f32_simt_kernel<<<grid, 256, 0, S(stream)>>>(a, sam, sak, b, sbn, sbk, M, N, K, ep);
    return check_launch("gemm_f32");
  }
  if (dtype != LSS_BF16) return fail(LSS_ERR_ARG, "gemm: dtype %d", dtype);
  if (N % 32 || ep.seg_width % 32) return fail(LSS_ERR_UNSUPPORTED, "gemm bf16: N=%d seg=%d not multiples of 32", N, ep.seg_width);
  if (K % 8 || lda % 8 || ldb % 8 || (a_mn_major && M % 8) || (b_mn_major && N % 8))
    return fail(LSS_ERR_UNSUPPORTED, "gemm bf16: 16-byte row alignment required");
  if (!aligned16(A) || !aligned16(B)) return fail(LSS_ERR_UNSUPPORTED, "gemm bf16: operands not 16B aligned");
  CUtensorMap ma, mb;
  int rc;
  {
    uint64_t dims[2], str[1] = {(uint64_t)lda};
    uint32_t box[2];
    if (a_mn_major) { dims[0] = M; dims[1] = K; box[0] = 64; box[1] = 64; }
    else            { dims[0] = K; dims[1] = M; box[0] = 64; box[1] = GEMM_BM; }
    if ((rc = make_map(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 2, A, dims, str, box,
                       CU_TENSOR_MAP_SWIZZLE_128B)))
      return rc;
  }
  // CTA pairs (cta_group::2, 256 x 256 tiles) for the long-K products, where the
  // mainloop dominates (A/B on B200, l=50112: dx K=3E 233 -> 208 us, dWqkv K=l 278 -> 267;
  // the K=E projections with their heavier epilogues: QKV 307 -> 303, out-proj 213 -> 226)
  const bool pair = LSS_GEMM_2CTA && M >= 4 * GEMM_BM && K >= 2048;
  {
    uint64_t dims[2], str[1] = {(uint64_t)ldb};
    uint32_t box[2];
    if (b_mn_major) { dims[0] = N; dims[1] = K; box[0] = 64; box[1] = 64; }
    else            { dims[0] = K; dims[1] = N; box[0] = 64; box[1] = pair ? GEMM_BN / 2 : GEMM_BN; }
    if ((rc = make_map(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 2, B, dims, str, box,
                       CU_TENSOR_MAP_SWIZZLE_128B)))
      return rc;
  }
  if (pair) {
    const int pairs = ((M + 2 * GEMM_BM - 1) / (2 * GEMM_BM)) * ((N + GEMM_BN - 1) / GEMM_BN);
    const int clusters = pairs < num_sms() / 2 ? pairs : num_sms() / 2;
#define LSS_GEMM2_LAUNCH(AM, BM_)                                                                      \
  do {                                                                                                  \
    if ((rc = set_smem(gemm_bf16_tc2_kernel<AM, BM_>, GEMM2_SMEM_BYTES))) return rc;                  \
    gemm_bf16_tc2_kernel<AM, BM_><<<2 * clusters, GEMM_THREADS, GEMM2_SMEM_BYTES, S(stream)>>>(ma, mb, M, N, K, ep); \
  } while (0)
    if (!a_mn_major && !b_mn_major) LSS_GEMM2_LAUNCH(0, 0);
    else if (!a_mn_major && b_mn_major) LSS_GEMM2_LAUNCH(0, 1);
    else if (a_mn_major && !b_mn_major) LSS_GEMM2_LAUNCH(1, 0);
    else LSS_GEMM2_LAUNCH(1, 1);
#undef LSS_GEMM2_LAUNCH
    return check_launch("gemm_bf16_tc2");
  }
  const int tiles = ((M + GEMM_BM - 1) / GEMM_BM) * ((N + GEMM_BN - 1) / GEMM_BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
#define LSS_GEMM_LAUNCH(AM, BM_)                                                                  \
  do {                                                                                             \
    if ((rc = set_smem(gemm_bf16_tc_kernel<AM, BM_>, GEMM_SMEM_BYTES))) return rc;                \
    gemm_bf16_tc_kernel<AM, BM_><<<grid, GEMM_THREADS, GEMM_SMEM_BYTES, S(stream)>>>(ma, mb, M, N, K, ep); \
  } while (0)
  if (!a_mn_major && !b_mn_major) LSS_GEMM_LAUNCH(0, 0);
  else if (!a_mn_major && b_mn_major) LSS_GEMM_LAUNCH(0, 1);
  else if (a_mn_major && !b_mn_major) LSS_GEMM_LAUNCH(1, 0);
  else LSS_GEMM_LAUNCH(1, 1);
#undef LSS_GEMM_LAUNCH
  return check_launch("gemm_bf16_tc");
}

int lss_stage_weights(int dtype, const float* wq, const float* wk, const float* wv, const float* wo,
                      const float* bq, const float* bk, const float* bv, void* wqkv_t, void* wqkv,
                      void* wo_t, void* wo_n, float* bqkv, int embed, void* stream) {
  if (!wq || !wk || !wv || !wo || !wqkv_t || !wqkv || !wo_t || !wo_n || !bqkv)
    return fail(LSS_ERR_ARG, "stage_weights: null pointer");
  dim3 grid((embed + 31) / 32, (embed + 31) / 32, 4), block(32, 8);
  if (dtype == LSS_BF16)
    weight_stage_kernel<__nv_bfloat16><<<grid, block, 0, S(stream)>>>(
        wq, wk, wv, wo, bq, bk, bv, reinterpret_cast<__nv_bfloat16*>(wqkv_t),
        reinterpret_cast<__nv_bfloat16*>(wqkv), reinterpret_cast<__nv_bfloat16*>(wo_t),
        reinterpret_cast<__nv_bfloat16*>(wo_n), bqkv, embed);
  else if (dtype == LSS_F32)
    weight_stage_kernel<float><<<grid, block, 0, S(stream)>>>(
        wq, wk, wv, wo, bq, bk, bv, reinterpret_cast<float*>(wqkv_t), reinterpret_cast<float*>(wqkv),
        reinterpret_cast<float*>(wo_t), reinterpret_cast<float*>(wo_n), bqkv, embed);
  else
    return fail(LSS_ERR_ARG, "stage_weights: dtype %d", dtype);
  return check_launch("stage_weights");
}

int lss_cat_cast_colsum(int out_dtype, const float* const* srcs, const long* lds, const int* cols,
                        int nsrc, void* dst, long ld_dst, float* colsum, float alpha, long rows,
                        void* stream) {
  return lss_cat_cast_colsum_ex(out_dtype, srcs, lds, cols, nullptr, nullptr, nullptr, nsrc, dst, ld_dst, colsum,
                                alpha, rows, stream);
}

int lss_cat_cast_colsum_ex(int out_dtype, const float* const* srcs, const long* lds, const int* cols,
                           const int* nslots, const unsigned int* masks, const long* slot_strides, int nsrc,
                           void* dst, long ld_dst, float* colsum, float alpha, long rows, void* stream) {
  if (nsrc < 1 || nsrc > 3 || !srcs || !lds || !cols) return fail(LSS_ERR_ARG, "cat_cast_colsum: bad sources");
  CatSrc cs;
  int total = 0;
  for (int i = 0; i < 3; ++i) {
    cs.ptr[i] = i < nsrc ? srcs[i] : nullptr;
    cs.ld[i] = i < nsrc ? lds[i] : 0;
    cs.cols[i] = i < nsrc ? cols[i] : 0;
    cs.nslot[i] = (i < nsrc && nslots) ? nslots[i] : 1;
    cs.mask[i] = (i < nsrc && masks) ? masks[i] : 1u;
    cs.slot_stride[i] = (i < nsrc && slot_strides) ? slot_strides[i] : 0;
    if (cs.nslot[i] > 32 || (cs.nslot[i] > 1 && cs.slot_stride[i] % 4))
      return fail(LSS_ERR_UNSUPPORTED, "cat_cast_colsum: source %d slots", i);
    if (i < nsrc) {
      if (!srcs[i] || cols[i] % 4 || lds[i] % 4) return fail(LSS_ERR_UNSUPPORTED, "cat_cast_colsum: source %d", i);
      total += cols[i];
    }
  }
  cs.n = nsrc;
  if (rows <= 0) return LSS_OK;
  const int threads = 128;
  const bool det = g_deterministic != 0 && colsum;
  dim3 grid((total / 4 + threads - 1) / threads, (rows + CAT_ROWS - 1) / CAT_ROWS);
  float* cs_atomic = det ? nullptr : colsum;
  if (dst || !det) {
    if (out_dtype == LSS_BF16)
      cat_cast_colsum_kernel<__nv_bfloat16><<<grid, threads, 0, S(stream)>>>(
          cs, reinterpret_cast<__nv_bfloat16*>(dst), ld_dst, cs_atomic, alpha, rows);
    else
      cat_cast_colsum_kernel<float><<<grid, threads, 0, S(stream)>>>(cs, reinterpret_cast<float*>(dst), ld_dst,
                                                                     cs_atomic, alpha, rows);
  }
  if (det)  // one writer per column, fixed order (bitwise repeatable)
    colsum_det_kernel<<<(total + DET_COLS - 1) / DET_COLS, DET_COLS * DET_LANES, 0, S(stream)>>>(cs, colsum, alpha,
                                                                                                  rows);
  return check_launch("cat_cast_colsum");
}

static int attn_check(int dtype, int batch, int rows, int workers, int seg_len, int heads, int head_dim) {
  if (batch <= 0 || rows <= 0 || workers <= 0 || seg_len <= 0 || heads <= 0 || head_dim <= 0)
    return fail(LSS_ERR_SHAPE, "attention: non-positive extent");
  if (dtype == LSS_BF16 && head_dim != ATT_D)
    return fail(LSS_ERR_UNSUPPORTED, "attention bf16: head_dim %d (tcgen05 path supports 64)", head_dim);
  if (dtype == LSS_F32 && head_dim > 128)
    return fail(LSS_ERR_UNSUPPORTED, "attention f32: head_dim %d > 128", head_dim);
  if (dtype != LSS_BF16 && dtype != LSS_F32) return fail(LSS_ERR_ARG, "attention: dtype %d", dtype);
  return LSS_OK;
}

}  // extern "C"

// Forward launcher shared by lss_attn_fwd_ex (splits = 1) and lss_attn_fwd_split.
static int attn_fwd_launch(int dtype, const void* q, int rows, long q_bstride, const void* k, const void* v,
                           long ld_kv, void* o, long o_bstride, float* lse2, int lse_pitch, int batch, int workers,
                           int seg_len, int heads, int head_dim, long offset, int causal, int g_begin, int g_end,
                           const lss_dropout* dropout, int splits, void* o_part, long o_part_stride,
                           float* lse_part, long lse_part_stride, const unsigned int* seg_ready,
                           unsigned int ready_seq, int own_seg, void* stream) {
  int rc = attn_check(dtype, batch, rows, workers, seg_len, heads, head_dim);
  if (rc) return rc;
  if (!q || !k || !v || !o || !lse2) return fail(LSS_ERR_ARG, "attn_fwd: null pointer");
  const int E = heads * head_dim;
  if (ld_kv < E) return fail(LSS_ERR_SHAPE, "attn_fwd: ld_kv %ld < embed %d", ld_kv, E);
  if (causal && offset < 0) return fail(LSS_ERR_DEGENERATE, "attn_fwd: negative offset leaves rows fully masked");
  if (g_begin < 0 || g_end > workers || g_begin >= g_end) return fail(LSS_ERR_SHAPE, "attn_fwd: bad segment range");
  const int m_pad = (int)lss_rows_pad(rows);
  if (lse_pitch < m_pad) return fail(LSS_ERR_SHAPE, "attn_fwd: lse pitch %d < %d", lse_pitch, m_pad);
  if (q_bstride < (long)rows * E || o_bstride < (long)rows * E) return fail(LSS_ERR_SHAPE, "attn_fwd: batch stride");
  const float scale = 1.0f / sqrtf((float)head_dim);
  if (dtype == LSS_F32) {
    if (dropout && dropout->active) return fail(LSS_ERR_UNSUPPORTED, "attn_fwd f32: dropout is bf16-path only");
    if (splits != 1) return fail(LSS_ERR_UNSUPPORTED, "attn_fwd f32: key splits are bf16-only");
    if (g_begin != 0 || g_end != workers || q_bstride != (long)rows * E || o_bstride != (long)rows * E ||
        lse_pitch != m_pad)
      return fail(LSS_ERR_UNSUPPORTED, "attn_fwd f32: partial/strided attention is bf16-only");
    dim3 grid((rows + 3) / 4, heads, batch);
    attn_fwd_f32_kernel<<<grid, 128, 0, S(stream)>>>(
        reinterpret_cast<const float*>(q), reinterpret_cast<const float*>(k), reinterpret_cast<const float*>(v),
        ld_kv, reinterpret_cast<float*>(o), lse2, batch, rows, m_pad, workers, seg_len, heads, head_dim, offset,
        causal, scale);
    return check_launch("attn_fwd_f32");
  }
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || ld_kv % 8 || q_bstride % 8 ||
      o_bstride % 8)
    return fail(LSS_ERR_UNSUPPORTED, "attn_fwd: 16B alignment");
  CUtensorMap mq, mk, mv;
  {
    uint64_t dims[3] = {(uint64_t)E, (uint64_t)rows, (uint64_t)batch};
    uint64_t str[2] = {(uint64_t)E, (uint64_t)q_bstride};
    uint32_t box[3] = {64, 128, 1};
    if ((rc = make_map(&mq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 3, q, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)))
      return rc;
  }
  if ((rc = map_rows(&mk, k, E, ld_kv, seg_len, batch, workers, 4))) return rc;
  if ((rc = map_rows(&mv, v, E, ld_kv, seg_len, batch, workers, 4))) return rc;
  AttnFwdParams p;
  p.B = batch; p.m = rows; p.m_pad = m_pad; p.G = workers; p.seg_len = seg_len; p.H = heads;
  p.g_begin = g_begin; p.g_end = g_end;
  p.offset = offset; p.causal = causal;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.o = reinterpret_cast<__nv_bfloat16*>(o);
  p.o_bstride = o_bstride;
  p.lse2 = lse2;
  p.lse_pitch = lse_pitch;
  const bool drop = dropout && dropout->active;
  p.drop_site = drop ? dropout->site_key : 0;
  p.drop_thresh = drop ? dropout->thresh : 0;
  p.drop_scale = drop ? dropout->scale : 1.f;
  p.splits = splits;
  p.o_part = reinterpret_cast<__nv_bfloat16*>(o_part);
  p.o_part_stride = o_part_stride;
  p.lse_part = lse_part;
  p.lse_part_stride = lse_part_stride;
  p.seg_ready = seg_ready;
  p.ready_seq = ready_seq;
  p.own_seg = own_seg;
  dim3 grid((unsigned)((rows + 2 * ATT_BM - 1) / (2 * ATT_BM)) * heads * batch * splits);
#ifdef LSS_FWD_PLAIN
  const bool part = splits > 1 || seg_ready != nullptr;
#else
  // the PART instance (incremental top-down tile walk) measured 2.5% faster than the
  // plain one even for a single resident segment (N=1: 6.12 vs 6.27 ms), so it runs always
  const bool part = true;
#endif
  auto launch = [&](auto kern) -> int {
    int r = set_smem(kern, ATT_FWD_SMEM);
    if (r) return r;
    kern<<<grid, ATT_FWD_THREADS, ATT_FWD_SMEM, S(stream)>>>(mq, mk, mv, p);
    return LSS_OK;
  };
  if (drop)
    rc = part ? launch(attn_fwd_tc_kernel<true, true>) : launch(attn_fwd_tc_kernel<true, false>);
  else
    rc = part ? launch(attn_fwd_tc_kernel<false, true>) : launch(attn_fwd_tc_kernel<false, false>);
  if (rc) return rc;
  if ((rc = check_launch("attn_fwd_tc"))) return rc;
  if (splits > 1) {
    const long warps = (long)batch * rows;
    attn_merge_n_kernel<<<(warps * 32 + 255) / 256, 256, 0, S(stream)>>>(
        reinterpret_cast<__nv_bfloat16*>(o), lse2, reinterpret_cast<const __nv_bfloat16*>(o_part), lse_part,
        splits - 1, o_part_stride, lse_part_stride, batch, rows, heads, o_bstride, lse_pitch);
    return check_launch("attn_merge_n");
  }
  return LSS_OK;
}

extern "C" {

int lss_attn_fwd_ex(int dtype, const void* q, int rows, long q_bstride, const void* k, const void* v, long ld_kv,
                    void* o, long o_bstride, float* lse2, int lse_pitch, int batch, int workers, int seg_len,
                    int heads, int head_dim, long offset, int causal, int g_begin, int g_end,
                    const lss_dropout* dropout, void* stream) {
  return attn_fwd_launch(dtype, q, rows, q_bstride, k, v, ld_kv, o, o_bstride, lse2, lse_pitch, batch, workers,
                         seg_len, heads, head_dim, offset, causal, g_begin, g_end, dropout, 1, nullptr, 0, nullptr,
                         0, nullptr, 0, -1, stream);
}

int lss_attn_fwd_split(int dtype, const void* q, int rows, long q_bstride, const void* k, const void* v,
                       long ld_kv, void* o, long o_bstride, float* lse2, int lse_pitch, int batch, int workers,
                       int seg_len, int heads, int head_dim, long offset, int causal, int g_begin, int g_end,
                       const lss_dropout* dropout, int splits, void* o_part, long o_part_stride, float* lse_part,
                       long lse_part_stride, const unsigned int* seg_ready, unsigned int ready_seq, int own_seg,
                       void* stream) {
  if (splits < 1 || splits > ATT_MERGE_MAX + 1)
    return fail(LSS_ERR_ARG, "attn_fwd_split: %d splits (1..%d)", splits, ATT_MERGE_MAX + 1);
  if (splits > 1) {
    if (!o_part || !lse_part) return fail(LSS_ERR_ARG, "attn_fwd_split: null partial buffers");
    const long o_span = (long)(batch - 1) * o_bstride + (long)rows * heads * head_dim;  // one slot's extent
    if (!aligned16(o_part) || o_part_stride % 8 || o_part_stride < o_span ||
        lse_part_stride < (long)(batch * heads - 1) * lse_pitch + rows)
      return fail(LSS_ERR_SHAPE, "attn_fwd_split: partial slot stride");
  }
  return attn_fwd_launch(dtype, q, rows, q_bstride, k, v, ld_kv, o, o_bstride, lse2, lse_pitch, batch, workers,
                         seg_len, heads, head_dim, offset, causal, g_begin, g_end, dropout, splits, o_part,
                         o_part_stride, lse_part, lse_part_stride, seg_ready, ready_seq, own_seg, stream);
}

int lss_attn_fwd(int dtype, const void* q, const void* k, const void* v, long ld_kv, void* o, float* lse2,
                 int batch, int rows, int workers, int seg_len, int heads, int head_dim, long offset, int causal,
                 void* stream) {
  const long E = (long)heads * head_dim;
  return lss_attn_fwd_ex(dtype, q, rows, rows * E, k, v, ld_kv, o, rows * E, lse2, (int)lss_rows_pad(rows), batch,
                         workers, seg_len, heads, head_dim, offset, causal, 0, workers, nullptr, stream);
}

int lss_attn_delta(int dtype, const void* o, const void* grad_o, float* delta, int batch, int rows, int heads,
                   int head_dim, int scaled, void* stream) {
  if (!o || !grad_o || !delta) return fail(LSS_ERR_ARG, "attn_delta: null pointer");
  if (batch <= 0 || rows <= 0 || heads <= 0 || head_dim <= 0) return fail(LSS_ERR_SHAPE, "attn_delta: extent");
  const int E = heads * head_dim;
  const int m_pad = (int)lss_rows_pad(rows);
  const float scale = scaled ? 1.0f / sqrtf((float)head_dim) : 1.0f;
  const long total = (long)batch * m_pad * heads;
  const int threads = 256;
  if (dtype == LSS_BF16 && head_dim == 64 && E % 256 == 0) {
    const long warps = (long)batch * m_pad;
    attn_delta_bf16_d64_kernel<<<(warps * 32 + threads - 1) / threads, threads, 0, S(stream)>>>(
        reinterpret_cast<const __nv_bfloat16*>(grad_o), reinterpret_cast<const __nv_bfloat16*>(o), delta, batch,
        rows, m_pad, heads, scale);
  } else if (dtype == LSS_BF16) {
    attn_delta_kernel<__nv_bfloat16><<<(total + threads - 1) / threads, threads, 0, S(stream)>>>(
        reinterpret_cast<const __nv_bfloat16*>(grad_o), reinterpret_cast<const __nv_bfloat16*>(o), delta, batch,
        rows, m_pad, heads, head_dim, scale);
  } else {
    attn_delta_kernel<float><<<(total + threads - 1) / threads, threads, 0, S(stream)>>>(
        reinterpret_cast<const float*>(grad_o), reinterpret_cast<const float*>(o), delta, batch, rows, m_pad, heads,
        head_dim, scale);
  }
  return check_launch("attn_delta");
}

// Shared launcher of the multi-source backward.  dK|dV of key segment g go to
// seg_tab[g] (peer memory allowed) when seg_tab != null, else to
// grad_k + g*B*seg_len*ld_dkv; dV sits dv_off elements after dK in either case.
static int attn_bwd_launch(const void* k, const void* v, long ld_kv, const lss_bwd_source* srcs, int nsrc,
                           float* grad_k, long dv_off, float* const* seg_tab, int peer, long ld_dkv, int batch,
                           int workers, int seg_len, int heads, int head_dim, int causal, const lss_dropout* dropout,
                           void* stream) {
  int rc = attn_check(LSS_BF16, batch, 1, workers, seg_len, heads, head_dim);
  if (rc) return rc;
  if (!k || !v || !srcs || (!grad_k && !seg_tab)) return fail(LSS_ERR_ARG, "attn_bwd_ex: null pointer");
  if (nsrc < 1 || nsrc > ATB_MAX_SRC) return fail(LSS_ERR_ARG, "attn_bwd_ex: %d sources (1..%d)", nsrc, ATB_MAX_SRC);
  const int E = heads * head_dim;
  if (ld_kv < E || ld_dkv < E) return fail(LSS_ERR_SHAPE, "attn_bwd_ex: row strides smaller than embed");
  if (dv_off % 4 || (dv_off < E && dv_off > -E)) return fail(LSS_ERR_SHAPE, "attn_bwd_ex: dK/dV column blocks overlap");
  if (!aligned16(k) || !aligned16(v) || ld_kv % 8 || ld_dkv % 4)
    return fail(LSS_ERR_UNSUPPORTED, "attn_bwd_ex: 16B alignment");
  if (seg_tab) {
    if (workers > ATB_MAX_SEG) return fail(LSS_ERR_UNSUPPORTED, "attn_bwd_p2p: %d workers (max %d)", workers, ATB_MAX_SEG);
    for (int g = 0; g < workers; ++g)
      if (!seg_tab[g] || !aligned16(seg_tab[g])) return fail(LSS_ERR_ARG, "attn_bwd_p2p: segment %d destination", g);
  } else if (!aligned16(grad_k)) {
    return fail(LSS_ERR_UNSUPPORTED, "attn_bwd_ex: 16B alignment");
  }
  const float scale = 1.0f / sqrtf((float)head_dim);
  AttnBwdParams p;
  memset(&p, 0, sizeof(p));
  BwdMaps maps;
  memset(&maps, 0, sizeof(maps));
  for (int i = 0; i < nsrc; ++i) {
    const lss_bwd_source& sr = srcs[i];
    const bool fixed = sr.grad_q_fixed != nullptr;
    if (fixed != (srcs[0].grad_q_fixed != nullptr))
      return fail(LSS_ERR_ARG, "source %d: fixed-point dQ for all sources or none", i);
    if (!sr.q || !sr.grad_o || (!sr.grad_q && !fixed) || !sr.lse2 || !sr.delta)
      return fail(LSS_ERR_ARG, "source %d: null", i);
    if (fixed && !aligned16(sr.grad_q_fixed)) return fail(LSS_ERR_UNSUPPORTED, "source %d: 16B alignment", i);
    if (sr.row0 < 0 || sr.rows <= 0 || sr.row0 + sr.rows > sr.m_src || sr.row0 % ATT_BM ||
        (sr.rows % ATT_BM && sr.row0 + sr.rows != sr.m_src))
      return fail(LSS_ERR_SHAPE, "source %d: rows [%d,%d) of %d must be 128-row aligned", i, sr.row0,
                  sr.row0 + sr.rows, sr.m_src);
    if (sr.g_begin < 0 || sr.g_end > workers || sr.g_begin >= sr.g_end)
      return fail(LSS_ERR_SHAPE, "source %d: bad segment range", i);
    if (sr.pitch < lss_rows_pad(sr.m_src)) return fail(LSS_ERR_SHAPE, "source %d: lse pitch", i);
    if (!aligned16(sr.q) || !aligned16(sr.grad_o) || (!fixed && !aligned16(sr.grad_q)))
      return fail(LSS_ERR_UNSUPPORTED, "source %d: 16B alignment", i);
    if ((rc = map_rows(&maps.q[i], sr.q, E, E, sr.m_src, batch, 1, 3))) return rc;
    if ((rc = map_rows(&maps.dO[i], sr.grad_o, E, E, sr.m_src, batch, 1, 3))) return rc;
    uint64_t dims[3] = {(uint64_t)E, (uint64_t)sr.m_src, (uint64_t)batch};
    uint64_t str[2] = {(uint64_t)E, (uint64_t)sr.m_src * E};
    uint32_t box[3] = {32, 128, 1};
    if (!fixed && (rc = make_map(&maps.dq[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 3, sr.grad_q, dims, str, box,
                                 CU_TENSOR_MAP_SWIZZLE_128B)))
      return rc;
    p.src[i].row0 = sr.row0;
    p.src[i].rows = sr.rows;
    p.src[i].pos0 = sr.pos0;
    p.src[i].g_begin = sr.g_begin;
    p.src[i].g_end = sr.g_end;
    p.src[i].lse2 = sr.lse2;
    p.src[i].delta = sr.delta;
    p.src[i].pitch = sr.pitch;
    p.src[i].m_src = sr.m_src;
    p.src[i].dq = sr.grad_q;
    p.src[i].dq_fixed = sr.grad_q_fixed;
    p.src[i].ready = sr.ready;
    p.src[i].ready_seq = sr.ready_seq;
  }
  CUtensorMap mk, mv;
  if ((rc = map_rows(&mk, k, E, ld_kv, seg_len, batch, workers, 4))) return rc;
  if ((rc = map_rows(&mv, v, E, ld_kv, seg_len, batch, workers, 4))) return rc;
  p.B = batch; p.G = workers; p.seg_len = seg_len; p.H = heads; p.nsrc = nsrc; p.causal = causal;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.scale = scale;
  p.dkv = grad_k; p.seg_stride = (long)batch * seg_len * ld_dkv; p.dv_off = dv_off; p.ld_dkv = ld_dkv;
  p.peer = peer;
  const bool drop = dropout && dropout->active;
  p.drop_site = drop ? dropout->site_key : 0;
  p.drop_thresh = drop ? dropout->thresh : 0;
  p.drop_scale = drop ? dropout->scale : 1.f;
  if (seg_tab)
    for (int g = 0; g < workers; ++g) p.seg_tab[g] = seg_tab[g];
  if (drop) {
    if ((rc = set_smem(attn_bwd_tc_kernel<true>, ATB_SMEM))) return rc;
  } else if ((rc = set_smem(attn_bwd_tc_kernel<false>, ATB_SMEM))) {
    return rc;
  }
  const int tps = (seg_len + ATT_BN - 1) / ATT_BN;
  // fused reduce-scatter: only the key segments some source reads get a CTA (the
  // owners sum just their writers' slots, lss_sum_slots_mask); the local layout
  // (NCCL reduce-scatter input) is fully written, zeros included
  int g_lo = 0, g_hi = workers;
  if (seg_tab) {
    g_lo = workers;
    g_hi = 0;
    for (int i = 0; i < nsrc; ++i) {
      g_lo = std::min(g_lo, srcs[i].g_begin);
      g_hi = std::max(g_hi, srcs[i].g_end);
    }
  }
  p.g_lo = g_lo;
  dim3 grid((g_hi - g_lo) * tps, heads, batch);
  if (drop)
    attn_bwd_tc_kernel<true><<<grid, ATB_THREADS, ATB_SMEM, S(stream)>>>(mk, mv, maps, p);
  else
    attn_bwd_tc_kernel<false><<<grid, ATB_THREADS, ATB_SMEM, S(stream)>>>(mk, mv, maps, p);
  return check_launch("attn_bwd_tc");
}

int lss_attn_bwd_ex(int dtype, const void* k, const void* v, long ld_kv, const lss_bwd_source* srcs, int nsrc,
                    float* grad_k, float* grad_v, long ld_dkv, int batch, int workers, int seg_len, int heads,
                    int head_dim, int causal, const lss_dropout* dropout, void* stream) {
  if (dtype != LSS_BF16) return fail(LSS_ERR_UNSUPPORTED, "attn_bwd_ex: bf16 only");
  if (!grad_k || !grad_v || !aligned16(grad_v)) return fail(LSS_ERR_ARG, "attn_bwd_ex: dK/dV buffers");
  return attn_bwd_launch(k, v, ld_kv, srcs, nsrc, grad_k, (long)(grad_v - grad_k), nullptr, 0, ld_dkv, batch, workers,
                         seg_len, heads, head_dim, causal, dropout, stream);
}

int lss_attn_bwd_p2p(int dtype, const void* k, const void* v, long ld_kv, const lss_bwd_source* srcs, int nsrc,
                     float* const* seg_dst, int peer, long ld_dkv, int batch, int workers, int seg_len, int heads,
                     int head_dim, int causal, const lss_dropout* dropout, void* stream) {
  if (dtype != LSS_BF16) return fail(LSS_ERR_UNSUPPORTED, "attn_bwd_p2p: bf16 only");
  if (!seg_dst) return fail(LSS_ERR_ARG, "attn_bwd_p2p: null segment table");
  return attn_bwd_launch(k, v, ld_kv, srcs, nsrc, nullptr, heads * head_dim, seg_dst, peer, ld_dkv, batch, workers,
                         seg_len, heads, head_dim, causal, dropout, stream);
}

int lss_sum_slots(float* dst, const float* src, int nslots, long slot_elems, long n, void* stream) {
  if (nslots < 1 || nslots > 32) return fail(LSS_ERR_SHAPE, "sum_slots: %d slots (1..32)", nslots);
  return lss_sum_slots_mask(dst, src, nslots, nslots == 32 ? 0xFFFFFFFFu : ((1u << nslots) - 1u), slot_elems, n,
                            stream);
}

int lss_sum_slots_mask(float* dst, const float* src, int nslots, unsigned int mask, long slot_elems, long n,
                       void* stream) {
  if (!dst || !src) return fail(LSS_ERR_ARG, "sum_slots: null pointer");
  if (nslots > 32) return fail(LSS_ERR_SHAPE, "sum_slots: %d slots (max 32)", nslots);
  if (nslots < 1 || n < 0 || n > slot_elems || n % 4 || slot_elems % 4 || !aligned16(dst) || !aligned16(src))
    return fail(LSS_ERR_SHAPE, "sum_slots: %d slots of %ld (n %ld) must be float4 aligned", nslots, slot_elems, n);
  if (n == 0) return LSS_OK;
  const int threads = 256;
  const long n4 = n / 4;
  const int blocks = (int)std::min<long>((n4 + threads - 1) / threads, (long)num_sms() * 8);
  sum_slots_kernel<<<blocks, threads, 0, S(stream)>>>(reinterpret_cast<float4*>(dst),
                                                       reinterpret_cast<const float4*>(src), nslots, mask,
                                                       slot_elems / 4, n4);
  return check_launch("sum_slots");
}

int lss_sgd_update(float* params, const float* grads, long n, float lr, void* stream) {
  if (!params || !grads) return fail(LSS_ERR_ARG, "sgd_update: null pointer");
  if (n <= 0) return n == 0 ? LSS_OK : fail(LSS_ERR_SHAPE, "sgd_update: n %ld", n);
  const int threads = 256;
  const int blocks = (int)std::min<long>((n + threads - 1) / threads, (long)num_sms() * 8);
  sgd_update_kernel<<<blocks, threads, 0, S(stream)>>>(params, grads, n, lr);
  return check_launch("sgd_update");
}

int lss_adam_update(float* params, const float* grads, float* m, float* v, long n, float lr, float beta1,
                    float beta2, float eps, int step, void* stream) {
  if (!params || !grads || !m || !v) return fail(LSS_ERR_ARG, "adam_update: null pointer");
  if (step < 1) return fail(LSS_ERR_ARG, "adam_update: step %d (1-based)", step);
  if (n <= 0) return n == 0 ? LSS_OK : fail(LSS_ERR_SHAPE, "adam_update: n %ld", n);
  const float inv_bc1 = (float)(1.0 / (1.0 - std::pow((double)beta1, step)));
  const float inv_bc2 = (float)(1.0 / (1.0 - std::pow((double)beta2, step)));
  const int threads = 256;
  const int blocks = (int)std::min<long>((n + threads - 1) / threads, (long)num_sms() * 8);
  adam_update_kernel<<<blocks, threads, 0, S(stream)>>>(params, grads, m, v, n, lr, beta1, beta2, eps, inv_bc1,
                                                        inv_bc2);
  return check_launch("adam_update");
}

int lss_embed_fwd(const int* tokens, const float* token_table, const float* pos_table, float* x, int batch,
                  int rows, int embed, void* stream) {
  if (!tokens || !token_table || !pos_table || !x) return fail(LSS_ERR_ARG, "embed_fwd: null pointer");
  if (batch <= 0 || rows <= 0 || embed <= 0 || embed % 4) return fail(LSS_ERR_SHAPE, "embed_fwd: shape");
  if (!aligned16(token_table) || !aligned16(pos_table) || !aligned16(x))
    return fail(LSS_ERR_UNSUPPORTED, "embed_fwd: 16B alignment");
  const long n = (long)batch * rows;
  embed_fwd_kernel<<<(unsigned)((n + 7) / 8), 256, 0, S(stream)>>>(tokens, token_table, pos_table, x, n, rows, embed);
  return check_launch("embed_fwd");
}

int lss_embed_bwd(const int* tokens, const float* grad_x, float* grad_token_table, float* grad_pos, int batch,
                  int rows, int embed, float alpha_token, float alpha_pos, void* stream) {
  if (!tokens || !grad_x || !grad_token_table || !grad_pos) return fail(LSS_ERR_ARG, "embed_bwd: null pointer");
  if (batch <= 0 || rows <= 0 || embed <= 0) return fail(LSS_ERR_SHAPE, "embed_bwd: shape");
  embed_bwd_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, S(stream)>>>(tokens, grad_x, grad_token_table, grad_pos,
                                                                      batch, rows, embed, alpha_token, alpha_pos);
  return check_launch("embed_bwd");
}

int lss_cross_entropy(const float* logits, long ld, const int* targets, long n, int vocab, float scale,
                      float* loss_rows, float* grad, long ld_grad, void* stream) {
  if (!logits || !targets || !loss_rows) return fail(LSS_ERR_ARG, "cross_entropy: null pointer");
  if (n < 0 || vocab <= 0 || ld < vocab || (grad && ld_grad < vocab)) return fail(LSS_ERR_SHAPE, "cross_entropy: shape");
  if (n == 0) return LSS_OK;
  cross_entropy_kernel<<<(unsigned)n, 256, 0, S(stream)>>>(logits, ld, targets, vocab, scale, loss_rows, grad, ld_grad);
  return check_launch("cross_entropy");
}

int lss_dropout_rows(int dtype, const void* x, long ldx, void* out, long ldo, const float* residual, long ld_res,
                     long rows, int cols, int rows_per_sample, long offset, unsigned long long site_key,
                     unsigned long long thresh, float scale, void* stream) {
  if (!x || !out) return fail(LSS_ERR_ARG, "dropout_rows: null pointer");
  if (rows < 0 || cols <= 0 || rows_per_sample <= 0 || ldx < cols || ldo < cols || (residual && ld_res < cols))
    return fail(LSS_ERR_SHAPE, "dropout_rows: shape");
  if (rows == 0) return LSS_OK;
  dim3 grid((unsigned)std::min(8, (cols + 255) / 256), (unsigned)std::min(rows, 65535L));
  if (dtype == LSS_BF16)
    dropout_rows_kernel<__nv_bfloat16><<<grid, 256, 0, S(stream)>>>(
        reinterpret_cast<const __nv_bfloat16*>(x), ldx, reinterpret_cast<__nv_bfloat16*>(out), ldo, residual, ld_res,
        rows, cols, rows_per_sample, offset, site_key, thresh, scale);
  else
    dropout_rows_kernel<float><<<grid, 256, 0, S(stream)>>>(reinterpret_cast<const float*>(x), ldx,
                                                           reinterpret_cast<float*>(out), ldo, residual, ld_res, rows,
                                                           cols, rows_per_sample, offset, site_key, thresh, scale);
  return check_launch("dropout_rows");
}

// ------------------------------------------------------------------ peer memory (CUDA IPC)
int lss_copy_d2d(void* dst, const void* src, long bytes, void* stream) {
  if (!dst || !src || bytes < 0) return fail(LSS_ERR_ARG, "copy_d2d: arguments");
  if (bytes == 0) return LSS_OK;
  cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, S(stream));
  if (e != cudaSuccess) return fail(LSS_ERR_CUDA, "copy_d2d: %s", cudaGetErrorString(e));
  return LSS_OK;
}

using PFN_getAddressRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

int lss_ipc_export(const void* dev_ptr, unsigned char* handle, long* offset) {
  if (!dev_ptr || !handle || !offset) return fail(LSS_ERR_ARG, "ipc_export: null pointer");
  static PFN_getAddressRange range_fn = nullptr;
  if (!range_fn) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fp)
      return fail(LSS_ERR_CUDA, "cuMemGetAddressRange unavailable");
    range_fn = reinterpret_cast<PFN_getAddressRange>(fp);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(LSS_ERR_CUDA, "ipc_export: not a device allocation");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail(LSS_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  memcpy(handle, &h, sizeof(h));
  *offset = (long)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return LSS_OK;
}

}  // extern "C"

// A peer allocation may back several exported buffers (the caching allocator
// sub-allocates segments) but can be opened only once per process: mappings are
// shared and reference-counted by handle.
struct IpcMapping {
  void* base;
  int refs;
};
static std::mutex g_ipc_mu;
static std::map<std::string, IpcMapping> g_ipc_maps;

extern "C" {

int lss_ipc_import(const unsigned char* handle, long offset, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(LSS_ERR_ARG, "ipc_import: null pointer");
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  const std::string key(reinterpret_cast<const char*>(handle), sizeof(cudaIpcMemHandle_t));
  auto it = g_ipc_maps.find(key);
  if (it == g_ipc_maps.end()) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(LSS_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    it = g_ipc_maps.emplace(key, IpcMapping{base, 0}).first;
  }
  it->second.refs++;
  *dev_ptr = static_cast<char*>(it->second.base) + offset;
  return LSS_OK;
}

int lss_ipc_close(void* dev_ptr, long offset) {
  if (!dev_ptr) return fail(LSS_ERR_ARG, "ipc_close: null pointer");
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  void* base = static_cast<char*>(dev_ptr) - offset;
  for (auto it = g_ipc_maps.begin(); it != g_ipc_maps.end(); ++it) {
    if (it->second.base != base) continue;
    if (--it->second.refs > 0) return LSS_OK;
    g_ipc_maps.erase(it);
    cudaError_t e = cudaIpcCloseMemHandle(base);
    if (e != cudaSuccess) return fail(LSS_ERR_CUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return LSS_OK;
  }
  return fail(LSS_ERR_ARG, "ipc_close: address was not imported");
}

// Stream memory operations (executed by the GPU front-end, no SM): cross-process
// signals through IPC-mapped flag words.
typedef CUresult (*PFN_streamValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_streamValue32 stream_value_fn(const char* name) {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fp, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<PFN_streamValue32>(fp);
}

int lss_stream_signal(unsigned int* flag, unsigned int value, void* stream) {
  static PFN_streamValue32 fn = stream_value_fn("cuStreamWriteValue32");
  if (!flag) return fail(LSS_ERR_ARG, "stream_signal: null flag");
  if (!fn) return fail(LSS_ERR_UNSUPPORTED, "cuStreamWriteValue32 unavailable");
  // default flags: a memory fence orders every prior write of the stream before the flag
  CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value, 0);
  if (r != CUDA_SUCCESS) return fail(LSS_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
  return LSS_OK;
}

int lss_stream_wait(const unsigned int* flag, unsigned int value, void* stream) {
  static PFN_streamValue32 fn = stream_value_fn("cuStreamWaitValue32");
  if (!flag) return fail(LSS_ERR_ARG, "stream_wait: null flag");
  if (!fn) return fail(LSS_ERR_UNSUPPORTED, "cuStreamWaitValue32 unavailable");
  // (int32)(*flag - value) >= 0: wrap-safe monotonic sequence numbers
  CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                  CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(LSS_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
  return LSS_OK;
}

// Bounded stream wait: one thread spins (system-scope acquire loads, nanosleep) until
// every flag word except `skip` reaches `value`, the wait deadline passes or the host
// aborts -- the cuStreamWaitValue32 wait cannot time out or be released.
__global__ void wait_flags_kernel(const unsigned int* flags, int count, int skip, unsigned int value) {
  for (int i = 0; i < count; ++i)
    if (i != skip && !wait_flag_geq(flags + i, value)) break;
}

int lss_stream_wait_bounded(const unsigned int* flags, int count, int skip, unsigned int value, void* stream) {
  if (!flags || count < 1) return fail(LSS_ERR_ARG, "stream_wait_bounded: no flags");
  wait_flags_kernel<<<1, 32, 0, S(stream)>>>(flags, count, skip, value);
  return check_launch("stream_wait_bounded");
}

// Guarded front-end wait: the stream waits in the GPU front-end (cuStreamWaitValue32, no
// SM, released the moment the flag lands), and a one-warp guard kernel on a private
// high-priority stream watches the same flags: past the deadline, or on a host abort,
// it raises the status word and writes the flags itself, so the parked stream drains.
__global__ void guard_flags_kernel(unsigned int* flags, int count, int skip, unsigned int value) {
  bool ok = true;
  for (int i = 0; i < count && ok; ++i)
    if (i != skip) ok = wait_flag_geq(flags + i, value);
  if (!ok && threadIdx.x == 0)
    for (int i = 0; i < count; ++i)
      if (i != skip)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags + i), "r"(value + 0x40000000u) : "memory");
}

int lss_stream_wait_guarded(unsigned int* flags, int count, int skip, unsigned int value, void* stream) {
  if (!flags || count < 1) return fail(LSS_ERR_ARG, "stream_wait_guarded: no flags");
  static PFN_streamValue32 fn = stream_value_fn("cuStreamWaitValue32");
  if (!fn) return fail(LSS_ERR_UNSUPPORTED, "cuStreamWaitValue32 unavailable");
  static std::mutex mu;
  static std::map<int, cudaStream_t> guards;  // one high-priority guard stream per device
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t gs;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = guards.find(dev);
    if (it == guards.end()) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      if (cudaStreamCreateWithPriority(&gs, cudaStreamNonBlocking, hi) != cudaSuccess)
        return fail(LSS_ERR_CUDA, "stream_wait_guarded: guard stream creation failed");
      guards[dev] = gs;
    } else {
      gs = it->second;
    }
  }
  // the guard is launched BEFORE the waits: streams share the front-end's hardware
  // queues, and a guard queued behind its own parked wait could never run
  guard_flags_kernel<<<1, 32, 0, gs>>>(flags, count, skip, value);
  int rc = check_launch("stream_wait_guarded");
  if (rc) return rc;
  for (int i = 0; i < count; ++i) {
    if (i == skip) continue;
    CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flags + i), value,
                    CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return fail(LSS_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
  }
  return LSS_OK;
}

int lss_peer_access(int device, int peer) {
  if (device == peer) return 1;  // two processes on one GPU: CUDA IPC maps the memory directly
  int ok = 0;
  if (cudaDeviceCanAccessPeer(&ok, device, peer) != cudaSuccess) return 0;
  return ok;
}

int lss_attn_bwd(int dtype, const void* q, const void* k, const void* v, long ld_kv, const void* o,
                 const void* grad_o, const float* lse2, float* delta_ws, float* grad_q, float* grad_k,
                 float* grad_v, long ld_dkv, int batch, int rows, int workers, int seg_len, int heads,
                 int head_dim, long offset, int causal, void* stream) {
  int rc = attn_check(dtype, batch, rows, workers, seg_len, heads, head_dim);
  if (rc) return rc;
  if (!q || !k || !v || !o || !grad_o || !lse2 || !delta_ws || !grad_q || !grad_k || !grad_v)
    return fail(LSS_ERR_ARG, "attn_bwd: null pointer");
  const int E = heads * head_dim;
  if (ld_kv < E || ld_dkv < E) return fail(LSS_ERR_SHAPE, "attn_bwd: row strides smaller than embed");
  const int m_pad = (int)lss_rows_pad(rows);
  const float scale = 1.0f / sqrtf((float)head_dim);
  if ((rc = lss_attn_delta(dtype, o, grad_o, delta_ws, batch, rows, heads, head_dim, dtype == LSS_BF16, stream)))
    return rc;
  if (dtype == LSS_F32) {
    const float* qf = reinterpret_cast<const float*>(q);
    const float* kf = reinterpret_cast<const float*>(k);
    const float* vf = reinterpret_cast<const float*>(v);
    const float* gof = reinterpret_cast<const float*>(grad_o);
    dim3 g1((rows + 3) / 4, heads, batch);
    attn_bwd_dq_f32_kernel<<<g1, 128, 0, S(stream)>>>(qf, kf, vf, ld_kv, gof, lse2, delta_ws, grad_q, batch, rows,
                                                     m_pad, workers, seg_len, heads, head_dim, offset, causal, scale);
    if ((rc = check_launch("attn_bwd_dq_f32"))) return rc;
    const long t = (long)workers * seg_len;
    dim3 g2((t + 3) / 4, heads, batch);
    attn_bwd_dkv_f32_kernel<<<g2, 128, 0, S(stream)>>>(qf, kf, vf, ld_kv, gof, lse2, delta_ws, grad_k, grad_v,
                                                      ld_dkv, batch, rows, m_pad, workers, seg_len, heads, head_dim,
                                                      offset, causal, scale);
    return check_launch("attn_bwd_dkv_f32");
  }
  if (!aligned16(grad_q)) return fail(LSS_ERR_UNSUPPORTED, "attn_bwd: 16B alignment");
  cudaError_t e = cudaMemsetAsync(grad_q, 0, sizeof(float) * (size_t)batch * rows * E, S(stream));
  if (e != cudaSuccess) return fail(LSS_ERR_CUDA, "attn_bwd memset: %s", cudaGetErrorString(e));
  lss_bwd_source src;
  src.q = q; src.grad_o = grad_o; src.grad_q = grad_q; src.m_src = rows; src.row0 = 0; src.rows = rows;
  src.pos0 = offset; src.g_begin = 0; src.g_end = workers; src.lse2 = lse2; src.delta = delta_ws; src.pitch = m_pad;
  src.ready = nullptr; src.ready_seq = 0; src.grad_q_fixed = nullptr;
  return lss_attn_bwd_ex(dtype, k, v, ld_kv, &src, 1, grad_k, grad_v, ld_dkv, batch, workers, seg_len, heads,
                         head_dim, causal, nullptr, stream);
}

int lss_attn_merge(const void* o_a, const float* lse_a, const void* o_b, const float* lse_b, void* o_out,
                   float* lse_out, int batch, int rows, int heads, long o_bstride, int lse_pitch, void* stream) {
  if (!o_a || !lse_a || !o_b || !lse_b || !o_out || !lse_out) return fail(LSS_ERR_ARG, "attn_merge: null pointer");
  if (heads <= 0) return fail(LSS_ERR_SHAPE, "attn_merge: heads");
  if (rows <= 0) return LSS_OK;
  const long warps = (long)batch * rows;
  attn_merge_kernel<<<(warps * 32 + 255) / 256, 256, 0, S(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(o_a), lse_a, reinterpret_cast<const __nv_bfloat16*>(o_b), lse_b,
      reinterpret_cast<__nv_bfloat16*>(o_out), lse_out, batch, rows, heads, o_bstride, lse_pitch);
  return check_launch("attn_merge");
}

// Diagnostic: the GPU's global nanosecond timer, stream-ordered (cross-rank timelines).
__global__ void timestamp_kernel(unsigned long long* dst) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *dst = t;
}

int lss_timestamp(unsigned long long* dst, void* stream) {
  if (!dst) return fail(LSS_ERR_ARG, "timestamp: null pointer");
  timestamp_kernel<<<1, 1, 0, S(stream)>>>(dst);
  return check_launch("timestamp");
}

// ---------------------------------------------------------------- runtime status / failure semantics

namespace {
unsigned int* g_status_host = nullptr;  // mapped pinned host words, see common.cuh
std::mutex g_status_mu;

int status_words() {
  std::lock_guard<std::mutex> lock(g_status_mu);
  if (g_status_host) return LSS_OK;
  void* p = nullptr;
  cudaError_t e = cudaHostAlloc(&p, 64, cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) return fail(LSS_ERR_CUDA, "cudaHostAlloc(status): %s", cudaGetErrorString(e));
  memset(p, 0, 64);
  g_status_host = static_cast<unsigned int*>(p);
  return LSS_OK;
}
}  // namespace

__global__ void check_finite_f32_kernel(const float4* x, long n4) {
  bool bad = false;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    const float4 v = x[i];
    bad |= nonfinite(v.x) | nonfinite(v.y) | nonfinite(v.z) | nonfinite(v.w);
  }
  report_nonfinite(bad);
}
__global__ void check_finite_bf16_kernel(const uint4* x, long n8) {
  bool bad = false;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n8; i += (long)gridDim.x * blockDim.x) {
    const uint4 v = x[i];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)  // bf16 NaN / Inf: exponent bits all ones
      bad |= ((w[j] & 0x7F80u) == 0x7F80u) | ((w[j] & 0x7F800000u) == 0x7F800000u);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) status_raise(1);
}

int lss_runtime_config(unsigned long long wait_timeout_ns, int flags) {
  const int numerics_check = (flags & LSS_RT_NUMERICS) ? 1 : 0;
  g_deterministic = (flags & LSS_RT_DETERMINISTIC) ? 1 : 0;
  int rc = status_words();
  if (rc) return rc;
  unsigned int* dev_words = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev_words), g_status_host, 0);
  if (e != cudaSuccess) return fail(LSS_ERR_CUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e));
  if (cudaMemcpyToSymbol(g_status_word, &dev_words, sizeof(dev_words)) != cudaSuccess ||
      cudaMemcpyToSymbol(g_wait_timeout_ns, &wait_timeout_ns, sizeof(wait_timeout_ns)) != cudaSuccess ||
      cudaMemcpyToSymbol(g_numerics_check, &numerics_check, sizeof(numerics_check)) != cudaSuccess)
    return fail(LSS_ERR_CUDA, "runtime_config: cudaMemcpyToSymbol failed");
  return LSS_OK;
}

int lss_status(unsigned int* out, int clear) {
  if (!out) return fail(LSS_ERR_ARG, "status: null pointer");
  int rc = status_words();
  if (rc) return rc;
  volatile unsigned int* w = g_status_host;
  out[0] = w[0];
  out[1] = w[1];
  if (clear) {
    w[0] = 0;
    w[1] = 0;
  }
  return LSS_OK;
}

int lss_check_finite(const void* x, long n, int dtype, void* stream) {
  if (!x) return fail(LSS_ERR_ARG, "check_finite: null pointer");
  if (n <= 0) return LSS_OK;
  const int per = dtype == LSS_BF16 ? 8 : 4;
  if (n % per || !aligned16(x)) return fail(LSS_ERR_UNSUPPORTED, "check_finite: %ld elements not 16-byte vectors", n);
  const long vec = n / per;
  const int threads = 256;
  const long blocks = std::min<long>((vec + threads - 1) / threads, 4L * num_sms());
  if (dtype == LSS_BF16)
    check_finite_bf16_kernel<<<blocks, threads, 0, S(stream)>>>(reinterpret_cast<const uint4*>(x), vec);
  else
    check_finite_f32_kernel<<<blocks, threads, 0, S(stream)>>>(reinterpret_cast<const float4*>(x), vec);
  return check_launch("check_finite");
}

int lss_abort_waits(int on) {
  int rc = status_words();
  if (rc) return rc;
  reinterpret_cast<volatile unsigned int*>(g_status_host)[2] = on ? 1u : 0u;
  return LSS_OK;
}

int lss_fixed_to_f32(float* dst, const long long* src, long n, int accumulate, void* stream) {
  if (!dst || !src) return fail(LSS_ERR_ARG, "fixed_to_f32: null pointer");
  if (n <= 0) return LSS_OK;
  const int threads = 256;
  const long blocks = std::min<long>((n + threads - 1) / threads, 8L * num_sms());
  fixed_to_f32_kernel<<<blocks, threads, 0, S(stream)>>>(dst, src, n, accumulate);
  return check_launch("fixed_to_f32");
}

int lss_flag_release(unsigned int* flags, long count, unsigned int value) {
  if (!flags) return fail(LSS_ERR_ARG, "flag_release: null pointer");
  // a private non-blocking stream: the caller's streams may be parked in a stream wait
  static cudaStream_t rs = nullptr;
  if (!rs && cudaStreamCreateWithFlags(&rs, cudaStreamNonBlocking) != cudaSuccess)
    return fail(LSS_ERR_CUDA, "flag_release: stream creation failed");
  static PFN_streamValue32 fn = stream_value_fn("cuStreamWriteValue32");
  if (!fn) return fail(LSS_ERR_UNSUPPORTED, "cuStreamWriteValue32 unavailable");
  for (long i = 0; i < count; ++i)
    if (fn(reinterpret_cast<CUstream>(rs), reinterpret_cast<CUdeviceptr>(flags + i), value, 0) != CUDA_SUCCESS)
      return fail(LSS_ERR_CUDA, "flag_release: cuStreamWriteValue32 failed");
  return LSS_OK;
}

int lss_add_f32(float* y, const float* x, long n, void* stream) {
  if (!y || !x) return fail(LSS_ERR_ARG, "add_f32: null pointer");
  if (n <= 0) return LSS_OK;
  const long threads = 256, per = threads * 4;
  add_f32_kernel<<<(n + per - 1) / per, threads, 0, S(stream)>>>(y, x, n);
  return check_launch("add_f32");
}

}  // extern "C"

#ifdef LSS_BWD_TRACE
extern "C" int lss_debug_bwd_trace(long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, g_bwd_trace, sizeof(long long) * 20 * 512) == cudaSuccess ? 0 : 5;
}
#endif

#ifdef LSS_FWD_TRACE
extern "C" int lss_debug_fwd_trace(long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, g_fwd_trace, sizeof(long long) * 8 * 1024) == cudaSuccess ? 0 : 5;
}
#endif
