/*
 * lss.h — C ABI of the B200-native LSS sequence-distributed attention path.
 *
 * Drop-in boundary for the attention half of the reference's transformer layer
 * (reference: /root/reference/pkg/src/seqpar).  Every entry point replaces one
 * numpy function of the reference's hot path; the citation next to each entry
 * names it.  All pointers are DEVICE pointers owned by the caller (no
 * allocation inside the library except cached launch metadata); every call is
 * stream-ordered on `stream` (a cudaStream_t) and never synchronises the host.
 *
 * Layouts (row-major, the reference's (batch, rows, features) convention,
 * model.py:16-19; head h <-> feature columns [h*d, (h+1)*d), model.py:309):
 *   activations  [batch][rows][embed]
 *   packed K/V   [workers][batch][seg_len][2*embed]   K in columns [0,embed),
 *                V in [embed, 2*embed); this is the rank-ordered all-gather of
 *                every rank's [K_r | V_r] (sharded.py:144-154, collectives.py:340)
 *   weights      reference layout [d_in][d_out] (nnops.py:172-177), y = x W + b
 *   lse2         [batch][heads][rows_pad], rows_pad = lss_rows_pad(rows),
 *                base-2 log-sum-exp of each softmax row
 *
 * Return value: LSS_OK (0) or an error code; lss_last_error() describes the
 * last failure of the calling thread.  Error codes map onto the reference's
 * exception taxonomy (errors.py:8-29).
 */
#ifndef LSS_H_
#define LSS_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSS_ABI_VERSION 10

enum lss_status {
  LSS_OK = 0,
  LSS_ERR_SHAPE = 1,        /* errors.ShapeError          (errors.py:8)  */
  LSS_ERR_PARTITION = 2,    /* errors.PartitionError      (errors.py:12) */
  LSS_ERR_DEGENERATE = 3,   /* errors.DegenerateRowError  (errors.py:16) */
  LSS_ERR_NUMERICS = 4,     /* errors.NumericsError       (errors.py:20) */
  LSS_ERR_CUDA = 5,         /* CUDA launch / driver failure              */
  LSS_ERR_UNSUPPORTED = 6,  /* shape outside what the sm_100a kernels do */
  LSS_ERR_ARG = 7           /* null pointer / bad enum                   */
};

enum lss_dtype {
  LSS_BF16 = 0, /* bf16 operands, fp32 accumulation: tcgen05/TMEM/TMA kernels */
  LSS_F32 = 1   /* fp32 check mode: FFMA kernels (<= 1e-4 vs the fp64 oracle) */
};

int lss_abi_version(void);
const char* lss_last_error(void);
/* rows rounded up to the 128-row query tile (size of the lse2 / delta rows) */
long lss_rows_pad(long rows);

/* nnops.layernorm_fwd (nnops.py:199-208) as called by model.norm3 (model.py:248-251).
 * x [rows][embed] fp32 -> y (bf16 or fp32 per y_dtype), mean/rstd [rows] cache. */
int lss_layernorm_fwd(const float* x, const float* gain, const float* bias, void* y, int y_dtype,
                      float* mean, float* rstd, long rows, int embed, float eps, void* stream);

/* nnops.layernorm_bwd (nnops.py:211-227) fused with the residual add of
 * model.layer_bwd (model.py:485-486): grad_x = grad_res + LN'(grad_xh).
 * grad_gain/grad_bias are ACCUMULATED (+= alpha * column sums). grad_res may be null. */
int lss_layernorm_bwd(const float* grad_xh, const float* x, const float* mean, const float* rstd,
                      const float* gain, const float* grad_res, float* grad_x, float* grad_gain,
                      float* grad_bias, float alpha, long rows, int embed, void* stream);

/* Products of nnops.linear_fwd / linear_bwd (nnops.py:180-193):
 *   C[M][N] = act(alpha * A . B^T (+ bias[N]) (+ residual[M][N]))
 * A is [M][K] (a_mn_major=0, row stride lda) or stored [K][M] (a_mn_major=1);
 * B is [N][K] (b_mn_major=0) or stored [K][N] (b_mn_major=1).
 * dtype LSS_BF16: A/B bf16, tcgen05 GEMM; LSS_F32: A/B fp32, FFMA GEMM (fp32 out).
 * Output columns are split into up to 3 segments of seg_width columns, segment
 * s written to out[s] with leading dimension ldo[s] (e.g. Q and packed K|V). */
typedef struct lss_gemm_epilogue {
  void* out[3];
  long ldo[3];
  int seg_width;
  int out_dtype; /* LSS_BF16 or LSS_F32 */
  float alpha;
  const float* bias;     /* [N] fp32 or null */
  const float* residual; /* [M][ld_res] fp32 or null */
  long ld_res;
  /* FFN activation (model.ffn_fwd / ffn_bwd, model.py:371-390; nnops.gelu_fwd /
   * gelu_bwd, nnops.py:235-245):
   *   LSS_ACT_GELU      out = gelu_tanh(v); pre (may be null) receives v, in out's dtype
   *   LSS_ACT_GELU_BWD  out = v * gelu_tanh'(aux[row][col]); aux dtype aux_dtype */
  int act;
  void* pre;
  long ld_pre;
  const void* aux;
  long ld_aux;
  int aux_dtype;
} lss_gemm_epilogue;
enum lss_act { LSS_ACT_NONE = 0, LSS_ACT_GELU = 1, LSS_ACT_GELU_BWD = 2 };

int lss_gemm(int dtype, const void* A, long lda, int a_mn_major, const void* B, long ldb,
             int b_mn_major, int M, int N, int K, const lss_gemm_epilogue* ep, void* stream);

/* Stage the attention weights (model.LayerParams attn_q/k/v/out, model.py:83-94)
 * in the GEMM operand layouts: wqkv_t [3E][E] = [Wq|Wk|Wv]^T, wqkv [E][3E],
 * wo_t [E][E] = Wo^T, wo [E][E], bqkv [3E] = [bq|bk|bv]. */
int lss_stage_weights(int dtype, const float* wq, const float* wk, const float* wv,
                      const float* wo, const float* bq, const float* bk, const float* bv,
                      void* wqkv_t, void* wqkv, void* wo_t, void* wo_n, float* bqkv, int embed,
                      void* stream);

/* Column-concatenate up to 3 fp32 blocks into dst (bf16/fp32, may be null) and
 * ACCUMULATE alpha * column sums into colsum (may be null): bias gradients
 * (nnops.py:192) fused with the operand casts of the backward GEMMs. */
int lss_cat_cast_colsum(int out_dtype, const float* const* srcs, const long* lds, const int* cols,
                        int nsrc, void* dst, long ld_dst, float* colsum, float alpha, long rows,
                        void* stream);

/* Same, where source i (nslots[i] > 1) is the ascending sum of the slots set in
 * masks[i], slot k at srcs[i] + k * slot_strides[i]: the fused reduce-scatter's
 * owner sum (lss_sum_slots_mask) folded into the cast (arrays may be NULL). */
int lss_cat_cast_colsum_ex(int out_dtype, const float* const* srcs, const long* lds, const int* cols,
                           const int* nslots, const unsigned int* masks, const long* slot_strides, int nsrc,
                           void* dst, long ld_dst, float* colsum, float alpha, long rows, void* stream);

/* model.scores_fwd (model.py:280-326): this rank's query rows (global
 * positions offset..offset+rows-1) against the whole sequence, whose keys and
 * values are given as `workers` segments of seg_len rows, row layout
 * [workers][batch][seg_len][ld_kv] (elements).  The packed all-gather buffer
 * [workers][batch][seg_len][2*embed] is k = kv, v = kv + embed, ld_kv = 2*embed;
 * a single (batch, t, embed) tensor is workers = 1, seg_len = t, ld_kv = embed.
 * Causal keep-mask key <= query position (model.py:301-304).  Writes ctx `o`
 * [batch][rows][embed] and lse2. */
int lss_attn_fwd(int dtype, const void* q, const void* k, const void* v, long ld_kv, void* o,
                 float* lse2, int batch, int rows, int workers, int seg_len, int heads,
                 int head_dim, long offset, int causal, void* stream);

/* Attention-probability dropout (model.scores_fwd / scores_bwd, model.py:313-317,
 * 350-352; nnops.keep_mask, nnops.py:124-135): site_key = mix(mix(seed, 2), layer+1),
 * the row key of query (b, h, q_pos) is mix(mix(mix(site_key, b+1), h+1), q_pos) and
 * (q_pos, k_pos) is kept iff (mix(row key, k_pos) >> 11) >= thresh, thresh =
 * ceil(rate * 2^53); kept probabilities are scaled by scale = 1/(1-rate).  Pass
 * null (or active = 0) for no dropout; bf16 path only. */
typedef struct lss_dropout {
  unsigned long long site_key;
  unsigned long long thresh;
  float scale;
  int active;
} lss_dropout;

/* Partial / strided form of lss_attn_fwd: q rows [0, rows) with batch stride
 * q_bstride (elements), attending only key segments [g_begin, g_end); ctx is
 * written normalised with batch stride o_bstride and lse2 with row pitch
 * lse_pitch.  Rows that see no key of the range get ctx = 0, lse2 = -inf.
 * Used by the balanced causal schedule, whose partial results are combined
 * with lss_attn_merge.  (bf16 only for partial ranges.) */
int lss_attn_fwd_ex(int dtype, const void* q, int rows, long q_bstride, const void* k, const void* v,
                    long ld_kv, void* o, long o_bstride, float* lse2, int lse_pitch, int batch,
                    int workers, int seg_len, int heads, int head_dim, long offset, int causal,
                    int g_begin, int g_end, const lss_dropout* dropout, void* stream);

/* Fused all-gather: with seg_ready != NULL, key segment g != own_seg is read only
 * after seg_ready[g] reaches ready_seq (wrap-safe >=) -- the gatherer signals each
 * segment as its copy lands (lss_stream_signal) and the kernel's TMA producer
 * waits per segment, so the transfer overlaps the math tile by tile.  Segments
 * are visited from the highest visible one down (diagonal first, then the
 * nearest remote ones).
 *
 * lss_attn_fwd_ex with the key range split `splits` ways (1..16) inside ONE
 * launch: split s attends key tiles [s*n/S, (s+1)*n/S) of each CTA's n visible
 * tiles; split 0 writes (o, lse2), split s > 0 the caller's scratch slot s-1 at
 * o_part + (s-1)*o_part_stride / lse_part + (s-1)*lse_part_stride (same batch
 * stride and lse pitch as o / lse2), and an N-way log-sum-exp merge folds the
 * slots into (o, lse2) on the same stream.  For launches with few query tiles
 * over a long key range (a rank's remote segments at N >= 4), where one CTA per
 * query-tile pair would leave most of the 148 SMs idle in the last wave.
 * Same result as lss_attn_fwd_ex up to the bf16 rounding of the partials. */
int lss_attn_fwd_split(int dtype, const void* q, int rows, long q_bstride, const void* k, const void* v,
                       long ld_kv, void* o, long o_bstride, float* lse2, int lse_pitch, int batch,
                       int workers, int seg_len, int heads, int head_dim, long offset, int causal,
                       int g_begin, int g_end, const lss_dropout* dropout, int splits, void* o_part,
                       long o_part_stride, float* lse_part, long lse_part_stride,
                       const unsigned int* seg_ready, unsigned int ready_seq, int own_seg, void* stream);

/* log-sum-exp combine of two partial attentions over disjoint key ranges:
 * lse = log2(2^la + 2^lb), ctx = 2^(la-lse) ctx_a + 2^(lb-lse) ctx_b (bf16, head_dim 64).
 * o_out / lse_out may alias o_a / lse_a. */
int lss_attn_merge(const void* o_a, const float* lse_a, const void* o_b, const float* lse_b,
                   void* o_out, float* lse_out, int batch, int rows, int heads, long o_bstride,
                   int lse_pitch, void* stream);

/* delta[b][h][row] = rowsum(grad_o * o) over the head's columns (x 1/sqrt(d) when scaled),
 * the softmax-backward row term of model.scores_bwd (model.py:355); [B][H][lss_rows_pad(rows)]. */
int lss_attn_delta(int dtype, const void* o, const void* grad_o, float* delta, int batch, int rows,
                   int heads, int head_dim, int scaled, void* stream);

/* model.scores_bwd (model.py:329-359).  grad_q [batch][rows][embed] fp32 is
 * overwritten; grad_k / grad_v (fp32, layout [workers][batch][seg_len][ld_dkv])
 * are fully written: this rank's partial dK, dV over the WHOLE sequence (the
 * reduce-scatter input; packed [dK|dV] when grad_v = grad_k + embed, ld = 2E).
 * delta_ws: workspace of batch*heads*lss_rows_pad(rows) floats. */
int lss_attn_bwd(int dtype, const void* q, const void* k, const void* v, long ld_kv, const void* o,
                 const void* grad_o, const float* lse2, float* delta_ws, float* grad_q,
                 float* grad_k, float* grad_v, long ld_dkv, int batch, int rows, int workers,
                 int seg_len, int heads, int head_dim, long offset, int causal, void* stream);

/* One query-row source of the multi-source backward: rows [row0, row0+rows)
 * (128-aligned; the last source may end at m_src) of [batch][m_src][embed]
 * Q / dO (bf16) and dQ (fp32, ACCUMULATED: zero it first) whose row 0 is at
 * global position pos0, attending key segments [g_begin, g_end); lse2 and the
 * scaled delta (lss_attn_delta(..., scaled=1)) are [batch][heads][pitch]. */
typedef struct lss_bwd_source {
  const void* q;
  const void* grad_o;
  float* grad_q;
  int m_src;
  int row0, rows;
  long pos0;
  int g_begin, g_end;
  const float* lse2;
  const float* delta;
  int pitch;
  /* optional (NULL = resident): the source's q / grad_o / lse2 / delta are read only
   * after (int32)(*ready - ready_seq) >= 0 -- a partner pushes them and signals
   * (lss_stream_signal), and the kernel processes the sources before it meanwhile */
  const unsigned int* ready;
  unsigned int ready_seq;
  /* optional (ABI v10, deterministic mode): when non-NULL (for every source of the
   * launch), dQ is accumulated here instead of grad_q -- int64 [batch][m_src][embed],
   * round(dQ * 2^32), added with integer bulk reductions, so the sum over key tiles is
   * bitwise identical whatever order they finish in; zero it first, convert with
   * lss_fixed_to_f32.  grad_q may then be NULL. */
  long long* grad_q_fixed;
} lss_bwd_source;

/* Backward over up to 3 sources in ONE launch: every key tile accumulates dK/dV
 * from all sources, so grad_k / grad_v rows have a single writer (fully written). */
int lss_attn_bwd_ex(int dtype, const void* k, const void* v, long ld_kv, const lss_bwd_source* srcs,
                    int nsrc, float* grad_k, float* grad_v, long ld_dkv, int batch, int workers,
                    int seg_len, int heads, int head_dim, int causal, const lss_dropout* dropout, void* stream);

/* y += x (fp32), used to fold a partner's dQ rows into the owner's. */
int lss_add_f32(float* y, const float* x, long n, void* stream);

/* Cross-process stream signals (stream memory operations: executed by the GPU
 * front-end, no SM, no NCCL kernel).  lss_stream_signal writes `value` to *flag
 * after every prior operation of `stream` (memory fence included); flag may be
 * an IPC-mapped word of a peer GPU.  lss_stream_wait blocks `stream` until
 * (int32)(*flag - value) >= 0 (monotonic sequence numbers).  They replace the
 * reference's point-to-point sends / barriers of the balanced causal schedule
 * (sharded.py:144-154 exchanges) on one NVLink domain. */
int lss_stream_signal(unsigned int* flag, unsigned int value, void* stream);
int lss_stream_wait(const unsigned int* flag, unsigned int value, void* stream);
/* Bounded form (ABI v10, the engine fabric's default): a one-warp kernel on
 * `stream` spins until flags[i] >= value for every i < count except i == skip (-1:
 * none), with the lss_runtime_config deadline and the host abort word
 * (lss_abort_waits) -- a dead peer raises CommTimeout / an abort CommAborted
 * instead of parking the stream forever (collectives.py:200-253). */
int lss_stream_wait_bounded(const unsigned int* flags, int count, int skip, unsigned int value, void* stream);
/* Guarded form: the front-end waits of
 * lss_stream_wait (no SM; released as soon as the flags land) plus a one-warp guard
 * kernel on a private high-priority stream that watches the same flags with the
 * deadline and the abort word, and on failure raises the status word and writes the
 * flags itself so the parked stream drains.  The guard is launched before the waits
 * (streams share the front-end's hardware queues).  Measured 2-3% slower than the
 * spin-kernel form at N=2/4. */
int lss_stream_wait_guarded(unsigned int* flags, int count, int skip, unsigned int value, void* stream);

/* Diagnostic: stream-ordered write of the GPU global timer (ns) to *dst. */
int lss_timestamp(unsigned long long* dst, void* stream);

/* ---- dK|dV reduce-scatter fused into the backward (NVLink / NVSwitch peer memory)
 *
 * Replaces the sharded.backward -> collectives.reduce_scatter pair
 * (sharded.py:192-199, collectives.py:362-372): instead of writing the partial
 * [dK|dV] of every key segment locally and reduce-scattering it, the kernel's
 * epilogue stores segment g's partial into seg_dst[g] — the owner's receive
 * slot for this rank, [batch][seg_len][ld_dkv] fp32 with dK at column h*d and dV
 * at embed + h*d — so the transfer overlaps the attention math tile by tile.
 * Stores leave the SM as whole 256-byte row segments.  peer marks seg_dst as
 * peer memory; ordering comes from kernel completion followed by a device-side
 * barrier, after which the owner sums its writers' slots with lss_sum_slots_mask.  Only key
 * segments [min g_begin, max g_end) of the sources are written (no zero tiles for
 * segments no source reads).  Same sources and numerics as lss_attn_bwd_ex; workers <= 16. */
int lss_attn_bwd_p2p(int dtype, const void* k, const void* v, long ld_kv, const lss_bwd_source* srcs,
                     int nsrc, float* const* seg_dst, int peer, long ld_dkv, int batch, int workers,
                     int seg_len, int heads, int head_dim, int causal, const lss_dropout* dropout,
                     void* stream);

/* Whole-model edges.  tokens / targets are int32.
 * model.embed_fwd (model.py:517-533): x[b][i] = token_table[tokens[b][i]] + pos_table[i]
 * (pos_table = this block's rows).  model.embed_bwd (536-540): grad_pos[i] = alpha_pos *
 * sum_b grad_x[b][i] (written); grad_token_table[id] += alpha_token * grad_x rows
 * (accumulated; the alphas carry the folded gradient scales, sharded.py:207-208).
 * nnops.cross_entropy (nnops.py:274-299) per row of logits [n][ld] (first vocab
 * columns): loss_rows[r] = logsumexp - logit[target]; grad (optional, [n][ld_grad],
 * columns >= vocab zeroed) = (softmax - onehot) * scale (scale = 1/rows of the mean). */
int lss_embed_fwd(const int* tokens, const float* token_table, const float* pos_table, float* x, int batch,
                  int rows, int embed, void* stream);
int lss_embed_bwd(const int* tokens, const float* grad_x, float* grad_token_table, float* grad_pos, int batch,
                  int rows, int embed, float alpha_token, float alpha_pos, void* stream);
int lss_cross_entropy(const float* logits, long ld, const int* targets, long n, int vocab, float scale,
                      float* loss_rows, float* grad, long ld_grad, void* stream);

/* nnops.dropout_fwd / dropout_bwd (nnops.py:143-166) on a (rows, cols) activation
 * whose row r is (sample r / rows_per_sample, position offset + r % rows_per_sample):
 * out = x * keep * scale (+ residual fp32), keep from the site key
 * mix(mix(seed, tag), layer+1) (see lss_dropout).  x / out bf16 or fp32 (dtype). */
int lss_dropout_rows(int dtype, const void* x, long ldx, void* out, long ldo, const float* residual, long ld_res,
                     long rows, int cols, int rows_per_sample, long offset, unsigned long long site_key,
                     unsigned long long thresh, float scale, void* stream);

/* Parameter updates after the gradient all-reduce, over flat fp32 buffers:
 * model.sgd_step (model.py:621-623) p -= lr * g, and optim.adam_step
 * (optim.py:35-53) with bias correction (step is 1-based). */
int lss_sgd_update(float* params, const float* grads, long n, float lr, void* stream);
int lss_adam_update(float* params, const float* grads, float* m, float* v, long n, float lr, float beta1,
                    float beta2, float eps, int step, void* stream);

/* dst[i] = sum_{s < nslots} src[s * slot_elems + i] for i < n (fp32, n % 4 == 0). */
int lss_sum_slots(float* dst, const float* src, int nslots, long slot_elems, long n, void* stream);

/* Same over the slots whose bit is set in mask (ascending; mask 0 -> zeros): the
 * owner's half of the fused reduce-scatter, whose writers are the ranks that
 * attend any key of its segment (lss_attn_bwd_p2p writes only segments
 * [min g_begin, max g_end) of its sources). */
int lss_sum_slots_mask(float* dst, const float* src, int nslots, unsigned int mask, long slot_elems, long n,
                       void* stream);

/* CUDA IPC for the peer buffers above: export a device pointer (any address
 * inside an allocation) as a 64-byte handle + offset; import it in another
 * process of the node (lazy peer access); close an imported pointer. */
#define LSS_IPC_HANDLE_BYTES 64
int lss_ipc_export(const void* dev_ptr, unsigned char* handle, long* offset);
int lss_ipc_import(const unsigned char* handle, long offset, void** dev_ptr);
int lss_ipc_close(void* dev_ptr, long offset);
/* Stream-ordered device-to-device copy on the copy engines (no SMs); src may be a
 * peer's memory imported with lss_ipc_import: the K/V gather pulls each peer's
 * [K_p|V_p] slot this way (replaces collectives.all_gather, collectives.py:325-344). */
int lss_copy_d2d(void* dst, const void* src, long bytes, void* stream);
/* 1 if `device` can load/store `peer`'s memory directly (NVLink / PCIe P2P, or the
 * same device in another process). */
int lss_peer_access(int device, int peer);

/* ---- failure semantics (ABI v9)
 *
 * The reference's communicator never hangs: a rendezvous past its timeout raises
 * CommTimeout and aborts the group (collectives.py:200-253, errors.py:24-29); every
 * matmul / softmax output is checked for NaN / Inf -> NumericsError
 * (tensor.py:79-95, 118, 131).  On B200:
 *  - lss_runtime_config sets, on the caller's current device, the deadline of every
 *    in-kernel cross-GPU wait (fused gather segment flags, pushed backward sources;
 *    0 = unbounded) and the flags: LSS_RT_NUMERICS, the opt-in NaN / Inf check in the
 *    epilogues of the GEMM and attention kernels; LSS_RT_DETERMINISTIC (process-wide,
 *    ABI v10), column sums (lss_cat_cast_colsum*, lss_layernorm_bwd) with one writer
 *    per column in a fixed order instead of atomics -- with the fixed-point dQ of
 *    lss_bwd_source.grad_q_fixed every result is bitwise repeatable run to run
 *    (the reference's ascending-rank folds, collectives.py:5-7).  A wait past its
 *    deadline gives up and raises status word 0; a non-finite output raises word 1.
 *  - lss_status copies the two process-wide status words into out[2] (mapped pinned
 *    host memory: no device synchronisation) and optionally clears them.
 *  - lss_check_finite raises word 1 if any of n fp32 / bf16 elements is NaN / Inf
 *    (n a multiple of 4 / 8, 16-byte aligned): the check for outputs of the other
 *    kernels (LayerNorm, fp32 check mode).
 *  - lss_flag_release writes `value` to `count` flag words from a private
 *    non-blocking stream: a host watchdog releases stream waits (lss_stream_wait)
 *    whose peer is dead, so the caller's streams drain and the host raises CommTimeout. */
int lss_runtime_config(unsigned long long wait_timeout_ns, int flags);
int lss_status(unsigned int* out, int clear);
int lss_check_finite(const void* x, long n, int dtype, void* stream);
int lss_flag_release(unsigned int* flags, long count, unsigned int value);
/* Host-side abort (1) / re-arm (0): every bounded wait (lss_stream_wait_bounded and the
 * in-kernel waits) returns at once while set (Communicator.abort, collectives.py:200-209). */
int lss_abort_waits(int on);
#define LSS_RT_NUMERICS 1
#define LSS_RT_DETERMINISTIC 2
/* dst (=, or += when accumulate) src * 2^-32: the fixed-point dQ of the deterministic mode. */
int lss_fixed_to_f32(float* dst, const long long* src, long n, int accumulate, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LSS_H_ */
