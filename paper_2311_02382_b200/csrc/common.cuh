// Blackwell (sm_100a) PTX helpers shared by the LSS kernels:
// mbarriers, TMA (cp.async.bulk.tensor), tcgen05 (TMEM alloc / mma / ld / st),
// UMMA descriptors.  Raw inline PTX; no CUTLASS/CuTe dependency.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define LSS_DEV __device__ __forceinline__

namespace lss {

// ---------------------------------------------------------------- basics
LSS_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

LSS_DEV uint32_t warp_id() { return __shfl_sync(0xffffffffu, threadIdx.x / 32, 0); }
LSS_DEV uint32_t lane_id() { return threadIdx.x % 32; }

LSS_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- mbarrier
LSS_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
LSS_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
LSS_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
LSS_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
LSS_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
LSS_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ---------------------------------------------------------------- shared memory (32-bit addresses)
LSS_DEV void st_shared_v2(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
LSS_DEV void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
LSS_DEV float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

// ---------------------------------------------------------------- fences
LSS_DEV void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
LSS_DEV void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// System scope: the flag words are written by a peer GPU's stream (NVLink) or by
// this GPU's copy engine after a pull from peer memory.
LSS_DEV uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
LSS_DEV unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------- runtime status
// Two words of mapped pinned host memory shared by every kernel of the process
// (lss_runtime_config / lss_status in include/lss.h): [0] a cross-GPU wait ran past
// its deadline (the host raises CommTimeout, collectives.py:242-252), [1] a kernel
// produced NaN / Inf while the numerics check is on (NumericsError, tensor.py:79-95).
// Plain system-scope stores (no host atomics needed).  Device globals are per device:
// lss_runtime_config sets them on the caller's current device.
__device__ unsigned int* g_status_word = nullptr;
__device__ unsigned long long g_wait_timeout_ns = 0;  // 0: unbounded
__device__ int g_numerics_check = 0;

LSS_DEV void status_raise(int which) {
  unsigned int* w = g_status_word;
  if (w) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(w + which), "r"(1u) : "memory");
}
LSS_DEV bool nonfinite(float x) { return !(fabsf(x) <= 3.402823466e38f); }  // NaN or +-Inf
// warp-aggregated report; every lane of the warp must call it
LSS_DEV void report_nonfinite(bool bad) {
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) status_raise(1);
}

// Word [2] is written by the HOST: a communicator abort (collectives.py:200-209)
// releases every wait at once.
LSS_DEV bool host_aborted() {
  const unsigned int* w = g_status_word;
  unsigned int v = 0;
  if (w) asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(w + 2) : "memory");
  return v != 0;
}

// Spin until the stream-signalled word reaches seq (wrap-safe), then order later
// async-proxy (TMA) reads after it.  Bounded: past g_wait_timeout_ns the wait gives
// up and raises the comm-timeout status word, and a host abort ends it at once (a
// dead or out-of-step peer turns into CommTimeout / CommAborted on the host instead
// of a hung GPU; the results of that step are void).
LSS_DEV bool wait_flag_geq(const uint32_t* p, uint32_t seq) {
  bool ok = true;
  if ((int)(ld_acquire_sys(p) - seq) < 0) {
    const unsigned long long lim = g_wait_timeout_ns, t0 = globaltimer_ns();
    for (uint32_t n = 1;; ++n) {
      __nanosleep(128);
      if ((int)(ld_acquire_sys(p) - seq) >= 0) break;
      // the deadline and the host abort word (a read of mapped host memory) every
      // 256 polls (~50 us): polled every time, hundreds of waiting CTAs flooded the
      // system-memory path and slowed the fused gather
      if ((n & 255) == 0) {
        if (host_aborted()) {
          ok = false;
          break;
        }
        if (lim && globaltimer_ns() - t0 > lim) {
          status_raise(0);
          ok = false;
          break;
        }
      }
    }
  }
  fence_proxy_async_global();
  return ok;
}
LSS_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
LSS_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
LSS_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- TMA
LSS_DEV void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
LSS_DEV void tma_load_2d(const CUtensorMap* m, uint64_t* bar, void* smem, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
LSS_DEV void tma_load_3d(const CUtensorMap* m, uint64_t* bar, void* smem, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
LSS_DEV void tma_load_4d(const CUtensorMap* m, uint64_t* bar, void* smem, int c0, int c1, int c2,
                         int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3)
      : "memory");
}
// bulk (non-tensor) reduce-add of fp32 from shared to global; bytes % 16 == 0
LSS_DEV void bulk_reduce_add_f32(float* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile(
      "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst),
      "r"(smem_u32(ssrc)), "r"(bytes)
      : "memory");
}
// bulk (non-tensor) integer add of int64 (two's complement: .u64 add) from shared to global
LSS_DEV void bulk_reduce_add_u64(long long* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile(
      "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;" ::"l"(gdst),
      "r"(smem_u32(ssrc)), "r"(bytes)
      : "memory");
}
// tensor (TMA) reduce-add from shared to global, 3-D map
LSS_DEV void tma_reduce_add_3d(const CUtensorMap* m, const void* smem, int c0, int c1, int c2) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(m)),
      "r"(smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
LSS_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
LSS_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
LSS_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// ---------------------------------------------------------------- tcgen05: TMEM
// allocation (whole warp), result written to smem
LSS_DEV void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
LSS_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

// SMEM matrix descriptor for tcgen05.mma (SWIZZLE_128B canonical layouts).
//   K-major  : rows of 128B (64 bf16 along K), 8-row atoms at SBO (=1024B when dense)
//   MN-major : rows of 128B (64 bf16 along M/N) indexed by K, 8-row atoms at SBO,
//              64-element M/N chunks at LBO
LSS_DEV uint64_t smem_desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm100)
  d |= (uint64_t)2 << 61;  // layout = SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::f16, bf16 x bf16 -> f32
//  bits: c_format[4,6)=1(F32) a_fmt[7,10)=1(BF16) b_fmt[10,13)=1(BF16)
//        a_major[15] b_major[16] n_dim[17,23)=N>>3 m_dim[24,29)=M>>4
__host__ __device__ constexpr uint32_t idesc_bf16_f32(uint32_t M, uint32_t N, uint32_t a_mn_major,
                                                      uint32_t b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn_major << 15) | (b_mn_major << 16) |
         ((N >> 3) << 17) | ((M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]^T
LSS_DEV void mma_bf16_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// D[tmem] (+)= A[tmem] * B[smem]^T   (A K-major in TMEM: lane = row, 2 bf16 per column)
LSS_DEV void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive on an mbarrier when all previously issued tcgen05 ops of this thread complete
LSS_DEV void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// TMEM <-> registers.  tcgen05.ld/st are asynchronous with respect to the
// register file: the compiler must not touch the destination (ld) or source (st)
// registers until tcgen05.wait::{ld,st}.  Issuing the wait inside the SAME asm
// statement makes the registers' def/use points exact (a separate wait lets
// ptxas spill or copy the registers while the load is still in flight).
#define LSS_R8(b) "=r"(r[b + 0]), "=r"(r[b + 1]), "=r"(r[b + 2]), "=r"(r[b + 3]), \
                  "=r"(r[b + 4]), "=r"(r[b + 5]), "=r"(r[b + 6]), "=r"(r[b + 7])
#define LSS_W8(b) "r"(r[b + 0]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3]), \
                  "r"(r[b + 4]), "r"(r[b + 5]), "r"(r[b + 6]), "r"(r[b + 7])

// 32 lanes x 32 bits, 32 consecutive columns per thread, then wait
LSS_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : LSS_R8(0), LSS_R8(8), LSS_R8(16), LSS_R8(24)
      : "r"(taddr)
      : "memory");
}
// 64 consecutive columns per thread, then wait
LSS_DEV void tmem_ld64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : LSS_R8(0), LSS_R8(8), LSS_R8(16), LSS_R8(24), LSS_R8(32), LSS_R8(40), LSS_R8(48),
        LSS_R8(56)
      : "r"(taddr)
      : "memory");
}
// registers -> TMEM, 32 consecutive columns per thread, then wait
LSS_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n\t"
      "tcgen05.wait::st.sync.aligned;" ::"r"(taddr),
      LSS_W8(0), LSS_W8(8)
      : "memory");
}
LSS_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n\t"
      "tcgen05.wait::st.sync.aligned;" ::"r"(taddr),
      LSS_W8(0), LSS_W8(8), LSS_W8(16), LSS_W8(24)
      : "memory");
}

// ---------------------------------------------------------------- math
LSS_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
LSS_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---------------------------------------------------------------- register reconfiguration
template <uint32_t N>
LSS_DEV void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <uint32_t N>
LSS_DEV void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------- packed fp32x2 (FFMA2 / FADD2 / FMUL2)
LSS_DEV uint64_t f2_u64(float2 v) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
LSS_DEV float2 u64_f2(uint64_t r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
LSS_DEV float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_u64(a)), "l"(f2_u64(b)), "l"(f2_u64(c)));
  return u64_f2(d);
}
LSS_DEV float2 fadd2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_u64(a)), "l"(f2_u64(b)));
  return u64_f2(d);
}
LSS_DEV float2 fsub2(float2 a, float2 b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_u64(a)), "l"(f2_u64(b)));
  return u64_f2(d);
}
LSS_DEV float2 fmul2(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_u64(a)), "l"(f2_u64(b)));
  return u64_f2(d);
}

// Counter-based dropout bits (nnops.py:40-64 mix_key, the splitmix64 finaliser
// keyed by a running hash): every keep decision is a pure function of
// (seed, layer, site, sample, [head,] position, column), so a mask is recomputed
// in the backward instead of stored and is identical across sharding layouts.
constexpr uint64_t DROP_GOLDEN = 0x9E3779B97F4A7C15ull;
constexpr uint64_t DROP_MIX_A = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t DROP_MIX_B = 0x94D049BB133111EBull;
LSS_DEV uint64_t drop_mix(uint64_t h, uint64_t word) {
  uint64_t z = h + word * DROP_GOLDEN;
  z = (z ^ (z >> 30)) * DROP_MIX_A;
  z = (z ^ (z >> 27)) * DROP_MIX_B;
  return z ^ (z >> 31);
}
// keep iff uniform = (word >> 11) * 2^-53 >= rate  <=>  (word >> 11) >= thresh,
// thresh = ceil(rate * 2^53) computed exactly on the host (nnops.keep_mask)
LSS_DEV bool drop_keep(uint64_t row_key, uint64_t col, uint64_t thresh) {
  return (drop_mix(row_key, col) >> 11) >= thresh;
}

// 2^x on the FMA pipe for x in [-125, 127] (x is clamped below, so -inf -> ~2^-125,
// never a wrapped exponent: p(f) < 1 at f = 0 would underflow the exponent field
// at -127): Cody-Waite split
// x = j + f, |f| <= 1/2 via the 1.5*2^23 rounding trick, degree-3 minimax for
// 2^f (max rel. error 1.0e-4, far below the bf16 rounding of P), exponent
// added as an integer.  Offloads MUFU.EX2, the softmax's binding unit.
// DEG 2: a quadratic (one FFMA2 less; 2.0e-3, half a bf16 ulp) for the forward,
// where the FMA pipe is the co-bottleneck; DEG 3 for the backward.
template <int DEG = 3>
LSS_DEV float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = fadd2(x, magic);            // round(x) in the low mantissa bits
  const float2 f = fsub2(x, fsub2(t, magic));  // x - round(x)
  float2 pl;
  if constexpr (DEG == 2) {
    // minimax quadratic for 2^f on [-1/2, 1/2], p(0) = 1 pinned: max relative error 2.0e-3
    pl = ffma2(make_float2(0.23986403f, 0.23986403f), f, make_float2(0.70294179f, 0.70294179f));
    pl = ffma2(pl, f, make_float2(1.0f, 1.0f));
  } else {
    // minimax cubic for 2^f on [-1/2, 1/2] with p(0) = 1 pinned (2^n exact, so
    // e.g. equal scores give exactly uniform rows); max relative error 1.0e-4
    pl = ffma2(make_float2(0.05500906f, 0.05500906f), f, make_float2(0.24221097f, 0.24221097f));
    pl = ffma2(pl, f, make_float2(0.69328290f, 0.69328290f));
    pl = ffma2(pl, f, make_float2(1.0f, 1.0f));
  }
  return make_float2(__uint_as_float(__float_as_uint(pl.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(pl.y) + (__float_as_uint(t.y) << 23)));
}

}  // namespace lss
