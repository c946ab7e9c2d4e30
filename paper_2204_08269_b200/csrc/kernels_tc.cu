// KD on the 5th-generation tensor cores (tcgen05, sm_100a): the frequential
// contraction of the joint stage (Eq. (1) psi_{beta,theta}(lambda), Eq. (2) separable
// joint wavelet) fused with the complex modulus and phi_T pooling of
// Eq. (3).
//
// Per active alpha, the exact frequential operator is the complex matrix A[M][K]
// (plan.cpp).  With Y'' the planar Y2_alpha tile (rows 2l / 2l+1 = Re / Im Y2[l],
// K' = 2K rows, Nt time columns), two real products per 128-row M-block
//   D_re[128 x Nt] = A_re''[128 x K'] Y'',   D_im[128 x Nt] = A_im''[128 x K'] Y''
// give Re Z and Im Z of the same complex row in the same TMEM lane (columns
// [0, Nt) and [Nt, 2Nt) of the block's accumulator), so the epilogue needs no
// cross-lane exchange: |Z| = sqrt(D_re^2 + D_im^2) lane-locally.
//
// Arithmetic: kind::f16 with a two-term fp16 split of both operands,
//   x s = hi + lo,  hi = rn16(x s),  lo = rn16(x s - hi),
//   D = A_hi Y_hi + A_hi Y_lo + A_lo Y_hi   (fp32 accumulation in TMEM),
// relative error ~2^-21 per product, like fp32 (precision budget).
// The scales are powers of two (exact): s_m per A row (max |A''_m| s_m in
// [2^13, 2^14), plan.cpp), s_Y per Y'' tile (max |Y''| s_Y in [2^13, 2^14), KY
// below); |Z| = |D| / (s_m s_Y), applied to the pooled partials.
//
// KY (k_ky): Y2_alpha fp32 tiles -> s_Y and the fp16 hi / lo planes [2][K16][L].
// KD (k_kd_tc): CTA = 11 warps (TMEM 512 columns), persistent over work units
// (signal, time chunk, M-part), tiles of Nt columns inside a unit:
//   warp 10     B producer: TMA of the fp16 hi / lo tile (MN-major SWIZZLE_128B,
//               exactly the UMMA B image) + bulk copy of the tile's phi_T taps
//   warp 8      A producer: A'' K-records (pre-tiled fp16 SWIZZLE_32B images, 16 KiB
//               each, 2 per 32 KiB stage of an S-ring), lane s serves ring slot s
//   warp 9      TMEM allocator + tcgen05.mma issuer (one elected lane)
//   warps 0..7  epilogue, two sets of 4 warps; both sets take every M-block, set s
//               the columns [s Nt/2, (s+1) Nt/2): tcgen05.ld (re, im) -> |Z| -> phi_T
//               pooling at the retained frames (packed FFMA2) -> per-row
//               accumulators in registers -> global partials [slice][Mpad][frames]
//               at the end of a unit (slice = 2 chunk + set; KE sums the slices).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "jtfs_internal.h"
#include "kernels.h"

#ifndef JTFS_KD_FMA_SQRT_COLS
#define JTFS_KD_FMA_SQRT_COLS 0
#endif

namespace jtfs {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, parity)) {
    if (clock64() - t0 > 20000000000LL) __trap();  // ~10 s at 2 GHz
  }
}

// wait (+ accumulate the waited cycles into acc when instrumented: the JTFS_KD_PROF plan flag selects
// the PROF = true kernel instantiation; the clock reads are compiled out otherwise)
template <bool PROF>
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity, long long& acc) {
  if constexpr (PROF) {
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    acc += clock64() - t0;
  } else {
    mbar_wait(bar, parity);
  }
}
template <bool PROF>
__device__ __forceinline__ long long clk() {
  if constexpr (PROF) return clock64();
  return 0;
}

// ---- TMA ----
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ---- bulk copy (non-tensor TMA): contiguous global -> smem, completes on an mbarrier ----
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// ---- CTA pairs (cluster of 2, tcgen05 cta_group::2) ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// arrive on a barrier of another CTA of the cluster.  Default (.release, .cta) semantics:
// the only ordering needed is that of the preceding tcgen05.ld's (tcgen05.fence::
// before_thread_sync); a .cluster-scope release costs ~1k cycles per arrive (measured: the
// pair epilogue 1.6x slower with it)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
// tensor copies of a CTA pair completing on the LEADER's mbarrier (bar: shared::cluster address)
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                                 int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2 [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2 [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

// ---- tcgen05 ----
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// commit of the pair's MMAs, arriving on the same barrier in both CTAs
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// an epilogue warp frees an accumulator buffer: on its own barrier, or (pair) on the leader's
template <bool PAIR>
__device__ __forceinline__ void acc_release(uint64_t* bar) {
  if constexpr (PAIR)
    mbar_arrive_cluster(map_rank(bar, 0));
  else
    mbar_arrive(bar);
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// ties the loaded registers to a point after tcgen05.wait::ld (volatile asm order), so
// the compiler cannot hoist their uses above the wait
__device__ __forceinline__ void reg_fence(uint32_t (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(v[i]));
}

// UMMA shared-memory descriptor (sm_100 version bit), lbo / sbo in bytes.
//  A, K-major fp16, SWIZZLE_32B (layout 6): 8-row x 32 B atoms, sbo = 256, lbo unused.
//  B, MN-major fp16, SWIZZLE_128B (layout 2): 8 K-rows x 128 B atoms (64 MN
//  elements), lbo = stride between 64-element MN groups, sbo = 1024 between 8-row
//  K groups.  (Both verified bit-exact with tools/tc_unit16.cu.)
constexpr uint32_t kLayoutSW128 = 2, kLayoutSW32 = 6;
constexpr int kRec = 8192;     // one A'' K-record: 128 pair rows x 16 fp16 x {Re, Im}
constexpr int kImg = 4096;     // one 128 x 16 fp16 image inside a record
constexpr int kMaxRps = 4;     // K-records per A ring stage: 1, 2 or 4 (TcParams::rps)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)layout << 61;
  return d;
}

// instruction descriptor: kind::f16, D f32, A/B fp16, A K-major, B MN-major, M (128, or 256 for
// a CTA pair), N = n
__host__ __device__ constexpr uint32_t idesc_f16(int n, int m = 128) {
  return (1u << 4) | (0u << 7) | (0u << 10) | (0u << 15) | (1u << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ float sqrt_fast(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// packed FP32x2 FMA (FFMA2): d = a * (s, s) + c
__device__ __forceinline__ float2 ffma2(float2 a, float s, float2 c) {
  unsigned long long r, ua, us, uc;
  ua = *reinterpret_cast<unsigned long long*>(&a);
  uc = *reinterpret_cast<unsigned long long*>(&c);
  const float2 ss = make_float2(s, s);
  us = *reinterpret_cast<const unsigned long long*>(&ss);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(ua), "l"(us), "l"(uc));
  return *reinterpret_cast<float2*>(&r);
}

// one elected lane of a converged warp (operands stay warp-uniform -> UR registers)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 %%rx;\n\t.reg .pred %%px;\n\t"
      "elect.sync %%rx|%%px, %1;\n\t"
      "@%%px mov.s32 %0, 1;\n\t}"
      : "+r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }


// tcgen05.ld 32x32b.x16: 16 consecutive accumulator columns of this warp's 32 lanes
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void reg_fence16(uint32_t (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) asm volatile("" : "+r"(v[i]));
}

// ---- packed FP32x2 arithmetic (FFMA2 / FMUL2 / FADD2: two lanes per instruction; a
// scalar or an immediate operand is broadcast to both halves) ----
__device__ __forceinline__ unsigned long long f2_u64(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 u64_f2(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_u64(a)), "l"(f2_u64(b)), "l"(f2_u64(c)));
  return u64_f2(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_u64(a)), "l"(f2_u64(b)));
  return u64_f2(r);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_u64(a)), "l"(f2_u64(b)));
  return u64_f2(r);
}

// (sqrt q.x, sqrt q.y) on the FMA pipe (to offload MUFU, 16 / clk / SM): the classic
// magic-constant rsqrt seed (integer ALU), two packed Newton steps y <- y (3/2 - q/2 y^2),
// s = q y and one Heron correction s <- s - y (s^2 - q) / 2; <= 1.5 ulp (checked against
// fp64 over 60 decades), exactly 0 for q = 0.  Deterministic, like MUFU.SQRT.
__device__ __forceinline__ float2 sqrt2_fma(float2 q) {
  float2 y = make_float2(__uint_as_float(0x5f3759dfu - (__float_as_uint(q.x) >> 1)),
                         __uint_as_float(0x5f3759dfu - (__float_as_uint(q.y) >> 1)));
  const float2 h = mul2(q, make_float2(-0.5f, -0.5f));
#pragma unroll
  for (int it = 0; it < 2; ++it) y = mul2(y, fma2(mul2(h, y), y, make_float2(1.5f, 1.5f)));
  const float2 sq = mul2(q, y);
  const float2 r = fma2(sq, sq, add2(h, h));  // s^2 - q
  return fma2(mul2(y, r), make_float2(-0.5f, -0.5f), sq);
}

// columns of each 8-column group whose moduli take the FMA-pipe square root (the rest
// take MUFU.SQRT): balances the MUFU and FMA pipes of the epilogue
constexpr int kFmaSqrtCols = JTFS_KD_FMA_SQRT_COLS;

// Both spins of a pair row from its four real products at 8 time columns:
// v1 = acc1 (Re A . [Yr, Yi]), v2 = acc2 (Im A . [Yr, Yi]), interleaved (Yr, Yi) per column:
//   Z_-1 = A Y      = (P1 - P2) + i (P3 + P4),   Z_+1 = conj(A) Y = (P1 + P2) + i (P3 - P4)
// with P1 = Re A Yr, P2 = Im A Yi, P3 = Re A Yi, P4 = Im A Yr (h_{+1} = conj h_{-1}, R10).
// Packed per column: X = (Re Z_-, Re Z_+) = (-1, 1) P2 + P1, Y = (Im Z_-, Im Z_+) = (1, -1) P4
// + P3, Q = X X + Y Y = (|Z_-|^2, |Z_+|^2): four FP32x2 instructions, then two MUFU.SQRT.
// mz[j] = (|Z_-|, |Z_+|) of column j.
template <int NC>
__device__ __forceinline__ void spin_mags(const uint32_t (&v1)[2 * NC], const uint32_t (&v2)[2 * NC],
                                          float2 (&mz)[NC]) {
  const float2 cm = make_float2(-1.f, 1.f), cp = make_float2(1.f, -1.f);
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const float p1 = __uint_as_float(v1[2 * j]), p3 = __uint_as_float(v1[2 * j + 1]);
    const float p4 = __uint_as_float(v2[2 * j]), p2 = __uint_as_float(v2[2 * j + 1]);
    const float2 X = fma2(cm, make_float2(p2, p2), make_float2(p1, p1));
    const float2 Y = fma2(cp, make_float2(p4, p4), make_float2(p3, p3));
    const float2 Q = fma2(X, X, mul2(Y, Y));
    mz[j] = ((j & 7) >= 8 - kFmaSqrtCols) ? sqrt2_fma(Q) : make_float2(sqrt_fast(Q.x), sqrt_fast(Q.y));
  }
}
// ---------------------------------------------------------------------------------
// fp32 Y2 -> KD's fp16 operand (validation entry jtfs_debug_joint only; the forward's KC
// writes the operand directly, kernels.cu ProbFold16).  k_y2max: exact max |Re|, |Im| of
// Y2_alpha per (signal, alpha) -> the same power-of-two scale rule as k_yscale; k_ky: the
// packed rows [Y_hi (K); Y_lo (K); Y_hi (K)] of [K16][2L] fp16, (re, im) interleaved.
// ---------------------------------------------------------------------------------
struct KYParams {
  const float* y2;     // planar Y2 of signal 0 at alpha's offset; signal stride y2_stride floats
  int64_t y2_stride;
  __half* y16;         // Y16 of signal 0 at alpha's offset; signal stride y16_stride halves
  int64_t y16_stride;
  float* ysc;          // scale of (signal 0, alpha); signal stride ys_stride
  float* ysi;          // inverse scale
  int64_t ys_stride;
  int K, L;
};

__global__ void __launch_bounds__(256) k_y2max(KYParams p) {
  __shared__ uint32_t red[8];
  const int b = blockIdx.x;
  const float* Y = p.y2 + (int64_t)b * p.y2_stride;
  float mx = 0.f;
  for (int64_t i = threadIdx.x; i < (int64_t)2 * p.K * p.L; i += 256) mx = fmaxf(mx, fabsf(__ldg(Y + i)));
  const uint32_t w = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t mbits = 0;
    for (int i = 0; i < 8; ++i) mbits = max(mbits, red[i]);
    int E = (int)(mbits >> 23) - 127;
    E = max(E, -100);
    p.ysc[(int64_t)b * p.ys_stride] = __uint_as_float((uint32_t)(13 - E + 127) << 23);
    p.ysi[(int64_t)b * p.ys_stride] = __uint_as_float((uint32_t)(E - 13 + 127) << 23);
  }
}

__global__ void __launch_bounds__(256) k_ky(KYParams p) {
  const int b = blockIdx.y;
  const float* Y = p.y2 + (int64_t)b * p.y2_stride;
  const float s = __ldg(p.ysc + (int64_t)b * p.ys_stride);
  __half* row0 = p.y16 + (int64_t)b * p.y16_stride;
  const int64_t rs = 2 * (int64_t)p.L;  // row stride (halves)
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < (int64_t)p.K * p.L; i += (int64_t)gridDim.x * 256) {
    const int l = (int)(i / p.L), c = (int)(i % p.L);
    const float yr = __ldg(Y + (int64_t)(2 * l) * p.L + c) * s;
    const float yi = __ldg(Y + (int64_t)(2 * l + 1) * p.L + c) * s;
    const __half2 h = __floats2half2_rn(yr, yi);
    const float2 f = __half22float2(h);
    const __half2 lo = __floats2half2_rn(yr - f.x, yi - f.y);
    *reinterpret_cast<__half2*>(row0 + (int64_t)l * rs + 2 * c) = h;
    *reinterpret_cast<__half2*>(row0 + (int64_t)(p.K + l) * rs + 2 * c) = lo;
    *reinterpret_cast<__half2*>(row0 + (int64_t)(2 * p.K + l) * rs + 2 * c) = h;
  }
}

struct TcParams {
  int K16;         // B tile rows (3K rounded up to 16)
  int nkc;         // 16-wide K chunks
  int Nt;          // time columns per tile (64 or 32)
  int BRk, nbr;    // B TMA box rows, row boxes
  int NBB;         // fp16 B tile buffers (1 or 2)
  int S;           // A ring stages
  int rps;         // K-records (8 KiB) per A ring stage
  int tpu;         // tiles per work unit
  int nchunks;     // time chunks per signal (L / (Nt * tpu))
  const int32_t* chunk_sel;  // selected chunks (path sharding) or nullptr = all
  int nsel;        // number of selected chunks
  int n_mpart, n_mblk;  // M-parts and 128-pair-row M-blocks per part
  int stat;        // 1: A stationary (the CTA's part loaded once; grid % n_mpart == 0), 0: A ring
  // CTA pairs (PAIR kernels): n_mblk counts M-block PAIRS per part; CTA rank r of a pair owns
  // the blocks 2 i + r (M = 256 MMAs: rows 0..127 from the leader's A, 128..255 from the peer's)
  int L, nframes, Mpp;
  int nsig;
  unsigned long long* prof;  // measurement only (JTFS_KD_PROF flag): per-role wait-cycle counters or nullptr
  const uint16_t* A;   // A''_alpha records [Mpp / 128][nkc] x 8 KiB ([Re | Im] images)
  const float* ainv;   // 1 / s_p per pair row [Mpp]
  const float* wtab;   // phi_T pooling table: taps [L][NF] (pool_mode 0) or cubic moments [L/32][4][NF] (1)
  int pool_mode;
  const float* ys;     // 1 / s_Y of (signal, this alpha): ys[b * ys_stride]
  int64_t ys_stride;
  float* part;
  int64_t part_off, part_stride;
};

constexpr int kThreads = 352;
// warp roles: 0..7 epilogue, 8 A producer, 9 MMA issuer, 10 B producer
constexpr int kProdWarp = 8, kMmaWarp = 9, kBWarp = 10;
constexpr int kNbuf = 2;  // TMEM accumulator buffers, each [acc1 | acc2] of 2 x 2 Nt columns

// shared-memory carve-up (host and device agree through this function): B tile buffers,
// the A region (a ring of S stages of rps records, or the n_mblk x nkc records of the CTA's
// M-part when A is stationary), the pooling table buffers, the barriers (nab A barrier
// pairs: S ring slots or n_mblk stationary blocks)
struct SmemLayout {
  uint32_t b[4], ast, wt, bars, total;
};
__host__ __device__ inline SmemLayout smem_layout(int K16, int Nt, int NBB, uint32_t abytes, int nab, int NF,
                                                  int pool_mode, int pair = 0) {
  SmemLayout l{};
  auto up = [](uint32_t v, uint32_t a) { return (v + a - 1) / a * a; };
  uint32_t o = 0;
  // one fp16 K16 x 2Nt image ((re, im) along N); a CTA of a pair holds half of its columns
  const uint32_t bsz = (uint32_t)(K16 * 2 * Nt * 2) >> (pair ? 1 : 0);
  for (int i = 0; i < 4; ++i) {
    if (i < NBB) {
      l.b[i] = o;
      o = up(o + bsz, 1024);
    } else {
      l.b[i] = l.b[0];
    }
  }
  l.ast = o;
  o += abytes;
  l.wt = o;  // [2][Nt][NF] taps, or [2][Nt / 32][4][NF] moment coefficients
  o += (uint32_t)((NBB < 2 ? 2 : NBB) * Nt * (pool_mode ? NF / 8 : NF) * 4);  // max(2, NBB) table buffers
  l.bars = up(o, 8);
  o = l.bars + 8 * (16 + 2 * kNbuf + 2 * nab) + 16;
  l.total = o + 1024;  // + alignment slack of the dynamic smem base
  return l;
}

// one 8-column group of an epilogue set: both spins' |Z| -> phi_T pooling
template <int NF, int G>
__device__ __forceinline__ void epi_group_taps(uint32_t tb1, uint32_t tb2, const float* wt, float2 (&pm)[NF / 2],
                                               float2 (&pp)[NF / 2]) {
  uint32_t v1[16], v2[16];
  tmem_ld16(tb1 + 16 * G, v1);
  tmem_ld16(tb2 + 16 * G, v2);
  tmem_wait_ld();
  reg_fence16(v1);
  reg_fence16(v2);
  float2 mz[8];
  spin_mags<8>(v1, v2, mz);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4* w4 = reinterpret_cast<const float4*>(wt + (8 * G + j) * NF);
#pragma unroll
    for (int m4 = 0; m4 < NF / 4; ++m4) {
      const float4 w = w4[m4];
      pm[2 * m4 + 0] = ffma2(make_float2(w.x, w.y), mz[j].x, pm[2 * m4 + 0]);
      pm[2 * m4 + 1] = ffma2(make_float2(w.z, w.w), mz[j].x, pm[2 * m4 + 1]);
      pp[2 * m4 + 0] = ffma2(make_float2(w.x, w.y), mz[j].y, pp[2 * m4 + 0]);
      pp[2 * m4 + 1] = ffma2(make_float2(w.z, w.w), mz[j].y, pp[2 * m4 + 1]);
    }
  }
}
// moments of both spins, packed: S[k] = (sum_j |Z_-,j| u_j^k, sum_j |Z_+,j| u_j^k), u_j
// = (j - 15.5) / 16 compile-time (FFMA2 with an immediate operand).  The moments are taken
// over column pairs (j, 31 - j), where u_{31-j} = -u_j: with s = z_j + z_{31-j} and d = z_j -
// z_{31-j}, S0 += s, S1 += d u, S2 += s u^2, S3 += d u^3 -- 3 FMA-pipe instructions per
// column instead of 4 (the epilogue is bound by the FMA pipe: tools/ffma2_forms.cu).  So a
// group holds both columns of its pairs: group 0 the columns 0..7 and 24..31 of the 32-column
// block (two x16 TMEM loads per accumulator), group 1 the columns 8..23 (one x32).
template <int G>
__device__ __forceinline__ void epi_group_mom(uint32_t tb1, uint32_t tb2, float2 (&S)[4]) {
  uint32_t v1[32], v2[32];
  if constexpr (G == 0) {
    // accumulator columns 2t, 2t + 1 of time column t: t in [0, 8) -> [0, 16), t in [24, 32) -> [48, 64)
    tmem_ld16(tb1, *reinterpret_cast<uint32_t(*)[16]>(v1));
    tmem_ld16(tb1 + 48, *reinterpret_cast<uint32_t(*)[16]>(v1 + 16));
    tmem_ld16(tb2, *reinterpret_cast<uint32_t(*)[16]>(v2));
    tmem_ld16(tb2 + 48, *reinterpret_cast<uint32_t(*)[16]>(v2 + 16));
  } else {
    tmem_ld32(tb1 + 16, v1);  // t in [8, 24)
    tmem_ld32(tb2 + 16, v2);
  }
  tmem_wait_ld();
  reg_fence(v1);
  reg_fence(v2);
  float2 mz[16];  // G 0: columns 0..7, 24..31; G 1: columns 8..23
  spin_mags<16>(v1, v2, mz);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = (G == 0 ? 0 : 8) + i;  // column c pairs with 31 - c = mz[15 - i]
    const float u = ((float)c - 15.5f) * 0.0625f;  // compile-time
    const float2 sm = add2(mz[i], mz[15 - i]);
    const float2 df = fma2(mz[15 - i], make_float2(-1.f, -1.f), mz[i]);
    S[0] = add2(S[0], sm);
    S[1] = fma2(df, make_float2(u, u), S[1]);
    S[2] = fma2(sm, make_float2(u * u, u * u), S[2]);
    S[3] = fma2(df, make_float2(u * u * u, u * u * u), S[3]);
  }
}

// The CTA's tile sequence (unit u = blockIdx.x + i * gridDim.x, tiles 0..tpu-1 of each
// unit), walked incrementally: the unit's fields (runtime divisions) once per unit.
struct TileCursor {
  int tile, u, mpart, chunk, b;
  int cta = -1, ncta = 0;  // work-distribution index of this CTA (pair index for CTA pairs) and count
  __device__ __forceinline__ void unit_fields(const TcParams& p) {
    mpart = u % p.n_mpart;
    const int c = (u / p.n_mpart) % p.nsel;
    chunk = p.chunk_sel ? p.chunk_sel[c] : c;
    b = u / (p.n_mpart * p.nsel);
  }
  __device__ __forceinline__ void start(const TcParams& p, int cta_, int ncta_) {
    cta = cta_;
    ncta = ncta_;
    tile = 0;
    u = cta;
    unit_fields(p);
  }
  __device__ __forceinline__ void next(const TcParams& p) {
    if (++tile == p.tpu) {
      tile = 0;
      u += ncta;
      unit_fields(p);
    }
  }
};

// NTC: the tile width Nt as a compile-time constant (64 / 32: the epilogue's column loops
// unroll completely).  PROF: the instrumented variant (JTFS_KD_PROF plan flag).  PAIR: a
// cluster of two CTAs runs tcgen05.mma.cta_group::2 (M = 256 = one M-block per CTA, N = 2 Nt
// with each CTA holding half of the B tile's columns): per SM an MMA reads 4 KiB of A and
// 2 KiB of B instead of 4 + 4, the SS-mode shared-memory port limit of the N = 128 stream
// (tools/tc_rate2cta.cu mode 5).  The leader (rank 0) issues; both CTAs' tensor copies
// complete on the leader's barriers; commits multicast to both CTAs; both epilogues free the
// leader's accumulator barrier.
template <int NF, int MAXSLOT, bool PROF, int NTC, bool PAIR>
__global__ void __launch_bounds__(kThreads, 1)
    k_kd_tc(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmA, TcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B align by offsetting the __shared__ array itself (keeps the shared
  // address space visible to the compiler: LDS/STS instead of generic LD/ST)
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  constexpr int Nt = NTC;
  const int nab = p.stat ? p.n_mblk : p.S;  // A barrier pairs
  const SmemLayout lay = smem_layout(p.K16, Nt, p.NBB, p.stat ? (uint32_t)(p.n_mblk * p.nkc * kRec)
                                                              : (uint32_t)(p.S * p.rps * kRec),
                                     nab, NF, p.pool_mode, PAIR ? 1 : 0);
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int cta_id = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // work-distribution index
  const int ncta = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int wfl = Nt * (p.pool_mode ? NF / 8 : NF);  // taps / coefficients floats per buffer
  const int nwb = p.NBB < 2 ? 2 : p.NBB;             // table buffers (the producer runs NBB tiles ahead)
  uint8_t* Ast = base + lay.ast;
  float* Wt = reinterpret_cast<float*>(base + lay.wt);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + lay.bars);
  uint64_t* b_full = bars + 0;      // [NBB <= 4] B tile landed
  uint64_t* b_empty = bars + 4;     // [NBB] MMA done with the B tile
  uint64_t* w_full = bars + 8;      // [nwb] taps landed
  uint64_t* w_empty = bars + 12;    // [nwb] epilogue done with the taps
  uint64_t* acc_full = bars + 16;   // [kNbuf]
  uint64_t* acc_empty = bars + 16 + kNbuf;
  uint64_t* a_full = bars + 16 + 2 * kNbuf;  // [nab]
  uint64_t* a_empty = a_full + nab;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_empty + nab);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) {
      mbar_init(b_full + i, 1);
      mbar_init(b_empty + i, 1);
      mbar_init(w_full + i, 1);
      mbar_init(w_empty + i, 8);
    }
    for (int i = 0; i < kNbuf; ++i) {
      mbar_init(acc_full + i, 1);
      mbar_init(acc_empty + i, PAIR ? 16 : 8);  // pair: both CTAs' epilogues free the leader's buffer
    }
    for (int i = 0; i < nab; ++i) {
      mbar_init(a_full + i, 1);
      mbar_init(a_empty + i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // both CTAs' barriers exist before any remote arrive / copy
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int units = p.nsig * p.nsel * p.n_mpart;
  const int nst = (p.nkc + p.rps - 1) / p.rps;  // A'' stages (<= rps records of 16 K-columns) per M-block
  const uint32_t stage_bytes = (uint32_t)(p.rps * kRec);
  // the tile sequence of this CTA (pair): unit u = cta_id + i * ncta, tile 0..tpu-1
  const int my_units = (units - cta_id + ncta - 1) / ncta;
  const int my_tiles = my_units * p.tpu;

  if (warp == kBWarp) {
    // ===================== B producer: the packed fp16 tile + pooling table =====================
    // one copy per lane (copies issued by one thread complete one after another):
    // lane 0 the table, lanes 1.. the TMA boxes (64-column groups x row boxes)
    constexpr int ncg = PAIR ? 1 : 2 * Nt / 64;  // pair: this CTA's half = one 64-column group
    const int nboxes = ncg * p.nbr;
    const uint32_t btx = (uint32_t)(p.K16 * 2 * Nt * 2);  // the whole tile (pair: both halves, leader)
    const int wcol = p.pool_mode ? NF / 8 : NF;  // table floats per time column
    const uint32_t wbytes = (uint32_t)(Nt * wcol * 4);
    TileCursor cur;
    cur.start(p, cta_id, ncta);
    for (int gt = 0; gt < my_tiles; ++gt, cur.next(p)) {
      const int chunk = cur.chunk, b = cur.b;
      const int t0 = (chunk * p.tpu + cur.tile) * Nt;
      const int wi = gt % nwb, bi = gt % p.NBB;
      if (lane == 0) {
        mbar_wait(w_empty + wi, (uint32_t)((gt / nwb) + 1) & 1u);
        mbar_expect_tx(w_full + wi, wbytes);
        bulk_load(Wt + wi * wfl, p.wtab + (size_t)t0 * wcol, wbytes, w_full + wi);
        mbar_wait(b_empty + bi, (uint32_t)((gt / p.NBB) + 1) & 1u);
        if (rank == 0) mbar_expect_tx(b_full + bi, btx);
      }
      __syncwarp();
      for (int i = lane - 1; i >= 0 && i < nboxes; i += 31) {
        const int cg = i / p.nbr, rb = i % p.nbr;
        uint8_t* dst = base + lay.b[bi] + cg * (p.K16 * 128) + rb * (p.BRk * 128);
        if constexpr (PAIR)
          tma_load_3d_pair(dst, &tmB, map_rank(b_full + bi, 0), 2 * t0 + 64 * (int)rank, rb * p.BRk, b);
        else
          tma_load_3d(dst, &tmB, b_full + bi, 2 * t0 + cg * 64, rb * p.BRk, b);
      }
    }
  } else if (warp == kProdWarp) {
    // ===================== A producer =====================
    if (p.stat) {
      // stationary: the CTA (pair) always works on M-part cta_id % n_mpart (the grid's CTA
      // (pair) count is a multiple of n_mpart); lane mb copies M-block mb's nkc records once,
      // for the whole launch (pair: this CTA's block of pair mb, one tensor copy completing on
      // the leader's barrier, which expects both CTAs' bytes)
      const int mpart = cta_id % p.n_mpart;
      if (lane < p.n_mblk) {
        const uint32_t bytes = (uint32_t)(p.nkc * kRec);
        if constexpr (PAIR) {
          const int blk = (mpart * p.n_mblk + lane) * 2 + (int)rank;
          if (rank == 0) mbar_expect_tx(a_full + lane, 2u * bytes);
          tma_load_2d_pair(Ast + (size_t)lane * bytes, &tmA, map_rank(a_full + lane, 0), 0, blk * p.nkc * 8);
        } else {
          mbar_expect_tx(a_full + lane, bytes);
          bulk_load(Ast + (size_t)lane * bytes, p.A + (size_t)(mpart * p.n_mblk + lane) * p.nkc * (kRec / 2), bytes,
                    a_full + lane);
        }
      }
    } else if (lane < p.S) {
      // ring: bulk copies issued by one thread complete one after another (~600 cycles
      // each, measured with tools/bulk_bw.cu), so lane s serves ring slot s (S lanes issue in
      // parallel; a slot is always served by the same lane: unambiguous parity waits)
      uint32_t s = 0, ph = 0;
      TileCursor cur;
      cur.start(p, cta_id, ncta);
      for (int gt = 0; gt < my_tiles; ++gt, cur.next(p)) {
        const int mpart = cur.mpart;
        for (int mb = 0; mb < p.n_mblk; ++mb) {
          const int blk = PAIR ? (mpart * p.n_mblk + mb) * 2 + (int)rank : mpart * p.n_mblk + mb;
          const uint16_t* arec = p.A + (size_t)blk * p.nkc * (kRec / 2);
          for (int st = 0; st < nst; ++st) {
            if ((int)s == lane) {
              mbar_wait(a_empty + s, ph ^ 1);
              if constexpr (PAIR) {
                // full-stage boxes (rps records; a short last stage reads past its block, unused)
                // of this CTA's block, completing on the leader's barrier (expect: both CTAs)
                if (rank == 0) mbar_expect_tx(a_full + s, 2u * stage_bytes);
                tma_load_2d_pair(Ast + s * stage_bytes, &tmA, map_rank(a_full + s, 0), 0,
                                 (blk * p.nkc + p.rps * st) * 8);
              } else {
                const uint32_t bytes = (uint32_t)(min(p.rps, p.nkc - p.rps * st) * kRec);
                mbar_expect_tx(a_full + s, bytes);
                bulk_load(Ast + s * stage_bytes, arec + (size_t)(p.rps * st) * (kRec / 2), bytes, a_full + s);
              }
            }
            if (++s == (uint32_t)p.S) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == kMmaWarp && (!PAIR || rank == 0)) {
    // ===================== MMA issuer (warp-wide loop, one elected lane issues) =====================
    // per M-block and 16-wide K chunk: acc1 += Re A'' . B, acc2 += Im A'' . B (N = 2 Nt)
    // (pair: the leader issues M = 256 for both CTAs' M-blocks; the peer's MMA warp idles)
    uint32_t s = 0, ph = 0, cnt = 0;
    long long w_b = 0, w_acc = 0, w_a = 0;
    const long long t_start = clk<PROF>();
    const uint32_t idesc = idesc_f16(2 * Nt, PAIR ? 256 : 128);
    const uint32_t colstride = (uint32_t)(p.K16 * 128);
    const uint64_t dA0 = sdesc(smem_u32(Ast), 16, 256, kLayoutSW32);
    for (int gt = 0; gt < my_tiles; ++gt) {
      const int bi = gt % p.NBB;
      mbar_wait_t<PROF>(b_full + bi, (uint32_t)(gt / p.NBB) & 1u, w_b);
      tc_fence_after();
      const uint64_t dB = sdesc(smem_u32(base + lay.b[bi]), colstride, 1024, kLayoutSW128);
      for (int mb = 0; mb < p.n_mblk; ++mb, ++cnt) {
        const uint32_t ab = cnt % (uint32_t)kNbuf, use = cnt / (uint32_t)kNbuf;
        mbar_wait_t<PROF>(acc_empty + ab, (use + 1) & 1, w_acc);
        tc_fence_after();
        const uint32_t d1 = tmem_base + ab * 4u * (uint32_t)Nt, d2 = d1 + 2u * (uint32_t)Nt;
        if (p.stat) {
          // the M-block's records stay resident: wait once for their copy (phase 0)
          mbar_wait_t<PROF>(a_full + mb, 0u, w_a);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t a0 = dA0 + (uint64_t)(((uint32_t)mb * (uint32_t)p.nkc * kRec) >> 4);
            for (int kc = 0; kc < p.nkc; ++kc) {
              const uint64_t a = a0 + (uint64_t)((kc * kRec) >> 4);
              const uint64_t yo = (uint64_t)((kc * 2048) >> 4);  // 16 K-rows x 128 B
              const uint32_t acc0 = kc > 0 ? 1u : 0u;
              if constexpr (PAIR) {
                mma_f16_pair(d1, a, dB + yo, idesc, acc0);
                mma_f16_pair(d2, a + (uint64_t)(kImg >> 4), dB + yo, idesc, acc0);
              } else {
                mma_f16(d1, a, dB + yo, idesc, acc0);                         // Re A'' . B
                mma_f16(d2, a + (uint64_t)(kImg >> 4), dB + yo, idesc, acc0);  // Im A'' . B
              }
            }
          }
          __syncwarp();
        } else {
          for (int st = 0; st < nst; ++st) {
            mbar_wait_t<PROF>(a_full + s, ph, w_a);
            tc_fence_after();
            if (elect_one()) {
              const uint64_t dst = dA0 + (uint64_t)((s * stage_bytes) >> 4);
#pragma unroll
              for (int r = 0; r < kMaxRps; ++r) {
                const int kc = p.rps * st + r;
                if (r < p.rps && kc < p.nkc) {
                  const uint64_t a = dst + (uint64_t)((r * kRec) >> 4);
                  const uint64_t yo = (uint64_t)((kc * 2048) >> 4);  // 16 K-rows x 128 B
                  const uint32_t acc0 = kc > 0 ? 1u : 0u;
                  if constexpr (PAIR) {
                    mma_f16_pair(d1, a, dB + yo, idesc, acc0);
                    mma_f16_pair(d2, a + (uint64_t)(kImg >> 4), dB + yo, idesc, acc0);
                  } else {
                    mma_f16(d1, a, dB + yo, idesc, acc0);                         // Re A'' . B
                    mma_f16(d2, a + (uint64_t)(kImg >> 4), dB + yo, idesc, acc0);  // Im A'' . B
                  }
                }
              }
              if constexpr (PAIR)
                mma_commit_pair(a_empty + s);
              else
                mma_commit(a_empty + s);
            }
            __syncwarp();
            if (++s == (uint32_t)p.S) {
              s = 0;
              ph ^= 1;
            }
          }
        }
        if (elect_one()) {
          if constexpr (PAIR)
            mma_commit_pair(acc_full + ab);
          else
            mma_commit(acc_full + ab);
        }
        __syncwarp();
      }
      if (elect_one()) {
        if constexpr (PAIR)
          mma_commit_pair(b_empty + bi);
        else
          mma_commit(b_empty + bi);
      }
      __syncwarp();
    }
    if (PROF && p.prof && lane == 0) {
      atomicAdd(p.prof + 0, (unsigned long long)(clk<PROF>() - t_start));
      atomicAdd(p.prof + 1, (unsigned long long)w_b);
      atomicAdd(p.prof + 2, (unsigned long long)w_acc);
      atomicAdd(p.prof + 3, (unsigned long long)w_a);
    }
  } else if (warp < kMmaWarp) {
    // ===================== epilogue (warps 0..7) =====================
    const int eset = warp >> 2;  // column half
    const int q = warp & 3;      // TMEM lane quarter (warp_id % 4)
    constexpr int half = Nt / 2;
    const int cbeg = eset * half;
    long long e_w = 0, e_acc = 0, e_math = 0;
    const long long e_start = clk<PROF>();
    uint32_t cnt = 0;
    float2 accm[MAXSLOT][NF / 2], accp[MAXSLOT][NF / 2];  // pooled partials of both spins of my pair rows
    TileCursor cur;
    cur.start(p, cta_id, ncta);
    float inv = 0.f;  // 1 / s_Y of the unit's signal (loaded once per unit, off the per-tile path)
    for (int gt = 0; gt < my_tiles; ++gt, cur.next(p)) {
      const int mpart = cur.mpart, chunk = cur.chunk, b = cur.b, tile = cur.tile;
      if (tile == 0) {
        inv = __ldg(p.ys + (int64_t)b * p.ys_stride);
#pragma unroll
        for (int k = 0; k < MAXSLOT; ++k)
#pragma unroll
          for (int m = 0; m < NF / 2; ++m) accm[k][m] = accp[k][m] = make_float2(0.f, 0.f);
      }
      const int wi = gt % nwb;
      mbar_wait_t<PROF>(w_full + wi, (uint32_t)(gt / nwb) & 1u, e_w);
      const float* wt = Wt + wi * wfl + cbeg * NF;
#pragma unroll 1
      for (int mb = 0; mb < p.n_mblk; ++mb, ++cnt) {
        const uint32_t ab = cnt % (uint32_t)kNbuf;
        mbar_wait_t<PROF>(acc_full + ab, (cnt / (uint32_t)kNbuf) & 1u, e_acc);
        const long long tm0 = clk<PROF>();
        tc_fence_after();
        // accumulator columns 2t / 2t+1 = (Yr, Yi) products of time column t; this set's
        // columns [cbeg, cbeg + Nt/2) start at TMEM column 2 cbeg of acc1 / acc2
        const uint32_t tb1 = tmem_base + ((uint32_t)(q * 32) << 16) + ab * 4u * (uint32_t)Nt + 2u * (uint32_t)cbeg;
        const uint32_t tb2 = tb1 + 2u * (uint32_t)Nt;
        float2 pm[NF / 2], pp[NF / 2];
#pragma unroll
        for (int m = 0; m < NF / 2; ++m) pm[m] = pp[m] = make_float2(0.f, 0.f);
        if (p.pool_mode == 1) {
          // moment form (Nt = 64: this set's 32 columns are one 32-column block):
          // S_k = sum_j |Z_j| u_j^k (k <= 3, u_j compile-time), then part += G_k S_k
          float2 S[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
          if constexpr (half == 32) {
            epi_group_mom<0>(tb1, tb2, S);
            epi_group_mom<1>(tb1, tb2, S);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) acc_release<PAIR>(acc_empty + ab);  // accumulator buffer read: back to the MMA
          const float4* g4 = reinterpret_cast<const float4*>(Wt + wi * wfl + (cbeg / 32) * 4 * NF);
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int m4 = 0; m4 < NF / 4; ++m4) {
              const float4 w = g4[k * (NF / 4) + m4];
              pm[2 * m4 + 0] = ffma2(make_float2(w.x, w.y), S[k].x, pm[2 * m4 + 0]);
              pm[2 * m4 + 1] = ffma2(make_float2(w.z, w.w), S[k].x, pm[2 * m4 + 1]);
              pp[2 * m4 + 0] = ffma2(make_float2(w.x, w.y), S[k].y, pp[2 * m4 + 0]);
              pp[2 * m4 + 1] = ffma2(make_float2(w.z, w.w), S[k].y, pp[2 * m4 + 1]);
            }
        } else {
          epi_group_taps<NF, 0>(tb1, tb2, wt, pm, pp);
          epi_group_taps<NF, 1>(tb1, tb2, wt, pm, pp);
          if constexpr (half == 32) {
            epi_group_taps<NF, 2>(tb1, tb2, wt, pm, pp);
            epi_group_taps<NF, 3>(tb1, tb2, wt, pm, pp);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) acc_release<PAIR>(acc_empty + ab);
        }
        e_math += clk<PROF>() - tm0;
        // warp-uniform branch to the M-block's slot (a predicated loop over all
        // MAXSLOT slots would issue MAXSLOT x NF FMAs)
        switch (mb) {
#define JTFS_ACC_SLOT(K)                                                                         \
  case K:                                                                                        \
    if constexpr (K < MAXSLOT) {                                                                 \
      _Pragma("unroll") for (int m = 0; m < NF / 2; ++m) {                                       \
        accm[K][m] = ffma2(pm[m], inv, accm[K][m]);                                              \
        accp[K][m] = ffma2(pp[m], inv, accp[K][m]);                                              \
      }                                                                                          \
    }                                                                                            \
    break;
          JTFS_ACC_SLOT(0) JTFS_ACC_SLOT(1) JTFS_ACC_SLOT(2) JTFS_ACC_SLOT(3) JTFS_ACC_SLOT(4)
#undef JTFS_ACC_SLOT
          default: break;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(w_empty + wi);  // this warp is done with the tile's taps
      if (tile == p.tpu - 1) {
        // unit done: my pair rows' pooled partials of this (time chunk, column half) slice,
        // theta = -1 (and phi_F) at row p, theta = +1 at row Mpp + p
        float* dst = p.part + (int64_t)b * p.part_stride + p.part_off +
                     (int64_t)(2 * chunk + eset) * (2 * p.Mpp) * p.nframes;
#pragma unroll
        for (int k = 0; k < MAXSLOT; ++k) {
          if (k < p.n_mblk) {
            const int row = (PAIR ? (mpart * p.n_mblk + k) * 2 + (int)rank : mpart * p.n_mblk + k) * 128 + q * 32 + lane;
            const float ia = __ldg(p.ainv + row);
            float* d0 = dst + (int64_t)row * p.nframes;
            float* d1 = dst + (int64_t)(p.Mpp + row) * p.nframes;
#pragma unroll
            for (int m = 0; m < NF / 2; ++m) {
              if (2 * m < p.nframes) {
                d0[2 * m] = accm[k][m].x * ia;
                d1[2 * m] = accp[k][m].x * ia;
              }
              if (2 * m + 1 < p.nframes) {
                d0[2 * m + 1] = accm[k][m].y * ia;
                d1[2 * m + 1] = accp[k][m].y * ia;
              }
            }
          }
        }
      }
    }
    if (PROF && p.prof && lane == 0) {
      atomicAdd(p.prof + 4, (unsigned long long)(clk<PROF>() - e_start));
      atomicAdd(p.prof + 5, (unsigned long long)e_w);
      atomicAdd(p.prof + 6, (unsigned long long)e_acc);
      atomicAdd(p.prof + 7, (unsigned long long)e_math);
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // no remote arrive / MMA into the peer is still in flight
  if (warp == kMmaWarp) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

}  // namespace tc

// =================================================================================
// host side
// =================================================================================
namespace {
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encoder() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

bool encode(CUtensorMap* m, CUtensorMapDataType dt, void* base, int rank, const cuuint64_t* dims,
            const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle swz) {
  PFN_encodeTiled fn = get_encoder();
  if (!fn) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return fn(m, dt, rank, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int nf_of(int nframes) { return nframes <= 8 ? 8 : nframes <= 16 ? 16 : 32; }
size_t tc_smem(const AlphaKD& d, int nf) {
  const uint32_t abytes = d.tc_stat ? (uint32_t)(d.tc_mblk * d.tc_nkc * tc::kRec) : (uint32_t)(d.tc_S * d.tc_rps * tc::kRec);
  return tc::smem_layout(d.tc_K16, d.tc_Nt, d.tc_NBB, abytes, d.tc_stat ? d.tc_mblk : d.tc_S, nf, d.pool_mode,
                         d.tc_pair)
      .total;
}
}  // namespace

// choose the per-alpha tensor-core tiling (called by build_plan): the first of
// (Nt, B buffers, min stages) = (128, 2, 3), (128, 2, 2), (128, 1, 3), (128, 1, 2),
// (64, 2, 2), (64, 1, 2), (32, 1, 2) that fits, then as many A'' ring stages of rps
// records as fit (<= 24 records).  Every choice is a function of the plan alone (no
// environment knobs: output bytes depend only on (plan, x)).  Returns "" or the reason
// an alpha cannot be tiled (the plan then fails unless JTFS_KD_SIMT was requested).
std::string plan_tc(Plan& P) {
  const int NF = nf_of(P.n_frames);
  const size_t budget = 227 * 1024;
  P.tc_n_mblk = P.Mpp / 128 / P.tc_n_mpart;
  // A ring stages of rps 8 KiB K-records, as equal as possible with <= 4 records per
  // stage (nkc = 5 -> 3 + 2, not 4 + 1: a 1-record stage is consumed in 2 MMAs, too fast
  // for the next 4-record copy into its slot).  Measured on c3 (round 1): uniform
  // rps = 1 / 2 / 4 -> 2156 / 2459 / 2542 signals/s (per-copy overhead), so stages stay
  // at <= 32 KiB.  The ring holds at most 24 records (192 KiB).
  constexpr int rec_max = 24;
  for (auto& d : P.kd) {
    d.tc_K2 = 3 * d.K;
    d.tc_K16 = (d.tc_K2 + 15) / 16 * 16;
    d.tc_nkc = d.tc_K16 / 16;
    d.tc_nbr = (d.tc_K16 + 255) / 256;
    d.tc_BRk = (d.tc_K16 / d.tc_nbr + 7) / 8 * 8;
    {
      const int nst = (d.tc_nkc + 3) / 4;
      d.tc_rps = (d.tc_nkc + nst - 1) / nst;
    }
    // Nt = 64 time columns (two accumulators of N = 2 Nt = 128 columns per M-block, two
    // TMEM buffers); two B buffers when they fit next to >= 2 stages of A records.  The
    // moment-form epilogue needs Nt = 64 (its 32-column blocks are one epilogue set's
    // columns): a narrower tile (L < 64 or no fit) falls back to the exact taps.
    auto choose = [&]() {
      const int cand[4][3] = {{64, 2, 3}, {64, 2, 2}, {64, 1, 2}, {32, 1, 2}};
      for (const auto& c : cand) {
        if (c[0] > d.L) continue;
        d.tc_Nt = c[0];
        d.tc_NBB = c[1];
        d.tc_S = c[2];
        if (tc_smem(d, NF) > budget) continue;
        while ((d.tc_S + 1) * d.tc_rps <= rec_max && tc_smem(d, NF) + (size_t)d.tc_rps * tc::kRec <= budget)
          ++d.tc_S;
        return true;
      }
      return false;
    };
    // A stationary: each CTA keeps its M-part's n_mblk x nkc records resident for the whole
    // launch, so A never streams from L2.  Used only where it fits with two B buffers and at
    // most two M-parts (measured on c3: alpha 0 22.3 -> 20.9 ms per step; alphas 2-4, which
    // need one B buffer or 5-10 parts re-reading every B tile, got 15-35 % slower).
    auto choose_stat = [&]() {
      const int nblocks = P.Mpp / 128, maxslot = NF == 8 ? 5 : NF == 16 ? 2 : 1;
      if (d.L < 64) return false;
      for (int np = 1; np <= std::min(2, nblocks); ++np) {
        if (nblocks % np || nblocks / np > maxslot) continue;
        for (int nbb = 2; nbb >= 2; --nbb) {
          d.tc_stat = 1;
          d.tc_mpart = np;
          d.tc_mblk = nblocks / np;
          d.tc_Nt = 64;
          d.tc_NBB = nbb;
          d.tc_S = 0;
          if (tc_smem(d, NF) <= budget) return true;
        }
      }
      d.tc_stat = 0;
      return false;
    };
    bool ok = choose_stat();
    if (!ok) {
      d.tc_mpart = P.tc_n_mpart;
      d.tc_mblk = P.tc_n_mblk;
      d.tc_pair = 0;
      ok = choose();
      if (ok && d.pool_mode && d.tc_Nt != 64) {
        d.pool_mode = 0;
        ok = choose();
      }
      // CTA pairs (cta_group::2): the ring alphas whose M-blocks split into pairs with
      // <= MAXSLOT blocks per CTA and an Nt = 64 tile (half of its B columns per CTA).
      // Not where the A'' ring's L2 stream bounds the single-CTA kernel (10..15 K-chunks:
      // measured on c3, tools/pair_check.py, 64 signals: alpha 2 / 3 (nkc 10 / 13) 1.78 ->
      // 2.13 / 1.28 -> 1.33 ms with pairs, as each SM still streams 8 KiB of A'' per two
      // MMAs, ~40 B/cycle/SM at the chip's L2 limit, and the pair adds the coupling of two
      // streams; alpha 1 (nkc 7) 2.92 -> 2.65 and alpha 4-6 (nkc 16-22, where the single CTA
      // fits one B buffer or few A stages) 1.47 -> 1.30 ms gain)
      const int nblocks = P.Mpp / 128, maxslot = NF == 8 ? 5 : NF == 16 ? 2 : 1;
      const bool a_stream_bound = d.tc_nkc >= 10 && d.tc_nkc < 16;
      bool pair_stat = false;
#ifndef JTFS_PAIRSTAT_ALL
#define JTFS_PAIRSTAT_ALL 0
#endif
      if (ok && !(P.prm.flags & JTFS_KD_NOPAIR) && (a_stream_bound || JTFS_PAIRSTAT_ALL) && d.tc_Nt == 64 &&
          nblocks % 2 == 0 && d.tc_nkc <= 32) {
        // stationary pairs first: each CTA keeps its M-blocks of the pair's part resident
        // (the A'' stream never touches L2 again; the B tile's halves are re-read once per
        // part), the fewest parts whose blocks fit next to two B half-buffers
        const AlphaKD keep = d;
        const int npair = nblocks / 2;
        for (int np = 1; np <= npair && !pair_stat; ++np) {
          if (npair % np || npair / np > maxslot) continue;
          d.tc_pair = 1;
          d.tc_stat = 1;
          d.tc_mpart = np;
          d.tc_mblk = npair / np;
          d.tc_Nt = 64;
          d.tc_NBB = 2;
          d.tc_S = 0;
          pair_stat = tc_smem(d, NF) <= budget;
          // a few M-blocks per CTA consume a B tile fast: up to 4 B half-buffers keep the
          // tile copies (L2 latency) ahead of the MMAs
          while (pair_stat && d.tc_NBB < 4) {
            ++d.tc_NBB;
            if (tc_smem(d, NF) > budget) {
              --d.tc_NBB;
              break;
            }
          }
        }
        if (!pair_stat) d = keep;
      }
      if (ok && !pair_stat && !(P.prm.flags & JTFS_KD_NOPAIR) && !a_stream_bound && d.tc_Nt == 64 &&
          nblocks % 2 == 0) {
        const AlphaKD keep = d;
        const int npair = nblocks / 2;
        int np = (npair + maxslot - 1) / maxslot;
        while (npair % np) ++np;
        d.tc_pair = 1;
        d.tc_mpart = np;
        d.tc_mblk = npair / np;
        if (!choose() || d.tc_Nt != 64) d = keep;
      }
    }
    if (!ok) return "tensor-core KD: no tile of alpha " + std::to_string(d.alpha) + " fits shared memory";
    // time chunk per work unit: the largest power of two <= 4096 that still gives
    // about 4 units per SM for a full micro-batch (partials are per chunk; measured on
    // c3, round 1: 4096 / 8192 / 16384-column chunks equal within noise)
    const int64_t sig = (P.prm.flags & JTFS_LATENCY) ? 1 : P.mb;  // signals per KD launch
    const int64_t target = sig * d.tc_mpart * d.L / (4 * (d.tc_pair ? 74 : 148));  // units per SM (pair)
    int ch = 4096;
    while (ch > d.tc_Nt && ch > target) ch /= 2;  // (JTFS_LATENCY: one signal per launch)
    d.chunk = std::min(ch, d.L);
    if (d.chunk < d.tc_Nt) d.chunk = d.tc_Nt;
    d.nchunks = d.L / d.chunk;
    d.tc_tpu = d.chunk / d.tc_Nt;
    // the KY / KD per-tile scale slots (plan.cpp sizes L / 32 per alpha and signal)
    if (d.L / d.tc_Nt > std::max(1, d.L / 32)) return "internal: tensor-core KD tile scales exceed their slots";
    if (d.L < 32) return "tensor-core KD: alpha " + std::to_string(d.alpha) + " has fewer than 32 time columns";
    if (d.chunk % d.tc_Nt || d.nchunks * d.chunk != d.L) return "internal: tensor-core KD chunking";
    if (d.tc_nbr * d.tc_BRk != d.tc_K16) return "internal: tensor-core KD B boxes";
  }
  return "";
}

cudaError_t tc_setup_device(Plan& P) {
  if (P.kd_impl != 1) return cudaSuccess;
  // The persistent KD launches of the slow alphas (few work units) leave SMs idle; they
  // run on a second stream, overlapping the tails of the fast alphas' launches.
  // The first 5 active alphas (the long, fast ones: >= 90 % of KD's work in c3) run on
  // the caller's stream, the rest on the side stream.
  {
#ifndef JTFS_KD_SIDE_FROM
#define JTFS_KD_SIDE_FROM 5
#endif
    const int split = JTFS_KD_SIDE_FROM;
    if (split > 0 && split < (int)P.kd.size()) {
      cudaStream_t s = nullptr;
      cudaError_t es = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (es != cudaSuccess) return es;
      P.kd_side_stream = (void*)s;
      P.kd_side_from = split;
    }
  }
  const int NF = nf_of(P.n_frames);
  size_t mx = 0;
  for (auto& d : P.kd) mx = std::max(mx, tc_smem(d, NF));
  cudaError_t e = cudaSuccess;
  auto set = [&](auto kern) {
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
  };
#define JTFS_SET_KD(NF_, MS_)                                                                      \
  set(tc::k_kd_tc<NF_, MS_, false, 64, false>); set(tc::k_kd_tc<NF_, MS_, false, 32, false>);      \
  set(tc::k_kd_tc<NF_, MS_, true, 64, false>); set(tc::k_kd_tc<NF_, MS_, true, 32, false>);        \
  set(tc::k_kd_tc<NF_, MS_, false, 64, true>); set(tc::k_kd_tc<NF_, MS_, true, 64, true>);
  if (NF == 8) { JTFS_SET_KD(8, 5) }
  else if (NF == 16) { JTFS_SET_KD(16, 2) }
  else { JTFS_SET_KD(32, 1) }
#undef JTFS_SET_KD
  return e;
}

int launch_y16_from_y2(Plan& P, const float* y2, int nsig, uint16_t* y16, float* ys, cudaStream_t st) {
  const int na = (int)P.kd.size();
  for (int i = 0; i < na; ++i) {
    const auto& d = P.kd[i];
    tc::KYParams q{};
    q.y2 = y2 + 2 * d.y2_off;
    q.y2_stride = 2 * P.y2_total;
    q.y16 = reinterpret_cast<__half*>(y16) + d.y16_off;
    q.y16_stride = P.y16_total;
    q.ysc = ys + i;
    q.ysi = ys + (int64_t)nsig * na + i;
    q.ys_stride = na;
    q.K = d.K;
    q.L = d.L;
    tc::k_y2max<<<nsig, 256, 0, st>>>(q);
    tc::k_ky<<<dim3(std::max(1, std::min(64, d.K * d.L / 4096)), nsig), 256, 0, st>>>(q);
  }
  return 2 * na;
}

int launch_kd_tc(Plan& P, const uint16_t* y16, const float* ysi, int nsig, float* part, cudaStream_t st,
                 int* err, const UnitSel* sel) {
  const int NF = nf_of(P.n_frames);
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int launches = 0;
  *err = 0;
  cudaStream_t main_st = st;
  // profiling (jtfs_profile_enable) serialises every alpha on the caller's stream, so each
  // launch's event pair measures that launch alone (not the wait for SMs it shares)
  cudaStream_t side = P.prof ? nullptr : (cudaStream_t)P.kd_side_stream;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (side) {
    // per-call events: concurrent forwards on one plan stay correctly paired
    cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming);
    cudaEventRecord(ev_fork, main_st);
    cudaStreamWaitEvent(side, ev_fork, 0);
  }
  for (size_t i = 0; i < P.kd.size(); ++i) {
    const auto& d = P.kd[i];
    const int nsel = sel ? sel->cnt[i] : d.nchunks;
    if (nsel == 0) continue;
    st = (side && (int)i >= P.kd_side_from) ? side : main_st;
    CUtensorMap tmB;
    // K' = 3K packed rows (the buffer is allocated with K16 rows): the box rows beyond K'
    // are out of bounds and arrive zero-filled (the MMA's K padding)
    cuuint64_t dims[3] = {(cuuint64_t)(2 * d.L), (cuuint64_t)d.tc_K2, (cuuint64_t)nsig};
    cuuint64_t strides[2] = {(cuuint64_t)d.L * 4, (cuuint64_t)P.y16_total * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)d.tc_BRk, 1};
    if (!encode(&tmB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, const_cast<uint16_t*>(y16) + d.y16_off, 3, dims, strides, box,
                CU_TENSOR_MAP_SWIZZLE_128B)) {
      *err = 1;
      break;  // the join below still orders the side stream before the caller's
    }
    // pair: A'' records as rows of 1 KiB (8 rows per record), one box = one ring stage,
    // copied verbatim (the records are pre-swizzled); a short last stage reads past the
    // alpha's records (zero fill) or into the next block's (never multiplied)
    CUtensorMap tmA;
    std::memset(&tmA, 0, sizeof(tmA));
    if (d.tc_pair) {
      const int64_t nrec = (int64_t)(P.Mpp / 128) * d.tc_nkc;
      cuuint64_t adims[2] = {256, (cuuint64_t)(nrec * 8)};
      cuuint64_t astr[1] = {1024};
      cuuint32_t abox[2] = {256, (cuuint32_t)(8 * (d.tc_stat ? d.tc_nkc : d.tc_rps))};  // stationary: one block
      if (!encode(&tmA, CU_TENSOR_MAP_DATA_TYPE_UINT32, const_cast<uint16_t*>(P.d_A16 + d.tc_a16_off), 2, adims, astr,
                  abox, CU_TENSOR_MAP_SWIZZLE_NONE)) {
        *err = 1;
        break;
      }
    }
    tc::TcParams p{};
    p.K16 = d.tc_K16;
    p.nkc = d.tc_nkc;
    p.Nt = d.tc_Nt;
    p.BRk = d.tc_BRk;
    p.nbr = d.tc_nbr;
    p.NBB = d.tc_NBB;
    p.S = d.tc_S;
    p.rps = d.tc_rps;
    p.tpu = d.tc_tpu;
    p.nchunks = d.nchunks;
    p.chunk_sel = sel ? sel->d_sel + sel->off[i] : nullptr;
    p.nsel = nsel;
    p.n_mpart = d.tc_mpart;
    p.n_mblk = d.tc_mblk;
    p.stat = d.tc_stat;
    p.L = d.L;
    p.nframes = P.n_frames;
    p.Mpp = P.Mpp;
    p.nsig = nsig;
    p.A = P.d_A16 + d.tc_a16_off;
    p.ainv = P.d_Ainv + d.tc_ainv_off;
    p.wtab = P.d_wtab + d.wtab_off;
    p.pool_mode = d.pool_mode;
    p.ys = ysi + d.ys_off;
    p.ys_stride = P.ys_total;
    static unsigned long long* prof = nullptr;
    const bool do_prof = (P.prm.flags & JTFS_KD_PROF) != 0;  // measurement-only plan flag
    if (do_prof && !prof) cudaMalloc(&prof, 16 * 8);
    if (do_prof) cudaMemsetAsync(prof, 0, 16 * 8, st);
    p.prof = do_prof ? prof : nullptr;
    p.part = part;
    p.part_off = d.part_off;
    p.part_stride = P.part_total;
    const int units = nsig * nsel * d.tc_mpart;
    // stationary A: a multiple of n_mpart CTAs, so CTA b always gets M-part b % n_mpart
    const int grid = d.tc_stat && d.tc_pair
                         ? 2 * std::max(d.tc_mpart, std::min(units, sms / 2) / d.tc_mpart * d.tc_mpart)
                     : d.tc_stat ? std::max(d.tc_mpart, std::min(units, sms) / d.tc_mpart * d.tc_mpart)
                     : d.tc_pair ? 2 * std::min(units, sms / 2)
                                 : std::min(units, sms);
    const size_t sm = tc_smem(d, NF);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (P.prof) {
      if (P.prof_kd.size() < P.kd.size()) P.prof_kd.resize(P.kd.size());
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
      P.prof_kd[i].push_back({(void*)e0, (void*)e1});
    }
    auto go = [&](auto kern) { kern<<<grid, tc::kThreads, sm, st>>>(tmB, tmA, p); };
    auto go_pair = [&](auto kern) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(tc::kThreads);
      cfg.dynamicSmemBytes = sm;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, kern, tmB, tmA, p);
    };
#define JTFS_GO_KD(NF_, MS_)                                                                        \
  if (d.tc_pair) { if (do_prof) go_pair(tc::k_kd_tc<NF_, MS_, true, 64, true>); else go_pair(tc::k_kd_tc<NF_, MS_, false, 64, true>); } \
  else if (d.tc_Nt == 64) { if (do_prof) go(tc::k_kd_tc<NF_, MS_, true, 64, false>); else go(tc::k_kd_tc<NF_, MS_, false, 64, false>); } \
  else { if (do_prof) go(tc::k_kd_tc<NF_, MS_, true, 32, false>); else go(tc::k_kd_tc<NF_, MS_, false, 32, false>); }
    if (NF == 8) { JTFS_GO_KD(8, 5) }
    else if (NF == 16) { JTFS_GO_KD(16, 2) }
    else { JTFS_GO_KD(32, 1) }
#undef JTFS_GO_KD
    ++launches;
    if (P.prof) cudaEventRecord(e1, st);
    if (do_prof) {
      unsigned long long h[16];
      cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const double nm = (double)grid, ne = (double)grid * 8;
      std::fprintf(stderr,
                   "KDPROF alpha %zu pair %d stat %d nkc %d mpart %d mblk %d Nt %d NBB %d S %d rps %d | mma: total %.0f wait_b %.0f wait_acc %.0f wait_a %.0f | "
                   "epi: total %.0f wait_w %.0f wait_acc %.0f math %.0f (kcycles/CTA)\n",
                   i, d.tc_pair, d.tc_stat, d.tc_nkc, d.tc_mpart, d.tc_mblk, d.tc_Nt, d.tc_NBB, d.tc_S, d.tc_rps, h[0] / nm / 1e3, h[1] / nm / 1e3, h[2] / nm / 1e3, h[3] / nm / 1e3,
                   h[4] / ne / 1e3, h[5] / ne / 1e3, h[6] / ne / 1e3, h[7] / ne / 1e3);
    }
  }
  if (side) {
    cudaEventRecord(ev_join, side);
    cudaStreamWaitEvent(main_st, ev_join, 0);
    cudaEventDestroy(ev_fork);  // released once the recorded work has completed
    cudaEventDestroy(ev_join);
  }
  return launches;
}

}  // namespace jtfs
