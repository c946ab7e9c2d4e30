// KD on the 5th-generation tensor cores (tcgen05, sm_100a): the frequential
// contraction of the joint stage (Eq. (1) psi_{beta,theta}(lambda), Eq. (2) separable
// joint wavelet) fused with the complex modulus and phi_T pooling of
// Eq. (3).
//
// Per active alpha, the exact frequential operator is the complex matrix
// A[M][K] (plan.cpp).  Real embedding (rows re/im interleaved per TMEM quarter):
//   D[128 lanes x Nt] += A''[128 x K'] * Y''[K' x Nt],   K' = 2K,
//   Y'' rows 2l / 2l+1 = Re / Im Y2_alpha[l]  (KC writes Y2 planar),
//   A'' row (lane q*32 + i): i < 16 -> Re, i >= 16 -> Im of complex row q*16 + i%16.
// 3xTF32: D = A_hi Y_hi + A_hi Y_lo + A_lo Y_hi (hi = fp32 with the low 13
// mantissa bits cleared, lo = x - hi exactly) keeps ~fp32 accuracy.
//
// CTA = 10 warps, persistent over work units (signal, time chunk, M-part):
//   warp 8      TMA producer: Y'' tile (MN-major, SWIZZLE_128B_BASE32B, loaded
//               once per tile and reused by every M-block) + A'' K-records of 16
//               (K-major, SWIZZLE_64B, pre-tiled; 2 per 32 KiB stage of an S-ring)
//   warp 9      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 0..7  epilogue, two sets of 4; set s owns TMEM buffer s and the M-blocks
//               mb = s, s+2, ...: tcgen05.ld -> re/im pairing by shuffle -> |Z| ->
//               phi_T pooling at the retained frames (packed FFMA2) -> per-row
//               accumulators in registers -> global partials at the end of a unit.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "jtfs_internal.h"
#include "kernels.h"

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

// wait + accumulate the waited cycles into acc (instrumentation)
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity, long long& acc) {
  const long long t0 = clock64();
  mbar_wait(bar, parity);
  acc += clock64() - t0;
}

// ---- TMA ----
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
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

// ---- tcgen05 ----
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
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

// UMMA shared-memory descriptor (sm_100 version bit), lbo / sbo in bytes.
//  A, K-major, SWIZZLE_64B (layout 4): 8-row x 64 B atoms, sbo = 512, lbo unused.
//  B, MN-major tf32, SWIZZLE_128B_BASE32B (layout 1, Swizzle<2,5,2>): 4-row x 128 B
//  atoms (32 MN elements), lbo = stride between 32-element MN groups, sbo = 512
//  between 4-row K atoms.  (Plain SWIZZLE_128B MN-major tf32 reads as zeros on
//  sm_100a -- found with tools/tc_unit.cu.)
constexpr uint32_t kLayoutSW128Base32B = 1, kLayoutSW64 = 4;
constexpr int kRec = 16384;    // one A'' K-record: 128 rows x 16 fp32, hi + lo (SWIZZLE_64B images)
constexpr int kStage = 32768;  // one pipeline stage: up to two consecutive K-records
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)layout << 61;
  return d;
}

// instruction descriptor: kind::tf32, D f32, A K-major, B MN-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
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

struct TcParams {
  int K8;        // K' = 2K rounded up to 8: rows of Y'' used
  int nkc;       // 16-wide K chunks of A''
  int Nt;        // time columns per tile (32..256)
  int BR, nbox;  // TMA box rows, boxes per 32-column group
  int colstride; // bytes between 32-column groups of the Y'' tile
  int ybytes;    // bytes of one Y'' tile buffer (hi or lo)
  int S;         // A ring stages
  int tpu;       // tiles per work unit
  int nchunks;   // time chunks per signal (L / (Nt * tpu))
  int n_mpart, n_mblk;  // M-parts and 64-complex-row M-blocks per part
  int L, D, frame0, nframes, Mpad;
  int nsig;
  int expmode;     // measurement only (JTFS_TC_EXPMODE): 1 skip epilogue math, 2 skip TMEM loads too
  unsigned long long* prof;  // measurement only (JTFS_TC_PROF): per-role wait-cycle counters or nullptr
  const float* A;  // A''_alpha pre-tiled 16 KiB chunk records [2 Mpad / 128][nkc]
  const float* g;  // phi_T taps g_alpha[L]
  float* part;
  int64_t part_off, part_stride;
};

constexpr int kThreads = 320;
// warp roles: 0..7 epilogue, 8 TMA producer, 9 MMA issuer (highest warp id: the
// issue arbiter favours high warp ids, so the single MMA thread is never starved)
constexpr int kProdWarp = 8, kMmaWarp = 9;

template <int NF, int MAXSLOT>
__global__ void __launch_bounds__(kThreads, 1) k_kd_tc(const __grid_constant__ CUtensorMap tmY, TcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B align by offsetting the __shared__ array itself (keeps the shared
  // address space visible to the compiler: LDS/STS instead of generic LD/ST)
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  float* Yhi = reinterpret_cast<float*>(base);
  float* Ylo = reinterpret_cast<float*>(base + p.ybytes);
  uint8_t* Ast = base + 2 * p.ybytes;
  float* Wt = reinterpret_cast<float*>(Ast + p.S * kStage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(Wt + p.Nt * NF);
  uint64_t* y_full = bars + 0;
  uint64_t* y_ready = bars + 1;
  uint64_t* y_empty = bars + 2;
  uint64_t* acc_full = bars + 3;   // [2]
  uint64_t* acc_empty = bars + 5;  // [2]
  uint64_t* a_full = bars + 7;     // [S]
  uint64_t* a_empty = bars + 7 + p.S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 7 + 2 * p.S);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(y_full, 1);
    mbar_init(y_ready, 1);
    mbar_init(y_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(acc_full + i, 1);
      mbar_init(acc_empty + i, 4);
    }
    for (int i = 0; i < p.S; ++i) {
      mbar_init(a_full + i, 1);
      mbar_init(a_empty + i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int units = p.nsig * p.nchunks * p.n_mpart;
  const int ngroups = p.Nt / 32;
  const int nst = (p.nkc + 1) / 2;  // A'' stages (<= 2 records of 16 K-columns) per M-block

  if (warp == kProdWarp) {
    // ===================== TMA producer =====================
    // Bulk copies issued by one thread complete one after another (~600 cycles
    // each, measured with tools/bulk_bw.cu), so kIssuers lanes issue in parallel:
    // A'' stage j goes through lane j % kIssuers; the Y'' boxes are spread too.
    // Issuer lanes must divide S so that every ring slot is always served by the
    // same lane (parity waits cannot tell laps apart).
    const int kIssuers = (p.S % 4 == 0) ? 4 : (p.S % 3 == 0) ? 3 : (p.S % 2 == 0) ? 2 : 1;
    if (lane < kIssuers) {
      uint32_t tile_cnt = 0, j = 0, s = 0, ph = 0;
      const uint32_t ytx = (uint32_t)(ngroups * p.nbox * p.BR * 128);
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int mpart = u % p.n_mpart;
        const int chunk = (u / p.n_mpart) % p.nchunks;
        const int b = u / (p.n_mpart * p.nchunks);
        for (int tile = 0; tile < p.tpu; ++tile, ++tile_cnt) {
          mbar_wait(y_empty, (tile_cnt + 1) & 1);
          const int t0 = (chunk * p.tpu + tile) * p.Nt;
          if (p.expmode >= 4) {  // measurement only: no Y'' load
            if (lane == 0) mbar_arrive(y_full);
          } else {
            if (lane == 0) mbar_expect_tx(y_full, ytx);
            __syncwarp((1u << kIssuers) - 1);
            for (int i = lane; i < ngroups * p.nbox; i += kIssuers) {
              const int cg = i / p.nbox, bx = i % p.nbox;
              tma_load_3d(reinterpret_cast<uint8_t*>(Yhi) + cg * p.colstride + bx * p.BR * 128, &tmY, y_full,
                          t0 + cg * 32, bx * p.BR, b);
            }
          }
          for (int mb = 0; mb < p.n_mblk; ++mb) {
            const float* arec = p.A + (size_t)(mpart * p.n_mblk + mb) * p.nkc * (kRec / 4);
            for (int st = 0; st < nst; ++st) {
              if ((int)(j % kIssuers) == lane) {
                mbar_wait(a_empty + s, ph ^ 1);
                if (p.expmode >= 3) {  // measurement only: no A'' load
                  mbar_arrive(a_full + s);
                } else {
                  const uint32_t bytes = (uint32_t)(min(2, p.nkc - 2 * st) * kRec);
                  mbar_expect_tx(a_full + s, bytes);
                  bulk_load(Ast + s * kStage, arec + (size_t)(2 * st) * (kRec / 4), bytes, a_full + s);
                }
              }
              ++j;
              if (++s == (uint32_t)p.S) {
                s = 0;
                ph ^= 1;
              }
            }
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (warp-wide loop, one elected lane issues) =====================
    {
      uint32_t tile_cnt = 0, s = 0, ph = 0;
      uint32_t use0 = 0, use1 = 0;  // per-accumulator-buffer use counters
      long long w_y = 0, w_acc = 0, w_a = 0;
      const long long t_start = clock64();
      const uint32_t idesc = idesc_tf32(p.Nt);
      const int ksteps = p.K8 / 8;
      // descriptor templates; per MMA only the 14-bit start-address field changes
      const uint64_t dA0 = sdesc(smem_u32(Ast), 16, 512, kLayoutSW64);
      const uint64_t dYh0 = sdesc(smem_u32(Yhi), p.colstride, 512, kLayoutSW128Base32B);
      const uint64_t dYl0 = sdesc(smem_u32(Ylo), p.colstride, 512, kLayoutSW128Base32B);
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        for (int tile = 0; tile < p.tpu; ++tile, ++tile_cnt) {
          mbar_wait_t(y_ready, tile_cnt & 1, w_y);
          tc_fence_after();
          for (int mb = 0; mb < p.n_mblk; ++mb) {
            const int ab = mb & 1;  // M-block parity fixes the TMEM buffer and the epilogue set
            const uint32_t use = ab ? use1++ : use0++;
            mbar_wait_t(acc_empty + ab, (use + 1) & 1, w_acc);
            tc_fence_after();
            const uint32_t d = tmem_base + (uint32_t)(ab * p.Nt);
            for (int st = 0; st < nst; ++st) {
              mbar_wait_t(a_full + s, ph, w_a);
              tc_fence_after();
              if (elect_one()) {
                const uint64_t dst = dA0 + (uint64_t)((s * kStage) >> 4);
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                  const uint64_t ah = dst + (uint64_t)((r * kRec) >> 4);
                  const uint64_t al = ah + (uint64_t)((kRec / 2) >> 4);
#pragma unroll
                  for (int ks = 0; ks < 2; ++ks) {
                    const int kstep = 4 * st + 2 * r + ks;
                    if (kstep < ksteps) {
                      const uint64_t ko = (uint64_t)((ks * 32) >> 4), yo = (uint64_t)((kstep * 1024) >> 4);
                      mma_tf32(d, ah + ko, dYh0 + yo, idesc, kstep > 0 ? 1u : 0u);
                      mma_tf32(d, ah + ko, dYl0 + yo, idesc, 1u);
                      mma_tf32(d, al + ko, dYh0 + yo, idesc, 1u);
                    }
                  }
                }
                mma_commit(a_empty + s);
              }
              __syncwarp();
              if (++s == (uint32_t)p.S) {
                s = 0;
                ph ^= 1;
              }
            }
            if (elect_one()) mma_commit(acc_full + ab);
            __syncwarp();
          }
          if (elect_one()) mma_commit(y_empty);
          __syncwarp();
        }
      }
      if (p.prof && lane == 0) {
        atomicAdd(p.prof + 0, (unsigned long long)(clock64() - t_start));
        atomicAdd(p.prof + 1, (unsigned long long)w_y);
        atomicAdd(p.prof + 2, (unsigned long long)w_acc);
        atomicAdd(p.prof + 3, (unsigned long long)w_a);
      }
    }
  } else {
    // ===================== epilogue (warps 0..7) =====================
    const int etid = threadIdx.x;            // 0..255
    const int eset = warp >> 2;              // TMEM accumulator buffer handled
    const int q = warp & 3;                  // TMEM lane quarter (warp_id % 4)
    const bool im = lane >= 16;
    const int rloc = q * 16 + (lane & 15);   // complex row inside an M-block
    uint32_t tile_cnt = 0, use = 0;
    const int yfloats = ngroups * p.colstride / 4;
    long long e_bar = 0, e_y = 0, e_split = 0, e_acc = 0, e_math = 0;
    const long long e_start = clock64();
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int mpart = u % p.n_mpart;
      const int chunk = (u / p.n_mpart) % p.nchunks;
      const int b = u / (p.n_mpart * p.nchunks);
      float2 accr[MAXSLOT][NF / 2];  // pooled partials of my rows (M-blocks eset, eset+2, ...)
#pragma unroll
      for (int k = 0; k < MAXSLOT; ++k)
#pragma unroll
        for (int m = 0; m < NF / 2; ++m) accr[k][m] = make_float2(0.f, 0.f);
      for (int tile = 0; tile < p.tpu; ++tile, ++tile_cnt) {
        long long tb0 = clock64();
        named_bar(1, 256);  // every epilogue warp is done with the previous tile's W
        e_bar += clock64() - tb0;
        mbar_wait_t(y_full, tile_cnt & 1, e_y);
        tb0 = clock64();
        // 3xTF32 split of the Y'' tile, in place (elementwise: layout-agnostic)
        for (int i = etid; i < yfloats; i += 256) {
          const float v = Yhi[i];
          const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
          Yhi[i] = h;
          Ylo[i] = v - h;
        }
        // phi_T pooling taps of this tile, stored [c][NF/2 re-lane pairs | NF/2 im-lane pairs]
        const int t0 = (chunk * p.tpu + tile) * p.Nt;
        for (int i = etid; i < p.Nt * NF; i += 256) {
          const int c = i / NF, m = i % NF;
          float w = 0.f;
          if (m < p.nframes) {
            int t = ((p.frame0 + m) * p.D - (t0 + c)) % p.L;
            if (t < 0) t += p.L;
            w = __ldg(p.g + t);
          }
          Wt[i] = w;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        named_bar(1, 256);
        e_split += clock64() - tb0;
        if (etid == 0) mbar_arrive(y_ready);
        for (int mb = eset; mb < p.n_mblk; mb += 2, ++use) {
          const int ab = eset;
          mbar_wait_t(acc_full + ab, use & 1, e_acc);
          const long long tm0 = clock64();
          tc_fence_after();
          const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * p.Nt);
          float2 part[NF / 2];
#pragma unroll
          for (int m = 0; m < NF / 2; ++m) part[m] = make_float2(0.f, 0.f);
          // re lane (i < 16) takes the even columns, im lane (i + 16) the odd ones
          const float2* wcol = reinterpret_cast<const float2*>(Wt) + (im ? NF / 2 : 0);
          for (int c0 = 0; c0 < p.Nt; c0 += 32) {
            if (p.expmode >= 2) break;
            uint32_t v[32];
            tmem_ld32(tb + c0, v);
            tmem_wait_ld();
            if (p.expmode == 1) {
              part[0].x += __uint_as_float(v[0] ^ v[31]);
              continue;
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float a = __uint_as_float(v[2 * j]), bb = __uint_as_float(v[2 * j + 1]);
              const float recv = __shfl_xor_sync(0xffffffffu, im ? a : bb, 16);
              const float own = im ? bb : a;
              const float mag = sqrt_fast(fmaf(own, own, recv * recv));
              const float4* w4 = reinterpret_cast<const float4*>(wcol + (c0 + 2 * j) * (NF / 2));
#pragma unroll
              for (int m4 = 0; m4 < NF / 4; ++m4) {
                const float4 w = w4[m4];
                part[2 * m4 + 0] = ffma2(make_float2(w.x, w.y), mag, part[2 * m4 + 0]);
                part[2 * m4 + 1] = ffma2(make_float2(w.z, w.w), mag, part[2 * m4 + 1]);
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty + ab);
          e_math += clock64() - tm0;
#pragma unroll
          for (int m = 0; m < NF / 2; ++m) {
            part[m].x += __shfl_xor_sync(0xffffffffu, part[m].x, 16);
            part[m].y += __shfl_xor_sync(0xffffffffu, part[m].y, 16);
          }
          const int slot = mb >> 1;
#pragma unroll
          for (int k = 0; k < MAXSLOT; ++k)
            if (k == slot) {
#pragma unroll
              for (int m = 0; m < NF / 2; ++m)
                accr[k][m] = make_float2(accr[k][m].x + part[m].x, accr[k][m].y + part[m].y);
            }
        }
      }
      // unit done: my rows' pooled partials of this time chunk -> global
      if (!im) {
        float* dst = p.part + (int64_t)b * p.part_stride + p.part_off +
                     ((int64_t)chunk * p.Mpad + (int64_t)mpart * p.n_mblk * 64) * p.nframes;
#pragma unroll
        for (int k = 0; k < MAXSLOT; ++k) {
          const int mb = 2 * k + eset;
          if (mb < p.n_mblk) {
            float* d = dst + (int64_t)(mb * 64 + rloc) * p.nframes;
#pragma unroll
            for (int m = 0; m < NF / 2; ++m) {
              if (2 * m < p.nframes) d[2 * m] = accr[k][m].x;
              if (2 * m + 1 < p.nframes) d[2 * m + 1] = accr[k][m].y;
            }
          }
        }
      }
    }
    if (p.prof && lane == 0) {
      atomicAdd(p.prof + 4, (unsigned long long)(clock64() - e_start));
      atomicAdd(p.prof + 5, (unsigned long long)e_bar);
      atomicAdd(p.prof + 6, (unsigned long long)e_y);
      atomicAdd(p.prof + 7, (unsigned long long)e_split);
      atomicAdd(p.prof + 8, (unsigned long long)e_acc);
      atomicAdd(p.prof + 9, (unsigned long long)e_math);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
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

bool encode(CUtensorMap* m, void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
            const cuuint32_t* box, CUtensorMapSwizzle swz) {
  PFN_encodeTiled fn = get_encoder();
  if (!fn) return false;
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t tc_smem(const AlphaKD& d, int nf) {
  return 1024 + 2 * (size_t)d.tc_ybytes + (size_t)d.tc_S * tc::kStage + (size_t)d.tc_Nt * nf * 4 +
         8 * (7 + 2 * d.tc_S) + 16;
}
int nf_of(int nframes) { return nframes <= 8 ? 8 : nframes <= 16 ? 16 : 32; }
}  // namespace

// choose the per-alpha tensor-core tiling (called by build_plan): the widest
// Y'' tile (Nt, power of two <= 256) that leaves room for >= 3 A'' stages, then as
// many 16 KiB A'' stages as fit (<= 8)
void plan_tc(Plan& P) {
  const int NF = nf_of(P.n_frames);
  const size_t budget = 227 * 1024;
  P.tc_n_mblk = P.Mpad / 64 / P.tc_n_mpart;
  // tuning overrides (measurement only): largest tile width / number of A'' stages
  const char* e_nt = std::getenv("JTFS_TC_NTMAX");
  const char* e_s = std::getenv("JTFS_TC_SMAX");
  const int nt_max = e_nt ? std::max(32, std::atoi(e_nt)) : 256;
  const int s_max = e_s ? std::max(2, std::min(6, std::atoi(e_s))) : 6;
  for (auto& d : P.kd) {
    const int K2 = 2 * d.K;
    d.tc_K8 = (K2 + 7) / 8 * 8;
    d.tc_Kst = (K2 + 15) / 16 * 16;
    d.tc_nkc = d.tc_Kst / 16;
    d.tc_nbox = (d.tc_K8 + 127) / 128;
    d.tc_BR = (d.tc_K8 + d.tc_nbox * 8 - 1) / (d.tc_nbox * 8) * 8;
    d.tc_colstride = d.tc_nbox * d.tc_BR * 128;
    int Nt = std::min(nt_max, d.L);
    for (; Nt > 32; Nt /= 2) {
      d.tc_Nt = Nt;
      d.tc_ybytes = (Nt / 32) * d.tc_colstride;
      d.tc_S = 2;
      if (tc_smem(d, NF) <= budget) break;
    }
    d.tc_Nt = Nt;
    d.tc_ybytes = (Nt / 32) * d.tc_colstride;
    d.tc_S = 2;
    while (d.tc_S < s_max && tc_smem(d, NF) + tc::kStage <= budget) ++d.tc_S;
    if (d.tc_S == 5) d.tc_S = 4;  // issuer lanes must divide S (kernels_tc.cu producer)
    // time chunk per work unit: the largest power of two <= 4096 that still gives
    // about 4 units per SM for a full micro-batch (partials are per chunk)
    {
      int64_t target = (int64_t)P.mb * P.tc_n_mpart * d.L / (4 * 148);
      int ch = 4096;
      while (ch > Nt && ch > target) ch /= 2;
      d.chunk = std::min(ch, d.L);
      if (d.chunk < Nt) d.chunk = Nt;
      d.nchunks = d.L / d.chunk;
    }
    d.tc_tpu = d.chunk / Nt;
    if (d.L < 32 || d.chunk % Nt || tc_smem(d, NF) > budget) P.kd_impl = 0;
  }
}

cudaError_t tc_setup_device(Plan& P) {
  const int NF = nf_of(P.n_frames);
  size_t mx = 0;
  for (auto& d : P.kd) mx = std::max(mx, tc_smem(d, NF));
  cudaError_t e = cudaSuccess;
  if (NF == 8) e = cudaFuncSetAttribute(tc::k_kd_tc<8, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
  else if (NF == 16)
    e = cudaFuncSetAttribute(tc::k_kd_tc<16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
  else e = cudaFuncSetAttribute(tc::k_kd_tc<32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
  if (e != cudaSuccess) return e;
  return cudaSuccess;
}

int launch_kd_tc(Plan& P, const float* y2, int nsig, float* part, cudaStream_t st, int* err) {
  const int NF = nf_of(P.n_frames);
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  for (size_t i = 0; i < P.kd.size(); ++i) {
    const auto& d = P.kd[i];
    CUtensorMap tmY;
    cuuint64_t dims[3] = {(cuuint64_t)d.L, (cuuint64_t)(2 * d.K), (cuuint64_t)nsig};
    cuuint64_t strides[2] = {(cuuint64_t)d.L * 4, (cuuint64_t)(2 * P.y2_total) * 4};
    cuuint32_t box[3] = {32, (cuuint32_t)d.tc_BR, 1};
    if (!encode(&tmY, const_cast<float*>(y2) + 2 * d.y2_off, 3, dims, strides, box,
                CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
      *err = 1;
      return (int)i;
    }
    tc::TcParams p{};
    p.K8 = d.tc_K8;
    p.nkc = (d.tc_K8 + 15) / 16;
    p.Nt = d.tc_Nt;
    p.BR = d.tc_BR;
    p.nbox = d.tc_nbox;
    p.colstride = d.tc_colstride;
    p.ybytes = d.tc_ybytes;
    p.S = d.tc_S;
    p.tpu = d.tc_tpu;
    p.nchunks = d.nchunks;
    p.n_mpart = P.tc_n_mpart;
    p.n_mblk = P.tc_n_mblk;
    p.L = d.L;
    p.D = d.D;
    p.frame0 = P.frame0;
    p.nframes = P.n_frames;
    p.Mpad = P.Mpad;
    p.nsig = nsig;
    p.A = P.d_A2 + d.tc_a2_off;
    {
      const char* e = std::getenv("JTFS_TC_EXPMODE");
      p.expmode = e ? std::atoi(e) : 0;
    }
    static unsigned long long* prof = nullptr;
    const bool do_prof = std::getenv("JTFS_TC_PROF") != nullptr;
    if (do_prof && !prof) cudaMalloc(&prof, 16 * 8);
    if (do_prof) cudaMemsetAsync(prof, 0, 16 * 8, st);
    p.prof = do_prof ? prof : nullptr;
    p.g = P.d_g + d.g_off;
    p.part = part;
    p.part_off = d.part_off;
    p.part_stride = P.part_total;
    const int units = nsig * d.nchunks * P.tc_n_mpart;
    const int grid = std::min(units, sms);
    const size_t sm = tc_smem(d, NF);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (P.prof) {
      if (P.prof_kd.size() < P.kd.size()) P.prof_kd.resize(P.kd.size());
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
      P.prof_kd[i].push_back({(void*)e0, (void*)e1});
    }
    if (NF == 8) tc::k_kd_tc<8, 9><<<grid, tc::kThreads, sm, st>>>(tmY, p);
    else if (NF == 16) tc::k_kd_tc<16, 4><<<grid, tc::kThreads, sm, st>>>(tmY, p);
    else tc::k_kd_tc<32, 2><<<grid, tc::kThreads, sm, st>>>(tmY, p);
    if (P.prof) cudaEventRecord(e1, st);
    if (do_prof) {
      unsigned long long h[16];
      cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const double nm = (double)grid, ne = (double)grid * 8;
      std::fprintf(stderr,
                   "KDPROF alpha %zu Nt %d S %d | mma: total %.0f wait_y %.0f wait_acc %.0f wait_a %.0f | "
                   "epi: total %.0f bar %.0f wait_y %.0f split %.0f wait_acc %.0f math %.0f (kcycles/CTA)\n",
                   i, d.tc_Nt, d.tc_S, h[0] / nm / 1e3, h[1] / nm / 1e3, h[2] / nm / 1e3, h[3] / nm / 1e3,
                   h[4] / ne / 1e3, h[5] / ne / 1e3, h[6] / ne / 1e3, h[7] / ne / 1e3, h[8] / ne / 1e3, h[9] / ne / 1e3);
    }
  }
  *err = 0;
  return (int)P.kd.size();
}

}  // namespace jtfs
