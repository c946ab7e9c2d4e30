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
//   warp 0      TMA producer: Y'' tile (MN-major, SWIZZLE_128B, loaded once per
//               tile and reused by every M-block) + A'' K-chunks (K-major,
//               SWIZZLE_128B, streamed from L2 through an S-stage ring)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..9  epilogue, two sets of 4 (one per TMEM accumulator buffer):
//               tcgen05.ld -> re/im pairing by shuffle -> |Z| -> phi_T pooling at
//               the retained frames -> per-row smem accumulators -> global partials.
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

// ---- TMA ----
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
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
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor (sm_100 version bit), lbo / sbo in bytes.
//  A, K-major, SWIZZLE_128B (layout 2): 8-row x 128 B atoms, sbo = 1024, lbo unused.
//  B, MN-major tf32, SWIZZLE_128B_BASE32B (layout 1, Swizzle<2,5,2>): 4-row x 128 B
//  atoms (32 MN elements), lbo = stride between 32-element MN groups, sbo = 512
//  between 4-row K atoms.  (Plain SWIZZLE_128B MN-major tf32 reads as zeros on
//  sm_100a -- found with tools/tc_unit.cu.)
constexpr uint32_t kLayoutSW128 = 2, kLayoutSW128Base32B = 1;
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

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct TcParams {
  int K8;        // K' = 2K rounded up to 8: rows of Y'' used
  int nkc;       // 32-wide K chunks of A''
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
  const float* g;  // phi_T taps g_alpha[L]
  float* part;
  int64_t part_off, part_stride;
  float* dbg;      // debug dump (JTFS_TC_DEBUG) or nullptr
};

constexpr int kThreads = 320;

template <int NF>
__global__ void __launch_bounds__(kThreads, 1)
    k_kd_tc(const __grid_constant__ CUtensorMap tmAhi, const __grid_constant__ CUtensorMap tmAlo,
            const __grid_constant__ CUtensorMap tmY, TcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B align by offsetting the __shared__ array itself (keeps the shared
  // address space visible to the compiler: LDS/STS instead of generic LD/ST)
  uint8_t* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  float* Yhi = reinterpret_cast<float*>(base);
  float* Ylo = reinterpret_cast<float*>(base + p.ybytes);
  uint8_t* Ast = base + 2 * p.ybytes;
  float* Wt = reinterpret_cast<float*>(Ast + p.S * 32768);
  float* acc = Wt + p.Nt * NF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(acc + p.n_mblk * 64 * NF);
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
  if (warp == 1) {
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

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      uint32_t tile_cnt = 0, a_cnt = 0;
      const uint32_t ytx = (uint32_t)(ngroups * p.nbox * p.BR * 128);
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int mpart = u % p.n_mpart;
        const int chunk = (u / p.n_mpart) % p.nchunks;
        const int b = u / (p.n_mpart * p.nchunks);
        for (int tile = 0; tile < p.tpu; ++tile, ++tile_cnt) {
          mbar_wait(y_empty, (tile_cnt + 1) & 1);
          mbar_expect_tx(y_full, ytx);
          const int t0 = (chunk * p.tpu + tile) * p.Nt;
          for (int cg = 0; cg < ngroups; ++cg)
            for (int bx = 0; bx < p.nbox; ++bx)
              tma_load_3d(reinterpret_cast<uint8_t*>(Yhi) + cg * p.colstride + bx * p.BR * 128, &tmY, y_full,
                          t0 + cg * 32, bx * p.BR, b);
          for (int mb = 0; mb < p.n_mblk; ++mb) {
            const int row0 = (mpart * p.n_mblk + mb) * 128;
            for (int kc = 0; kc < p.nkc; ++kc, ++a_cnt) {
              const int s = a_cnt % p.S;
              const uint32_t k = a_cnt / p.S;
              mbar_wait(a_empty + s, (k + 1) & 1);
              mbar_expect_tx(a_full + s, 32768);
              tma_load_2d(Ast + s * 32768, &tmAhi, a_full + s, kc * 32, row0);
              tma_load_2d(Ast + s * 32768 + 16384, &tmAlo, a_full + s, kc * 32, row0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      uint32_t tile_cnt = 0, a_cnt = 0, mb_cnt = 0;
      const uint32_t idesc = idesc_tf32(p.Nt);
      const uint32_t yhi = smem_u32(Yhi), ylo = smem_u32(Ylo), ast = smem_u32(Ast);
      const int ksteps = p.K8 / 8;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        for (int tile = 0; tile < p.tpu; ++tile, ++tile_cnt) {
          mbar_wait(y_ready, tile_cnt & 1);
          tc_fence_after();
          for (int mb = 0; mb < p.n_mblk; ++mb, ++mb_cnt) {
            const int ab = mb_cnt & 1;
            mbar_wait(acc_empty + ab, ((mb_cnt >> 1) + 1) & 1);
            tc_fence_after();
            const uint32_t d = tmem_base + (uint32_t)(ab * p.Nt);
            for (int kc = 0; kc < p.nkc; ++kc, ++a_cnt) {
              const int s = a_cnt % p.S;
              mbar_wait(a_full + s, (a_cnt / p.S) & 1);
              tc_fence_after();
              const uint32_t ah = ast + s * 32768, al = ah + 16384;
              for (int ks = 0; ks < 4; ++ks) {
                const int kstep = kc * 4 + ks;
                if (kstep >= ksteps) break;
                const uint64_t dah = sdesc(ah + ks * 32, 16, 1024, kLayoutSW128);
                const uint64_t dal = sdesc(al + ks * 32, 16, 1024, kLayoutSW128);
                const uint64_t dbh = sdesc(yhi + kstep * 1024, p.colstride, 512, kLayoutSW128Base32B);
                const uint64_t dbl = sdesc(ylo + kstep * 1024, p.colstride, 512, kLayoutSW128Base32B);
                mma_tf32(d, dah, dbh, idesc, kstep > 0 ? 1u : 0u);
                mma_tf32(d, dah, dbl, idesc, 1u);
                mma_tf32(d, dal, dbh, idesc, 1u);
              }
              mma_commit(a_empty + s);
            }
            mma_commit(acc_full + ab);
          }
          mma_commit(y_empty);
        }
      }
    }
  } else {
    // ===================== epilogue (warps 2..9) =====================
    const int etid = threadIdx.x - 64;       // 0..255
    const int eset = (warp - 2) >> 2;        // TMEM accumulator buffer handled
    const int q = warp & 3;                  // TMEM lane quarter (warp_id % 4)
    const bool im = lane >= 16;
    const int rloc = q * 16 + (lane & 15);   // complex row inside an M-block
    uint32_t tile_cnt = 0, mb_cnt = 0;
    const int yfloats = ngroups * p.colstride / 4;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int mpart = u % p.n_mpart;
      const int chunk = (u / p.n_mpart) % p.nchunks;
      const int b = u / (p.n_mpart * p.nchunks);
      for (int tile = 0; tile < p.tpu; ++tile, ++tile_cnt) {
        named_bar(1, 256);  // every epilogue warp is done with the previous tile (W, acc)
        if (tile == 0)
          for (int i = etid; i < p.n_mblk * 64 * NF; i += 256) acc[i] = 0.f;
        mbar_wait(y_full, tile_cnt & 1);
        // 3xTF32 split of the Y'' tile, in place (elementwise: layout-agnostic)
        for (int i = etid; i < yfloats; i += 256) {
          const float v = Yhi[i];
          const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
          Yhi[i] = h;
          Ylo[i] = v - h;
        }
        // phi_T pooling taps of this tile: Wt[c][m] = g[((frame0 + m) D - t) mod L]
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
        if (p.dbg && blockIdx.x == 0 && tile_cnt == 0)
          for (int i = etid; i < 8192 && i < yfloats; i += 256) p.dbg[i] = Yhi[i];
        if (etid == 0) mbar_arrive(y_ready);
        for (int mb = 0; mb < p.n_mblk; ++mb, ++mb_cnt) {
          const int ab = mb_cnt & 1;
          if (ab != eset) continue;
          mbar_wait(acc_full + ab, (mb_cnt >> 1) & 1);
          tc_fence_after();
          const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * p.Nt);
          if (p.dbg && blockIdx.x == 0 && mb_cnt == 0) {
            uint32_t v[16];
            tmem_ld16(tb, v);
            tmem_wait_ld();
            for (int j = 0; j < 16; ++j) p.dbg[8192 + (q * 32 + lane) * 16 + j] = __uint_as_float(v[j]);
            if (lane == 0 && q == 0) {
              for (int i = 0; i < 8192; ++i) p.dbg[8192 + 2048 + i] = reinterpret_cast<const float*>(Ast)[i];
            }
          }
          float2 part[NF / 2];
#pragma unroll
          for (int m = 0; m < NF / 2; ++m) part[m] = make_float2(0.f, 0.f);
          // re lane (i < 16) takes the even columns, im lane (i + 16) the odd ones
          const float2* wcol = reinterpret_cast<const float2*>(Wt) + (im ? NF / 2 : 0);
          for (int c0 = 0; c0 < p.Nt; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tb + c0, v);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
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
#pragma unroll
          for (int m = 0; m < NF / 2; ++m) {
            part[m].x += __shfl_xor_sync(0xffffffffu, part[m].x, 16);
            part[m].y += __shfl_xor_sync(0xffffffffu, part[m].y, 16);
          }
          if (!im) {
            float2* a = reinterpret_cast<float2*>(acc + (mb * 64 + rloc) * NF);
#pragma unroll
            for (int m = 0; m < NF / 2; ++m) a[m] = make_float2(a[m].x + part[m].x, a[m].y + part[m].y);
          }
        }
      }
      // unit done: write the M-part's pooled partials of this time chunk
      named_bar(1, 256);
      float* dst = p.part + (int64_t)b * p.part_stride + p.part_off +
                   ((int64_t)chunk * p.Mpad + (int64_t)mpart * p.n_mblk * 64) * p.nframes;
      for (int i = etid; i < p.n_mblk * 64 * p.nframes; i += 256) {
        const int r = i / p.nframes, m = i % p.nframes;
        dst[i] = acc[r * NF + m];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
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

size_t tc_smem(const AlphaKD& d, int nf, int n_mblk) {
  return 1024 + 2 * (size_t)d.tc_ybytes + (size_t)d.tc_S * 32768 + (size_t)d.tc_Nt * nf * 4 +
         (size_t)n_mblk * 64 * nf * 4 + 8 * (7 + 2 * d.tc_S) + 16;
}
int nf_of(int nframes) { return nframes <= 8 ? 8 : nframes <= 16 ? 16 : 32; }
}  // namespace

// choose the per-alpha tensor-core tiling (called by build_plan)
void plan_tc(Plan& P) {
  const int NF = nf_of(P.n_frames);
  const size_t budget = 227 * 1024;
  P.tc_n_mblk = P.Mpad / 64 / P.tc_n_mpart;
  for (auto& d : P.kd) {
    const int K2 = 2 * d.K;
    d.tc_K8 = (K2 + 7) / 8 * 8;
    d.tc_Kst = (K2 + 31) / 32 * 32;
    d.tc_nkc = d.tc_Kst / 32;
    d.tc_nbox = (d.tc_K8 + 127) / 128;
    d.tc_BR = (d.tc_K8 + d.tc_nbox * 8 - 1) / (d.tc_nbox * 8) * 8;
    d.tc_colstride = d.tc_nbox * d.tc_BR * 128;
    const size_t fixed = 1024 + (size_t)P.tc_n_mblk * 64 * NF * 4 + 256;
    int Nt = std::min(256, d.L);
    d.tc_S = 2;
    for (; Nt > 32; Nt /= 2) {
      const size_t y = 2 * (size_t)(Nt / 32) * d.tc_colstride;
      if (fixed + y + 2 * 32768 + (size_t)Nt * NF * 4 <= budget) break;
    }
    d.tc_Nt = Nt;
    d.tc_ybytes = (Nt / 32) * d.tc_colstride;
    while (d.tc_S < 4 && tc_smem(d, NF, P.tc_n_mblk) + 32768 <= budget) ++d.tc_S;
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
    if (d.L < 32 || d.chunk % Nt) P.kd_impl = 0;  // tiles need >= 32 time columns
  }
}

cudaError_t tc_setup_device(Plan& P) {
  const int NF = nf_of(P.n_frames);
  size_t mx = 0;
  for (auto& d : P.kd) mx = std::max(mx, tc_smem(d, NF, P.tc_n_mblk));
  cudaError_t e = cudaSuccess;
  if (NF == 8) e = cudaFuncSetAttribute(tc::k_kd_tc<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
  else if (NF == 16) e = cudaFuncSetAttribute(tc::k_kd_tc<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
  else e = cudaFuncSetAttribute(tc::k_kd_tc<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
  if (e != cudaSuccess) return e;
  // A'' tensor maps (constant per plan)
  P.tc_maps.resize(P.kd.size() * 2);
  for (size_t i = 0; i < P.kd.size(); ++i) {
    const auto& d = P.kd[i];
    cuuint64_t dims[2] = {(cuuint64_t)d.tc_Kst, (cuuint64_t)(2 * P.Mpad)};
    cuuint64_t strides[1] = {(cuuint64_t)d.tc_Kst * 4};
    cuuint32_t box[2] = {32, 128};
    if (!encode(reinterpret_cast<CUtensorMap*>(P.tc_maps[2 * i].b), P.d_A2hi + d.tc_a2_off, 2, dims, strides, box,
                CU_TENSOR_MAP_SWIZZLE_128B) ||
        !encode(reinterpret_cast<CUtensorMap*>(P.tc_maps[2 * i + 1].b), P.d_A2lo + d.tc_a2_off, 2, dims, strides,
                box, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

int launch_kd_tc(const Plan& P, const float* y2, int nsig, float* part, cudaStream_t st, int* err) {
  const int NF = nf_of(P.n_frames);
  static float* dbg = nullptr;
  const bool debug = std::getenv("JTFS_TC_DEBUG") != nullptr;
  if (debug && !dbg) cudaMalloc(&dbg, 65536 * 4);
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
    p.nkc = (d.tc_K8 + 31) / 32;
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
    p.g = P.d_g + d.g_off;
    p.part = part;
    p.part_off = d.part_off;
    p.part_stride = P.part_total;
    p.dbg = (debug && i == 0) ? dbg : nullptr;
    const int units = nsig * d.nchunks * P.tc_n_mpart;
    const int grid = std::min(units, sms);
    const size_t sm = tc_smem(d, NF, P.tc_n_mblk);
    const CUtensorMap* mA = reinterpret_cast<const CUtensorMap*>(P.tc_maps[2 * i].b);
    const CUtensorMap* mL = reinterpret_cast<const CUtensorMap*>(P.tc_maps[2 * i + 1].b);
    if (NF == 8) tc::k_kd_tc<8><<<grid, tc::kThreads, sm, st>>>(*mA, *mL, tmY, p);
    else if (NF == 16) tc::k_kd_tc<16><<<grid, tc::kThreads, sm, st>>>(*mA, *mL, tmY, p);
    else tc::k_kd_tc<32><<<grid, tc::kThreads, sm, st>>>(*mA, *mL, tmY, p);
    if (debug && i == 0) {
      std::vector<float> h(65536);
      cudaStreamSynchronize(st);
      cudaMemcpy(h.data(), dbg, 65536 * 4, cudaMemcpyDeviceToHost);
      FILE* f = std::fopen(std::getenv("JTFS_TC_DEBUG"), "wb");
      if (f) {
        std::fwrite(h.data(), 4, h.size(), f);
        std::fclose(f);
      }
    }
  }
  *err = 0;
  return (int)P.kd.size();
}

}  // namespace jtfs
