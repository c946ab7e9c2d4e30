// CTA-pair (cta_group::2) kind::f16 MMA microbenchmark for the KD pattern (round-2 groundwork).
//
//   mode 1: one CTA per SM, tcgen05.mma.cta_group::1, M = 128, N = 256 (the current KD)
//   mode 2: CTA pairs (cluster 2x1x1), tcgen05.mma.cta_group::2, M = 256, N = 256: each CTA
//           holds its 128 rows of A and 128 of the 256 columns of B, the leader (rank 0)
//           issues, the commit multicasts to both CTAs' barriers.
// Per 16-wide K chunk 3 MMAs (hi.hi, hi.lo, lo.hi as in KD); ideal 384 cycles per chunk per
// SM in both modes (each SM computes 128 x 256 x 16 per instruction).  A correctness
// check runs first: A = 1 + rank, B = 1 + 2 rank (fp16 constants) -> in CTA r' the
// accumulator columns [0,128) hold 48 n (1 + r') * 1 and [128,256) hold 48 n (1 + r') * 3
// if B is split along N across the pair (n = K chunks).
// Measured (B200, round 1): the check confirms the split (A rows from each CTA's own smem,
// B columns [0,128) from the leader's, [128,256) from the peer's; tcgen05.alloc.cta_group::2
// issued by one warp in each CTA).  Without a producer both modes run at 100 % of the MMA
// rate; with a 2-stage bulk-copy A ring, cta_group::1 reaches 94 % but cta_group::2 only
// 42 %: the peer's copies reach the leader's barrier through a relay arrive, whose latency
// a 2-stage ring cannot hide -- a KD port needs a deeper ring (or TMA .cta_group::2 loads).
//   mode 3: cta_group::1, 6 x N = 128 per K chunk into two accumulators (the layout a
//           spin-pair factorisation needs): 72 % without / 67 % with the ring -- each
//           N = 128 MMA reads 8 KB of smem per 64 cycles, the full port.
//   mode 4: mode 2 with the A ring filled by 2-D tensor copies with .cta_group::2 that
//           complete on the leader's barrier (tools/tma2cta_probe.cu): 93 % with the ring
//           (the relay of mode 2: 42 %).
//   mode 5: mode 4 with 6 x N = 128 into two accumulators (spin-pair layout on a CTA
//           pair): 322 cycles per chunk without / 374 with the ring against 384 for
//           mode 1 -- the pair removes the N = 128 penalty of mode 3 (each SM reads
//           4 KB of A + 2 KB of B per MMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tc_rate2cta tools/tc_rate2cta.cu && tools/tc_rate2cta
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ bool try_wait(uint64_t* bar, uint32_t ph) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(ph));
  return ok;
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k(int nchunks_total, int nkc, long long* out, float* check, const uint8_t* gsrc, int ring,
      const __grid_constant__ CUtensorMap tmA) {
  // MODE 4: MODE 2's pair, the A ring filled by 2-D tensor copies with .cta_group::2 that
  // complete on the leader's barrier (no relay; tools/tma2cta_probe.cu)
  extern __shared__ __align__(1024) unsigned char raw[];
  uint8_t* base = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  __shared__ uint64_t bar, afull[2], gbar[2], lfull[2];
  __shared__ uint32_t tslot;
  constexpr bool PAIR = MODE == 2 || MODE == 4 || MODE == 5;
  const uint32_t rank = PAIR ? cta_rank() : 0;
  constexpr int NN = (MODE == 3 || MODE == 5) ? 128 : 256;  // MMA N
  // A images (64 KB) = 1 + rank, B images (hi at 64 KB, lo at 128 KB) = 1 + 2 rank
  const uint32_t av = rank ? 0x40004000u : 0x3c003c00u;   // fp16 2.0 / 1.0
  const uint32_t bv = rank ? 0x42004200u : 0x3c003c00u;   // fp16 3.0 / 1.0
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)base)[i] = av;
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) ((uint32_t*)(base + 65536))[i] = bv;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 2; ++i) {
      // leader's ring-full barrier: own copy (expect_tx) + the peer's relay arrive in mode 2
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&afull[i])), "r"(MODE == 2 ? 2 : 1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&gbar[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&lfull[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (PAIR) cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  long long t0 = clock64();
  if (threadIdx.x < 32 && rank == 0) {
    const int M = PAIR ? 256 : 128;
    const uint32_t idesc = (1u << 4) | (1u << 16) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = smem_u32(base), bh0 = smem_u32(base + 65536), bl0 = smem_u32(base + 131072);
    // B image per CTA: K16 x (N per CTA) MN-major SW128: 64-column groups of nkc*16 rows x 128 B
    const uint32_t colstride = (uint32_t)(nkc * 16 * 128);
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\telect.sync rx|px, %1;\n\t@px mov.s32 %0, 1;\n\t}"
                 : "+r"(pred)
                 : "r"(0xffffffffu));
    if (pred) {
      for (int c = 0; c < nchunks_total; ++c) {
        const int kc = c % nkc, st = (c / 2) % 2, r = c % 2;
        if (ring && r == 0) {  // the stage's A records landed (both CTAs in mode 2)
          while (!try_wait(&afull[st], (uint32_t)((c / 4) & 1))) {
          }
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const uint32_t rec = ring ? a0 + st * 32768 + r * 8192 : a0 + (c % 4) * 8192;
        const uint64_t da = sdesc(rec, 16, 256, 6), dal = sdesc(rec + 4096, 16, 256, 6);
        const uint64_t bh = sdesc(bh0 + kc * 2048, colstride, 1024, 2), bl = sdesc(bl0 + kc * 2048, colstride, 1024, 2);
        const uint32_t acc = c > 0;
#define MMA2T(D, A, B, ACC)                                                                                   \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" :: \
                   "r"(D), "l"(A), "l"(B), "r"(idesc), "r"(ACC))
#define MMA3(D, A, B, ACC)                                                                                    \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" :: \
                   "r"(D), "l"(A), "l"(B), "r"(idesc), "r"(ACC))
        if (PAIR) {
#define MMA2(A, B, ACC)                                                                                       \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" :: \
                   "r"(tmem), "l"(A), "l"(B), "r"(idesc), "r"(ACC))
          MMA2(da, bh, acc);
          MMA2(da, bl, 1u);
          MMA2(dal, bh, 1u);
        } else if (MODE == 3) {
          // two N = 128 accumulators (columns [0,128) and [128,256)), A images of 4 KB each
          MMA3(tmem, da, bh, acc);
          MMA3(tmem, da, bl, 1u);
          MMA3(tmem, dal, bh, 1u);
          MMA3(tmem + 128, sdesc(rec + 8192 * 0 + 2048, 16, 256, 6), bh, acc);
          MMA3(tmem + 128, sdesc(rec + 2048, 16, 256, 6), bl, 1u);
          MMA3(tmem + 128, sdesc(rec + 4096 + 2048, 16, 256, 6), bh, 1u);
        } else {
#define MMA1(A, B, ACC)                                                                                       \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" :: \
                   "r"(tmem), "l"(A), "l"(B), "r"(idesc), "r"(ACC))
          MMA1(da, bh, acc);
          MMA1(da, bl, 1u);
          MMA1(dal, bh, 1u);
        }
        if (ring && r == 1) {  // stage consumed: free the ring slot in every CTA of the pair
          if (PAIR)
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    smem_u32(&gbar[st])),
                "h"((uint16_t)3));
          else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&gbar[st])));
        }
      }
      if (PAIR)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"((uint16_t)3));
      else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    __syncwarp();
  }
  if (ring && threadIdx.x >= 32 && threadIdx.x < 34) {  // one issuer lane per ring slot
    const int st = threadIdx.x - 32;
    const uint32_t bytes = 16384u;  // 2 records of 8 KB per stage (complex-in-N KD)
    const int nst = nchunks_total / 2;
    for (int j = st; j < nst; j += 2) {
      if (j >= 2)
        while (!try_wait(&gbar[st], (uint32_t)(((j - 2) / 2) & 1))) {
        }
      if (MODE == 4 || MODE == 5) {
        uint32_t lead;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(lead) : "r"(smem_u32(&afull[st])));
        if (rank == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&afull[st])),
                       "r"(2 * bytes));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2 [%0], [%1, {%3, %4}], [%2];" ::"r"(
                smem_u32(base + st * 32768)),
            "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(lead), "r"(0), "r"((j % 64) * 64)
            : "memory");
        continue;
      }
      // leader: completes on afull directly; peer: on a local barrier, relayed below
      uint64_t* fb = (MODE == 2 && rank) ? &lfull[st] : &afull[st];
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(fb)), "r"(bytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(base + st * 32768)),
                   "l"(gsrc + (size_t)((j % 64) * 32768)), "r"(bytes), "r"(smem_u32(fb)));
      if (MODE == 2 && rank) {  // relay: the records are in this CTA's smem -> arrive on the leader's afull
        while (!try_wait(&lfull[st], (uint32_t)((j / 2) & 1))) {
        }
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(&afull[st])));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
      }
    }
  }
  // every CTA waits for the accumulator (its own barrier: multicast commit in mode 2)
  while (!try_wait(&bar, 0)) {
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) out[blockIdx.x / (PAIR ? 2 : 1)] = t1 - t0;
  // correctness: warp w reads TMEM lanes 32w..32w+31, columns 0 and 128
  {
    const int w = threadIdx.x >> 5;
    uint32_t v0, v1;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v0) : "r"(tmem + ((uint32_t)(32 * w) << 16)));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                 : "=r"(v1)
                 : "r"(tmem + ((uint32_t)(32 * w) << 16) + 128u));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if ((threadIdx.x & 31) == 0 && blockIdx.x < 2) {
      check[blockIdx.x * 8 + 2 * w] = __uint_as_float(v0);
      check[blockIdx.x * 8 + 2 * w + 1] = __uint_as_float(v1);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (PAIR) cluster_sync();
  if (threadIdx.x < 32) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  long long* d;
  float* chk;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&chk, 16 * 4);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(k<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  uint8_t* gsrc;
  cudaMalloc(&gsrc, 64 * 32768 + 65536);
  cudaMemset(gsrc, 0, 64 * 32768 + 65536);
  CUtensorMap tmA;
  {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
    cuuint64_t dims[2] = {256, 64 * 32768 / 256}, strides[1] = {256};
    cuuint32_t box[2] = {256, 64}, es[2] = {1, 1};
    ((PFN_encodeTiled)fp)(&tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, gsrc, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  for (int ring = 0; ring < 2; ++ring)
  for (int nkc : {3, 7}) {
    for (int mode = 1; mode <= 5; ++mode) {
      for (int total : {100, 2400}) {
        if (ring && total == 100) continue;
        cudaMemset(chk, 0, 64);
        if (mode == 1) k<1><<<148, 128, 200000>>>(total, nkc, d, chk, gsrc, ring, tmA);
        else if (mode == 2) k<2><<<148, 128, 200000>>>(total, nkc, d, chk, gsrc, ring, tmA);
        else if (mode == 3) k<3><<<148, 128, 200000>>>(total, nkc, d, chk, gsrc, ring, tmA);
        else if (mode == 4) k<4><<<148, 128, 200000>>>(total, nkc, d, chk, gsrc, ring, tmA);
        else k<5><<<148, 128, 200000>>>(total, nkc, d, chk, gsrc, ring, tmA);
        cudaError_t e = cudaDeviceSynchronize();
        const int nrec = (mode == 2 || mode >= 4) ? 74 : 148;
        long long h[148];
        float c[16];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        cudaMemcpy(c, chk, sizeof(c), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < nrec; ++i) avg += h[i];
        avg /= nrec;
        printf("ring %d mode %d (%s) nkc %d chunks %d: %s  %.1f cycles per K chunk (ideal 384) -> %.0f%%\n", ring,
               mode, mode == 1 ? "cta_group::1 M=128 3xN=256" : mode == 2 ? "cta_group::2 M=256 3xN=256" : mode == 3 ? "cta_group::1 M=128 6xN=128" : mode == 4 ? "cta_group::2, TMA.cta_group::2 ring" : "cta_group::2 6xN=128, TMA ring", nkc, total, cudaGetErrorString(e),
               avg / total, 100.0 * 384.0 * total / avg);
        if (total == 100)
          printf("   check (48 n = %d): cta0 lane0 col0 %.0f col128 %.0f | cta1 lane0 col0 %.0f col128 %.0f\n",
                 48 * total, c[0], c[1], c[8], c[9]);
      }
    }
  }
  return 0;
}
