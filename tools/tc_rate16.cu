// kind::f16 MMA-stream microbenchmark of the KD pattern (one CTA per SM, all SMs):
//   mode 0 (current KD): per 16-wide K chunk 6 MMAs M=128 N=128 -- re: A0.Bh, A0.Bl, A1.Bh;
//          im: A2.Bh, A2.Bl, A3.Bh (A images 4 KB, K-major SW32; B MN-major SW128)
//   mode 1 (complex-in-N): per K chunk 3 MMAs M=128 N=256 -- A0.Bh, A0.Bl, A1.Bh
// Both do the same MACs per K chunk (ideal 384 cycles at 4096 MAC/clk).  Operands
// rotate over nkc chunks like an M-block; a commit every 2 chunks (a ring stage).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tc_rate16 tools/tc_rate16.cu && tools/tc_rate16
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(
          d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__global__ void k(int mode, int nchunks_total, int nkc, long long* out, const uint8_t* gsrc, int ring) {
  extern __shared__ __align__(1024) unsigned char raw[];
  uint8_t* base = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  __shared__ uint64_t bar, gbar[8], afull[2];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 200000 / 4 - 300; i += blockDim.x) ((uint32_t*)base)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&gbar[i])));
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&afull[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    const int N = mode == 0 ? 128 : 256;
    const uint32_t idesc = (1u << 4) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    // A ring: 2 stages x 32 KB at base; B: hi at base + 64 KB, lo at + 128 KB (K16 x N fp16 each <= 57 KB)
    const uint32_t a0 = smem_u32(base), bh0 = smem_u32(base + 65536), bl0 = smem_u32(base + 131072);
    const uint32_t colstride = (uint32_t)(nkc * 16 * 128);
    long long t0 = clock64();
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\telect.sync rx|px, %1;\n\t@px mov.s32 %0, 1;\n\t}"
                 : "+r"(pred)
                 : "r"(0xffffffffu));
    if (pred) {
      for (int c = 0; c < nchunks_total; ++c) {
        const int kc = c % nkc, st = (c / 2) % 2, r = c % 2;
        if (ring && r == 0) {  // wait for the stage's records (producer ring)
          const uint32_t ph = (uint32_t)((c / 4) & 1);
          uint32_t ok = 0;
          while (!ok)
            asm volatile(
                "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
                : "=r"(ok)
                : "r"(smem_u32(&afull[st])), "r"(ph));
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const uint32_t rec = a0 + st * 32768 + r * 16384;
        const uint64_t bh = sdesc(bh0 + kc * 2048, colstride, 1024, 2), bl = sdesc(bl0 + kc * 2048, colstride, 1024, 2);
        const uint32_t acc = kc > 0;
        if (mode == 0) {
          mma(tmem, sdesc(rec, 16, 256, 6), bh, idesc, acc);
          mma(tmem, sdesc(rec, 16, 256, 6), bl, idesc, 1);
          mma(tmem, sdesc(rec + 4096, 16, 256, 6), bh, idesc, 1);
          mma(tmem + 128, sdesc(rec + 8192, 16, 256, 6), bh, idesc, acc);
          mma(tmem + 128, sdesc(rec + 8192, 16, 256, 6), bl, idesc, 1);
          mma(tmem + 128, sdesc(rec + 12288, 16, 256, 6), bh, idesc, 1);
        } else {
          mma(tmem, sdesc(rec, 16, 256, 6), bh, idesc, acc);
          mma(tmem, sdesc(rec, 16, 256, 6), bl, idesc, 1);
          mma(tmem, sdesc(rec + 4096, 16, 256, 6), bh, idesc, 1);
        }
        if (r == 1) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(&gbar[st])));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    __syncwarp();
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  if (ring && threadIdx.x >= 32 && threadIdx.x < 34) {  // 2 issuer lanes, one per ring slot
    const int st = threadIdx.x - 32;
    const uint32_t bytes = mode == 0 ? 32768u : 16384u;  // 2 records of 16 KB (current) / 8 KB (complex-in-N)
    const int nst = nchunks_total / 2;
    for (int j = st; j < nst; j += 2) {
      if (j >= 2) {  // slot free once the MMAs of stage j - 2 completed
        const uint32_t ph = (uint32_t)(((j - 2) / 2) & 1);
        uint32_t ok = 0;
        while (!ok)
          asm volatile(
              "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
              : "=r"(ok)
              : "r"(smem_u32(&gbar[st])), "r"(ph));
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&afull[st])), "r"(bytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(base + st * 32768)),
                   "l"(gsrc + (size_t)((j % 64) * 32768)), "r"(bytes), "r"(smem_u32(&afull[st])));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  uint8_t* gsrc;
  cudaMalloc(&gsrc, 64 * 32768 + 65536);
  cudaMemset(gsrc, 0, 64 * 32768 + 65536);
  for (int ring = 0; ring < 2; ++ring)
  for (int nkc : {3, 7}) {
    for (int mode = 0; mode < 2; ++mode) {
      const int total = 2400;
      k<<<148, 128, 200000>>>(mode, total, nkc, d, gsrc, ring);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      printf("ring %d nkc %d %s: %s  %.1f cycles per K chunk (ideal 384) -> %.0f%%\n", ring, nkc,
             mode == 0 ? "6 x N=128 (re | im regions)" : "3 x N=256 (complex in N)   ", cudaGetErrorString(e),
             avg / total, 100.0 * 384.0 * total / avg);
    }
  }
  return 0;
}
