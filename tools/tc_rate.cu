// tcgen05 kind::tf32 issue-rate microbenchmark: NITER back-to-back MMAs M=128, N, K=8
// into one TMEM accumulator; A K-major SW64; B K-major SW128 (mode 0) or MN-major
// SWIZZLE_128B_BASE32B (mode 1).  Reports cycles per MMA (one CTA per SM, all SMs).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__global__ void k(int mode, int N, int niter, long long* out, int rot, int grp) {
  extern __shared__ __align__(1024) unsigned char raw[];
  uint8_t* base = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint64_t gbar[8];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) ((float*)base)[i] = 0.001f * (i % 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&gbar[i])));
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
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((mode == 1 ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint64_t da = sdesc(smem_u32(base), 16, 512, 4);
    const uint64_t db = mode == 1 ? sdesc(smem_u32(base + 65536), 8 * 128, 512, 1) : sdesc(smem_u32(base + 65536), 16, 1024, 2);
    long long t0 = clock64();
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\telect.sync rx|px, %1;\n\t@px mov.s32 %0, 1;\n\t}" : "+r"(pred) : "r"(0xffffffffu));
    if (pred) {
      for (int i = 0; i < niter; ++i) {
        // rot: rotate over distinct operand addresses (A: 4 KB steps in 48 KB, B: 1 KB k-steps)
        const uint64_t a_off = rot ? (uint64_t)(((i % 12) * 4096) >> 4) : 0;
        const uint64_t b_off = rot ? (uint64_t)(((i % 8) * 1024) >> 4) : 0;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(da + a_off), "l"(db + b_off), "r"(idesc), "r"(1u));
        if (grp && (i % 6) == 5) {
          // grp 1: commit to a ring barrier every 6 MMAs; grp 2: + fence::after_thread_sync;
          // grp 3: + wait for the commit of the group 4 back (like an S=4 ring)
          const int g = (i / 6) % 8;
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&gbar[g])));
          if (grp >= 2) asm volatile("tcgen05.fence::after_thread_sync;");
          if (grp >= 3 && i / 6 >= 4) {
            const int gp = (i / 6 - 4) % 8;
            const uint32_t ph = ((i / 6 - 4) / 8) & 1;
            uint32_t ok = 0;
            while (!ok) asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(smem_u32(&gbar[gp])), "r"(ph));
          }
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    __syncwarp();
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
  long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for (int grp = 0; grp < 4; ++grp)
  for (int rot = 1; rot < 2; ++rot)
  for (int mode = 1; mode < 2; ++mode)
    for (int N : {128, 256}) {
      const int niter = 4800;
      k<<<148, 128, 200000>>>(mode, N, niter, d, rot, grp);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      printf("grp %d rot %d %s B %s N=%3d: %.1f cycles/MMA (ideal %d) -> %.0f MAC/clk/SM\n", grp, rot, cudaGetErrorString(e),
             mode ? "MN-major BASE32B" : "K-major SW128  ", N, avg / niter, 128 * N / 256, 128.0 * N * 8 * niter / avg);
    }
  return 0;
}
