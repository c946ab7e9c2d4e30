// L2 -> smem bandwidth of cp.async.bulk: every CTA streams CH-byte chunks of an
// L2-resident buffer through an S-stage ring (mbarrier complete_tx), all SMs.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const char* src, size_t srcbytes, int CH, int S, int nchunks, long long* out, int nissuers) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const bool lanes_mode = nissuers < 0;
  const int ni = lanes_mode ? -nissuers : nissuers;
  const bool me = lanes_mode ? (threadIdx.x < ni) : (threadIdx.x % 32 == 0 && threadIdx.x / 32 < ni);
  if (me) {
    const int w = lanes_mode ? threadIdx.x : threadIdx.x / 32;
    nissuers = ni;
    long long t0 = clock64();
    size_t off = ((size_t)blockIdx.x * 7919 + w * 104729) * 256 % srcbytes;
    for (int c = w; c < nchunks + S; c += nissuers) {
      const int s = c % S;
      if (c >= S) {  // wait for chunk c - S
        uint32_t ok = 0, ph = ((c - S) / S) & 1;
        while (!ok) asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0,1,0,P;\n\t}" : "=r"(ok) : "r"(su(&bar[s])), "r"(ph));
      }
      if (c < nchunks) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(CH) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm + s * CH)),
                     "l"(src + off), "r"(CH), "r"(su(&bar[s])) : "memory");
        off = (off + CH) % (srcbytes - CH);
        off &= ~(size_t)255;
      }
    }
    if (w == 0) out[blockIdx.x] = clock64() - t0;
  }
}
int main() {
  size_t sb = 4 << 20; char* src; cudaMalloc(&src, sb); cudaMemset(src, 1, sb);
  long long* d; cudaMalloc(&d, 296 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int CH : {8192, 16384})
    for (int S : {4, 8}) 
      for (int ni : {1, 4, -4}) {
        if (S % ni) continue;
        const int nchunks = (64 << 20) / CH / 148 ;
        k<<<148, 128, CH * S>>>(src, sb, CH, S, nchunks, d, ni);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("%s CH=%6d S=%d issuers=%d: %.1f B/clk/SM (slowest CTA)\n", cudaGetErrorString(e), CH, S, ni, (double)CH * nchunks / mx);
      }
  return 0;
}
