// Bring-up test of the tcgen05 kind::f16 layouts planned for the fp16-split KD:
//   A: K-major, SWIZZLE_32B (8-row x 32 B atoms = 16 fp16 of K per row), one 4 KiB
//      image per 16-wide K chunk (128 rows), SBO = 256 B
//   B: MN-major, SWIZZLE_128B (8 K-rows x 128 B = 64 MN elements per atom),
//      LBO = stride between 64-element MN groups, SBO = 1024 B between 8-row K groups
// D = A[128 x K] * B[K x N] in fp32 (TMEM), read back with tcgen05.ld 32x32b.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tc_unit16 tools/tc_unit16.cu && tools/tc_unit16
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__device__ __forceinline__ uint32_t swz128(uint32_t o) { return o ^ (((o >> 7) & 7u) << 4); }
__device__ __forceinline__ uint32_t swz32(uint32_t o) { return o ^ (((o >> 7) & 1u) << 4); }

template <int N>
__global__ void k_test(const float* A, const float* B, float* D, int K, int layoutA) {
  extern __shared__ unsigned char raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int KC = (K + 15) / 16;
  uint8_t* As = base;                       // KC chunks x 4 KiB
  uint8_t* Bs = base + KC * 4096;           // (N/64) groups x (K16 rows x 128 B)
  const int colstride = KC * 16 * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * KC * 16; i += blockDim.x) {
    const int m = i / (KC * 16), k = i % (KC * 16);
    const int kc = k / 16, kk = k % 16;
    uint32_t off;
    if (layoutA == 6) off = kc * 4096 + swz32((m / 8) * 256 + (m % 8) * 32 + kk * 2);
    else off = kc * 4096 + (m / 8) * 256 + (m % 8) * 32 + kk * 2;  // unused variant
    *(__half*)(As + off) = __float2half_rn(k < K ? A[m * K + k] : 0.f);
  }
  for (int i = tid; i < KC * 16 * N; i += blockDim.x) {
    const int k = i / N, n = i % N;
    const uint32_t off = (n / 64) * colstride + swz128(k * 128 + (n % 64) * 2);
    *(__half*)(Bs + off) = __float2half_rn(k < K ? B[k * N + n] : 0.f);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (tid == 0) {
    // kind::f16: D f32 (bit 4), A/B f16 (0), A K-major, B MN-major (bit 16), N>>3, M>>4
    const uint32_t idesc = (1u << 4) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    for (int kc = 0; kc < KC; ++kc) {
      const uint64_t da = sdesc(smem_u32(As) + kc * 4096, 16, 256, 6);
      const uint64_t db = sdesc(smem_u32(Bs) + kc * 2048, colstride, 1024, 2);
      const uint32_t acc = kc > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar)));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid / 32, lane = tid % 32;
  if (warp < 4) {
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  constexpr int N = 128;
  int fails = 0;
  for (int K : {16, 36, 48}) {
    std::vector<float> A(128 * K), B(K * N), D(128 * N), R(128 * N, 0.f);
    for (int i = 0; i < 128 * K; ++i) A[i] = (float)((i * 7 + 3) % 11 - 5);
    for (int i = 0; i < K * N; ++i) B[i] = (float)((i * 5 + 1) % 9 - 4);
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) R[m * N + n] += A[m * K + k] * B[k * N + n];
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, D.size() * 4);
    cudaFuncSetAttribute(k_test<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    k_test<N><<<1, 128, 100000>>>(dA, dB, dD, K, 6);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int i = 0; i < 128 * N; ++i) {
      err = std::max(err, (double)std::fabs(D[i] - R[i]));
      mx = std::max(mx, (double)std::fabs(R[i]));
    }
    printf("f16 K %d: %s maxerr %.3g (max ref %.3g)  D[0..3]=%g %g %g %g ref %g %g %g %g\n", K, cudaGetErrorString(e),
           err, mx, D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3]);
    fails += !(e == cudaSuccess && err == 0.0);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
  }
  printf(fails ? "FAIL\n" : "PASS\n");
  return fails;
}
