// Bring-up test of the tcgen05 tf32 MMA path used by kernels_tc.cu:
// one CTA, smem operands written by threads with the SWIZZLE_128B pattern,
// one or more MMAs, tcgen05.ld readback, compare with host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tc_unit tools/tc_unit.cu && ./tc_unit
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
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

__device__ __forceinline__ uint32_t swz(uint32_t off) { return off ^ (((off >> 7) & 7u) << 4); }
__device__ __forceinline__ uint32_t swz32(uint32_t off) { return off ^ (((off >> 7) & 3u) << 5); }
__device__ __forceinline__ uint32_t swz64(uint32_t off) { return off ^ (((off >> 7) & 3u) << 4); }

// mode 0: A K-major SW128, B MN-major SW128 (the KD layout)
// mode 1: A K-major SW128, B K-major SW128
template <int N>
__global__ void k_test(const float* A, const float* B, float* D, int mode, int K) {
  extern __shared__ unsigned char raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* As = base;                 // 128 rows x 128 B, K <= 32
  uint8_t* Bs = base + 16384;         // MN-major: (N/32) groups x (K rows x 128 B); K-major: N rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  if (mode == 3) {  // A K-major SWIZZLE_64B: 16-float (64 B) rows, 8-row atoms of 512 B, K chunks of 16
    for (int i = tid; i < 128 * 32; i += blockDim.x) {
      const int m = i / 32, k = i % 32;
      const uint32_t off = (k / 16) * (128 * 64) + (m / 8) * 512 + (m % 8) * 64 + (k % 16) * 4;
      *(float*)(As + swz64(off)) = (k < K) ? A[m * K + k] : 0.f;
    }
  } else {
    for (int i = tid; i < 128 * 32; i += blockDim.x) {
      const int m = i / 32, k = i % 32;
      const uint32_t off = (m / 8) * 1024 + (m % 8) * 128 + k * 4;
      *(float*)(As + swz(off)) = (k < K) ? A[m * K + k] : 0.f;
    }
  }
  const int KR = (K + 7) / 8 * 8;
  for (int i = tid; i < KR * N; i += blockDim.x) {
    const int k = i / N, n = i % N;
    float v = (k < K) ? B[k * N + n] : 0.f;
    if (mode == 0) {
      const uint32_t off = (n / 32) * (KR * 128) + k * 128 + (n % 32) * 4;
      *(float*)(Bs + swz(off)) = v;
    } else if (mode == 2 || mode == 3) {
      const uint32_t off = (n / 32) * (KR * 128) + k * 128 + (n % 32) * 4;
      *(float*)(Bs + swz32(off)) = v;
    } else {
      const uint32_t off = (n / 8) * 1024 + (n % 8) * 128 + k * 4;
      *(float*)(Bs + swz(off)) = v;
    }
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
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((mode != 1 ? 1u : 0u) << 16) |
                           ((uint32_t)(N >> 3) << 17) | (8u << 24);
    for (int ks = 0; ks < KR / 8; ++ks) {
      uint64_t da = mode == 3 ? sdesc(smem_u32(As) + (ks / 2) * (128 * 64) + (ks % 2) * 32, 16, 512, 4)
                              : sdesc(smem_u32(As) + ks * 32, 16, 1024, 2);
      uint64_t db = mode == 0   ? sdesc(smem_u32(Bs) + ks * 1024, KR * 128, 1024, 2)
                    : mode >= 2 ? sdesc(smem_u32(Bs) + ks * 1024, KR * 128, 512, 1)
                                : sdesc(smem_u32(Bs) + ks * 32, 16, 1024, 2);
      uint32_t acc = ks > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
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
  constexpr int N = 64;
  for (int mode = 0; mode < 4; ++mode)
    for (int K : {8, 24}) {
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
      k_test<N><<<1, 128, 100000>>>(dA, dB, dD, mode, K);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0, mx = 0;
      int nz = 0;
      for (int i = 0; i < 128 * N; ++i) {
        err = std::max(err, (double)std::abs(D[i] - R[i]));
        mx = std::max(mx, (double)std::abs(R[i]));
        nz += D[i] != 0;
      }
      printf("mode %d K %d: %s maxerr %.3g (max ref %.3g) nonzero %d  D[0..3]=%g %g %g %g ref %g %g %g %g\n", mode, K,
             cudaGetErrorString(e), err, mx, nz, D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3]);
      cudaFree(dA);
      cudaFree(dB);
      cudaFree(dD);
    }
  return 0;
}
