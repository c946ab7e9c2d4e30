// Probe (round-2 groundwork): can the peer CTA of a CTA pair signal the LEADER's mbarrier
// when its tensor copy lands in its own shared memory?  cp.async.bulk.tensor with
// .cta_group::2: each CTA loads 16 KB of a global buffer into its own smem; both copies
// complete_tx on CTA 0's barrier (armed once with 32 KB); CTA 0 waits, then both CTAs
// check their data after a cluster barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma2cta_probe tools/tma2cta_probe.cu && tools/tma2cta_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int VARIANT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1)
    k(const __grid_constant__ CUtensorMap tm, int* result) {
  extern __shared__ __align__(1024) unsigned char raw[];
  uint8_t* buf = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) {
    uint32_t lead;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(lead) : "r"(smem_u32(&bar)));
    if (rank == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(32768));
    // both CTAs: 16 KB (box 256 B x 64 rows) at rows [64 rank, 64 rank + 64) into their own smem
    if (VARIANT == 0)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2 [%0], [%1, {%3, %4}], [%2];" ::"r"(
              smem_u32(buf)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(lead), "r"(0), "r"((int)(64 * rank))
          : "memory");
    else  // control: plain copy completing on the executing CTA's own barrier (leader only)
      if (rank == 0)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                smem_u32(buf)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&bar)), "r"(0), "r"(0)
            : "memory");
  }
  if (rank == 0 && threadIdx.x == 0) {
    uint32_t ok = 0;
    long long t0 = clock64();
    while (!ok && clock64() - t0 < 2000000000LL)
      asm volatile(
          "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar)));
    result[0] = ok ? 1 : -1;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (VARIANT == 0 || rank == 0) {
    // verify: byte b of row r holds (r * 7 + b) & 0xff
    int bad = 0;
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) {
      const int r = 64 * rank + i / 256, b = i % 256;
      if (buf[i] != (uint8_t)((r * 7 + b) & 0xff)) ++bad;
    }
    atomicAdd(result + 1 + rank, bad);
  }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  uint8_t h[128 * 256];
  for (int r = 0; r < 128; ++r)
    for (int b = 0; b < 256; ++b) h[r * 256 + b] = (uint8_t)((r * 7 + b) & 0xff);
  uint8_t* g;
  cudaMalloc(&g, sizeof(h));
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  CUtensorMap tm;
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
  cuuint64_t dims[2] = {256, 128}, strides[1] = {256};
  cuuint32_t box[2] = {256, 64}, es[2] = {1, 1};
  CUresult cr = ((PFN_encodeTiled)fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, g, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)cr);
  int* res;
  cudaMalloc(&res, 16);
  for (int variant : {1, 0}) {
    cudaMemset(res, 0, 16);
    if (variant == 0) {
      cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
      k<0><<<2, 64, 20000>>>(tm, res);
    } else {
      cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
      k<1><<<2, 64, 20000>>>(tm, res);
    }
    cudaError_t e = cudaDeviceSynchronize();
    int hr[4] = {0, 0, 0, 0};
    cudaMemcpy(hr, res, 16, cudaMemcpyDeviceToHost);
    printf("variant %d (%s): %s  barrier %d  bad bytes cta0 %d cta1 %d\n", variant,
           variant == 0 ? ".cta_group::2, leader barrier" : "control, own barrier", cudaGetErrorString(e), hr[0],
           hr[1], hr[2]);
    if (e != cudaSuccess) break;
  }
  return 0;
}
