// TMEM -> register read bandwidth by tcgen05.ld shape and number of reading warps
// (one CTA per SM, all SMs busy).  Prints bytes per SM-cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tmem_bw tools/tmem_bw.cu && tools/tmem_bw
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int SHAPE>
__device__ __forceinline__ uint32_t ld(uint32_t taddr) {
  uint32_t v[32];
  if constexpr (SHAPE == 0) {  // 32x32b.x32: 32 lanes x 32 columns, 32 regs
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
  } else if constexpr (SHAPE == 1) {  // 16x256b.x8: 16 lanes x 8x256 bits, 32 regs
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
  } else if constexpr (SHAPE == 2) {  // 16x128b.x16
    asm volatile(
        "tcgen05.ld.sync.aligned.16x128b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
  } else {  // 16x64b.x32
    asm volatile(
        "tcgen05.ld.sync.aligned.16x64b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) x ^= v[i];
  return x;
}

template <int SHAPE>
__global__ void k_bw(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  // warp w reads lane quarter w % 4 (32x32b) / lanes 32(w%4) + 16 ((w/4)%2) (16xNb)
  const uint32_t lane_base = SHAPE == 0 ? (uint32_t)((warp & 3) * 32) : (uint32_t)((warp & 3) * 32 + ((warp >> 2) & 1) * 16);
  const uint32_t colspan = SHAPE == 0 ? 32 : SHAPE == 1 ? 64 : SHAPE == 2 ? 64 : 64;  // columns per ld
  uint32_t x = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t col = (uint32_t)((it * colspan + (warp >> 3) * 128) & 511);
    x ^= ld<SHAPE>(tmem + (lane_base << 16) + col);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  if (x == 0x12345678u) sink[0] = x;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 4);
  const int iters = 4096;
  const char* names[4] = {"32x32b.x32", "16x256b.x8", "16x128b.x16", "16x64b.x32"};
  for (int shape = 0; shape < 4; ++shape)
    for (int warps : {4, 8, 12, 16}) {
      cudaMemset(cyc, 0, 8);
      void (*k)(int, unsigned long long*, uint32_t*) =
          shape == 0 ? k_bw<0> : shape == 1 ? k_bw<1> : shape == 2 ? k_bw<2> : k_bw<3>;
      k<<<148, warps * 32>>>(iters, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h = 0;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double cyc_per_cta = (double)h / 148.0;
      const double bytes = (double)warps * iters * 32 * 32 * 4;  // 32 regs x 32 threads x 4 B per ld
      printf("%-12s warps %2d: %s  %.1f B/cycle/SM  (%.0f cycles per ld per warp)\n", names[shape], warps,
             cudaGetErrorString(e), bytes / cyc_per_cta, cyc_per_cta / iters);
    }
  return 0;
}
