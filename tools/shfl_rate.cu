// Warp-shuffle vs shared-memory exchange throughput on the B200 (measurement only): the
// data movement of one FFT butterfly level between lanes.  A float2 exchanged by two
// shfl.sync.bfly (re, im) against a float2 written (STS.64) and read back (LDS.64) from a
// padded shared buffer, 32 warps per SM, 8 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/shfl_rate tools/shfl_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(1024) k(float* out, int iters) {
  __shared__ float2 buf[1024 * 4];
  float2 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = make_float2(threadIdx.x + i, i);
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (OP == 0) {  // butterfly partner across lanes: 2 x shfl.bfly per float2
        const int m = 1 << (i % 5);
        v[i].x = __shfl_xor_sync(0xffffffffu, v[i].x, m) + v[i].y;
        v[i].y = __shfl_xor_sync(0xffffffffu, v[i].y, m) - v[i].x;
      } else {  // the same exchange through shared memory: STS.64 + LDS.64 of the partner
        const int m = 1 << (i % 5);
        float2* b = buf + (i & 3) * 1024 + (threadIdx.x & ~31);
        b[lane] = v[i];
        __syncwarp();
        const float2 w = b[lane ^ m];
        __syncwarp();
        v[i].x = w.x + v[i].y;
        v[i].y = w.y - v[i].x;
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i].x + v[i].y;
  if (s == 12345.f) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 4);
  const int iters = 2048;
  const char* names[2] = {"shfl.bfly x2 (float2)", "STS.64 + LDS.64 (float2)"};
  for (int op = 0; op < 2; ++op) {
    auto run = [&](int blocks) {
      if (op == 0) k<0><<<blocks, 1024>>>(out, iters);
      else k<1><<<blocks, 1024>>>(out, iters);
    };
    run(sms);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) run(sms * 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    // float2 exchanges (one per thread per chain step)
    const double ex = 5.0 * sms * 2 * 1024.0 * iters * 8;
    const double per_clk_sm = ex / (ms * 1e-3) / sms / (clk * 1e3);
    std::printf("%-26s %.3f ms  %.1f float2 exchanges/clk/SM (%.0f B/clk/SM, at %.0f MHz nominal)\n", names[op], ms,
                per_clk_sm, per_clk_sm * 8, clk / 1e3);
  }
  return 0;
}
