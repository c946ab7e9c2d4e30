// FFMA2 (fma.rn.f32x2) throughput by operand form on the B200 (measurement only): the KD
// epilogue's packed FMAs use scalar-broadcast operands (make_float2(p, p) -> .F32 source),
// immediate pairs (compile-time u^k) and plain 64-bit register pairs.  32 warps per SM,
// 8 independent accumulators per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ffma2_forms tools/ffma2_forms.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 upk(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
  return upk(r);
}

template <int OP>
__global__ void __launch_bounds__(1024) k(float* out, const float* in, int iters) {
  float2 acc[8];
  float2 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    acc[i] = make_float2(i, -i);
    x[i] = make_float2(in[(threadIdx.x + i) & 255], in[(threadIdx.x + 3 * i) & 255]);
  }
  const float s = in[threadIdx.x & 255];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (OP == 0) acc[i] = fma2(x[i], x[(i + 1) & 7], acc[i]);                  // registers
      if constexpr (OP == 1) acc[i] = fma2(x[i], make_float2(0.3125f, 0.3125f), acc[i]);  // immediate
      if constexpr (OP == 2) acc[i] = fma2(x[i], make_float2(s, s), acc[i]);              // broadcast
      if constexpr (OP == 3)
        acc[i] = fma2(make_float2(x[i].x, x[i].x), make_float2(-1.f, 1.f), acc[i]);      // both
    }
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += acc[i].x + acc[i].y;
  if (r == 12345.f) out[0] = r;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out, *in;
  cudaMalloc(&out, 4);
  cudaMalloc(&in, 256 * 4);
  cudaMemset(in, 0, 256 * 4);
  const int iters = 4096;
  const char* names[4] = {"register pairs", "immediate pair", "scalar broadcast", "broadcast + immediate"};
  for (int op = 0; op < 4; ++op) {
    auto run = [&](int blocks) {
      switch (op) {
        case 0: k<0><<<blocks, 1024>>>(out, in, iters); break;
        case 1: k<1><<<blocks, 1024>>>(out, in, iters); break;
        case 2: k<2><<<blocks, 1024>>>(out, in, iters); break;
        default: k<3><<<blocks, 1024>>>(out, in, iters); break;
      }
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
    const double ins = 5.0 * sms * 2 * 1024.0 * iters * 8 / 32;  // warp instructions
    const double per_clk_smsp = ins / (ms * 1e-3) / (sms * 4.0) / (clk * 1e3);
    std::printf("FFMA2 %-22s %.3f ms  %.3f warp-instr/clk/SMSP (%.2f cycles each)\n", names[op], ms, per_clk_smsp,
                1.0 / per_clk_smsp);
  }
  return 0;
}
