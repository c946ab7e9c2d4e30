// MUFU throughput on the B200 (measurement only): sqrt.approx.ftz.f32, rsqrt.approx,
// ex2.approx, against FFMA, with 8 independent chains per thread and 32 warps per SM.
// The KD epilogue needs one sqrt per |Z| (16384 per 128 x 64 spin-pair block); this says
// which pipe bounds it.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_rate mufu_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters) {
  float v[8], w[8];
  unsigned long long w2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = 1.0f + 1e-3f * (threadIdx.x + i);
    w[i] = 0.5f * v[i];
    w2[i] = (unsigned long long)__float_as_uint(w[i]) * 0x100000001ull;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (OP == 0) asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      if constexpr (OP == 1) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      if constexpr (OP == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
      if constexpr (OP == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(v[i]));
      if constexpr (OP == 4) asm volatile("sqrt.approx.f32 %0, %0;" : "+f"(v[i]));
      if constexpr (OP == 5) {  // 1 sqrt : 8 FFMA (the KD epilogue's mix): max or sum of the two?
        asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
#pragma unroll
        for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(w[(i + k) & 7]));
      }
      if constexpr (OP == 6) {  // 1 sqrt : 4 FFMA2 (packed) -- the same lane-op mix
        asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          unsigned long long& r = w2[(i + k) & 7];
          asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(r));
        }
      }
      if constexpr (OP == 7) {  // the FFMA part of OP 5 alone
#pragma unroll
        for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(w[(i + k) & 7]));
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i] + w[i] + (float)(w2[i] & 1);
  if (s == 12345.f) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4);
  const char* names[8] = {"sqrt.approx.ftz", "rsqrt.approx.ftz", "ex2.approx.ftz", "fma.rn (FFMA)", "sqrt.approx",
                          "1 sqrt + 8 FFMA", "1 sqrt + 4 FFMA2", "8 FFMA (alone)"};
  const int iters = 4096;
  for (int op = 0; op < 8; ++op) {
    auto run = [&](int blocks) {
      switch (op) {
        case 0: k<0><<<blocks, 1024>>>(out, iters); break;
        case 1: k<1><<<blocks, 1024>>>(out, iters); break;
        case 2: k<2><<<blocks, 1024>>>(out, iters); break;
        case 3: k<3><<<blocks, 1024>>>(out, iters); break;
        case 4: k<4><<<blocks, 1024>>>(out, iters); break;
        case 5: k<5><<<blocks, 1024>>>(out, iters); break;
        case 6: k<6><<<blocks, 1024>>>(out, iters); break;
        default: k<7><<<blocks, 1024>>>(out, iters); break;
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
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ops = 5.0 * sms * 2 * 1024.0 * iters * 8;  // (per sqrt / per chain step)
    const double per_s = ops / (ms * 1e-3);
    // per-SM per-cycle at the nominal max clock (kHz attribute): a lower bound if clocks dip
    std::printf("%-20s %.3f ms  %.1f Gop/s  %.2f op/clk/SM (at %.0f MHz)\n", names[op], ms, per_s / 1e9,
                per_s / sms / (clk * 1e3), clk / 1e3);
  }
  return 0;
}
