// K-nearest-neighbour parameter regression on JTFS features.
//
// PAPER.md Sec. 3.5: for every example i, the K examples j != i with the
// smallest Euclidean feature distance (the greedy argmin recursion of P:201-209; ties
// to the smaller index, reading R23), and theta~_i = (1/K) sum_{j in N_K(i)} theta_j.
// Written from the paper; shares no code with oracle/knn.py.
//
//   k_knn_dist   D[i][j] = sum_d (F_i[d] - F_j[d])^2 in fp64 over fp32 features, 64 x 64
//                tiles of the upper triangle (j-tile >= i-tile) mirrored into the lower
//                one (the sum is symmetric term by term, so D is exactly symmetric)
//   k_knn_select one CTA per example: the row of D as (distance, index) keys in shared
//                memory, bitonic sort (lexicographic, so ties go to the smaller index),
//                first K indices (self excluded), theta~ and theta~ / theta in fp64
#include <cuda_runtime.h>

#include <cstdint>

namespace jtfs {
namespace knn {

constexpr int TD = 64;   // tile edge (examples)
constexpr int KC = 32;   // feature chunk

__global__ void __launch_bounds__(256) k_knn_dist(const float* __restrict__ F, int n, int d, int64_t ldf,
                                                  double* __restrict__ D) {
  // map the linear block id onto the upper-triangle tile (ti <= tj)
  const int nt = (n + TD - 1) / TD;
  int t = blockIdx.x, ti = 0;
  while (t >= nt - ti) {
    t -= nt - ti;
    ++ti;
  }
  const int tj = ti + t;
  const int i0 = ti * TD, j0 = tj * TD;
  __shared__ double As[KC][TD + 1];
  __shared__ double Bs[KC][TD + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int k0 = 0; k0 < d; k0 += KC) {
    for (int idx = threadIdx.x; idx < KC * TD; idx += 256) {
      const int r = idx / KC, k = idx % KC;  // consecutive threads along the feature axis
      const int gi = i0 + r, gj = j0 + r, gk = k0 + k;
      As[k][r] = (gi < n && gk < d) ? (double)__ldg(F + (int64_t)gi * ldf + gk) : 0.0;
      Bs[k][r] = (gj < n && gk < d) ? (double)__ldg(F + (int64_t)gj * ldf + gk) : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < KC; ++k) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = As[k][ty + 16 * q];
        b[q] = Bs[k][tx + 16 * q];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double e = a[p] - b[q];
          acc[p][q] = fma(e, e, acc[p][q]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int gi = i0 + ty + 16 * p, gj = j0 + tx + 16 * q;
      if (gi < n && gj < n) {
        D[(int64_t)gi * n + gj] = acc[p][q];
        D[(int64_t)gj * n + gi] = acc[p][q];
      }
    }
}

__device__ __forceinline__ bool key_less(double ka, int ia, double kb, int ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__global__ void __launch_bounds__(1024) k_knn_select(const double* __restrict__ D, int n, int npow2, int K,
                                                     const double* __restrict__ theta, int P,
                                                     int32_t* __restrict__ nbr, double* __restrict__ theta_hat,
                                                     double* __restrict__ ratio) {
  extern __shared__ double sm[];
  double* key = sm;                       // [npow2]
  int* id = (int*)(sm + npow2);           // [npow2]
  const int i = blockIdx.x;
  const double* row = D + (int64_t)i * n;
  for (int j = threadIdx.x; j < npow2; j += blockDim.x) {
    // self and padding sort last (+inf); ties keep index order
    key[j] = (j < n && j != i) ? row[j] : __longlong_as_double(0x7ff0000000000000LL);
    id[j] = j;
  }
  __syncthreads();
  for (int size = 2; size <= npow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < npow2 / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const double kl = key[lo], kh = key[hi];
        const int il = id[lo], ih = id[hi];
        if (key_less(kh, ih, kl, il) == up) {
          key[lo] = kh;
          key[hi] = kl;
          id[lo] = ih;
          id[hi] = il;
        }
      }
      __syncthreads();
    }
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) nbr[(int64_t)i * K + k] = id[k];
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < K; ++k) s += theta[(int64_t)id[k] * P + p];  // fixed order
    const double h = s / (double)K;
    if (theta_hat) theta_hat[(int64_t)i * P + p] = h;
    if (ratio) ratio[(int64_t)i * P + p] = h / theta[(int64_t)i * P + p];
  }
}

}  // namespace knn

size_t knn_workspace_bytes(int64_t n) { return (size_t)n * (size_t)n * sizeof(double); }

int knn_npow2(int n) {
  int p = 2;
  while (p < n) p <<= 1;
  return p;
}

cudaError_t launch_knn(const float* F, int n, int d, int64_t ldf, const double* theta, int P, int K, int32_t* nbr,
                       double* theta_hat, double* ratio, void* ws, cudaStream_t st) {
  using namespace knn;
  double* D = (double*)ws;
  const int nt = (n + TD - 1) / TD;
  k_knn_dist<<<nt * (nt + 1) / 2, 256, 0, st>>>(F, n, d, ldf, D);
  const int np2 = knn_npow2(n);
  const size_t sm = (size_t)np2 * (sizeof(double) + sizeof(int));
  cudaError_t e = cudaFuncSetAttribute(k_knn_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k_knn_select<<<n, 1024, sm, st>>>(D, n, np2, K, theta, P, nbr, theta_hat, ratio);
  return cudaGetLastError();
}

}  // namespace jtfs
