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

#include <algorithm>
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

// =================================================================================
// Isomap (Tenenbaum et al. 2000): the K-NN graph of k_knn_select,
// geodesic distances by blocked Floyd-Warshall (fp64, 64 x 64 tiles: diagonal tile,
// its row / column tiles, then every other tile), classical MDS (double centring of
// the squared geodesics), top eigenpairs by subspace iteration + Rayleigh-Ritz.
// =================================================================================
namespace iso {

constexpr int TB = 64;  // Floyd-Warshall tile

__global__ void k_graph(const double* __restrict__ D, const int32_t* __restrict__ nbr, int n, int npad, int K,
                        double* __restrict__ G) {
  const int64_t tot = (int64_t)npad * npad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / npad), j = (int)(e % npad);
    G[e] = (i == j) ? 0.0 : __longlong_as_double(0x7ff0000000000000LL);
  }
}

// symmetric edges: G[i][j] = G[j][i] = ||F_i - F_j|| for j in N_K(i) (D is exactly symmetric,
// so both writers of an edge write the same value)
__global__ void k_edges(const double* __restrict__ D, const int32_t* __restrict__ nbr, int n, int npad, int K,
                        double* __restrict__ G) {
  const int64_t tot = (int64_t)n * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / K), j = nbr[e];
    const double w = sqrt(D[(int64_t)i * n + j]);
    G[(int64_t)i * npad + j] = w;
    G[(int64_t)j * npad + i] = w;
  }
}

// phase 1: the diagonal tile kb, in shared memory
__global__ void __launch_bounds__(256) k_fw1(double* G, int npad, int kb) {
  __shared__ double t[TB][TB + 1];
  const int o = kb * TB;
  for (int e = threadIdx.x; e < TB * TB; e += 256) t[e / TB][e % TB] = G[(int64_t)(o + e / TB) * npad + o + e % TB];
  __syncthreads();
  for (int k = 0; k < TB; ++k) {
    for (int e = threadIdx.x; e < TB * TB; e += 256) {
      const int i = e / TB, j = e % TB;
      t[i][j] = fmin(t[i][j], t[i][k] + t[k][j]);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < TB * TB; e += 256) G[(int64_t)(o + e / TB) * npad + o + e % TB] = t[e / TB][e % TB];
}

// phase 2: the tiles of block row kb and block column kb (blockIdx.y = 0: row, 1: column)
__global__ void __launch_bounds__(256) k_fw2(double* G, int npad, int kb) {
  extern __shared__ double fsm[];
  double (*dg)[TB + 1] = reinterpret_cast<double (*)[TB + 1]>(fsm);
  double (*t)[TB + 1] = reinterpret_cast<double (*)[TB + 1]>(fsm + TB * (TB + 1));
  int b = blockIdx.x;
  if (b >= kb) ++b;  // skip the diagonal tile
  const bool row = blockIdx.y == 0;
  const int o = kb * TB;
  const int ti = row ? o : b * TB, tj = row ? b * TB : o;
  for (int e = threadIdx.x; e < TB * TB; e += 256) {
    dg[e / TB][e % TB] = G[(int64_t)(o + e / TB) * npad + o + e % TB];
    t[e / TB][e % TB] = G[(int64_t)(ti + e / TB) * npad + tj + e % TB];
  }
  __syncthreads();
  for (int k = 0; k < TB; ++k) {
    for (int e = threadIdx.x; e < TB * TB; e += 256) {
      const int i = e / TB, j = e % TB;
      t[i][j] = row ? fmin(t[i][j], dg[i][k] + t[k][j]) : fmin(t[i][j], t[i][k] + dg[k][j]);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < TB * TB; e += 256) G[(int64_t)(ti + e / TB) * npad + tj + e % TB] = t[e / TB][e % TB];
}

// phase 3: every tile outside block row / column kb; 4 x 4 elements per thread in registers
__global__ void __launch_bounds__(256) k_fw3(double* G, int npad, int kb) {
  extern __shared__ double fsm[];
  double (*a)[TB + 1] = reinterpret_cast<double (*)[TB + 1]>(fsm);             // tile (bi, kb)
  double (*c)[TB + 1] = reinterpret_cast<double (*)[TB + 1]>(fsm + TB * (TB + 1));  // tile (kb, bj)
  int bi = blockIdx.y, bj = blockIdx.x;
  if (bi >= kb) ++bi;
  if (bj >= kb) ++bj;
  const int o = kb * TB;
  for (int e = threadIdx.x; e < TB * TB; e += 256) {
    a[e / TB][e % TB] = G[(int64_t)(bi * TB + e / TB) * npad + o + e % TB];
    c[e / TB][e % TB] = G[(int64_t)(o + e / TB) * npad + bj * TB + e % TB];
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double v[4][4];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) v[p][q] = G[(int64_t)(bi * TB + ty + 16 * p) * npad + bj * TB + tx + 16 * q];
#pragma unroll 4
  for (int k = 0; k < TB; ++k) {
    double x[4], y[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      x[p] = a[ty + 16 * p][k];
      y[p] = c[k][tx + 16 * p];
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) v[p][q] = fmin(v[p][q], x[p] + y[q]);
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) G[(int64_t)(bi * TB + ty + 16 * p) * npad + bj * TB + tx + 16 * q] = v[p][q];
}

// row means of the squared geodesics (fixed-order fp64 sums) + disconnection flag
__global__ void __launch_bounds__(256) k_rowmean(const double* __restrict__ G, int n, int npad,
                                                 double* __restrict__ r, int* flag) {
  __shared__ double red[256];
  const int i = blockIdx.x;
  double s = 0.0;
  bool inf = false;
  for (int j = threadIdx.x; j < n; j += 256) {
    const double g = G[(int64_t)i * npad + j];
    inf |= isinf(g);
    s += g * g;
  }
  if (inf) atomicOr(flag, 1);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) r[i] = red[0] / n;
}

__global__ void __launch_bounds__(256) k_grandmean(const double* __restrict__ r, int n, double* __restrict__ m) {
  __shared__ double red[256];
  double s = 0.0;
  for (int j = threadIdx.x; j < n; j += 256) s += r[j];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *m = red[0] / n;
}

// B = -1/2 (G o G - r 1^T - 1 r^T + m)   (= -1/2 H (G o G) H), written over D
__global__ void k_center(const double* __restrict__ G, int n, int npad, const double* __restrict__ r,
                         const double* __restrict__ m, double* __restrict__ B) {
  const int64_t tot = (int64_t)n * n;
  const double mm = *m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    const double g = G[(int64_t)i * npad + j];
    B[e] = -0.5 * (g * g - r[i] - r[j] + mm);
  }
}

// deterministic start block: a counter-based hash per (row, column)
__global__ void k_vinit(double* V, int n, int p) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * p; e += gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)e * 2654435761u + 0x9e3779b9u;
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    V[e] = (double)h / 4294967296.0 - 0.5;
  }
}

// W = B V (B symmetric n x n, V column-major n x p): one warp per row
__global__ void __launch_bounds__(256) k_bv(const double* __restrict__ B, const double* __restrict__ V, int n, int p,
                                            double* __restrict__ W) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= n) return;
  double acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = 0.0;
  const double* b = B + (int64_t)row * n;
  for (int j = lane; j < n; j += 32) {
    const double x = b[j];
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c < p) acc[c] = fma(x, V[(int64_t)c * n + j], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    if (c >= p) break;
    double s = acc[c];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) W[(int64_t)c * n + row] = s;
  }
}

__device__ double block_sum(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double s = red[0];
  __syncthreads();
  return s;
}

// V = orthonormal basis of W's columns (modified Gram-Schmidt, twice for stability)
__global__ void __launch_bounds__(1024) k_orth(double* __restrict__ W, int n, int p, double* __restrict__ V) {
  __shared__ double red[1024];
  for (int a = 0; a < p; ++a) {
    double* wa = W + (int64_t)a * n;
    for (int pass = 0; pass < 2; ++pass) {
      for (int b = 0; b < a; ++b) {
        const double* vb = V + (int64_t)b * n;
        double d = 0.0;
        for (int j = threadIdx.x; j < n; j += blockDim.x) d = fma(vb[j], wa[j], d);
        d = block_sum(d, red);
        for (int j = threadIdx.x; j < n; j += blockDim.x) wa[j] -= d * vb[j];
        __syncthreads();
      }
    }
    double s = 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) s = fma(wa[j], wa[j], s);
    s = block_sum(s, red);
    const double inv = s > 0 ? 1.0 / sqrt(s) : 0.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) V[(int64_t)a * n + j] = wa[j] * inv;
    __syncthreads();
  }
}

// Rayleigh-Ritz: T = V^T W (W = B V), cyclic Jacobi on the p x p T (one block), Ritz
// vectors of the top c eigenvalues (descending), sign fixed so that the entry of
// largest magnitude is positive, embedding = vector * sqrt(max(lambda, 0))
__global__ void __launch_bounds__(1024) k_ritz(const double* __restrict__ V, const double* __restrict__ W, int n,
                                               int p, int c, double* __restrict__ emb, double* __restrict__ evals) {
  __shared__ double red[1024];
  __shared__ double T[16][16], Q[16][16];
  __shared__ int order[16];
  for (int a = 0; a < p; ++a)
    for (int b = 0; b < p; ++b) {
      double d = 0.0;
      for (int j = threadIdx.x; j < n; j += blockDim.x) d = fma(V[(int64_t)a * n + j], W[(int64_t)b * n + j], d);
      d = block_sum(d, red);
      if (threadIdx.x == 0) T[a][b] = d;
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int a = 0; a < p; ++a) {
      for (int b = 0; b < p; ++b) Q[a][b] = a == b ? 1.0 : 0.0;
      for (int b = a + 1; b < p; ++b) T[a][b] = T[b][a] = 0.5 * (T[a][b] + T[b][a]);
    }
    for (int sweep = 0; sweep < 60; ++sweep) {
      double off = 0.0;
      for (int a = 0; a < p; ++a)
        for (int b = a + 1; b < p; ++b) off += T[a][b] * T[a][b];
      if (off < 1e-300) break;
      for (int a = 0; a < p; ++a)
        for (int b = a + 1; b < p; ++b) {
          if (T[a][b] == 0.0) continue;
          const double th = (T[b][b] - T[a][a]) / (2.0 * T[a][b]);
          const double tt = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
          const double cs = 1.0 / sqrt(tt * tt + 1.0), sn = tt * cs;
          for (int k = 0; k < p; ++k) {  // T <- J^T T J
            const double x = T[k][a], y = T[k][b];
            T[k][a] = cs * x - sn * y;
            T[k][b] = sn * x + cs * y;
          }
          for (int k = 0; k < p; ++k) {
            const double x = T[a][k], y = T[b][k];
            T[a][k] = cs * x - sn * y;
            T[b][k] = sn * x + cs * y;
          }
          for (int k = 0; k < p; ++k) {
            const double x = Q[k][a], y = Q[k][b];
            Q[k][a] = cs * x - sn * y;
            Q[k][b] = sn * x + cs * y;
          }
        }
    }
    bool used[16] = {};
    for (int r = 0; r < c; ++r) {  // descending eigenvalues, ties -> smaller index
      int best = -1;
      for (int a = 0; a < p; ++a)
        if (!used[a] && (best < 0 || T[a][a] > T[best][best])) best = a;
      used[best] = true;
      order[r] = best;
      evals[r] = T[best][best];
    }
  }
  __syncthreads();
  for (int r = 0; r < c; ++r) {
    const int a = order[r];
    // Ritz vector y = V Q[:, a]; sign: largest |y_j| positive (ties -> smaller j)
    double best = 0.0;
    int bj = n;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double y = 0.0;
      for (int b = 0; b < p; ++b) y = fma(V[(int64_t)b * n + j], Q[b][a], y);
      if (fabs(y) > fabs(best) || (fabs(y) == fabs(best) && j < bj)) {
        best = y;
        bj = j;
      }
    }
    // block argmax by (|y|, -j)
    __shared__ double sb[1024];
    __shared__ int sj[1024];
    sb[threadIdx.x] = best;
    sj[threadIdx.x] = bj;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) {
        const double o = sb[threadIdx.x + w];
        const int oj = sj[threadIdx.x + w];
        if (fabs(o) > fabs(sb[threadIdx.x]) || (fabs(o) == fabs(sb[threadIdx.x]) && oj < sj[threadIdx.x])) {
          sb[threadIdx.x] = o;
          sj[threadIdx.x] = oj;
        }
      }
      __syncthreads();
    }
    const double sgn = sb[0] < 0 ? -1.0 : 1.0;
    const double sc = sgn * sqrt(fmax(T[a][a], 0.0));
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double y = 0.0;
      for (int b = 0; b < p; ++b) y = fma(V[(int64_t)b * n + j], Q[b][a], y);
      emb[(int64_t)j * c + r] = y * sc;
    }
    __syncthreads();
  }
}

}  // namespace iso

size_t isomap_workspace_bytes(int64_t n, int K) {
  const int64_t npad = (n + iso::TB - 1) / iso::TB * iso::TB;
  const size_t al = 256;
  auto up = [&](size_t v) { return (v + al - 1) / al * al; };
  return up((size_t)n * n * 8) + up((size_t)npad * npad * 8) + up((size_t)n * K * 4) + 3 * up((size_t)n * 16 * 8) +
         up((size_t)n * 8) + up(64);
}

// the iteration count of the subspace iteration (fixed: no host synchronisation inside)
constexpr int kIsoIters = 300;

cudaError_t launch_isomap(const float* F, int n, int d, int64_t ldf, int K, int c, double* emb, double* evals,
                          void* ws, cudaStream_t st, int* disconnected) {
  using namespace iso;
  const int npad = (n + TB - 1) / TB * TB;
  const size_t al = 256;
  auto up = [&](size_t v) { return (v + al - 1) / al * al; };
  char* w = (char*)ws;
  double* D = (double*)w; w += up((size_t)n * n * 8);
  double* G = (double*)w; w += up((size_t)npad * npad * 8);
  int32_t* nbr = (int32_t*)w; w += up((size_t)n * K * 4);
  double* V = (double*)w; w += up((size_t)n * 16 * 8);
  double* W = (double*)w; w += up((size_t)n * 16 * 8);
  w += up((size_t)n * 16 * 8);
  double* r = (double*)w; w += up((size_t)n * 8);
  double* m = (double*)w;
  int* flag = (int*)(m + 1);
  cudaError_t e = launch_knn(F, n, d, ldf, nullptr, 0, K, nbr, nullptr, nullptr, D, st);
  if (e != cudaSuccess) return e;
  k_graph<<<1184, 256, 0, st>>>(D, nbr, n, npad, K, G);
  k_edges<<<(int)std::min<int64_t>(((int64_t)n * K + 255) / 256, 1184), 256, 0, st>>>(D, nbr, n, npad, K, G);
  const int nb = npad / TB;
  const int fsm = 2 * TB * (TB + 1) * (int)sizeof(double);
  e = cudaFuncSetAttribute(k_fw2, cudaFuncAttributeMaxDynamicSharedMemorySize, fsm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fw3, cudaFuncAttributeMaxDynamicSharedMemorySize, fsm);
  if (e != cudaSuccess) return e;
  for (int kb = 0; kb < nb; ++kb) {
    k_fw1<<<1, 256, 0, st>>>(G, npad, kb);
    if (nb > 1) {
      k_fw2<<<dim3(nb - 1, 2), 256, fsm, st>>>(G, npad, kb);
      k_fw3<<<dim3(nb - 1, nb - 1), 256, fsm, st>>>(G, npad, kb);
    }
  }
  cudaMemsetAsync(flag, 0, sizeof(int), st);
  k_rowmean<<<n, 256, 0, st>>>(G, n, npad, r, flag);
  k_grandmean<<<1, 256, 0, st>>>(r, n, m);
  k_center<<<1184, 256, 0, st>>>(G, n, npad, r, m, D);
  const int p = std::min(n, std::max(2 * c, c + 6) > 16 ? 16 : std::max(2 * c, c + 6));
  k_vinit<<<64, 256, 0, st>>>(W, n, p);
  k_orth<<<1, 1024, 0, st>>>(W, n, p, V);
  for (int it = 0; it < kIsoIters; ++it) {
    k_bv<<<(n + 7) / 8, 256, 0, st>>>(D, V, n, p, W);
    k_orth<<<1, 1024, 0, st>>>(W, n, p, V);
  }
  k_bv<<<(n + 7) / 8, 256, 0, st>>>(D, V, n, p, W);
  k_ritz<<<1, 1024, 0, st>>>(V, W, n, p, c, emb, evals);
  int h = 0;
  e = cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  *disconnected = h;
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace jtfs
