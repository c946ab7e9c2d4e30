// CUDA kernels (sm_100a) of the forward JTFS hot path.
//
//   KA  reflect-pad + DFT of x                                  (R6)
//   KB  band-multiply psi_lambda + fold + IDFT + modulus -> U1, DFT(U1) -> U1hat
//       (scalogram X = |x * psi_lambda|, critically subsampled: P:71; R5)
//   KS  S0 / S1 / Y_phi: phi_T averaging at rate T by spectral folding
//   KC  U1hat * psi_alpha + fold + IDFT -> Y2_alpha (Eq. (1) temporal rate)
//   KD  frequential contraction along lambda with psi_{beta,theta} / phi_F (Eq. (1)
//       P:79, Eq. (2)) + complex modulus + phi_T pooling (Eq. (3))
//   KE  phi_F pooling along lambda, phi-only paths, out_3D packing
//
// Every spectral decimation is done by folding (aliasing-sum) the band-limited
// product spectrum to the decimated length before a shorter inverse FFT, which is
// the exact identity IDFT_L(X)[n d] = (1/d) IDFT_{L/d}(fold X)[n].
#include <cuda_fp16.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <type_traits>
#include <utility>

#include "fft.cuh"
#include "jtfs_internal.h"
#include "kernels.h"

namespace jtfs {
namespace dev {

// ---------------------------------------------------------------------------------
// gather: output bin i (of a length-L fold) of the band-limited product src * band
// ---------------------------------------------------------------------------------
__device__ __forceinline__ float2 fold_value(const float2* __restrict__ src, const FoldRow& d,
                                             const float* __restrict__ bandvals, int i, int L) {
  // first alias t0 = (i - m0) mod L handled without a loop (the common case has at
  // most one alias, so the loads of several bins can be in flight together); L is a
  // power of two (every FFT length), so the residue is a mask, not a division
  int t = (i - d.m0) & (L - 1);
  float2 acc = make_float2(0.f, 0.f);
  if (t < d.len) {
    int p = d.m0 + t;
    if (p >= d.Lsrc) p -= d.Lsrc;
    const float2 x = src[d.src_off + p];
    const float f = __ldg(bandvals + d.band_off + t);
    acc = make_float2(x.x * f, x.y * f);
    for (t += L; t < d.len; t += L) {
      p = d.m0 + t;
      if (p >= d.Lsrc) p -= d.Lsrc;
      const float2 y = src[d.src_off + p];
      const float g = __ldg(bandvals + d.band_off + t);
      acc.x = fmaf(y.x, g, acc.x);
      acc.y = fmaf(y.y, g, acc.y);
    }
  }
  return acc;
}

// ---------------------------------------------------------------------------------
// problems: load(rho, i) -> element i of input row rho; store(rho, o, v)
// ---------------------------------------------------------------------------------
struct ProbPad {  // KA (fp64): x_pad[b][i] = x[b][reflect(i - pad_left)]; X_hat rounded per bin
  using CT = double2;
  const float* x;
  float2* xhat;
  int N, N_pad, pad_left, periodic;
  __device__ double2 load(int b, int i) const {
    int n = i - pad_left;
    if (!periodic) {
      if (n < 0) n = -n;
      if (n >= N) n = 2 * (N - 1) - n;
    }
    return make_double2((double)__ldg(x + (int64_t)b * N + n), 0.0);
  }
  __device__ void store(int b, int o, double2 v) const {
    xhat[(int64_t)b * N_pad + o] = make_float2((float)v.x, (float)v.y);
  }
};

struct ProbFold {  // rows rho = b * nrows + r: band-multiply + fold gather
  using CT = float2;
  const float2* src;
  int64_t src_stride;
  const FoldRow* rows;
  int nrows;
  const float* bandvals;
  int L;
  // outputs
  float* dst_real;    // modulus output (U1) or nullptr
  float* dst_planar;  // planar complex output (Y2: re row at dst_off, im row at dst_off + L) or nullptr
  int64_t dst_stride;
  unsigned int* u1max = nullptr;  // first order: per (signal, lambda = rows[r].pad) max |U1| (float bits)
  int n1 = 0;
  __device__ float2 load(int rho, int i) const {
    const int b = rho / nrows, r = rho % nrows;
    return fold_value(src + (int64_t)b * src_stride, rows[r], bandvals, i, L);
  }
  __device__ void store(int rho, int o, float2 v) const {
    const int b = rho / nrows, r = rho % nrows;
    const FoldRow& d = rows[r];
    if (dst_real) {
      const float u = sqrtf(fmaf(v.x, v.x, v.y * v.y)) * d.scale;
      dst_real[(int64_t)b * dst_stride + d.dst_off + o] = u;
      if (u1max) atomicMax(u1max + (int64_t)b * n1 + d.pad, __float_as_uint(u));
    } else {
      float* row = dst_planar + (int64_t)b * dst_stride + d.dst_off;
      row[o] = v.x * d.scale;
      row[L + o] = v.y * d.scale;
    }
  }
};

// KC for the tensor-core KD: the Y2 row goes straight into KD's packed fp16 B layout,
// x s = hi + lo (hi = rn16(x s), lo = rn16(x s - hi)) with the per-(signal, alpha) power-of-
// two scale s of k_yscale, written as rows [hi; lo; hi] (segments y.seg halves apart) with
// (re, im) interleaved per time column (kernels_tc.cu)
struct ProbFold16 {
  using CT = float2;
  const float2* src;
  int64_t src_stride;
  const FoldRow* rows;
  int nrows;
  const float* bandvals;
  int L;
  const Y16Row* y16rows;
  __half* y16;
  int64_t y16_stride;
  const float* ysc;  // [signal][n_alpha] scales
  int nalpha;
  __device__ float2 load(int rho, int i) const {
    const int b = rho / nrows, r = rho % nrows;
    return fold_value(src + (int64_t)b * src_stride, rows[r], bandvals, i, L);
  }
  __device__ void store(int rho, int o, float2 v) const {
    const int b = rho / nrows, r = rho % nrows;
    const Y16Row y = y16rows[r];
    const float s = rows[r].scale * __ldg(ysc + (int64_t)b * nalpha + y.aslot);
    const float xr = v.x * s, xi = v.y * s;
    const __half2 hi = __floats2half2_rn(xr, xi);
    const float2 f = __half22float2(hi);
    const __half2 lo = __floats2half2_rn(xr - f.x, xi - f.y);
    __half* dst = y16 + (int64_t)b * y16_stride + y.off + 2 * o;
    *reinterpret_cast<__half2*>(dst) = hi;
    *reinterpret_cast<__half2*>(dst + y.seg) = lo;
    *reinterpret_cast<__half2*>(dst + 2 * y.seg) = hi;
  }
};

struct ProbRealFwd {  // U1 (real) -> U1hat
  using CT = float2;
  const float* u1;
  float2* u1hat;
  int64_t stride;
  const FoldRow* rows;
  int nrows;
  __device__ float2 load(int rho, int i) const {
    const int b = rho / nrows, r = rho % nrows;
    return make_float2(u1[(int64_t)b * stride + rows[r].dst_off + i], 0.f);
  }
  __device__ void store(int rho, int o, float2 v) const {
    const int b = rho / nrows, r = rho % nrows;
    u1hat[(int64_t)b * stride + rows[r].dst_off + o] = v;
  }
};

template <class T>
struct ProbPlain {  // jtfs_debug_fft: contiguous complex rows in -> rows out (the bare FFT engine)
  using CT = T;
  const T* in;
  T* out;
  int L;
  __device__ T load(int rho, int i) const { return in[(int64_t)rho * L + i]; }
  __device__ void store(int rho, int o, T v) const { out[(int64_t)rho * L + o] = v; }
};

// ---------------------------------------------------------------------------------
// row-bound accessors: kernels whose CTA works on one row rho (four-step passes) bind the
// problem to that row once, so the row's parameters (FoldRow, output offsets, scales)
// sit in registers.  Through the generic (rho, i) interface every element re-read them
// after the previous element's global store (the compiler cannot prove the tables and
// the outputs do not alias): one dependent L1/L2 load per stored element.
// ---------------------------------------------------------------------------------
template <class P>
struct BoundRow {  // generic: forwards to (rho, i) (a copy: no address of the kernel parameter)
  P p;
  int rho;
  __device__ __forceinline__ typename P::CT load(int i) const { return p.load(rho, i); }
  __device__ __forceinline__ void store(int o, typename P::CT v) const { p.store(rho, o, v); }
};
template <class P>
__device__ __forceinline__ BoundRow<P> bind_row(const P& p, int rho) {
  return BoundRow<P>{p, rho};
}

struct BoundFold {  // ProbFold / ProbFold16 loads: the band-limited fold gather of one row
  const float2* src;
  FoldRow d;
  const float* bandvals;
  int L;
  __device__ __forceinline__ float2 load(int i) const { return fold_value(src, d, bandvals, i, L); }
};

struct BoundFold16 : BoundFold {  // + KC's packed fp16 store
  __half* dst;  // hi segment of the row (lo at + seg, hi again at + 2 seg)
  int64_t seg;
  float s;
  __device__ __forceinline__ void store(int o, float2 v) const {
    const float xr = v.x * s, xi = v.y * s;
    const __half2 hi = __floats2half2_rn(xr, xi);
    const float2 f = __half22float2(hi);
    const __half2 lo = __floats2half2_rn(xr - f.x, xi - f.y);
    __half* q = dst + 2 * o;
    *reinterpret_cast<__half2*>(q) = hi;
    *reinterpret_cast<__half2*>(q + seg) = lo;
    *reinterpret_cast<__half2*>(q + 2 * seg) = hi;
  }
};
__device__ __forceinline__ BoundFold16 bind_row(const ProbFold16& p, int rho) {
  const int b = rho / p.nrows, r = rho % p.nrows;
  BoundFold16 x;
  x.src = p.src + (int64_t)b * p.src_stride;
  x.d = p.rows[r];
  x.bandvals = p.bandvals;
  x.L = p.L;
  const Y16Row y = p.y16rows[r];
  x.dst = p.y16 + (int64_t)b * p.y16_stride + y.off;
  x.seg = y.seg;
  x.s = x.d.scale * __ldg(p.ysc + (int64_t)b * p.nalpha + y.aslot);
  return x;
}

struct BoundFoldP : BoundFold {  // ProbFold: + its store (modulus + row max, or planar complex)
  float* real_row;    // dst_real row or nullptr
  float* planar_row;  // dst_planar row (re; im at + L) or nullptr
  unsigned int* umax; // the row's max |U1| slot or nullptr
  __device__ __forceinline__ void store(int o, float2 v) const {
    if (real_row) {
      const float u = sqrtf(fmaf(v.x, v.x, v.y * v.y)) * d.scale;
      real_row[o] = u;
      if (umax) atomicMax(umax, __float_as_uint(u));
    } else {
      planar_row[o] = v.x * d.scale;
      planar_row[L + o] = v.y * d.scale;
    }
  }
};
__device__ __forceinline__ BoundFoldP bind_row(const ProbFold& p, int rho) {
  const int b = rho / p.nrows, r = rho % p.nrows;
  BoundFoldP x;
  x.src = p.src + (int64_t)b * p.src_stride;
  x.d = p.rows[r];
  x.bandvals = p.bandvals;
  x.L = p.L;
  x.real_row = p.dst_real ? p.dst_real + (int64_t)b * p.dst_stride + x.d.dst_off : nullptr;
  x.planar_row = p.dst_planar ? p.dst_planar + (int64_t)b * p.dst_stride + x.d.dst_off : nullptr;
  x.umax = p.u1max ? p.u1max + (int64_t)b * p.n1 + x.d.pad : nullptr;
  return x;
}

struct BoundRealFwd {  // ProbRealFwd: one real row in, its spectrum out
  const float* in;
  float2* out;
  __device__ __forceinline__ float2 load(int i) const { return make_float2(in[i], 0.f); }
  __device__ __forceinline__ void store(int o, float2 v) const { out[o] = v; }
};
__device__ __forceinline__ BoundRealFwd bind_row(const ProbRealFwd& p, int rho) {
  const int b = rho / p.nrows, r = rho % p.nrows;
  const int64_t off = (int64_t)b * p.stride + p.rows[r].dst_off;
  return BoundRealFwd{p.u1 + off, p.u1hat + off};
}
// problems with a row-bound accessor of their own (the others keep the (rho, i) interface);
// k_fft_rows stages one per row in shared memory, kBoundRowBytes each
constexpr int kBoundRowBytes = 128;
template <class P>
constexpr bool kRowBound = !std::is_same<decltype(bind_row(std::declval<const P&>(), 0)), BoundRow<P>>::value;

// ---------------------------------------------------------------------------------
// single-CTA FFT of G rows per block
// ---------------------------------------------------------------------------------
template <int LOG2L, int G, int NT, int DIR, class P>
__global__ void __launch_bounds__(NT) k_fft_rows(P prob, int nrows, const typename P::CT* __restrict__ Wtab) {
  using CT = typename P::CT;
  constexpr int L = 1 << LOG2L, LS = pad_row(L), EPT = G * L / NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CT* smem = reinterpret_cast<CT*>(smem_raw);
  CT* Ws = smem + G * LS;
  stage_twiddles<LOG2L, NT>(Ws, Wtab + tw_offset(LOG2L));
  const int rho0 = blockIdx.x * G;
  if constexpr (LOG2L >= 3 && kRowBound<P>) {
    // the G rows' bound accessors staged once in shared memory (see bind_row)
    using BR = decltype(bind_row(prob, 0));
    static_assert(sizeof(BR) <= kBoundRowBytes, "bound row slot");
    BR* brs = reinterpret_cast<BR*>(Ws + L);  // after the twiddles (launch_rows adds G slots)
    if (threadIdx.x < G && rho0 + (int)threadIdx.x < nrows) brs[threadIdx.x] = bind_row(prob, rho0 + threadIdx.x);
    __syncthreads();
    auto ld = [&](int g, int e) -> CT { return (rho0 + g < nrows) ? brs[g].load(e) : CxT<CT>::make(0, 0); };
    auto st = [&](int g, int e, CT v) {
      if (rho0 + g < nrows) brs[g].store(e, v);
    };
    fft_fused<LOG2L, G, NT, DIR, LS, false, true, true>(smem, Ws, ld, st);
  } else if constexpr (LOG2L >= 3) {
    // first pass straight from global memory, last pass straight to global memory
    auto ld = [&](int g, int e) -> CT {
      return (rho0 + g < nrows) ? prob.load(rho0 + g, e) : CxT<CT>::make(0, 0);
    };
    auto st = [&](int g, int e, CT v) {
      if (rho0 + g < nrows) prob.store(rho0 + g, e, v);
    };
    fft_fused<LOG2L, G, NT, DIR, LS, false, true, true>(smem, Ws, ld, st);
  } else {
    CT v[EPT];  // all global loads of this thread in flight together
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int idx = threadIdx.x + i * NT, g = idx / L, e = idx % L;
      v[i] = (rho0 + g < nrows) ? prob.load(rho0 + g, e) : CxT<CT>::make(0, 0);
    }
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int idx = threadIdx.x + i * NT, g = idx / L, e = idx % L;
      smem[g * LS + padx(e)] = v[i];
    }
    __syncthreads();
    fft_smem<LOG2L, G, NT, DIR, LS>(smem, Ws);
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int idx = threadIdx.x + i * NT, g = idx / L, e = idx % L;
      if (rho0 + g < nrows) prob.store(rho0 + g, e, smem[g * LS + padx(e)]);
    }
  }
}

// fused first order for L1 <= 4096: fold -> IDFT -> |.| scale -> DFT -> U1hat (+U1)
template <int LOG2L, int G, int NT>
__global__ void __launch_bounds__(NT) k_u1_fused(ProbFold prob, float2* __restrict__ u1hat,
                                                 float* __restrict__ u1dbg, int nrows,
                                                 const float2* __restrict__ Wtab) {
  constexpr int L = 1 << LOG2L, LS = pad_row(L), EPT = G * L / NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* smem = reinterpret_cast<float2*>(smem_raw);
  float2* Ws = smem + G * LS;
  stage_twiddles<LOG2L, NT>(Ws, Wtab + tw_offset(LOG2L));
  const int rho0 = blockIdx.x * G;
  // the G rows' parameters staged once in shared memory (after the twiddles; launch_u1_fused
  // adds the slots): the fold gather, the scale, U1hat / U1 row pointers, the max slot
  struct U1Row {
    BoundFold fold;
    float2* hat;
    float* dbg;
    unsigned int* umax;
  };
  static_assert(sizeof(U1Row) <= kBoundRowBytes, "u1 row slot");
  U1Row* rr = reinterpret_cast<U1Row*>(Ws + L);
  if (threadIdx.x < G) {
    const int rho = min(rho0 + (int)threadIdx.x, nrows - 1);
    const int b = rho / prob.nrows, r = rho % prob.nrows;
    U1Row x;
    x.fold.src = prob.src + (int64_t)b * prob.src_stride;
    x.fold.d = prob.rows[r];
    x.fold.bandvals = prob.bandvals;
    x.fold.L = prob.L;
    x.hat = u1hat + (int64_t)b * prob.dst_stride + x.fold.d.dst_off;
    x.dbg = u1dbg ? u1dbg + (int64_t)b * prob.dst_stride + x.fold.d.dst_off : nullptr;
    x.umax = prob.u1max ? prob.u1max + (int64_t)b * prob.n1 + x.fold.d.pad : nullptr;
    rr[threadIdx.x] = x;
  }
  __syncthreads();
  auto modulus = [&]() {
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int idx = threadIdx.x + i * NT, g = idx / L, e = idx % L;
      const float sc = rr[g].fold.d.scale;
      const float2 v = smem[g * LS + padx(e)];
      const float u = sqrtf(fmaf(v.x, v.x, v.y * v.y)) * sc;
      smem[g * LS + padx(e)] = make_float2(u, 0.f);
      if (u1dbg && rho0 + g < nrows) rr[g].dbg[e] = u;
      if (prob.u1max) {  // per-row max |U1|: a warp's 32 elements share one row when L >= 32
        unsigned int* slot = rr[g].umax;
        if constexpr (L >= 32) {
          const unsigned int m = __reduce_max_sync(0xffffffffu, rho0 + g < nrows ? __float_as_uint(u) : 0u);
          if ((threadIdx.x & 31) == 0 && rho0 + g < nrows) atomicMax(slot, m);
        } else if (rho0 + g < nrows) {
          atomicMax(slot, __float_as_uint(u));
        }
      }
    }
    __syncthreads();
  };
  auto st = [&](int g, int e, float2 v) {
    if (rho0 + g < nrows) rr[g].hat[e] = v;
  };
  if constexpr (LOG2L >= 3) {
    // IDFT: first pass straight from the band fold (global), result left in smem;
    // modulus in smem; DFT of U1: last pass straight to U1hat (global)
    auto ld = [&](int g, int e) -> float2 {
      return (rho0 + g < nrows) ? rr[g].fold.load(e) : make_float2(0.f, 0.f);
    };
    auto none = [&](int, int, float2) {};
    fft_fused<LOG2L, G, NT, +1, LS, false, true, false>(smem, Ws, ld, none);
    modulus();
    auto nold = [&](int, int) -> float2 { return make_float2(0.f, 0.f); };
    fft_fused<LOG2L, G, NT, -1, LS, false, false, true>(smem, Ws, nold, st);
  } else {
    float2 v[EPT];
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int idx = threadIdx.x + i * NT, g = idx / L, e = idx % L;
      v[i] = (rho0 + g < nrows) ? rr[g].fold.load(e) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int idx = threadIdx.x + i * NT, g = idx / L, e = idx % L;
      smem[g * LS + padx(e)] = v[i];
    }
    __syncthreads();
    fft_smem<LOG2L, G, NT, +1, LS>(smem, Ws);
    modulus();
    fft_smem<LOG2L, G, NT, -1, LS>(smem, Ws);
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const int idx = threadIdx.x + i * NT, g = idx / L, e = idx % L;
      st(g, e, smem[g * LS + padx(e)]);
    }
  }
}

// ---------------------------------------------------------------------------------
// four-step FFT, L = La * Lb:  step A: column FFTs (length La) of x[na*Lb + nb] then
// twiddle W_L^{ka nb};  step B: row FFTs (length Lb) -> X[ka + La kb]
// ---------------------------------------------------------------------------------
template <int LOG2A, int LOG2B, int G, int NT, int DIR, class P>
__global__ void __launch_bounds__(NT) k_fft4_a(P prob, typename P::CT* __restrict__ tmp,
                                               const typename P::CT* __restrict__ Wtab, int rho0) {
  using CT = typename P::CT;
  constexpr int La = 1 << LOG2A, Lb = 1 << LOG2B, L = La * Lb;
  constexpr int LS = pad_row(La);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CT* smem = reinterpret_cast<CT*>(smem_raw);
  CT* Ws = smem + G * LS;
  stage_twiddles<LOG2A, NT>(Ws, Wtab + tw_offset(LOG2A));
  // inter-pass twiddle W_L^x, x = ka * nb < L, as W_L^{x_lo} * W_L^{x_hi 2^LOG2A}
  // (x_lo < La: the first La entries of the length-L table; x_hi < Lb: the
  // length-Lb table), both staged in shared memory
  CT* Wlo = Ws + La;
  CT* Whi = Wlo + La;
  {
    const CT* WL = Wtab + tw_offset(LOG2A + LOG2B);
    for (int t = threadIdx.x; t < La; t += NT) Wlo[t] = __ldg(WL + t);
    for (int t = threadIdx.x; t < Lb; t += NT) Whi[t] = __ldg(Wtab + tw_offset(LOG2B) + t);
  }
  constexpr int CPB = Lb / G;  // column groups per big row
  const int rho = rho0 + (int)(blockIdx.x / CPB);  // rows of this launch's group
  const int nb0 = (blockIdx.x % CPB) * G;
  CT* out = tmp + (int64_t)(rho - rho0) * L;
  // column g of this block = big-row column nb0 + g; consecutive threads take
  // consecutive columns (coalesced gathers and scatters), first / last pass fused
  const auto br = bind_row(prob, rho);
  auto ld = [&](int g, int na) -> CT { return br.load(na * Lb + nb0 + g); };
  auto st = [&](int g, int ka, CT v) {
    const int x = ka * (nb0 + g);
    const CT t = cmul(Wlo[x & (La - 1)], Whi[x >> LOG2A]);
    out[ka * Lb + nb0 + g] = cmul(v, DIR < 0 ? t : CxT<CT>::make(t.x, -t.y));
  };
  fft_fused<LOG2A, G, NT, DIR, LS, true, true, true>(smem, Ws, ld, st);
}

template <int LOG2A, int LOG2B, int G, int NT, int DIR, class P>
__global__ void __launch_bounds__(NT) k_fft4_b(P prob, const typename P::CT* __restrict__ tmp,
                                               const typename P::CT* __restrict__ Wtab, int rho0) {
  using CT = typename P::CT;
  constexpr int La = 1 << LOG2A, Lb = 1 << LOG2B, L = La * Lb;
  constexpr int LS = pad_row(Lb);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CT* smem = reinterpret_cast<CT*>(smem_raw);
  CT* Ws = smem + G * LS;
  stage_twiddles<LOG2B, NT>(Ws, Wtab + tw_offset(LOG2B));
  constexpr int RPB = La / G;
  const int rho = rho0 + (int)(blockIdx.x / RPB);
  const int ka0 = (blockIdx.x % RPB) * G;
  const CT* in = tmp + (int64_t)(rho - rho0) * L;
  // rows (ka0 + g) of the intermediate are contiguous: the first pass (row-major
  // threads) is fused with the loads; the last pass (column-major threads: consecutive
  // ka, i.e. consecutive output bins ka + La kb) with the stores
  auto ld = [&](int g, int e) -> CT { return in[(ka0 + g) * Lb + e]; };
  const auto br = bind_row(prob, rho);
  auto st = [&](int g, int kb, CT v) { br.store(ka0 + g + La * kb, v); };
  fft_fused<LOG2B, G, NT, DIR, LS, true, true, true, CT, decltype(ld), decltype(st), false>(smem, Ws, ld, st);
}

// ---------------------------------------------------------------------------------
// KB middle stage for four-step lengths (L = La Lb): the inverse DFT's pass B (rows ka of
// the pass-A intermediate, length Lb over kb), the modulus |.| / L1 of the scalogram row,
// and the forward DFT's first pass -- fused through shared memory, so U1 never leaves
// the chip.  The forward DFT is factorised the other way round (n = na' + La nb',
// k = kb' + Lb ka''): the G inverse-DFT outputs of this CTA, U1[ka + La kb] for its G
// values ka and every kb, are exactly the G columns na' = ka of the forward transform.
// Stage 2 is a length-Lb FFT over nb' per column, times W_L^{na' kb'}, written as rows
// kb' of length La; k_fft4_b<LOG2B, LOG2A> (ProbRealFwd) finishes with the length-La pass.
// ---------------------------------------------------------------------------------
template <int LOG2A, int LOG2B, int G, int NT>
__global__ void __launch_bounds__(NT) k_fft4_mid(ProbFold prob, const float2* __restrict__ tmp_in,
                                                 float2* __restrict__ tmp_out, const float2* __restrict__ Wtab,
                                                 int rho0) {
  constexpr int La = 1 << LOG2A, Lb = 1 << LOG2B, L = La * Lb;
  constexpr int LS = pad_row(Lb);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* s1 = reinterpret_cast<float2*>(smem_raw);
  float2* s2 = s1 + G * LS;
  float2* Ws = s2 + G * LS;        // per-pass twiddles of length Lb (both directions)
  float2* Wlo = Ws + Lb;           // W_L^t, t < Lb
  float2* Whi = Wlo + Lb;          // W_La^t, t < La  (= W_L^{Lb t})
  stage_twiddles<LOG2B, NT>(Ws, Wtab + tw_offset(LOG2B));
  {
    const float2* WL = Wtab + tw_offset(LOG2A + LOG2B);
    for (int t = threadIdx.x; t < Lb; t += NT) Wlo[t] = __ldg(WL + t);
    for (int t = threadIdx.x; t < La; t += NT) Whi[t] = __ldg(Wtab + tw_offset(LOG2A) + t);
  }
  constexpr int RPB = La / G;
  const int rho = rho0 + (int)(blockIdx.x / RPB);
  const int ka0 = (blockIdx.x % RPB) * G;
  const float2* in = tmp_in + (int64_t)(rho - rho0) * L;
  float2* out = tmp_out + (int64_t)(rho - rho0) * L;
  const float sc = prob.rows[rho % prob.nrows].scale;
  __syncthreads();  // twiddle tables
  // stage 1: inverse DFT over kb of rows ka0 + g; U1 = |.| sc into s2 row g, element kb
  auto ld1 = [&](int g, int e) -> float2 { return in[(ka0 + g) * Lb + e]; };
  auto st1 = [&](int g, int kb, float2 v) { s2[g * LS + padx(kb)] = make_float2(sqrtf(fmaf(v.x, v.x, v.y * v.y)) * sc, 0.f); };
  fft_fused<LOG2B, G, NT, +1, LS, true, true, true, float2, decltype(ld1), decltype(st1), false>(s1, Ws, ld1, st1);
  __syncthreads();
  // stage 2: forward DFT over nb' of columns na' = ka0 + g, twiddle W_L^{na' kb'}, rows kb'
  auto ld2 = [&](int, int) -> float2 { return make_float2(0.f, 0.f); };  // unused: input in s2
  auto st2 = [&](int g, int kb, float2 v) {
    const int x = kb * (ka0 + g);
    const float2 tw = cmul(Wlo[x & (Lb - 1)], Whi[x >> LOG2B]);
    out[kb * La + ka0 + g] = cmul(v, tw);
  };
  fft_fused<LOG2B, G, NT, -1, LS, true, false, true>(s2, Ws, ld2, st2);
}

// Real-pair variant: two scalogram rows (lambda = 2j, 2j + 1 of the group) share one
// complex forward DFT, z = U1_a + i U1_b; k_fft4_fin2 separates the spectra with
// U_a[k] = (Z[k] + conj Z[-k]) / 2, U_b[k] = (Z[k] - conj Z[-k]) / 2i.  Grid: (signal, pair, ka block).
template <int LOG2A, int LOG2B, int G, int NT>
__global__ void __launch_bounds__(NT) k_fft4_mid2(ProbFold prob, const float2* __restrict__ tmp_in,
                                                  float2* __restrict__ tmp_out, const float2* __restrict__ Wtab) {
  constexpr int La = 1 << LOG2A, Lb = 1 << LOG2B, L = La * Lb;
  constexpr int LS = pad_row(Lb);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* s1 = reinterpret_cast<float2*>(smem_raw);
  float2* s2 = s1 + G * LS;
  float2* Ws = s2 + G * LS;
  float2* Wlo = Ws + Lb;
  float2* Whi = Wlo + Lb;
  stage_twiddles<LOG2B, NT>(Ws, Wtab + tw_offset(LOG2B));
  {
    const float2* WL = Wtab + tw_offset(LOG2A + LOG2B);
    for (int t = threadIdx.x; t < Lb; t += NT) Wlo[t] = __ldg(WL + t);
    for (int t = threadIdx.x; t < La; t += NT) Whi[t] = __ldg(Wtab + tw_offset(LOG2A) + t);
  }
  constexpr int RPB = La / G;
  const int nr = prob.nrows, npair = (nr + 1) >> 1;
  const int q = (int)(blockIdx.x / RPB);  // pair id = b * npair + j
  const int ka0 = (blockIdx.x % RPB) * G;
  const int b = q / npair, j = q % npair;
  const bool two = 2 * j + 1 < nr;
  float2* out = tmp_out + (int64_t)q * L;
  __syncthreads();  // twiddle tables
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    float* s2f = reinterpret_cast<float*>(s2) + h;  // component h (re: row 2j, im: row 2j + 1)
    if (h == 1 && !two) {
      for (int idx = threadIdx.x; idx < G * Lb; idx += NT) s2f[2 * ((idx / Lb) * LS + padx(idx % Lb))] = 0.f;
      break;
    }
    const int rho = b * nr + 2 * j + h;
    const float2* in = tmp_in + (int64_t)rho * L;
    const float sc = prob.rows[2 * j + h].scale;
    float umax = 0.f;  // this thread's max |U1| of row 2j + h (KB's per-row max for KC's fp16 scale)
    auto ld1 = [&](int g, int e) -> float2 { return in[(ka0 + g) * Lb + e]; };
    auto st1 = [&](int g, int kb, float2 v) {
      const float u = sqrtf(fmaf(v.x, v.x, v.y * v.y)) * sc;
      umax = fmaxf(umax, u);
      s2f[2 * (g * LS + padx(kb))] = u;
    };
    fft_fused<LOG2B, G, NT, +1, LS, true, true, true, float2, decltype(ld1), decltype(st1), false>(s1, Ws, ld1, st1);
    if (prob.u1max) {
      const unsigned int m = __reduce_max_sync(0xffffffffu, __float_as_uint(umax));
      if ((threadIdx.x & 31) == 0) atomicMax(prob.u1max + (int64_t)b * prob.n1 + prob.rows[2 * j + h].pad, m);
    }
    __syncthreads();
  }
  __syncthreads();
  auto ld2 = [&](int, int) -> float2 { return make_float2(0.f, 0.f); };  // unused: input in s2
  auto st2 = [&](int g, int kb, float2 v) {
    const int x = kb * (ka0 + g);
    const float2 tw = cmul(Wlo[x & (Lb - 1)], Whi[x >> LOG2B]);
    out[kb * La + ka0 + g] = cmul(v, tw);
  };
  fft_fused<LOG2B, G, NT, -1, LS, true, false, true>(s2, Ws, ld2, st2);
}

// Final pass of the real-pair forward DFT: rows kb' (length La over na') of the packed
// intermediate, G rows per CTA chosen closed under kb' <-> Lb - kb' (rows 0 and Lb/2 pair
// with themselves), FFT in shared memory, then the two spectra are separated bin by bin.
template <int LOG2A, int LOG2B, int G, int NT>
__global__ void __launch_bounds__(NT) k_fft4_fin2(ProbRealFwd prob, const float2* __restrict__ tmp,
                                                  const float2* __restrict__ Wtab) {
  constexpr int La = 1 << LOG2A, Lb = 1 << LOG2B, L = La * Lb;  // rows kb' < Lb of length La
  constexpr int LS = pad_row(La);
  constexpr int H = G / 2;
  static_assert(G % 2 == 0 && G <= Lb, "paired rows");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* s = reinterpret_cast<float2*>(smem_raw);
  float2* Ws = s + G * LS;
  stage_twiddles<LOG2A, NT>(Ws, Wtab + tw_offset(LOG2A));
  constexpr int CPP = Lb / G;  // CTAs per pair
  const int q = (int)(blockIdx.x / CPP);
  const int c = blockIdx.x % CPP;
  const int nr = prob.nrows, npair = (nr + 1) >> 1;
  const int b = q / npair, j = q % npair;
  const bool two = 2 * j + 1 < nr;
  const float2* in = tmp + (int64_t)q * L;
  // slot g -> row: g < H: A = c H + g; g >= H: Lb - A (A = 0 -> Lb / 2)
  auto row_of = [&](int g) -> int {
    const int a = c * H + (g < H ? g : g - H);
    return g < H ? a : (a == 0 ? Lb / 2 : Lb - a);
  };
  __syncthreads();
  auto ld = [&](int g, int e) -> float2 { return in[row_of(g) * La + e]; };
  auto st = [&](int, int, float2) {};  // results stay in shared memory
  fft_fused<LOG2A, G, NT, -1, LS, false, true, false, float2, decltype(ld), decltype(st), false>(s, Ws, ld, st);
  float2* ua = prob.u1hat + (int64_t)b * prob.stride + prob.rows[2 * j].dst_off;
  float2* ub = two ? prob.u1hat + (int64_t)b * prob.stride + prob.rows[2 * j + 1].dst_off : nullptr;
  for (int idx = threadIdx.x; idx < G * La; idx += NT) {
    const int g = idx % G, e = idx / G;
    const int r = row_of(g);
    int gp, ep;
    if (r == 0) {
      gp = g;
      ep = (La - e) & (La - 1);
    } else if (r == Lb / 2) {
      gp = g;
      ep = La - 1 - e;
    } else {
      gp = g < H ? g + H : g - H;
      ep = La - 1 - e;
    }
    const float2 z = s[g * LS + padx(e)], zp = s[gp * LS + padx(ep)];
    const int k = r + Lb * e;
    ua[k] = make_float2(0.5f * (z.x + zp.x), 0.5f * (z.y - zp.y));
    if (ub) ub[k] = make_float2(0.5f * (z.y + zp.y), -0.5f * (z.x - zp.x));
  }
}

// ---------------------------------------------------------------------------------
// KS: phi_T averaging at rate T by folding the band-limited spectrum to NPT bins.
// One warp per (signal, row).  row < 0 denotes S0 (source X_hat on the N_pad grid).
// ---------------------------------------------------------------------------------
struct KSParams {
  const float2* xhat;
  const float2* u1hat;
  float* yphi;
  float* out;
  const float* bandvals;
  const float2* W;
  int log2Ntw;
  int n1, NPT, N_pad, frame0, n_frames;
  int64_t u1_stride, fps, off_s0, off_s1;
  const int64_t* u1_off;  // per lambda
  const int* k1;          // per lambda
  Band band_pad;          // phi_T on the N_pad grid
  const Band* band_L1;    // phi_T on grid N_pad >> k
  int nsig;
};

__global__ void __launch_bounds__(128) k_phi_first(KSParams p) {
  __shared__ float2 fold[4][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * 4 + warp;  // item = b * (n1 + 1) + (row + 1)
  const int per = p.n1 + 1;
  if (item >= p.nsig * per) return;
  const int b = item / per, row = item % per - 1;
  const float2* src;
  int Lsrc;
  Band bd;
  float scale;
  if (row < 0) {
    src = p.xhat + (int64_t)b * p.N_pad;
    Lsrc = p.N_pad;
    bd = p.band_pad;
    scale = 1.f / (float)p.N_pad;
  } else {
    src = p.u1hat + (int64_t)b * p.u1_stride + p.u1_off[row];
    const int k = p.k1[row];
    Lsrc = p.N_pad >> k;
    bd = p.band_L1[k];
    scale = 1.f / (float)Lsrc;
  }
  const int NPT = p.NPT;
  for (int i = lane; i < NPT; i += 32) {
    float2 acc = make_float2(0.f, 0.f);
    int t = (i - bd.m0) % NPT;
    if (t < 0) t += NPT;
    for (; t < bd.len; t += NPT) {
      int q = bd.m0 + t;
      if (q >= Lsrc) q -= Lsrc;
      const float2 x = src[q];
      const float f = __ldg(p.bandvals + bd.off + t);
      acc.x = fmaf(x.x, f, acc.x);
      acc.y = fmaf(x.y, f, acc.y);
    }
    fold[warp][i] = acc;
  }
  __syncwarp();
  const int shift = p.log2Ntw - (31 - __clz(NPT));
  for (int n = lane; n < NPT; n += 32) {
    float acc = 0.f;
    for (int m = 0; m < NPT; ++m) {  // Re of IDFT: sum_m F[m] e^{+2 pi i m n / NPT}
      const float2 w = twiddle<+1>(p.W, ((m * n) & (NPT - 1)) << shift);
      acc = fmaf(fold[warp][m].x, w.x, acc);
      acc = fmaf(-fold[warp][m].y, w.y, acc);
    }
    acc *= scale;
    if (row < 0) {
      const int m = n - p.frame0;
      if (m >= 0 && m < p.n_frames) p.out[(int64_t)b * p.fps + p.off_s0 + m] = acc;
    } else {
      p.yphi[((int64_t)b * p.n1 + row) * NPT + n] = acc;
      const int m = n - p.frame0;
      if (m >= 0 && m < p.n_frames)
        p.out[(int64_t)b * p.fps + p.off_s1 + (int64_t)row * p.n_frames + m] = acc;
    }
  }
}

// ---------------------------------------------------------------------------------
// KD (SIMT v1): per (signal, alpha, chunk, 64-row block): Z = A_alpha Y2_alpha over a
// 64 x 128 tile (complex fp32, 4 FFMA per complex MAC), |Z|, phi_T pooling into the
// retained frames with taps g_alpha; per-unit partials written in fixed order.
// ---------------------------------------------------------------------------------
template <int NF>
__global__ void __launch_bounds__(256) k_kd_simt(KDParams p) {
  __shared__ float2 As[8][64];
  __shared__ float2 Ys[8][128];
  __shared__ float gs[NF][128];
  const int nmb = p.Mpad / 64;
  int u = blockIdx.x;
  const int mblk = u % nmb;
  u /= nmb;
  const int ch = p.chunk_sel ? p.chunk_sel[u % p.nsel] : u % p.nsel;
  const int b = u / p.nsel;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const float* Y = p.y2 + (int64_t)b * p.y2_stride + p.y2_off;  // planar rows 2l (re), 2l+1 (im)
  const float2* A = p.A + mblk * 64;
  float part[4][NF];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int m = 0; m < NF; ++m) part[i][m] = 0.f;
  const int col_end = (ch + 1) * p.chunk;
  const int ntile = (p.chunk + 127) / 128;
  for (int tile = 0; tile < ntile; ++tile) {
    const int c0 = ch * p.chunk + tile * 128;
    // pooling taps for this tile
    for (int idx = threadIdx.x; idx < NF * 128; idx += 256) {
      const int m = idx / 128, c = idx % 128;
      float w = 0.f;
      if (m < p.nframes && c0 + c < col_end) {
        int t = ((p.frame0 + m) * p.D - (c0 + c)) % p.L;
        if (t < 0) t += p.L;
        w = __ldg(p.g + t);
      }
      gs[m][c] = w;
    }
    float2 acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = make_float2(0.f, 0.f);
    for (int k0 = 0; k0 < p.Kpad; k0 += 8) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int idx = threadIdx.x + q * 256;
        const int kk = idx / 64, r = idx % 64;
        As[kk][r] = A[(int64_t)(k0 + kk) * p.Mpad + r];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int idx = threadIdx.x + q * 256;
        const int kk = idx / 128, c = idx % 128;
        float2 y = make_float2(0.f, 0.f);
        if (k0 + kk < p.K && c0 + c < col_end) {
          const float* row = Y + (int64_t)(2 * (k0 + kk)) * p.L + c0 + c;
          y = make_float2(row[0], row[p.L]);
        }
        Ys[kk][c] = y;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        float2 a[4], y[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] = Ys[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            acc[i][j].x = fmaf(a[i].x, y[j].x, acc[i][j].x);
            acc[i][j].x = fmaf(-a[i].y, y[j].y, acc[i][j].x);
            acc[i][j].y = fmaf(a[i].x, y[j].y, acc[i][j].y);
            acc[i][j].y = fmaf(a[i].y, y[j].x, acc[i][j].y);
          }
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float w[NF];
#pragma unroll
      for (int m = 0; m < NF; ++m) w[m] = gs[m][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float mag = sqrtf(fmaf(acc[i][j].x, acc[i][j].x, acc[i][j].y * acc[i][j].y));
#pragma unroll
        for (int m = 0; m < NF; ++m) part[i][m] = fmaf(w[m], mag, part[i][m]);
      }
    }
    __syncthreads();  // gs reuse
  }
  // reduce over the 16 column lanes (fixed xor tree -> deterministic)
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int m = 0; m < NF; ++m) {
      float v = part[i][m];
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      part[i][m] = v;
    }
  if (tx == 0) {
    float* dst = p.part + (int64_t)b * p.part_stride + p.part_off +
                 ((int64_t)ch * p.Mpad + mblk * 64 + ty * 4) * p.nframes;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int m = 0; m < NF; ++m)
        if (m < p.nframes) dst[i * p.nframes + m] = part[i][m];
  }
}

// Eq. (adalog) of one S2 value: log(1 + S / (eps mu)); 0 where eps mu <= 0
__device__ __forceinline__ float mulog_val(float s, float den) { return den > 0.f ? log1pf(s / den) : 0.f; }

// ---------------------------------------------------------------------------------
// KE: lambda pooling (phi_F) of the pooled rows, phi-only paths, packing of S2.
// One block per (signal, path).
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_ke(KEParams p) {
  extern __shared__ float sm[];
  const int b = blockIdx.x;
  const int pi = blockIdx.y;
  const DevPath P = p.paths[pi];
  const int nf = p.n_frames;
  float* outp = p.out + (int64_t)b * p.fps + p.off_s2 + (int64_t)pi * p.lam_out * nf;
  if (P.kind == JTFS_PATH_PHI_T_PHI_F) {
    const float* yphi = p.yphi + (int64_t)b * p.n1 * p.NPT;
    for (int idx = threadIdx.x; idx < p.lam_out * nf; idx += blockDim.x) {
      const int q = idx / nf, m = idx % nf;
      float acc = 0.f;
      // circular tap index d = (q 2^k - l) mod N_fr, q 2^k < N_fr: two wrap-free ranges
      const int rp = q << p.k_phiphi;
      const float* ym = yphi + p.frame0 + m;
      const int l1 = min(p.n1, rp + 1);
      for (int l = 0; l < l1; ++l) acc = fmaf(__ldg(p.hphiF + (rp - l)), ym[l * p.NPT], acc);
      for (int l = l1; l < p.n1; ++l) acc = fmaf(__ldg(p.hphiF + (rp - l + p.N_fr)), ym[l * p.NPT], acc);
      outp[idx] = p.mu ? mulog_val(acc, p.mu_eps * __ldg(p.mu + pi)) : acc;
    }
    return;
  }
  const DevFilter f = p.filters[P.filter];
  float* Pm = sm;  // [nrows][nf]
  if (P.kind == JTFS_PATH_PHI_T_PSI_F) {
    const float* yphi = p.yphi + (int64_t)b * p.n1 * p.NPT;
    float* ys = sm + f.nrows * nf;           // [n1][NPT]
    float* u2 = ys + p.n1 * p.NPT;           // [nrows][NPT]
    for (int idx = threadIdx.x; idx < p.n1 * p.NPT; idx += blockDim.x) ys[idx] = yphi[idx];
    __syncthreads();
    const float2* h = p.hpsi + (int64_t)P.beta * p.N_fr;
    for (int idx = threadIdx.x; idx < f.nrows * p.NPT; idx += blockDim.x) {
      const int r = idx / p.NPT, n = idx % p.NPT;
      const int rp = p.rprime[f.rp_off + r] << f.k;
      float2 z = make_float2(0.f, 0.f);
      // circular tap index d = (r' 2^k - l) mod N_fr, r' 2^k < N_fr: two wrap-free ranges
      const int l1 = min(p.n1, rp + 1);
      for (int l = 0; l < l1; ++l) {
        const float2 hv = __ldg(h + (rp - l));
        const float yv = ys[l * p.NPT + n];
        z.x = fmaf(hv.x, yv, z.x);
        z.y = fmaf(hv.y, yv, z.y);
      }
      for (int l = l1; l < p.n1; ++l) {
        const float2 hv = __ldg(h + (rp - l + p.N_fr));
        const float yv = ys[l * p.NPT + n];
        z.x = fmaf(hv.x, yv, z.x);
        z.y = fmaf(hv.y, yv, z.y);
      }
      u2[idx] = sqrtf(fmaf(z.x, z.x, z.y * z.y));
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < f.nrows * nf; idx += blockDim.x) {
      const int r = idx / nf, m = idx % nf;
      float acc = 0.f;
      // d = (frame0 + m - n) mod NPT with frame0 + m < NPT: two wrap-free ranges
      const int base = p.frame0 + m;
      const float* ur = u2 + r * p.NPT;
      for (int n = 0; n <= base; ++n) acc = fmaf(__ldg(p.gT + (base - n)), ur[n], acc);
      for (int n = base + 1; n < p.NPT; ++n) acc = fmaf(__ldg(p.gT + (base - n + p.NPT)), ur[n], acc);
      Pm[idx] = acc;
    }
    __syncthreads();
  } else {
    // spinned or psi_t x phi_f: sum the KD partials over chunks in fixed order
    const DevAlpha a = p.alphas[P.alpha_slot];
    const float* part = p.part + (int64_t)b * p.part_stride + a.part_off;
    const int64_t cstride = (int64_t)p.Mpad * nf;
    const int nout = f.nrows * nf;
    if ((nf & 3) == 0) {
      // 16-byte loads (the block's rows are contiguous in every slice; row0 * nf * 4 and
      // the slice stride are multiples of 16 B): 4 outputs per thread, 8 slices in flight
      const int64_t cs4 = cstride / 4;
      const float4* src4 = reinterpret_cast<const float4*>(part + (int64_t)f.row0 * nf);
      for (int v = threadIdx.x; v < nout / 4; v += blockDim.x) {
        const float4* s = src4 + v;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        int c = 0;
        for (; c + 8 <= a.nchunks; c += 8) {  // sums in fixed (slice) order per output
          float4 x[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) x[j] = __ldg(s + (c + j) * cs4);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            acc.x += x[j].x;
            acc.y += x[j].y;
            acc.z += x[j].z;
            acc.w += x[j].w;
          }
        }
        for (; c < a.nchunks; ++c) {
          const float4 x = __ldg(s + c * cs4);
          acc.x += x.x;
          acc.y += x.y;
          acc.z += x.z;
          acc.w += x.w;
        }
        reinterpret_cast<float4*>(Pm)[v] = acc;
      }
    } else {
      for (int idx = threadIdx.x; idx < nout; idx += blockDim.x) {
        const float* src = part + (int64_t)f.row0 * nf + idx;  // (row0 + r) * nf + m
        float acc = 0.f;
        int c = 0;
        for (; c + 8 <= a.nchunks; c += 8) {  // 8 loads in flight, sums in fixed order
          float v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = __ldg(src + (c + j) * cstride);
#pragma unroll
          for (int j = 0; j < 8; ++j) acc += v[j];
        }
        for (; c < a.nchunks; ++c) acc += __ldg(src + c * cstride);
        Pm[idx] = acc;
      }
    }
    __syncthreads();
  }
  const float* Wf = p.W + f.w_off;
  for (int idx = threadIdx.x; idx < p.lam_out * nf; idx += blockDim.x) {
    const int q = idx / nf, m = idx % nf;
    const int2 band = __ldg(p.Wrange + f.wr_off + q);  // rows with |W| >= 1e-9 max (plan.cpp)
    const float* wq = Wf + (int64_t)q * f.nrows;
    float acc = 0.f;
    for (int r = band.x; r < band.y; ++r) acc = fmaf(__ldg(wq + r), Pm[r * nf + m], acc);
    outp[idx] = p.mu ? mulog_val(acc, p.mu_eps * __ldg(p.mu + pi)) : acc;
  }
}

// ---------------------------------------------------------------------------------
// NEXT-1.  Resynthesis loss E = ||S y - S x|| / ||S x|| and its gradient w.r.t.
// S y, dE/dSy = (S y - S x) / (||S y - S x|| ||S x||) (0 when S y = S x), one record: one
// block, fp64 sums in a fixed order (fixed shared tree), then the scaled difference.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_resynth_loss(const float* __restrict__ Sy, const float* __restrict__ Sx,
                                                      int64_t n, double* E, float* dout) {
  __shared__ double rr[256], xx[256];
  double a = 0.0, c = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) {
    const double d = (double)Sy[i] - (double)Sx[i], x = (double)Sx[i];
    a = fma(d, d, a);
    c = fma(x, x, c);
  }
  rr[threadIdx.x] = a;
  xx[threadIdx.x] = c;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      rr[threadIdx.x] += rr[threadIdx.x + h];
      xx[threadIdx.x] += xx[threadIdx.x + h];
    }
    __syncthreads();
  }
  const double nr = sqrt(rr[0]), nx = sqrt(xx[0]);
  if (threadIdx.x == 0) *E = nx > 0.0 ? nr / nx : 0.0;
  const double sc = (nr > 0.0 && nx > 0.0) ? 1.0 / (nr * nx) : 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) dout[i] = (float)(((double)Sy[i] - (double)Sx[i]) * sc);
}

// ---------------------------------------------------------------------------------
// NEXT-4.  mu(lambda_2) = (1/B) sum_b sum_{lambda,t} S2_b[p] (Eq. (adalog:mu)):
// one block per path, fp64 per-thread sums in a fixed index order, fixed shared tree.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_mulog_mu(const float* __restrict__ S, int64_t B, int64_t fps,
                                                  int64_t off_s2, int map, float* __restrict__ mu) {
  __shared__ double red[256];
  const int pi = blockIdx.x;
  double acc = 0.0;
  for (int64_t b = 0; b < B; ++b) {
    const float* src = S + b * fps + off_s2 + (int64_t)pi * map;
    for (int i = threadIdx.x; i < map; i += 256) acc += (double)__ldg(src + i);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) mu[pi] = (float)(red[0] / (double)B);
}

// Eq. (adalog) over whole records: S0/S1 copied, S2 compressed (reading R22)
__global__ void __launch_bounds__(256) k_mulog_apply(const float* S, int64_t n, int64_t fps, int64_t off_s2,
                                                     int map, const float* __restrict__ mu, float eps,
                                                     float* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i % fps;
    const float v = S[i];
    out[i] = j < off_s2 ? v : mulog_val(v, eps * __ldg(mu + (j - off_s2) / map));
  }
}

// Scale-rate map of one psi_t path (Fig. 1; reading R21): |Z| before Phi.
// grid (column blocks, rows, signals); the row's taps are block-uniform (broadcast),
// Y2 rows are read coalesced along time.
struct U2MapParams {
  const float* y2;      // micro-batch Y2 base, planar rows 2l (re), 2l+1 (im), per alpha [2K][L]
  const float2* hc;     // complex taps [N_fr] (psi path), or nullptr
  const float* hr;      // real taps [N_fr] (phi_F path), or nullptr
  float* out;           // [nsig][rows][cols]
  int64_t y2_off, y2_stride;
  int K, L, N_fr, k, c0, rows, cols, conj;
};

__global__ void __launch_bounds__(256) k_u2_map(U2MapParams p) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  const int r = blockIdx.y;
  const int b = blockIdx.z;
  if (c >= p.cols) return;
  const float* Y = p.y2 + (int64_t)b * p.y2_stride + p.y2_off + p.c0 + c;
  const int rp = r << p.k;
  float zr = 0.f, zi = 0.f;
  for (int l = 0; l < p.K; ++l) {
    int d = (rp - l) % p.N_fr;
    if (d < 0) d += p.N_fr;
    float hr, hi;
    if (p.hc) {
      const float2 h = __ldg(p.hc + d);
      hr = h.x;
      hi = p.conj ? -h.y : h.y;
    } else {
      hr = __ldg(p.hr + d);
      hi = 0.f;
    }
    const float yr = __ldg(Y + (int64_t)(2 * l) * p.L), yi = __ldg(Y + (int64_t)(2 * l + 1) * p.L);
    zr = fmaf(hr, yr, zr);
    zr = fmaf(-hi, yi, zr);
    zi = fmaf(hr, yi, zi);
    zi = fmaf(hi, yr, zi);
  }
  p.out[((int64_t)b * p.rows + r) * p.cols + c] = sqrtf(fmaf(zr, zr, zi * zi));
}

// check for NaN / Inf in x
__global__ void k_check_finite(const float* x, int64_t n, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) atomicOr(flag, 1);
}

// backward (VJP) kernels -- see backward.inc
#include "backward.inc"

}  // namespace dev

// =================================================================================
// host launchers
// =================================================================================
using namespace dev;

namespace {
template <int LOG2L>
constexpr int rows_G() { return (LOG2L >= 11) ? 1 : (2048 >> LOG2L); }
template <int LOG2L>
constexpr int rows_NT() { return (rows_G<LOG2L>() << LOG2L) / 8 < 32 ? 32 : (rows_G<LOG2L>() << LOG2L) / 8; }

template <int LOG2L, int DIR, class P>
void launch_rows(const P& prob, int nrows, const typename P::CT* W, int, cudaStream_t st) {
  constexpr int G = rows_G<LOG2L>();
  constexpr int NT = rows_NT<LOG2L>();
  const int grid = (nrows + G - 1) / G;
  const size_t sm = ((size_t)G * pad_row(1 << LOG2L) + (1 << LOG2L)) * sizeof(typename P::CT) +
                    (size_t)G * kBoundRowBytes;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft_rows<LOG2L, G, NT, DIR, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  k_fft_rows<LOG2L, G, NT, DIR, P><<<grid, NT, sm, st>>>(prob, nrows, W);
}

template <int LOG2L>
void launch_u1_fused(const ProbFold& prob, float2* u1hat, float* u1dbg, int nrows, const float2* W, int,
                     cudaStream_t st) {
  constexpr int G = rows_G<LOG2L>();
  constexpr int NT = rows_NT<LOG2L>();
  const int grid = (nrows + G - 1) / G;
  const size_t sm = ((size_t)G * pad_row(1 << LOG2L) + (1 << LOG2L)) * sizeof(float2) + (size_t)G * kBoundRowBytes;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_u1_fused<LOG2L, G, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  k_u1_fused<LOG2L, G, NT><<<grid, NT, sm, st>>>(prob, u1hat, u1dbg, nrows, W);
}

template <int LOG2L, int DIR, class PA, class PB>
void launch_fft4(const PA& pa, const PB& pb, int nbig, typename PA::CT* tmp, const typename PA::CT* W, int,
                 cudaStream_t st) {
  using CT = typename PA::CT;
  constexpr int ELEMS = sizeof(CT) == 8 ? 4096 : 2048;  // 32 KiB of smem per CTA
  constexpr int LOG2A = (LOG2L + 1) / 2, LOG2B = LOG2L / 2;
  constexpr int La = 1 << LOG2A, Lb = 1 << LOG2B;
  // pass A gathers columns (stride Lb): 16 columns per CTA when the column is
  // long enough (128 B contiguous per row of the gather), else ELEMS / La
  constexpr int GA0 = ELEMS / La;
  constexpr int GA = (GA0 < 16 && 16 <= Lb && sizeof(CT) == 8 && La >= 256) ? 16 : GA0;
  constexpr int GB = ELEMS / Lb;
  constexpr int NT = ELEMS / 8;
  static_assert(GA >= 1 && GB >= 1 && GA <= Lb && GB <= La, "four-step tile");
  const size_t sma = ((size_t)GA * pad_row(La) + 2 * La + Lb) * sizeof(CT);
  const size_t smb = ((size_t)GB * pad_row(Lb) + Lb) * sizeof(CT);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft4_a<LOG2A, LOG2B, GA, NT, DIR, PA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    cudaFuncSetAttribute(k_fft4_b<LOG2A, LOG2B, GB, NT, DIR, PB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    attr = true;
  }
  // One launch pair over all rows.  (Measured on c3, round 1: splitting the rows into
  // 32 / 64 / 96 MiB groups whose intermediate stays L2-resident made KB 16.5 -> 20.3 /
  // 18.5 / 18.4 ms per step -- the passes are not HBM-bound, so the extra launches and
  // tails cost more than the DRAM round trip of the intermediate.)
  {
    const int r0 = 0, nr = nbig;
    k_fft4_a<LOG2A, LOG2B, GA, NT, DIR, PA><<<nr * (Lb / GA), NT, sma, st>>>(pa, tmp, W, r0);
    k_fft4_b<LOG2A, LOG2B, GB, NT, DIR, PB><<<nr * (La / GB), NT, smb, st>>>(pb, tmp, W, r0);
  }
}

// KB four-step with the fused middle stage: inverse pass A (ProbFold) -> k_fft4_mid ->
// forward pass B' (k_fft4_b<LOG2B, LOG2A>, ProbRealFwd).  tmp2: a second intermediate.
template <int LOG2L>
void launch_fft4_u1(const ProbFold& pf, const ProbRealFwd& prf, int nbig, float2* tmp, float2* tmp2,
                    const float2* W, cudaStream_t st) {
  constexpr int ELEMS = 4096;
  constexpr int LOG2A = (LOG2L + 1) / 2, LOG2B = LOG2L / 2;
  constexpr int La = 1 << LOG2A, Lb = 1 << LOG2B;
  constexpr int GA0 = ELEMS / La;
  constexpr int GA = (GA0 < 16 && 16 <= Lb && La >= 256) ? 16 : GA0;  // as launch_fft4
  constexpr int GM = ELEMS / Lb;   // middle stage: rows ka per CTA
  constexpr int GB = ELEMS / La;   // final pass: rows kb' (length La) per CTA
  constexpr int NT = ELEMS / 8;
  static_assert(GA >= 1 && GM >= 1 && GB >= 1 && GM <= La && GB <= Lb, "four-step tile");
  const size_t sma = ((size_t)GA * pad_row(La) + 2 * La + Lb) * sizeof(float2);
  const size_t smm = ((size_t)2 * GM * pad_row(Lb) + 2 * Lb + La) * sizeof(float2);
  const size_t smb = ((size_t)GB * pad_row(La) + La) * sizeof(float2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft4_a<LOG2A, LOG2B, GA, NT, +1, ProbFold>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    cudaFuncSetAttribute(k_fft4_mid<LOG2A, LOG2B, GM, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_fft4_b<LOG2B, LOG2A, GB, NT, -1, ProbRealFwd>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  k_fft4_a<LOG2A, LOG2B, GA, NT, +1, ProbFold><<<nbig * (Lb / GA), NT, sma, st>>>(pf, tmp, W, 0);
  // real pairs: rows (2j, 2j + 1) of the group share one complex forward DFT
  static bool attr2 = false;
  constexpr int GF = GB < 2 ? 2 : GB;
  const size_t smf = ((size_t)GF * pad_row(La) + La) * sizeof(float2);
  if (!attr2) {
    cudaFuncSetAttribute(k_fft4_mid2<LOG2A, LOG2B, GM, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_fft4_fin2<LOG2A, LOG2B, GF, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    attr2 = true;
  }
  const int nsig = nbig / pf.nrows, npair = (pf.nrows + 1) / 2;
  k_fft4_mid2<LOG2A, LOG2B, GM, NT><<<nsig * npair * (La / GM), NT, smm, st>>>(pf, tmp, tmp2, W);
  k_fft4_fin2<LOG2A, LOG2B, GF, NT><<<nsig * npair * (Lb / GF), NT, smf, st>>>(prf, tmp2, W);
}

template <class F>
void dispatch_log2(int lg, F&& f) {
  switch (lg) {
#define JTFS_CASE(n) \
  case n: f(std::integral_constant<int, n>{}); break;
    JTFS_CASE(1) JTFS_CASE(2) JTFS_CASE(3) JTFS_CASE(4) JTFS_CASE(5) JTFS_CASE(6)
    JTFS_CASE(7) JTFS_CASE(8) JTFS_CASE(9) JTFS_CASE(10) JTFS_CASE(11) JTFS_CASE(12)
    JTFS_CASE(13) JTFS_CASE(14) JTFS_CASE(15) JTFS_CASE(16) JTFS_CASE(17) JTFS_CASE(18)
#undef JTFS_CASE
    default: break;
  }
}
}  // namespace

// ---------------------------------------------------------------------------------
// FP32 SIMT peak probe (jtfs_measure_fp32_peak; "the bench must measure
// it with an FFMA loop"): 8 independent FMA chains per thread, scalar FFMA or packed
// FFMA2 (fma.rn.f32x2), enough warps per SM to hide the 4-cycle latency.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k_ffma_peak(float* out, int iters, float b, float c) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = (float)(threadIdx.x + j) * 1e-3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], b, c);
  }
  float t = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) t += a[j];
  if (t == 1234.5f) out[threadIdx.x] = t;  // keeps the chains live
}

__global__ void __launch_bounds__(512) k_ffma2_peak(float* out, int iters, float b, float c) {
  unsigned long long a[8];
  const float2 bb = make_float2(b, b), cc = make_float2(c, c);
  const unsigned long long ub = *reinterpret_cast<const unsigned long long*>(&bb);
  const unsigned long long uc = *reinterpret_cast<const unsigned long long*>(&cc);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 v = make_float2((float)(threadIdx.x + j) * 1e-3f, (float)j * 1e-3f);
    a[j] = *reinterpret_cast<const unsigned long long*>(&v);
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(ub), "l"(uc));
  }
  float t = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 v = *reinterpret_cast<const float2*>(&a[j]);
    t += v.x + v.y;
  }
  if (t == 1234.5f) out[threadIdx.x] = t;
}

cudaError_t measure_fp32_peak(double* tflops_ffma, double* tflops_ffma2) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  cudaError_t e = cudaMalloc(&out, 512 * sizeof(float));
  if (e != cudaSuccess) return e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 2, threads = 512, iters = 4096;
  const double fl = (double)blocks * threads * iters * 16 * 8 * 2;  // FMA = 2 flops
  for (int v = 0; v < 2; ++v) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {  // rep 0 warms the clocks up
      cudaEventRecord(e0);
      if (v == 0) k_ffma_peak<<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f);
      else k_ffma2_peak<<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0) best = std::min(best, ms);
    }
    const double t = fl * (v == 0 ? 1.0 : 2.0) / (best * 1e-3) / 1e12;
    if (v == 0) *tflops_ffma = t;
    else *tflops_ffma2 = t;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  e = cudaGetLastError();
  cudaFree(out);
  return e;
}

// workspace guard check (JTFS_WS_GUARDS builds): any byte != pattern in the bands -> flag
__global__ void k_guard_check(const unsigned char* ws, const int64_t* starts, int n, int64_t len, int* flag) {
  const unsigned char* g = ws + starts[blockIdx.y];
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < len; i += (int64_t)gridDim.x * 256)
    if (g[i] != 0xA5) atomicOr(flag, 1 << min((int)blockIdx.y, 30));
}
void launch_guard_check(const void* ws, const int64_t* d_starts, int n, int64_t len, int* flag, cudaStream_t st) {
  k_guard_check<<<dim3(16, n), 256, 0, st>>>((const unsigned char*)ws, d_starts, n, len, flag);
}

// jtfs_debug_fft: the FFT engine on plain rows (fp32: both directions, lengths 2^1..2^18;
// fp64: forward, 2^1..2^18), with the plan's twiddle tables (L <= N_pad)
int launch_debug_fft(const Plan& P, int log2L, int dir, bool fp64, const void* in, void* out, int nrows, void* tmp,
                     cudaStream_t st) {
  const int ltw = ilog2_exact(P.N_tw);
  int n = 0;
  dispatch_log2(log2L, [&](auto c) {
    constexpr int LG = decltype(c)::value;
    if (fp64) {
      ProbPlain<double2> pr{(const double2*)in, (double2*)out, 1 << LG};
      const double2* W = (const double2*)P.d_twiddle64;
      if constexpr (LG <= 11) launch_rows<LG, -1>(pr, nrows, W, ltw, st);
      else launch_fft4<LG, -1>(pr, pr, nrows, (double2*)tmp, W, ltw, st);
    } else {
      ProbPlain<float2> pr{(const float2*)in, (float2*)out, 1 << LG};
      const float2* W = (const float2*)P.d_twiddle;
      if constexpr (LG <= 12) {
        if (dir < 0) launch_rows<LG, -1>(pr, nrows, W, ltw, st);
        else launch_rows<LG, +1>(pr, nrows, W, ltw, st);
      } else {
        if (dir < 0) launch_fft4<LG, -1>(pr, pr, nrows, (float2*)tmp, W, ltw, st);
        else launch_fft4<LG, +1>(pr, pr, nrows, (float2*)tmp, W, ltw, st);
      }
    }
    n = LG <= (fp64 ? 11 : 12) ? 1 : 2;
  });
  return n;
}

int launch_pad_fft(const Plan& P, const float* x, int nsig, float2* xhat, float2* tmp, cudaStream_t st) {
  // fp64 DFT of the padded signal: a fp32 FFT's roundoff is proportional to the
  // global spectral norm and would swamp the weak high-frequency bands that the
  // top first-order filters select (precision budget).
  ProbPad pr{x, xhat, P.N, P.N_pad, P.pad_left, P.prm.pad_mode == JTFS_PAD_PERIODIC};
  const double2* W = (const double2*)P.d_twiddle64;
  const int ltw = ilog2_exact(P.N_tw);
  dispatch_log2(ilog2_exact(P.N_pad), [&](auto c) {
    constexpr int LG = decltype(c)::value;
    if constexpr (LG <= 11) {
      launch_rows<LG, -1>(pr, nsig, W, ltw, st);
    } else {
      launch_fft4<LG, -1>(pr, pr, nsig, (double2*)tmp, W, ltw, st);
    }
  });
  return ilog2_exact(P.N_pad) <= 11 ? 1 : 2;
}

int launch_first_order(const Plan& P, const float2* xhat, int nsig, float* u1, float2* u1hat, float2* tmp,
                       bool keep_u1, cudaStream_t st, float2* tmp2, unsigned int* u1max) {
  const float2* W = (const float2*)P.d_twiddle;
  const int ltw = ilog2_exact(P.N_tw);
  int n = 0;
  const bool fuse = tmp2 && !keep_u1;
  for (const auto& g : P.u1_groups) {
    n += g.log2L <= 12 ? 1 : (fuse ? 3 : 4);
    const int nr = (int)g.rows.size();
    ProbFold pf{xhat, P.N_pad, g.d_rows, nr, P.d_bandvals, 1 << g.log2L, u1, nullptr, P.u1_total, u1max, P.n1};
    ProbRealFwd prf{u1, u1hat, P.u1_total, g.d_rows, nr};
    dispatch_log2(g.log2L, [&](auto c) {
      constexpr int LG = decltype(c)::value;
      if constexpr (LG <= 12) {
        launch_u1_fused<LG>(pf, u1hat, keep_u1 ? u1 : nullptr, nsig * nr, W, ltw, st);
      } else if (fuse) {
        ProbRealFwd prf2 = prf;  // reads nothing from U1 (its input comes from tmp2)
        launch_fft4_u1<LG>(pf, prf2, nsig * nr, tmp, tmp2, W, st);
      } else {
        launch_fft4<LG, +1>(pf, pf, nsig * nr, tmp, W, ltw, st);
        launch_fft4<LG, -1>(prf, prf, nsig * nr, tmp, W, ltw, st);
      }
    });
  }
  return n;
}

int launch_phi_first(const Plan& P, const float2* xhat, const float2* u1hat, int nsig, float* yphi, float* out,
                      int64_t fps, int64_t off_s0, int64_t off_s1, const int64_t* d_u1_off, const int* d_k1,
                      const Band* d_band_L1, cudaStream_t st) {
  KSParams p{};
  p.xhat = xhat;
  p.u1hat = u1hat;
  p.yphi = yphi;
  p.out = out;
  p.bandvals = P.d_bandvals;
  p.W = (const float2*)P.d_twiddle + dev::tw_offset(ilog2_exact(P.N_tw));
  p.log2Ntw = ilog2_exact(P.N_tw);
  p.n1 = P.n1;
  p.NPT = P.NPT;
  p.N_pad = P.N_pad;
  p.frame0 = P.frame0;
  p.n_frames = P.n_frames;
  p.u1_stride = P.u1_total;
  p.fps = fps;
  p.off_s0 = off_s0;
  p.off_s1 = off_s1;
  p.u1_off = d_u1_off;
  p.k1 = d_k1;
  p.band_pad = P.band_phiT_pad;
  p.band_L1 = d_band_L1;
  p.nsig = nsig;
  const int items = nsig * (P.n1 + 1);
  k_phi_first<<<(items + 3) / 4, 128, 0, st>>>(p);
  return 1;
}

// ---------------------------------------------------------------------------------
// per-(signal, alpha) power-of-two scale of KD's fp16 operand (read by KC's fp16 store and
// KD): s = 2^(13 - E), bound = max_{lambda < K} ybound[alpha][lambda] max|U1_lambda| in
// [2^E, 2^(E+1)) -- a true upper bound of |Y2_alpha| (plan.cpp), so |Y2| s < 2^14 fits
// fp16, and every value above 2^-27 of the bound keeps the split's 2^-22 relative error.
// One warp per (signal, alpha); fixed-order max (exact, order-independent anyway).
// ---------------------------------------------------------------------------------
__global__ void k_yscale(const unsigned int* __restrict__ u1max, const float* __restrict__ ybound,
                         const DevAlpha* __restrict__ alphas, int n1, int nalpha, float* ysc, float* ysi) {
  const int b = blockIdx.x, a = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (a >= nalpha) return;
  const int K = alphas[a].pad;
  float m = 0.f;
  for (int l = lane; l < K; l += 32)
    m = fmaxf(m, __uint_as_float(__ldg(u1max + (int64_t)b * n1 + l)) * __ldg(ybound + (int64_t)a * n1 + l));
  const unsigned int mb = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
  if (lane == 0) {
    int E = (int)(mb >> 23) - 127;
    E = max(E, -100);
    ysc[(int64_t)b * nalpha + a] = __uint_as_float((uint32_t)(13 - E + 127) << 23);
    ysi[(int64_t)b * nalpha + a] = __uint_as_float((uint32_t)(E - 13 + 127) << 23);
  }
}

int launch_yscale(const Plan& P, const unsigned int* u1max, int nsig, float* ys, cudaStream_t st) {
  const int na = (int)P.kd.size();
  k_yscale<<<nsig, 32 * na, 0, st>>>(u1max, P.d_ybound, (const DevAlpha*)P.d_alphas, P.n1, na, ys,
                                     ys + (int64_t)nsig * na);
  return 1;
}

// KC in the tensor-core KD's fp16 layout (ProbFold16): no fp32 Y2, no separate conversion
int launch_second_order16(const Plan& P, const float2* u1hat, int nsig, uint16_t* y16, const float* ysc,
                          float2* tmp, cudaStream_t st) {
  const float2* W = (const float2*)P.d_twiddle;
  const int ltw = ilog2_exact(P.N_tw);
  int n = 0;
  for (const auto& g : P.y2_groups) {
    n += g.log2L <= 12 ? 1 : 2;
    const int nr = (int)g.rows.size();
    ProbFold16 pf{u1hat, P.u1_total, g.d_rows, nr, P.d_bandvals, 1 << g.log2L, g.d_y16rows,
                  reinterpret_cast<__half*>(y16), P.y16_total, ysc, (int)P.kd.size()};
    dispatch_log2(g.log2L, [&](auto c) {
      constexpr int LG = decltype(c)::value;
      if constexpr (LG <= 12) {
        launch_rows<LG, +1>(pf, nsig * nr, W, ltw, st);
      } else {
        launch_fft4<LG, +1>(pf, pf, nsig * nr, tmp, W, ltw, st);
      }
    });
  }
  return n;
}

// modulus: store |Y2| (times the row scale) in the real row's place instead of the planar
// complex row (Scattering1D needs only the modulus: half the bytes written by KC and read by KT)
int launch_second_order(const Plan& P, const float2* u1hat, int nsig, float* y2, float2* tmp, cudaStream_t st,
                        bool modulus) {
  const float2* W = (const float2*)P.d_twiddle;
  const int ltw = ilog2_exact(P.N_tw);
  int n = 0;
  for (const auto& g : P.y2_groups) {
    n += g.log2L <= 12 ? 1 : 2;
    const int nr = (int)g.rows.size();
    ProbFold pf{u1hat, P.u1_total, g.d_rows, nr, P.d_bandvals, 1 << g.log2L, modulus ? y2 : nullptr,
                modulus ? nullptr : y2, 2 * P.y2_total};
    dispatch_log2(g.log2L, [&](auto c) {
      constexpr int LG = decltype(c)::value;
      if constexpr (LG <= 12) {
        launch_rows<LG, +1>(pf, nsig * nr, W, ltw, st);
      } else {
        launch_fft4<LG, +1>(pf, pf, nsig * nr, tmp, W, ltw, st);
      }
    });
  }
  return n;
}

// ---------------------------------------------------------------------------------
// KT: second-order time scattering (Scattering1D):
// S2_t[alpha][lambda][m] = sum_t g_alpha[(frame0 + m) D - t mod L] |Y2_alpha[lambda](t)|
// -- the phi_T pooling of |Y2| at the retained frames, no lambda convolution.  KC stored
// |Y2| itself (launch_second_order, modulus mode) in the place of each row's real part.
// The pooling weights come from KD's per-alpha table (plan.cpp): exact taps [L][NF]
// (one float4 row per column, no index arithmetic), or, where the plan verified it to fp32
// accuracy, the cubic-moment form [L/32][4][NF] (per 32-column block S_k = sum_j |Y| u_j^k,
// then sum_k G_k,m S_k).  One CTA per (signal, lambda row), 8 warps; fixed-order
// reductions (bit-stable).
// ---------------------------------------------------------------------------------
struct KTParams {
  const float* y2;    // |Y2| rows of signal 0 at alpha's offset (row l at 2 l L); signal stride y2_stride
  const float* wtab;  // alpha's phi_T pooling table (taps or moment coefficients)
  float* out;         // out record of signal 0 at row0's first frame; signal stride fps
  int64_t y2_stride, fps;
  int L, nframes, K, pool_mode;
  int nsplit;         // k_time_scat_rows: column splits (partials [signal][split][K][NF] in part)
  float* part;
};

template <int NF>
__global__ void __launch_bounds__(256) k_time_scat(KTParams p) {
  __shared__ float red[8][NF];
  const int b = blockIdx.x / p.K, l = blockIdx.x % p.K;
  const float* re = p.y2 + (int64_t)b * p.y2_stride + (int64_t)(2 * l) * p.L;  // |Y2| row
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (p.pool_mode == 1) {
    // warp w takes the 32-column blocks w, w + 8, ...; lane j = column j of the block
    const float u = ((float)lane - 15.5f) * 0.0625f;
    float accm = 0.f;  // lane m < NF: frame m
    for (int blk = warp; blk < p.L / 32; blk += 8) {
      const int t = blk * 32 + lane;
      const float mag = __ldg(re + t);
      float S[4] = {mag, mag * u, mag * u * u, mag * u * u * u};
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) S[k] += __shfl_xor_sync(0xffffffffu, S[k], o);
      if (lane < NF) {
        const float* G = p.wtab + (int64_t)blk * 4 * NF + lane;
        accm = fmaf(__ldg(G), S[0], accm);
        accm = fmaf(__ldg(G + NF), S[1], accm);
        accm = fmaf(__ldg(G + 2 * NF), S[2], accm);
        accm = fmaf(__ldg(G + 3 * NF), S[3], accm);
      }
    }
    if (lane < NF) red[warp][lane] = accm;
  } else {
    float acc[NF];
#pragma unroll
    for (int m = 0; m < NF; ++m) acc[m] = 0.f;
    for (int t = threadIdx.x; t < p.L; t += 256) {
      const float mag = __ldg(re + t);
      const float4* w4 = reinterpret_cast<const float4*>(p.wtab + (int64_t)t * NF);
#pragma unroll
      for (int m4 = 0; m4 < NF / 4; ++m4) {
        const float4 w = __ldg(w4 + m4);
        acc[4 * m4 + 0] = fmaf(w.x, mag, acc[4 * m4 + 0]);
        acc[4 * m4 + 1] = fmaf(w.y, mag, acc[4 * m4 + 1]);
        acc[4 * m4 + 2] = fmaf(w.z, mag, acc[4 * m4 + 2]);
        acc[4 * m4 + 3] = fmaf(w.w, mag, acc[4 * m4 + 3]);
      }
    }
#pragma unroll
    for (int m = 0; m < NF; ++m) {
      float v = acc[m];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp][m] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < NF && threadIdx.x < p.nframes) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
    p.out[(int64_t)b * p.fps + (int64_t)l * p.nframes + threadIdx.x] = v;
  }
}

// KT, thread = row: a CTA takes 32 rows (one per lane) of one (signal, alpha); its 8 warps
// split the columns in 32-column blocks (warp w: blocks w, w + 8, ...).  Each lane reads its
// row's 32 columns of a block (16 B vector loads), forms |Y2| and pools them in registers:
// with the cubic-moment form S_k = sum_j |Y2_j| u_j^k (k <= 3) and then pooled += G_k S_k
// (the block's 4 x NF coefficients, a broadcast shared-memory read), else with the exact taps
// (NF FMAs per column, taps [32][NF] of the block broadcast from shared memory).  The 8
// warps' partial sums are combined in fixed order (bit-stable).
template <int NF>
__global__ void __launch_bounds__(256) k_time_scat_rows(KTParams p) {
  constexpr int TB = 8;  // 32-column blocks staged per round (one per warp)
  constexpr int NTAB = TB * 32 * NF, NRED = 8 * 32 * (NF + 1);
  __shared__ __align__(16) float sbuf[NTAB > NRED ? NTAB : NRED];
  float(*tab)[32][NF] = reinterpret_cast<float(*)[32][NF]>(sbuf);       // per block: taps [32][NF] or moments [4][NF]
  float(*red)[32][NF + 1] = reinterpret_cast<float(*)[32][NF + 1]>(sbuf);  // the warps' partial sums (after the loop)
  const int ngrp = (p.K + 31) / 32;
  const int split = blockIdx.x % p.nsplit;
  const int b = blockIdx.x / (p.nsplit * ngrp), grp = (blockIdx.x / p.nsplit) % ngrp;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = grp * 32 + lane;
  const bool active = r < p.K;
  const float* re = p.y2 + (int64_t)b * p.y2_stride + (int64_t)(2 * (active ? r : 0)) * p.L;  // |Y2| row
  // this CTA's 32-column blocks: split `split` of nsplit equal ranges
  const int nblk_all = p.L / 32;
  const int per = (nblk_all + p.nsplit - 1) / p.nsplit;
  const int bbeg = split * per, nblk = min(nblk_all, bbeg + per);
  const int wblk = p.pool_mode ? 4 * NF : 32 * NF;  // table floats per block
  float acc[NF];
#pragma unroll
  for (int m = 0; m < NF; ++m) acc[m] = 0.f;
  for (int blk0 = bbeg; blk0 < nblk; blk0 += TB) {
    __syncthreads();
    const int nb = min(TB, nblk - blk0);
    for (int idx = threadIdx.x; idx < nb * wblk; idx += 256)
      (&tab[0][0][0])[(idx / wblk) * 32 * NF + idx % wblk] = __ldg(p.wtab + (int64_t)blk0 * wblk + idx);
    __syncthreads();
    if (warp < nb && active) {
      const int t0 = (blk0 + warp) * 32;
      const float* tb = &tab[warp][0][0];
      if (p.pool_mode) {
        float S0 = 0.f, S1 = 0.f, S2 = 0.f, S3 = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 a = __ldg(reinterpret_cast<const float4*>(re + t0) + q);
          const float mg[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float u = ((float)(4 * q + e) - 15.5f) * 0.0625f;  // compile-time
            S0 += mg[e];
            S1 = fmaf(mg[e], u, S1);
            S2 = fmaf(mg[e], u * u, S2);
            S3 = fmaf(mg[e], u * u * u, S3);
          }
        }
#pragma unroll
        for (int m = 0; m < NF; ++m) {
          float v = acc[m];
          v = fmaf(tb[m], S0, v);
          v = fmaf(tb[NF + m], S1, v);
          v = fmaf(tb[2 * NF + m], S2, v);
          v = fmaf(tb[3 * NF + m], S3, v);
          acc[m] = v;
        }
      } else {
#pragma unroll 2
        for (int q = 0; q < 8; ++q) {
          const float4 a = __ldg(reinterpret_cast<const float4*>(re + t0) + q);
          const float mg[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float4* w4 = reinterpret_cast<const float4*>(tb + (4 * q + e) * NF);
#pragma unroll
            for (int m4 = 0; m4 < NF / 4; ++m4) {
              const float4 w = w4[m4];
              acc[4 * m4 + 0] = fmaf(w.x, mg[e], acc[4 * m4 + 0]);
              acc[4 * m4 + 1] = fmaf(w.y, mg[e], acc[4 * m4 + 1]);
              acc[4 * m4 + 2] = fmaf(w.z, mg[e], acc[4 * m4 + 2]);
              acc[4 * m4 + 3] = fmaf(w.w, mg[e], acc[4 * m4 + 3]);
            }
          }
        }
      }
    }
  }
  __syncthreads();  // the table buffer becomes the reduction buffer
#pragma unroll
  for (int m = 0; m < NF; ++m) red[warp][lane][m] = acc[m];
  __syncthreads();
  for (int idx = threadIdx.x; idx < 32 * NF; idx += 256) {
    const int rl = idx / NF, m = idx % NF;
    const int row = grp * 32 + rl;
    if (row < p.K && m < p.nframes) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) v += red[w][rl][m];
      if (p.nsplit == 1) p.out[(int64_t)b * p.fps + (int64_t)row * p.nframes + m] = v;
      else p.part[(((int64_t)b * p.nsplit + split) * p.K + row) * NF + m] = v;
    }
  }
}

// sum of k_time_scat_rows' column-split partials in fixed split order
template <int NF>
__global__ void k_time_scat_sum(KTParams p, int nsig) {
  const int64_t i = blockIdx.x * 256 + threadIdx.x;
  if (i >= (int64_t)nsig * p.K * p.nframes) return;
  const int m = (int)(i % p.nframes);
  const int row = (int)((i / p.nframes) % p.K);
  const int b = (int)(i / ((int64_t)p.nframes * p.K));
  float v = 0.f;
  for (int sp = 0; sp < p.nsplit; ++sp) v += p.part[(((int64_t)b * p.nsplit + sp) * p.K + row) * NF + m];
  p.out[(int64_t)b * p.fps + (int64_t)row * p.nframes + m] = v;
}

int launch_time_scat(const Plan& P, const float* y2, int nsig, float* out, int64_t fps, int64_t off_s2,
                     cudaStream_t st, float* scratch, size_t scratch_floats) {
  int row0 = 0, n = 0;
  for (const auto& d : P.kd) {
    KTParams k{};
    k.y2 = y2 + 2 * d.y2_off;
    k.wtab = P.d_wtab + d.wtab_off;
    k.out = out + off_s2 + (int64_t)row0 * P.n_frames;
    k.y2_stride = 2 * P.y2_total;
    k.fps = fps;
    k.L = d.L;
    k.nframes = P.n_frames;
    k.K = d.K;
    k.pool_mode = (d.pool_mode == 1 && d.L % 32 == 0) ? 1 : 0;
    // the table's frame stride NF = 8 / 16 / 32 (plan.cpp, n_frames <= 32); blocks of 32
    // columns (L is a power of two >= 32 for every alpha that reaches KT: L / 32 >= 1)
    if (d.L % 32 == 0) {
      // enough CTAs for the machine (>= 4 per SM): split the columns, >= 8 blocks each
      const int ngrp = (d.K + 31) / 32, NF = P.n_frames <= 8 ? 8 : P.n_frames <= 16 ? 16 : 32;
      int nsplit = std::max(1, std::min(d.L / 32 / 8, (4 * 148 + nsig * ngrp - 1) / (nsig * ngrp)));
      while (nsplit > 1 && (size_t)nsig * nsplit * d.K * NF > scratch_floats) --nsplit;
      k.nsplit = nsplit;
      k.part = scratch;
      const int grid = nsig * ngrp * nsplit;
      if (P.n_frames <= 8) k_time_scat_rows<8><<<grid, 256, 0, st>>>(k);
      else if (P.n_frames <= 16) k_time_scat_rows<16><<<grid, 256, 0, st>>>(k);
      else k_time_scat_rows<32><<<grid, 256, 0, st>>>(k);
      if (nsplit > 1) {
        const int sg = (int)(((int64_t)nsig * d.K * P.n_frames + 255) / 256);
        if (P.n_frames <= 8) k_time_scat_sum<8><<<sg, 256, 0, st>>>(k, nsig);
        else if (P.n_frames <= 16) k_time_scat_sum<16><<<sg, 256, 0, st>>>(k, nsig);
        else k_time_scat_sum<32><<<sg, 256, 0, st>>>(k, nsig);
        ++n;
      }
    } else {
      const int grid = nsig * d.K;
      if (P.n_frames <= 8) k_time_scat<8><<<grid, 256, 0, st>>>(k);
      else if (P.n_frames <= 16) k_time_scat<16><<<grid, 256, 0, st>>>(k);
      else k_time_scat<32><<<grid, 256, 0, st>>>(k);
    }
    row0 += d.K;
    ++n;
  }
  return n;
}

int launch_kd(const Plan& P, const float* y2, int nsig, float* part, cudaStream_t st, const UnitSel* sel) {
  int n = 0;
  for (size_t i = 0; i < P.kd.size(); ++i) {
    const auto& d = P.kd[i];
    KDParams k{};
    k.chunk_sel = sel ? sel->d_sel + sel->off[i] : nullptr;
    k.nsel = sel ? sel->cnt[i] : d.nchunks;
    if (k.nsel == 0) continue;
    k.A = (const float2*)P.d_A + d.a_off;
    k.y2 = y2;
    k.g = P.d_g + d.g_off;
    k.part = part;
    k.K = d.K;
    k.Kpad = d.Kpad;
    k.Mpad = P.Mpad;
    k.L = d.L;
    k.D = d.D;
    k.frame0 = P.frame0;
    k.nframes = P.n_frames;
    k.chunk = d.chunk;
    k.nchunks = d.nchunks;
    k.y2_off = 2 * d.y2_off;
    k.part_off = d.part_off;
    k.y2_stride = 2 * P.y2_total;
    k.part_stride = P.part_total;
    const int grid = nsig * k.nsel * (P.Mpad / 64);
    if (P.n_frames <= 8) k_kd_simt<8><<<grid, 256, 0, st>>>(k);
    else if (P.n_frames <= 16) k_kd_simt<16><<<grid, 256, 0, st>>>(k);
    else k_kd_simt<32><<<grid, 256, 0, st>>>(k);
    ++n;
  }
  return n;
}

size_t ke_smem_bytes(const Plan& P) {
  int maxrows = 0;
  for (const auto& f : P.fr) maxrows = std::max(maxrows, f.nrows);
  return (size_t)(maxrows * P.n_frames + P.n1 * P.NPT + maxrows * P.NPT) * sizeof(float);
}

int launch_ke(const Plan& P, const KEParams& kp, int nsig, cudaStream_t st) {
  const size_t sm = ke_smem_bytes(P);
  dim3 grid(nsig, (unsigned)P.paths.size());
  k_ke<<<grid, 256, sm, st>>>(kp);
  return 1;
}

cudaError_t ke_set_smem(const Plan& P) {
  return cudaFuncSetAttribute(k_ke, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ke_smem_bytes(P));
}

void launch_resynth_loss(const float* Sy, const float* Sx, int64_t n, double* E, float* dout, cudaStream_t st) {
  dev::k_resynth_loss<<<1, 256, 0, st>>>(Sy, Sx, n, E, dout);
}

int launch_mulog_mu(const Plan& P, const float* S, int64_t B, float* mu, cudaStream_t st) {
  const int64_t off_s2 = P.n_frames + (int64_t)P.n1 * P.n_frames;
  const int map = P.lam_out * P.n_frames;
  const int64_t fps = off_s2 + (int64_t)P.paths.size() * map;
  k_mulog_mu<<<(unsigned)P.paths.size(), 256, 0, st>>>(S, B, fps, off_s2, map, mu);
  return 1;
}

int launch_mulog_apply(const Plan& P, const float* S, int64_t B, const float* mu, float eps, float* out,
                       cudaStream_t st) {
  const int64_t off_s2 = P.n_frames + (int64_t)P.n1 * P.n_frames;
  const int map = P.lam_out * P.n_frames;
  const int64_t fps = off_s2 + (int64_t)P.paths.size() * map;
  const int64_t n = B * fps;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_mulog_apply<<<(unsigned)blocks, 256, 0, st>>>(S, n, fps, off_s2, map, mu, eps, out);
  return 1;
}

int launch_u2_map(const Plan& P, const float* y2, int nsig, int path, int rows, int cols, float* out,
                  cudaStream_t st) {
  const jtfs_path_t& ph = P.paths[path];
  const FrFilter& f = P.fr[P.path_filter[path]];
  int slot = -1;
  for (size_t i = 0; i < P.kd.size(); ++i)
    if (P.kd[i].alpha == ph.alpha) slot = (int)i;
  const AlphaKD& d = P.kd[slot];
  const int nbeta = (int)P.bf.xi.size();
  U2MapParams k{};
  k.y2 = y2;
  if (f.kind == 0) {
    // stored taps are psi_{beta,+1}; psi_{beta,-1} = their conjugate (psi_hat real, reading R10)
    k.hc = (const float2*)P.d_hphi + (size_t)f.beta * P.N_fr;
    k.conj = f.theta == -1;
  } else {
    k.hr = P.d_hphi + (size_t)2 * nbeta * P.N_fr;
  }
  k.out = out;
  k.y2_off = 2 * d.y2_off;
  k.y2_stride = 2 * P.y2_total;
  k.K = d.K;
  k.L = d.L;
  k.N_fr = P.N_fr;
  k.k = f.k;
  k.c0 = (P.pad_left + (1 << d.k_alpha) - 1) >> d.k_alpha;
  k.rows = rows;
  k.cols = cols;
  k_u2_map<<<dim3((cols + 255) / 256, rows, nsig), 256, 0, st>>>(k);
  return 1;
}

void launch_check_finite(const float* x, int64_t n, int* flag, cudaStream_t st) {
  k_check_finite<<<296, 256, 0, st>>>(x, n, flag);
}


// =================================================================================
// backward (VJP) orchestration, see backward.inc
// =================================================================================
int launch_backward(Plan& P, const float* x, int nb, const float* dout, float* dx, const BwdWs& w,
                    cudaStream_t st) {
  int n = 0;
  const float2* W32 = (const float2*)P.d_twiddle;
  const int ltw = ilog2_exact(P.N_tw);
  // ---- forward recompute of the intermediates (X_hat, U1hat, Y_phi, Y2) ----
  n += launch_pad_fft(P, x, nb, w.xhat, w.tmp, st);
  n += launch_first_order(P, w.xhat, nb, w.u1, w.u1hat, w.tmp, false, st);
  jtfs_layout_t lay{};
  {
    int64_t off_s1 = P.n_frames, off_s2 = off_s1 + (int64_t)P.n1 * P.n_frames;
    lay.off_s0 = 0;
    lay.off_s1 = off_s1;
    lay.off_s2 = off_s2;
    lay.floats_per_signal = off_s2 + (int64_t)P.paths.size() * P.lam_out * P.n_frames;
  }
  n += launch_phi_first(P, w.xhat, w.u1hat, nb, w.yphi, w.scratch_out, lay.floats_per_signal, lay.off_s0,
                        lay.off_s1, P.d_u1_off, P.d_k1, (const Band*)P.d_band_L1, st);
  n += launch_second_order(P, w.u1hat, nb, w.y2, w.tmp, st);
  // ---- KE^T ----
  const int NF = P.n_frames <= 8 ? 8 : P.n_frames <= 16 ? 16 : P.n_frames <= 32 ? 32 : 64;
  const int64_t dP_stride = (int64_t)P.kd.size() * P.Mpad * P.n_frames;
  cudaMemsetAsync(w.dP, 0, (size_t)nb * dP_stride * 4, st);
  {
    BwdKEParams k{};
    k.paths = (const DevPath*)P.d_paths;
    k.filters = (const DevFilter*)P.d_fr;
    k.W = P.d_W;
    k.Wrange = (const int2*)P.d_Wrange;
    k.dout = dout;
    k.dP = w.dP;
    k.fps = lay.floats_per_signal;
    k.off_s2 = lay.off_s2;
    k.dP_stride = dP_stride;
    k.lam_out = P.lam_out;
    k.n_frames = P.n_frames;
    k.Mpad = P.Mpad;
    k_bwd_ke<<<dim3(nb, (unsigned)P.paths.size()), 256, 0, st>>>(k);
    ++n;
  }
  {
    BwdPhiParams k{};
    k.paths = (const DevPath*)P.d_paths;
    k.filters = (const DevFilter*)P.d_fr;
    k.rprime = P.d_rprime;
    k.W = P.d_W;
    k.Wrange = (const int2*)P.d_Wrange;
    const int nbeta = (int)P.bf.xi.size();
    k.hpsi = (const float2*)P.d_hphi;
    k.hphiF = P.d_hphi + (size_t)2 * nbeta * P.N_fr;
    k.gT = k.hphiF + P.N_fr;
    k.yphi = w.yphi;
    k.dout = dout;
    k.dyphi = w.dyphi;
    k.fps = lay.floats_per_signal;
    k.off_s2 = lay.off_s2;
    k.n_paths = (int)P.paths.size();
    k.n1 = P.n1;
    k.NPT = P.NPT;
    k.N_fr = P.N_fr;
    k.lam_out = P.lam_out;
    k.n_frames = P.n_frames;
    k.frame0 = P.frame0;
    k.k_phiphi = P.prm.average_fr ? P.log2F : 0;
    int maxrows = 0;
    for (const auto& f : P.fr) maxrows = std::max(maxrows, f.nrows);
    const size_t sm = (size_t)2 * P.n1 * P.NPT * 4 + (size_t)maxrows * P.NPT * 8;
    cudaFuncSetAttribute(k_bwd_phi, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    k_bwd_phi<<<nb, 256, sm, st>>>(k);
    ++n;
  }
  // ---- KD^T per alpha ----
  for (size_t a = 0; a < P.kd.size(); ++a) {
    const auto& d = P.kd[a];
    BwdKDParams k{};
    k.A = (const float2*)P.d_A + d.a_off;
    k.y2 = w.y2 + 2 * d.y2_off;
    k.dP = w.dP + (int64_t)a * P.Mpad * P.n_frames;
    k.g = P.d_g + d.g_off;
    k.gy2 = w.gy2 + 2 * d.y2_off;
    k.y2_stride = 2 * P.y2_total;
    k.dP_stride = dP_stride;
    k.K = d.K;
    k.Kpad = d.Kpad;
    k.Mpad = P.Mpad;
    k.L = d.L;
    k.D = d.D;
    k.frame0 = P.frame0;
    k.nframes = P.n_frames;
    const size_t sm = (size_t)d.Kpad * 32 * 8 + (size_t)d.Kpad * 64 * 8 + 64 * 32 * 8 + 32 * NF * 4 + 64 * NF * 4;
    const int grid = nb * (d.L / 32);
    auto go = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      kern<<<grid, 256, sm, st>>>(k);
    };
    if (d.Kpad <= 64) {
      if (NF == 8) go(k_bwd_kd<8, 64>); else if (NF == 16) go(k_bwd_kd<16, 64>); else go(k_bwd_kd<32, 64>);
    } else if (d.Kpad <= 128) {
      if (NF == 8) go(k_bwd_kd<8, 128>); else if (NF == 16) go(k_bwd_kd<16, 128>); else go(k_bwd_kd<32, 128>);
    } else {
      if (NF == 8) go(k_bwd_kd<8, 192>); else if (NF == 16) go(k_bwd_kd<16, 192>); else go(k_bwd_kd<32, 192>);
    }
    ++n;
  }
  // ---- KC^T: G = DFT(dY2) per y2 row ----
  for (const auto& g : P.y2_groups) {
    const int nr = (int)g.rows.size();
    ProbPlanarC2C pc{w.gy2, w.G, 2 * P.y2_total, P.y2_total, g.d_rows, nr, 1 << g.log2L};
    dispatch_log2(g.log2L, [&](auto c) {
      constexpr int LG = decltype(c)::value;
      if constexpr (LG <= 12) launch_rows<LG, -1>(pc, nb * nr, W32, ltw, st);
      else launch_fft4<LG, -1>(pc, pc, nb * nr, w.tmp, W32, ltw, st);
    });
    n += g.log2L <= 12 ? 1 : 2;
  }
  {
    BwdU1Params k{};
    k.rows = P.d_bw_rows;
    k.rowoff = P.d_bw_rowoff;
    k.G = w.G;
    k.G_stride = P.y2_total;
    k.bandvals = P.d_bandvals;
    k.u1_off = P.d_u1_off;
    k.k1 = P.d_k1;
    k.band_L1 = (const Band*)P.d_band_L1;
    k.dout = dout;
    k.dyphi = w.dyphi;
    k.gu1hat = w.gu1hat;
    k.u1_total = P.u1_total;
    k.fps = lay.floats_per_signal;
    k.off_s1 = lay.off_s1;
    k.n1 = P.n1;
    k.N_pad = P.N_pad;
    k.NPT = P.NPT;
    k.frame0 = P.frame0;
    k.n_frames = P.n_frames;
    k.total = (int64_t)nb * P.u1_total;
    k_bwd_gather_u1hat<<<(unsigned)((k.total + 255) / 256), 256, 0, st>>>(k);
    ++n;
  }
  // ---- KB^T ----
  for (const auto& g : P.u1_groups) {
    const int nr = (int)g.rows.size();
    ProbC2RealRow pr{w.gu1hat, w.gu1, P.u1_total, g.d_rows, nr, 1.f};
    ProbFoldComplex pw{w.xhat, P.N_pad, g.d_rows, nr, P.d_bandvals, 1 << g.log2L, w.wb, P.u1_total};
    ProbGradMod pg{w.gu1, w.wb, w.gw, P.u1_total, g.d_rows, nr};
    dispatch_log2(g.log2L, [&](auto c) {
      constexpr int LG = decltype(c)::value;
      if constexpr (LG <= 12) {
        launch_rows<LG, +1>(pr, nb * nr, W32, ltw, st);
        launch_rows<LG, +1>(pw, nb * nr, W32, ltw, st);
        launch_rows<LG, -1>(pg, nb * nr, W32, ltw, st);
      } else {
        launch_fft4<LG, +1>(pr, pr, nb * nr, w.tmp, W32, ltw, st);
        launch_fft4<LG, +1>(pw, pw, nb * nr, w.tmp, W32, ltw, st);
        launch_fft4<LG, -1>(pg, pg, nb * nr, w.tmp, W32, ltw, st);
      }
    });
    n += g.log2L <= 12 ? 3 : 6;
  }
  {
    BwdXParams k{};
    k.rows = P.u1_rows_flat;
    k.k1 = P.d_k1;
    k.GW = w.gw;
    k.u1_total = P.u1_total;
    k.fps = lay.floats_per_signal;
    k.off_s0 = lay.off_s0;
    k.bandvals = P.d_bandvals;
    k.band_pad = P.band_phiT_pad;
    k.dout = dout;
    k.gxhat = w.gxhat;
    k.n1 = P.n1;
    k.N_pad = P.N_pad;
    k.NPT = P.NPT;
    k.frame0 = P.frame0;
    k.n_frames = P.n_frames;
    k_bwd_gather_xhat<<<dim3((P.N_pad + 255) / 256, nb), 256, 0, st>>>(k);
    ++n;
  }
  // ---- KA^T ----
  {
    ProbPadAdj pa{w.gxhat, w.gxpad, P.N_pad};
    dispatch_log2(ilog2_exact(P.N_pad), [&](auto c) {
      constexpr int LG = decltype(c)::value;
      if constexpr (LG <= 12) launch_rows<LG, +1>(pa, nb, W32, ltw, st);
      else launch_fft4<LG, +1>(pa, pa, nb, w.tmp, W32, ltw, st);
    });
    n += ilog2_exact(P.N_pad) <= 12 ? 1 : 2;
    const int64_t total = (int64_t)nb * P.N;
    k_bwd_unpad<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(w.gxpad, dx, P.N, P.N_pad, P.pad_left,
                                                                 P.prm.pad_mode == JTFS_PAD_PERIODIC, total);
    ++n;
  }
  return n;
}

}  // namespace jtfs
