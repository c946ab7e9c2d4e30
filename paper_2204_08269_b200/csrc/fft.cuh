// Shared-memory Stockham FFT for sm_100a (radix-8 passes + one radix-2/4 pass),
// generic over the complex type CT = float2 (fp32) or double2 (fp64).
//
// G rows of length L = 2^LOG2L live in shared memory at s[g*LS + e] (LS >= L is
// the row stride; LS = L + 1 breaks the bank conflicts of column gathers).  NT
// threads run each pass: every thread loads its butterflies' inputs into
// registers, barrier, twiddle + in-register radix-R DFT, store to the Stockham
// output positions, barrier (one buffer, in place).  Twiddles come from a table
// W[t] = exp(-2 pi i t / N_tw) built in fp64 on the host.
// DIR = -1: forward DFT  sum_n x[n] e^{-2 pi i k n / L};  DIR = +1: unnormalised inverse.
#pragma once
#include <cuda_runtime.h>

namespace jtfs {
namespace dev {

template <class CT> struct CxT;
template <> struct CxT<float2> {
  using R = float;
  __device__ static __forceinline__ float2 make(float a, float b) { return make_float2(a, b); }
};
template <> struct CxT<double2> {
  using R = double;
  __device__ static __forceinline__ double2 make(double a, double b) { return make_double2(a, b); }
};

template <class CT>
__device__ __forceinline__ CT cadd(CT a, CT b) { return CxT<CT>::make(a.x + b.x, a.y + b.y); }
template <class CT>
__device__ __forceinline__ CT csub(CT a, CT b) { return CxT<CT>::make(a.x - b.x, a.y - b.y); }
// fp32: one packed FP32x2 instruction (FADD2) per complex add / subtract -- the compiler
// does not pair float2 adds by itself; each lane rounds exactly like add.rn.f32
template <>
__device__ __forceinline__ float2 cadd<float2>(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
template <>
__device__ __forceinline__ float2 csub<float2>(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
template <class CT>
__device__ __forceinline__ CT cmul(CT a, CT b) {
  return CxT<CT>::make(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// fp32: a b = a b.x + (a.y, a.x) (-b.y, b.y) as FMUL2 + FFMA2 -- ptxas folds the lane
// swap, the one-lane negation and the broadcasts into operand modifiers (2 instructions
// instead of 4; each lane is one rounded product + one fused multiply-add)
__device__ __forceinline__ unsigned long long pk2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
template <>
__device__ __forceinline__ float2 cmul<float2>(float2 a, float2 b) {
  unsigned long long t, r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk2(a.y, a.x)), "l"(pk2(-b.y, b.y)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.x)), "l"(t));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }

template <int DIR, class CT>
__device__ __forceinline__ CT twiddle(const CT* __restrict__ W, int u) {
  const CT w = __ldg(W + u);
  return DIR < 0 ? w : CxT<CT>::make(w.x, -w.y);
}

// cos(2 pi j / 16), j in [0, 8]
__device__ __forceinline__ double c16(int j) {
  switch (j) {
    case 0: return 1.0;
    case 1: return 0.92387953251128675613;
    case 2: return 0.70710678118654752440;
    case 3: return 0.38268343236508977173;
    case 4: return 0.0;
    case 5: return -0.38268343236508977173;
    case 6: return -0.70710678118654752440;
    case 7: return -0.92387953251128675613;
    default: return -1.0;
  }
}

// multiply by exp(DIR * 2 pi i j / 16), j in [0, 8) a compile-time constant after
// unrolling; sin(2 pi j / 16) = cos(2 pi |j - 4| / 16)
template <int DIR, class CT>
__device__ __forceinline__ CT rot16(CT a, int j) {
  using R = typename CxT<CT>::R;
  if (j == 0) return a;
  if (j == 4) return DIR < 0 ? CxT<CT>::make(a.y, -a.x) : CxT<CT>::make(-a.y, a.x);
  const R c = (R)c16(j);
  const R s = (R)(DIR * c16(j < 4 ? 4 - j : j - 4));
  return cmul(a, CxT<CT>::make(c, s));
}

// Shared-memory index padding: one pad element after every 16 (breaks the bank
// conflicts of the stride-R writes of the early Stockham passes).
__host__ __device__ constexpr int padx(int e) { return e + (e >> 4); }
// padded row stride for rows of length L (odd when >= 16, for column gathers)
__host__ __device__ constexpr int pad_row(int L) { return L < 16 ? L : L + (L >> 4) + 1; }

__host__ __device__ constexpr int bitrev(int v, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((v >> i) & 1) << (bits - 1 - i);
  return r;
}
__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }

// In-register R-point DFT (R = 2, 4, 8, 16): radix-2 decimation in frequency,
// then the bit-reversal permutation so that v[r] = X[r] on exit.
template <int R, int DIR, class CT>
__device__ __forceinline__ void dft_reg(CT (&v)[R]) {
#pragma unroll
  for (int span = R / 2; span >= 1; span >>= 1) {
#pragma unroll
    for (int start = 0; start < R; start += 2 * span) {
#pragma unroll
      for (int k = 0; k < span; ++k) {
        const CT a = v[start + k], b = v[start + k + span];
        v[start + k] = cadd(a, b);
        v[start + k + span] = rot16<DIR>(csub(a, b), k * (16 / (2 * span)));
      }
    }
  }
  constexpr int bits = ilog2c(R);
  CT t[R];
#pragma unroll
  for (int r = 0; r < R; ++r) t[r] = v[bitrev(r, bits)];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = t[r];
}

// One Stockham pass of radix R over G rows of length L held in smem s[g*LS + padx(e)].
// Wp: this pass's twiddles in shared memory, Wp[(r - 1) * Ns + k] = exp(-2 pi i r k / (R Ns))
// (k = j mod Ns is contiguous across a warp: conflict-free or broadcast reads).
template <int LOG2L, int R, int G, int NT, int DIR, int LS, class CT>
__device__ __forceinline__ void stockham_pass(CT* s, int log2Ns, const CT* Wp) {
  constexpr int L = 1 << LOG2L;
  constexpr int LR = L / R;
  constexpr int NBF = G * LR;
  constexpr int BPT = (NBF + NT - 1) / NT;
  const int Ns = 1 << log2Ns;
  CT v[BPT][R];
  int base[BPT];
#pragma unroll
  for (int i = 0; i < BPT; ++i) {
    const int bf = threadIdx.x + i * NT;
    base[i] = -1;
    if ((NBF % NT == 0) || bf < NBF) {
      const int g = bf / LR, j = bf % LR;
      const CT* row = s + g * LS;
#pragma unroll
      for (int r = 0; r < R; ++r) v[i][r] = row[padx(j + r * LR)];
      const int k = j & (Ns - 1);
      if (Ns > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          const CT w = Wp[(r - 1) * Ns + k];
          v[i][r] = cmul(v[i][r], DIR < 0 ? w : CxT<CT>::make(w.x, -w.y));
        }
      }
      dft_reg<R, DIR>(v[i]);
      base[i] = g * LS + (j - k) * R + k;  // row start + unpadded offset of r = 0
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < BPT; ++i) {
    if (base[i] >= 0) {
      const int g = (threadIdx.x + i * NT) / LR;
      const int e0 = base[i] - g * LS;
#pragma unroll
      for (int r = 0; r < R; ++r) s[g * LS + padx(e0 + r * Ns)] = v[i][r];
    }
  }
  __syncthreads();
}

// Stage the per-pass twiddle tables of a length-L FFT into shared memory (at
// most L entries): for every pass with Ns > 1 (same pass sequence as fft_smem),
// Ws[off + (r - 1) * Ns + k] = W_L[(r k) << (LOG2L - log2Ns - log2R)], read from
// the contiguous length-L table Wg (exp(-2 pi i t / L)).
template <int LOG2L, int NT, class CT>
__device__ __forceinline__ void stage_twiddles(CT* Ws, const CT* __restrict__ Wg) {
  constexpr int REM = LOG2L % 3;
  int off = 0, log2Ns = REM;  // the radix-2^REM pass runs at Ns = 1 (no twiddles)
  if constexpr (LOG2L >= 3) {
    for (int p = 0; p < LOG2L / 3; ++p, log2Ns += 3) {
      const int Ns = 1 << log2Ns;
      if (Ns > 1) {
        const int sh = LOG2L - log2Ns - 3;
        for (int idx = threadIdx.x; idx < 7 * Ns; idx += NT) {
          const int r = idx / Ns + 1, k = idx % Ns;
          Ws[off + idx] = __ldg(Wg + ((r * k) << sh));
        }
        off += 7 * Ns;
      }
    }
  }
}

// Full FFT of G rows in smem (caller has __syncthreads()'d after filling s and the
// shared per-pass twiddle tables Ws built by stage_twiddles<LOG2L>).
template <int LOG2L, int G, int NT, int DIR, int LS = pad_row(1 << LOG2L), class CT>
__device__ __forceinline__ void fft_smem(CT* s, const CT* Ws) {
  constexpr int REM = LOG2L % 3;
  int log2Ns = 0, off = 0;
  if constexpr (REM != 0) {
    stockham_pass<LOG2L, (1 << REM), G, NT, DIR, LS>(s, 0, Ws);
    log2Ns = REM;
  }
  if constexpr (LOG2L >= 3) {
#pragma unroll 1
    for (int p = 0; p < LOG2L / 3; ++p) {
      stockham_pass<LOG2L, 8, G, NT, DIR, LS>(s, log2Ns, Ws + off);
      if (log2Ns > 0) off += 7 << log2Ns;
      log2Ns += 3;
    }
  }
}

// ---------------------------------------------------------------------------------
// Fused variant: the first pass takes its inputs straight from global memory
// (load(g, e)) and the last pass writes straight to global memory (store(g, e, v)),
// which saves one shared-memory round trip (and one barrier) at each end.  COLMAJOR
// maps consecutive threads to consecutive rows g (coalesced column gathers of the
// four-step pass A); otherwise to consecutive elements of a row.
// Preconditions: LOG2L >= 3; the shared per-pass twiddles are staged and visible
// (the caller's barrier after stage_twiddles -- the first pass uses none).
// ---------------------------------------------------------------------------------
template <int LOG2L, int R, int G, int NT, int DIR, int LS, bool COLMAJOR, bool FROM_G, bool TO_G, class CT,
          class LF, class SF>
__device__ __forceinline__ void stockham_pass_x(CT* s, int log2Ns, const CT* Wp, const LF& load, const SF& store) {
  constexpr int L = 1 << LOG2L;
  constexpr int LR = L / R;
  constexpr int NBF = G * LR;
  constexpr int BPT = (NBF + NT - 1) / NT;
  const int Ns = 1 << log2Ns;
  CT v[BPT][R];
  int gg[BPT], e0s[BPT];
#pragma unroll
  for (int i = 0; i < BPT; ++i) {
    const int bf = threadIdx.x + i * NT;
    gg[i] = -1;
    if ((NBF % NT == 0) || bf < NBF) {
      const int g = COLMAJOR ? bf % G : bf / LR, j = COLMAJOR ? bf / G : bf % LR;
      if constexpr (FROM_G) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[i][r] = load(g, j + r * LR);
      } else {
        const CT* row = s + g * LS;
#pragma unroll
        for (int r = 0; r < R; ++r) v[i][r] = row[padx(j + r * LR)];
      }
      gg[i] = g;
      e0s[i] = j;
    }
  }
#pragma unroll
  for (int i = 0; i < BPT; ++i) {
    if (gg[i] >= 0) {
      const int j = e0s[i];
      const int k = j & (Ns - 1);
      if (Ns > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          const CT w = Wp[(r - 1) * Ns + k];
          v[i][r] = cmul(v[i][r], DIR < 0 ? w : CxT<CT>::make(w.x, -w.y));
        }
      }
      dft_reg<R, DIR>(v[i]);
      e0s[i] = (j - k) * R + k;
    }
  }
  if constexpr (!FROM_G && !TO_G) __syncthreads();  // in place: all reads before any write
#pragma unroll
  for (int i = 0; i < BPT; ++i) {
    if (gg[i] >= 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (TO_G) store(gg[i], e0s[i] + r * Ns, v[i][r]);
        else s[gg[i] * LS + padx(e0s[i] + r * Ns)] = v[i][r];
      }
    }
  }
  if constexpr (!TO_G) __syncthreads();
}

// Full fused FFT of G rows: inputs from load (FUSE_IN) or from smem (the caller has
// filled it and synchronised), outputs to store (FUSE_OUT) or left in smem in
// natural order.  Pass order: radix-2^REM at Ns = 1 (if LOG2L % 3), then radix-8.
template <int LOG2L, int G, int NT, int DIR, int LS, bool COLMAJOR, bool FUSE_IN, bool FUSE_OUT, class CT,
          class LF, class SF, bool COL_FIRST = COLMAJOR>
__device__ __forceinline__ void fft_fused(CT* s, const CT* Ws, const LF& load, const SF& store) {
  // COL_FIRST: thread mapping of the first pass (the loads); COLMAJOR: of the others
  static_assert(LOG2L >= 3, "fused FFT needs at least one radix-8 pass");
  constexpr int REM = LOG2L % 3;
  constexpr int NP8 = LOG2L / 3;
  int log2Ns = 0, off = 0;
  if constexpr (REM != 0) {
    stockham_pass_x<LOG2L, (1 << REM), G, NT, DIR, LS, COL_FIRST, FUSE_IN, false>(s, 0, Ws, load, store);
    log2Ns = REM;
  }
#pragma unroll
  for (int p = 0; p < NP8; ++p) {
    const bool first = (REM == 0 && p == 0), last = (p == NP8 - 1);
    const CT* Wp = Ws + off;
    if (first && last) {
      stockham_pass_x<LOG2L, 8, G, NT, DIR, LS, COL_FIRST, FUSE_IN, FUSE_OUT>(s, log2Ns, Wp, load, store);
    } else if (first) {
      stockham_pass_x<LOG2L, 8, G, NT, DIR, LS, COL_FIRST, FUSE_IN, false>(s, log2Ns, Wp, load, store);
    } else if (last) {
      stockham_pass_x<LOG2L, 8, G, NT, DIR, LS, COLMAJOR, false, FUSE_OUT>(s, log2Ns, Wp, load, store);
    } else {
      stockham_pass_x<LOG2L, 8, G, NT, DIR, LS, COLMAJOR, false, false>(s, log2Ns, Wp, load, store);
    }
    if (log2Ns > 0) off += 7 << log2Ns;
    log2Ns += 3;
  }
}

// offset of the length-L table inside the concatenated per-length twiddle tables
// (lengths 2, 4, ..., 2^k stored back to back: offset(L) = L - 2)
__host__ __device__ constexpr int tw_offset(int log2L) { return (1 << log2L) - 2; }

}  // namespace dev
}  // namespace jtfs
