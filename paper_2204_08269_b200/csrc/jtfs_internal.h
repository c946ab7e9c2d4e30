// Internal plan of the B200 JTFS path.  Host-side schedule + device tables.
// Written from PAPER.md Sec. 2 and DESIGN.md §3 readings; shares no
// code with oracle/ (the fp64 numpy oracle).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/jtfs.h"

namespace jtfs {

// ---- filter generator G(J', Q')  (R1, R2, R5) --------------------------
struct Bank {
  std::vector<double> xi, sigma;  // cycles/sample (or cycles/bin), descending xi
  std::vector<int> j;             // critical subsampling exponent
};
Bank morlet_bank(int J, int Q);
void morlet_hat(double xi, double sigma, int L, int n_grid, double* out);
void gauss_hat(double sigma, int L, int n_grid, double* out);

// A circular arc [m0, m0+len) (mod grid length) of a sampled spectrum whose
// values are stored in Plan::bandvals[off .. off+len).
struct Band {
  int32_t m0 = 0, len = 0;
  int64_t off = 0;
};

// One FFT row of a fused band-multiply + fold + FFT launch (per signal).
struct FoldRow {
  int64_t src_off;   // complex offset of the source spectrum row inside one signal's source buffer
  int32_t Lsrc;      // source grid length
  int32_t m0, len;   // band arc on the source grid
  int64_t band_off;  // offset into bandvals
  int64_t dst_off;   // offset of the output row inside one signal's destination buffer
  float scale;       // output scale
  int32_t pad;
};

// Where KC's fp16 store puts one Y2 row (tensor-core KD layout, kernels_tc.cu): the row's
// hi / lo / hi segments of alpha's packed [3K][2L] block (KC writes them directly).
struct Y16Row {
  int64_t off;   // halves: row lambda of the hi segment inside one signal's Y16 buffer
  int64_t seg;   // halves between the segments (K rows x 2L)
  int32_t aslot; // active-alpha index (per-(signal, alpha) scale)
  int32_t pad;
};

// A launch group: all rows (per signal) that share one FFT length.
struct FoldGroup {
  int log2L;
  std::vector<FoldRow> rows;
  FoldRow* d_rows = nullptr;
  std::vector<Y16Row> y16rows;  // y2 groups: the fp16 destinations of the same rows
  Y16Row* d_y16rows = nullptr;
};

// One active second-order temporal wavelet psi_alpha and its KD problem.
struct AlphaKD {
  int alpha;        // index in bank 2
  int K;            // admissible lambda rows [0, K)
  int k_alpha;      // time exponent
  int L;            // time length N_pad >> k_alpha
  int D;            // pooling stride 2^(log2T - k_alpha)
  int64_t y2_off;   // complex offset of Y2_alpha in one signal's Y2 buffer
  int Kpad;         // K rounded up to the contraction chunk
  int64_t a_off;    // complex offset of A_alpha^T [Kpad][Mpad] in the A table
  int64_t g_off;    // float offset of the time-pooling taps g_alpha[L]
  int chunk;        // time columns per KD work unit
  int nchunks;      // L / chunk
  int64_t part_off; // float offset of partials [nchunks][Mpad][n_frames] in one signal
  // tensor-core (tcgen05 kind::f16, fp16 two-term split) tiling, see kernels_tc.cu
  int tc_K2 = 0;        // K' = 3K packed contraction length ([hi | hi | lo] x [Y_hi; Y_lo; Y_hi])
  int tc_K16 = 0;       // K' rounded up to the MMA K-step (16)
  int tc_nkc = 0;       // 16-wide K chunks (A records per M-block)
  int tc_nbr = 1, tc_BRk = 0;  // TMA row boxes / rows per box of the fp16 B tile
  int tc_Nt = 0;        // time columns per tile (64 or 128)
  int tc_NBB = 2;       // fp16 B-operand tile buffers
  int tc_S = 2, tc_tpu = 1;
  int tc_rps = 1;       // K-records per A ring stage
  int tc_stat = 0;      // 1: A stationary per CTA (its M-part's records resident), 0: A ring
  int tc_mpart = 1, tc_mblk = 1;  // M-parts of this alpha's KD and 128-pair-row M-blocks per part
                                  // (pair: M-block pairs per part, one block per CTA)
  int tc_pair = 0;      // 1: CTA pairs (cluster of 2, tcgen05 cta_group::2, M = 256)
  int64_t tc_a16_off = 0;   // uint16 offset of A''_alpha's 16 KiB records in A16
  int64_t tc_ainv_off = 0;  // float offset of the per-row inverse A scales in Ainv
  int64_t y16_off = 0;  // fp16 offset of Y16_alpha [K16][2L] in one signal's Y16 buffer (KY output)
  int64_t ys_off = 0;   // slot of the per-(signal, alpha) Y scale in one signal's ys (= active-alpha index)
  int64_t wtab_off = 0; // float offset of the phi_T pooling table in wtab
  int pool_mode = 0;    // 0: taps [L][NF]; 1: cubic-moment coefficients [L/32][4][NF] (kernels_tc.cu)
  int nslices = 0;      // KD partial slices per signal and alpha (time chunks x epilogue sets)
};

struct TmapBlob {
  alignas(64) unsigned char b[128];
};

// A frequential filter f of the joint stage (rows of every A_alpha).
struct FrFilter {
  int kind;         // 0 psi_beta (spin), 1 phi_F
  int theta;        // -1/+1 for psi
  int beta;
  int k;            // lambda decimation exponent
  int R;            // N_fr >> k
  int row0, nrows;  // row block inside the M rows of every alpha
  std::vector<int> rprime;  // the retained rows r' (decimated grid indices)
  int64_t w_off;    // float offset of the lambda-pooling matrix W [lambda_out][nrows]
  int64_t wr_off;   // offset (int pairs) of the per-output band [first, last] of W's row q in Wrange
};

struct Plan {
  jtfs_params prm{};
  // derived scalars
  int N = 0, N_pad = 0, pad_left = 0, T = 0, log2T = 0, F = 0, log2F = 0;
  int n1 = 0, N_fr = 0, frame0 = 0, n_frames = 0, lam_out = 0, NPT = 0;  // NPT = N_pad / T
  Bank b1, b2, bf;
  std::vector<int> k1, L1;
  std::vector<int64_t> u1_off;   // per lambda offset in U1 / U1hat (per signal)
  int64_t u1_total = 0;          // sum of L1
  std::vector<AlphaKD> kd;       // active alphas in bank order
  int64_t y2_total = 0;          // complex elements of Y2 per signal
  int M = 0;                     // joint-stage output rows per alpha (all filters)
  int Mpp_rows = 0, Mpp = 0;     // spin-pair rows (KD) and their padding to whole M-blocks
  int Mpad = 0;                  // rows of the full (spin-major) layout: 2 Mpp
  int tc_n_mpart = 1, tc_n_mblk = 1;  // M-parts per KD work unit, 128-row M-blocks per part
  int kd_impl = 1;               // 1: tcgen05 (default), 0: SIMT (plan flag JTFS_KD_SIMT, validation)
  std::vector<FrFilter> fr;      // frequential filters: theta=-1 (beta), theta=+1 (beta), phi_F
  std::vector<jtfs_path_t> paths;
  std::vector<int> path_filter;  // path -> fr index (or -1)
  int64_t part_total = 0;        // floats of KD partials per signal

  // ---- host tables (fp32 unless noted) ----
  std::vector<float> bandvals;
  std::vector<Band> band_psi1;           // per lambda, on the N_pad grid
  Band band_phiT_pad;                    // phi_T on the N_pad grid (S0)
  std::vector<Band> band_phiT_L1;        // phi_T on the grid N_pad >> k, k = 0..log2T
  std::vector<FoldGroup> u1_groups;      // first-order IFFT rows grouped by L1
  std::vector<FoldGroup> y2_groups;      // second-order rows grouped by L_alpha
  std::vector<float> A;                  // complex interleaved A_alpha^T tables (SIMT KD)
  std::vector<uint16_t> A16;             // A''_alpha re/im, row-scaled fp16 hi/lo, pre-tiled/swizzled (tcgen05 KD)
  std::vector<float> Ainv;               // per alpha and row: 1 / (power-of-two row scale of A16)
  std::vector<float> wtab;               // per alpha: phi_T pooling table (taps or moment coefficients)
  int64_t y16_total = 0, ys_total = 0;   // per signal: fp16 elements of Y16, scale slots (one per alpha)
  std::vector<float> ybound;             // [n_alpha][n1]: sqrt(sum psi_hat_alpha^2) of the band row lambda
                                         // uses (Cauchy-Schwarz: |Y2| <= ybound * max|U1_lambda|)
  std::vector<float> g;                  // time pooling taps per alpha
  std::vector<float> W;                  // lambda pooling matrices per filter
  std::vector<int32_t> Wrange;           // per filter and output row q: first, last + 1 row of |W| >= 1e-9 max
  std::vector<float> hphi;               // phi_t paths: [n_beta][N_fr] complex psi_{beta,+1} taps,
                                         // then [N_fr] real phi_F taps, then [NPT] real phi_T taps
  std::vector<float> twiddle;            // per-length tables exp(-2 pi i t / L), L = 2..N_tw, at offset L - 2
  std::vector<double> twiddle64;         // the same in fp64 (KA)
  int N_tw = 0;

  // ---- device copies ----
  int device = -1;
  float* d_bandvals = nullptr;
  float* d_A = nullptr;
  uint16_t* d_A16 = nullptr;
  float* d_Ainv = nullptr;
  float* d_wtab = nullptr;
  float* d_ybound = nullptr;
  float* d_g = nullptr;
  float* d_W = nullptr;
  int32_t* d_Wrange = nullptr;
  float* d_hphi = nullptr;
  float* d_twiddle = nullptr;
  double* d_twiddle64 = nullptr;
  void* d_alphas = nullptr;    // DevAlpha[n_alpha]
  void* d_fr = nullptr;        // DevFilter[n_filters]
  int32_t* d_rprime = nullptr; // concatenated retained rows of every filter
  void* d_paths = nullptr;     // DevPath[n_paths]
  int64_t* d_u1_off = nullptr; // per lambda
  int32_t* d_k1 = nullptr;     // per lambda
  Band* d_band_L1 = nullptr;   // phi_T bands per k
  // backward (VJP) tables: per lambda its (alpha, lambda) Y2 rows (pad = log2 L_alpha),
  // offsets [n1 + 1]; the first-order rows in lambda order
  FoldRow* d_bw_rows = nullptr;
  int32_t* d_bw_rowoff = nullptr;
  FoldRow* u1_rows_flat = nullptr;
  std::vector<void*> allocations;

  int mb = 16;                 // signals per micro-batch
  // a second stream for the KD launches of the slower alphas (kernels_tc.cu), created
  // with the device tables; fork / join events are created per call
  void* kd_side_stream = nullptr;
  int kd_side_from = 1 << 30;  // first active-alpha index launched on the side stream

  // ---- profiling (the only mutable state; see jtfs_profile_enable) ----
  bool prof = false;
  std::vector<std::pair<void*, void*>> prof_events[6];  // cudaEvent_t pairs per stage
  int64_t launches[6] = {0, 0, 0, 0, 0, 0};
  std::vector<std::vector<std::pair<void*, void*>>> prof_kd;  // per active alpha
};

// plan.cpp
std::string build_plan(const jtfs_params& p, Plan& plan);   // returns "" or an error message
void a16_density(const Plan& P, double thr, std::vector<int64_t>& out);  // 6 values per alpha
int ilog2_exact(int64_t v);  // -1 if not a power of two

// workspace guard bands (validation builds: -DJTFS_WS_GUARDS, abi.cu checks them after
// every forward; 0 in production builds)
#ifdef JTFS_WS_GUARDS
constexpr size_t kWsGuard = 65536;
#else
constexpr size_t kWsGuard = 0;
#endif

// workspace layout (per micro-batch of mb signals), in bytes
struct WsLayout {
  size_t xhat, tmp, tmp2, u1, u1hat, yphi, y2, y16, ys, u1max, part, sel, flag, total;
};
WsLayout ws_layout(const Plan& p, int64_t mb);

// tensor-core KD planning / device setup (kernels_tc.cu)
std::string plan_tc(Plan& P);  // "" or why an alpha cannot be tiled

// algorithmic per-signal cost per stage (jtfs_cost)
void stage_cost(const Plan& p, double flops[6], double bytes[6]);

}  // namespace jtfs
