// Launch interface between the C ABI (abi.cu) and the kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "jtfs_internal.h"

namespace jtfs {

struct KDParams {
  const float2* A;   // A_alpha^T [Kpad][Mpad]
  const float* y2;   // micro-batch Y2 base (planar complex rows)
  const float* g;    // time pooling taps g_alpha[L]
  float* part;       // micro-batch partials base
  int K, Kpad, Mpad, L, D, frame0, nframes, chunk, nchunks;
  int64_t y2_off, part_off, y2_stride, part_stride;
  const int32_t* chunk_sel;  // selected time chunks (path sharding) or nullptr = all
  int nsel;                  // number of selected chunks (= nchunks when chunk_sel is null)
};

// KD work-unit selection of jtfs_forward_units: per alpha, cnt[a] chunk ids at
// d_sel + off[a] (device); cnt[a] == 0 skips the alpha.
struct UnitSel {
  const int32_t* d_sel = nullptr;
  std::vector<int> off, cnt;
};

struct DevPath {
  int32_t kind, filter, alpha_slot, beta;
};
struct DevFilter {
  int32_t k, nrows, row0, rp_off;
  int64_t w_off;
  int64_t wr_off;  // [lam_out] int2 {first, last + 1} row of each output's phi_F band
};
struct DevAlpha {
  int32_t nchunks, pad;  // pad: K (admissible lambda rows)
  int64_t part_off;
};

struct KEParams {
  const DevPath* paths;
  const DevFilter* filters;
  const DevAlpha* alphas;
  const int32_t* rprime;
  const float* W;
  const int2* Wrange;
  const float2* hpsi;  // [n_beta][N_fr] psi_{beta,+1} taps
  const float* hphiF;  // [N_fr]
  const float* gT;     // [NPT]
  const float* part;
  const float* yphi;
  float* out;
  int64_t fps, off_s2, part_stride;
  int n1, NPT, N_fr, lam_out, n_frames, frame0, Mpad, k_phiphi;
  const float* mu;  // NEXT-4 fused mu-log (jtfs_forward_mulog): per path mu, or nullptr
  float mu_eps;
};

int launch_pad_fft(const Plan& P, const float* x, int nsig, float2* xhat, float2* tmp, cudaStream_t st);
// tmp2 (optional): a second four-step intermediate; with it (and keep_u1 false) the
// lengths > 4096 run the fused inverse-DFT / modulus / forward-DFT middle stage
int launch_first_order(const Plan& P, const float2* xhat, int nsig, float* u1, float2* u1hat, float2* tmp,
                        bool keep_u1, cudaStream_t st, float2* tmp2 = nullptr, unsigned int* u1max = nullptr);
// per-(signal, alpha) fp16 scales ys[nsig][n_alpha] and inverses ys + nsig n_alpha (KC -> KD)
int launch_yscale(const Plan& P, const unsigned int* u1max, int nsig, float* ys, cudaStream_t st);
// KC writing KD's packed fp16 operand directly (tensor-core KD forward)
int launch_second_order16(const Plan& P, const float2* u1hat, int nsig, uint16_t* y16, const float* ysc,
                          float2* tmp, cudaStream_t st);
// fp32 Y2 -> KD's fp16 operand with exact per-(signal, alpha) scales (jtfs_debug_joint)
int launch_y16_from_y2(Plan& P, const float* y2, int nsig, uint16_t* y16, float* ys, cudaStream_t st);
int launch_phi_first(const Plan& P, const float2* xhat, const float2* u1hat, int nsig, float* yphi, float* out,
                      int64_t fps, int64_t off_s0, int64_t off_s1, const int64_t* d_u1_off, const int* d_k1,
                      const Band* d_band_L1, cudaStream_t st);
int launch_second_order(const Plan& P, const float2* u1hat, int nsig, float* y2, float2* tmp, cudaStream_t st,
                        bool modulus = false);
int launch_kd(const Plan& P, const float* y2, int nsig, float* part, cudaStream_t st, const UnitSel* sel = nullptr);
size_t ke_smem_bytes(const Plan& P);
int launch_ke(const Plan& P, const KEParams& kp, int nsig, cudaStream_t st);
int launch_time_scat(const Plan& P, const float* y2, int nsig, float* out, int64_t fps, int64_t off_s2,
                     cudaStream_t st, float* scratch, size_t scratch_floats);
cudaError_t ke_set_smem(const Plan& P);
// KD on the tensor cores from KD's fp16 operand y16 and the inverse scales ysi [nsig][n_alpha]
int launch_kd_tc(Plan& P, const uint16_t* y16, const float* ysi, int nsig, float* part, cudaStream_t st, int* err,
                 const UnitSel* sel = nullptr);
cudaError_t tc_setup_device(Plan& P);

// backward (VJP) workspace pointers for one micro-batch (abi.cu carves them)
struct BwdWs {
  float2 *xhat, *tmp, *u1hat, *G, *gu1hat, *wb, *gw, *gxhat;
  float *u1, *yphi, *y2, *scratch_out, *dP, *dyphi, *gy2, *gu1, *gxpad;
};
int launch_backward(Plan& P, const float* x, int nb, const float* dout, float* dx, const BwdWs& w,
                    cudaStream_t st);
// NEXT-1: resynthesis loss and its gradient w.r.t. the record
void launch_resynth_loss(const float* Sy, const float* Sx, int64_t n, double* E, float* dout, cudaStream_t st);
// NEXT-4: mu-log (Eqs. (adalog:mu), (adalog)) and the scale-rate map (Fig. 1)
int launch_mulog_mu(const Plan& P, const float* S, int64_t B, float* mu, cudaStream_t st);
int launch_mulog_apply(const Plan& P, const float* S, int64_t B, const float* mu, float eps, float* out,
                       cudaStream_t st);
int launch_u2_map(const Plan& P, const float* y2, int nsig, int path, int rows, int cols, float* out,
                  cudaStream_t st);
// NEXT-3: K-NN regression (knn.cu)
size_t knn_workspace_bytes(int64_t n);
cudaError_t launch_knn(const float* F, int n, int d, int64_t ldf, const double* theta, int P, int K, int32_t* nbr,
                       double* theta_hat, double* ratio, void* ws, cudaStream_t st);
size_t isomap_workspace_bytes(int64_t n, int K);
cudaError_t launch_isomap(const float* F, int n, int d, int64_t ldf, int K, int c, double* emb, double* evals,
                          void* ws, cudaStream_t st, int* disconnected);
void launch_check_finite(const float* x, int64_t n, int* flag, cudaStream_t st);
void launch_guard_check(const void* ws, const int64_t* d_starts, int n, int64_t len, int* flag, cudaStream_t st);
cudaError_t measure_fp32_peak(double* tflops_ffma, double* tflops_ffma2);  // synchronous probe
int launch_debug_fft(const Plan& P, int log2L, int dir, bool fp64, const void* in, void* out, int nrows, void* tmp,
                     cudaStream_t st);

}  // namespace jtfs
