// C ABI of libjtfs.so (declared in include/jtfs.h): plan lifecycle, queries,
// workspace, forward orchestration over micro-batches, debug taps.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "jtfs_internal.h"
#include "kernels.h"

struct jtfs_plan_s {
  jtfs::Plan P;
};

namespace {
thread_local std::string g_err;

jtfs_status fail(jtfs_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

jtfs_status cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return JTFS_ERR_CUDA;
}

bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

template <class T>
cudaError_t upload(jtfs::Plan& P, T** dst, const void* src, size_t bytes) {
  *dst = nullptr;
  if (bytes == 0) bytes = 16;
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, bytes);
  if (e != cudaSuccess) return e;
  P.allocations.push_back(d);
  if (src) e = cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice);
  *dst = (T*)d;
  return e;
}

void free_device(jtfs::Plan& P) {
  if (P.device >= 0) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(P.device);
    if (P.kd_side_stream) cudaStreamDestroy((cudaStream_t)P.kd_side_stream);
    P.kd_side_stream = nullptr;
    for (void* p : P.allocations) cudaFree(p);
    cudaSetDevice(cur);
  }
  P.allocations.clear();
}

// record the device tables of a host plan
jtfs_status upload_plan(jtfs::Plan& P) {
  using namespace jtfs;
  cudaError_t e;
#define UP(dst, src, bytes)                                    \
  do {                                                         \
    e = upload(P, &(dst), (src), (bytes));                     \
    if (e != cudaSuccess) return cuda_fail(e, "plan upload");  \
  } while (0)
  UP(P.d_bandvals, P.bandvals.data(), P.bandvals.size() * 4);
  UP(P.d_A, P.A.data(), P.A.size() * 4);
  UP(P.d_A16, P.A16.data(), P.A16.size() * 2);
  UP(P.d_Ainv, P.Ainv.data(), P.Ainv.size() * 4);
  UP(P.d_wtab, P.wtab.data(), P.wtab.size() * 4);
  UP(P.d_g, P.g.data(), P.g.size() * 4);
  UP(P.d_W, P.W.data(), P.W.size() * 4);
  UP(P.d_Wrange, P.Wrange.data(), P.Wrange.size() * 4);
  UP(P.d_hphi, P.hphi.data(), P.hphi.size() * 4);
  UP(P.d_twiddle, P.twiddle.data(), P.twiddle.size() * 4);
  UP(P.d_twiddle64, P.twiddle64.data(), P.twiddle64.size() * 8);
  for (auto& g : P.u1_groups) UP(g.d_rows, g.rows.data(), g.rows.size() * sizeof(FoldRow));
  for (auto& g : P.y2_groups) UP(g.d_rows, g.rows.data(), g.rows.size() * sizeof(FoldRow));
  for (auto& g : P.y2_groups) UP(g.d_y16rows, g.y16rows.data(), g.y16rows.size() * sizeof(Y16Row));
  UP(P.d_ybound, P.ybound.data(), P.ybound.size() * 4);
  {
    // backward tables (kernels.cu launch_backward)
    std::vector<FoldRow> u1flat;
    for (auto& g : P.u1_groups) u1flat.insert(u1flat.end(), g.rows.begin(), g.rows.end());
    UP(P.u1_rows_flat, u1flat.data(), u1flat.size() * sizeof(FoldRow));
    // y2 rows of (alpha, lambda): in each L group, alphas in kd order, K rows each
    std::vector<std::vector<FoldRow>> per(P.n1);
    for (auto& g : P.y2_groups) {
      size_t r = 0;
      for (const auto& d : P.kd) {
        if (ilog2_exact(d.L) != g.log2L) continue;
        for (int l = 0; l < d.K; ++l, ++r) {
          FoldRow fr = g.rows[r];
          fr.pad = g.log2L;
          per[l].push_back(fr);
        }
      }
    }
    std::vector<FoldRow> flat;
    std::vector<int32_t> off(1, 0);
    for (int l = 0; l < P.n1; ++l) {
      flat.insert(flat.end(), per[l].begin(), per[l].end());
      off.push_back((int32_t)flat.size());
    }
    UP(P.d_bw_rows, flat.data(), std::max<size_t>(flat.size(), 1) * sizeof(FoldRow));
    UP(P.d_bw_rowoff, off.data(), off.size() * 4);
  }
  UP(P.d_u1_off, P.u1_off.data(), P.u1_off.size() * 8);
  {
    std::vector<int32_t> k1(P.k1.begin(), P.k1.end());
    UP(P.d_k1, k1.data(), k1.size() * 4);
  }
  UP(P.d_band_L1, P.band_phiT_L1.data(), P.band_phiT_L1.size() * sizeof(Band));
  {
    std::vector<DevAlpha> da;
    for (const auto& d : P.kd) da.push_back(DevAlpha{d.nslices, d.K, d.part_off});
    UP(P.d_alphas, da.data(), da.size() * sizeof(DevAlpha));
  }
  {
    std::vector<DevFilter> df;
    std::vector<int32_t> rp;
    for (const auto& f : P.fr) {
      df.push_back(DevFilter{f.k, f.nrows, f.row0, (int32_t)rp.size(), f.w_off, f.wr_off});
      rp.insert(rp.end(), f.rprime.begin(), f.rprime.end());
    }
    UP(P.d_fr, df.data(), df.size() * sizeof(DevFilter));
    UP(P.d_rprime, rp.data(), rp.size() * 4);
  }
  {
    std::vector<DevPath> dp;
    for (size_t i = 0; i < P.paths.size(); ++i) {
      const auto& p = P.paths[i];
      int slot = -1;
      for (size_t a = 0; a < P.kd.size(); ++a)
        if (P.kd[a].alpha == p.alpha) slot = (int)a;
      dp.push_back(DevPath{p.kind, P.path_filter[i], slot, p.beta});
    }
    UP(P.d_paths, dp.data(), dp.size() * sizeof(DevPath));
  }
#undef UP
  e = jtfs::ke_set_smem(P);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(k_ke)");
  e = jtfs::tc_setup_device(P);
  if (e != cudaSuccess) return cuda_fail(e, "tcgen05 KD setup (tensor maps / smem)");
  return JTFS_OK;
}

struct WsPtrs {
  float2 *xhat, *tmp, *tmp2, *u1hat;
  float *u1, *yphi, *y2, *ys, *part;
  unsigned int* u1max;
  uint16_t* y16;
  int32_t* sel;
  int* flag;
};

WsPtrs carve(const jtfs::Plan& P, void* ws, int64_t mb) {
  const jtfs::WsLayout L = jtfs::ws_layout(P, mb);
  char* c = (char*)ws;
  WsPtrs w{};
  w.xhat = (float2*)c; c += L.xhat;
  w.tmp = (float2*)c; c += L.tmp;
  w.tmp2 = (float2*)c; c += L.tmp2;
  w.u1 = (float*)c; c += L.u1;
  w.u1hat = (float2*)c; c += L.u1hat;
  w.yphi = (float*)c; c += L.yphi;
  w.y2 = (float*)c; c += L.y2;
  w.y16 = (uint16_t*)c; c += L.y16;
  w.ys = (float*)c; c += L.ys;
  w.u1max = (unsigned int*)c; c += L.u1max;
  w.part = (float*)c; c += L.part;
  w.sel = (int32_t*)c; c += L.sel;
  w.flag = (int*)c;
  return w;
}

void layout_of(const jtfs::Plan& P, jtfs_layout_t* o) {
  o->n1 = P.n1;
  o->n_frames = P.n_frames;
  o->frame0 = P.frame0;
  o->lambda_out = P.lam_out;
  o->n_paths = (int32_t)P.paths.size();
  o->n_alpha = (int32_t)P.kd.size();
  o->n_beta = (int32_t)P.bf.xi.size();
  o->N_pad = P.N_pad;
  o->N_fr = P.N_fr;
  o->reserved = 0;
  o->off_s0 = 0;
  o->off_s1 = P.n_frames;
  o->off_s2 = o->off_s1 + (int64_t)P.n1 * P.n_frames;
  o->floats_per_signal = o->off_s2 + (int64_t)P.paths.size() * P.lam_out * P.n_frames;
}

// stage tracing (jtfs_profile_enable)
struct StageScope {
  jtfs::Plan& P;
  int stage;
  cudaStream_t st;
  cudaEvent_t e1 = nullptr;
  StageScope(jtfs::Plan& P_, int s, cudaStream_t st_) : P(P_), stage(s), st(st_) {
    static const char* const names[6] = {"KA pad+DFT", "KB first order", "KS phi_T averaging",
                                         "KC second order", "KD joint contraction", "KE phi_F pooling+pack"};
    nvtxRangePushA(names[stage]);  // host-side NVTX range around the stage's launches
    if (P.prof) {
      cudaEvent_t e0;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
      P.prof_events[stage].push_back({(void*)e0, (void*)e1});
    }
  }
  void done(int nlaunch) {
    P.launches[stage] += nlaunch;
    if (P.prof) cudaEventRecord(e1, st);
    nvtxRangePop();
  }
};

// enqueue every stage for one micro-batch of nb signals; returns "" or an error
// Options of jtfs_forward_units / jtfs_reduce_pack: KD restricted to a unit
// selection and writing an external partials buffer; KE skipped or run alone.
struct RunOpts {
  const jtfs::UnitSel* sel = nullptr;
  float* part = nullptr;  // KD partials target (default: the workspace's)
  bool skip_ke = false;
  const float* mu = nullptr;  // fused mu-log in KE (jtfs_forward_mulog)
  float mu_eps = 0.f;
  bool joint_only = false;  // jtfs_debug_joint: Y2 / Y_phi already in the workspace, run KD + KE only
};

void fill_ke_params(jtfs::Plan& P, jtfs::KEParams& kp, const float* part, const float* yphi, float* out);

std::string run_microbatch(jtfs::Plan& P, const float* x, int nb, float* out, const WsPtrs& w, bool keep_u1,
                           int upto_stage, cudaStream_t st, const RunOpts& o = RunOpts()) {
  using namespace jtfs;
  jtfs_layout_t lay;
  layout_of(P, &lay);
  // the tensor-core KD takes Y2 as its packed fp16 operand, written by KC (scale from KB's
  // per-row max |U1|); debug taps (keep_u1) and the SIMT validation KD take fp32 Y2
  const bool y16_path = P.kd_impl == 1 && !keep_u1;
  if (!o.joint_only) {
    { StageScope s(P, 0, st); s.done(launch_pad_fft(P, x, nb, w.xhat, w.tmp, st)); }
    if (upto_stage == 0) return "";
    {
      StageScope s(P, 1, st);
      if (y16_path) cudaMemsetAsync(w.u1max, 0, (size_t)nb * P.n1 * 4, st);
      s.done(launch_first_order(P, w.xhat, nb, w.u1, w.u1hat, w.tmp, keep_u1, st, w.tmp2,
                                y16_path ? w.u1max : nullptr));
    }
    {
      StageScope s(P, 2, st);
      s.done(launch_phi_first(P, w.xhat, w.u1hat, nb, w.yphi, out, lay.floats_per_signal, lay.off_s0, lay.off_s1,
                              P.d_u1_off, P.d_k1, P.d_band_L1, st));
    }
    if (upto_stage == 1) return "";
    {
      StageScope s(P, 3, st);
      if (y16_path)
        s.done(launch_yscale(P, w.u1max, nb, w.ys, st) + launch_second_order16(P, w.u1hat, nb, w.y16, w.ys, w.tmp, st));
      else
        s.done(launch_second_order(P, w.u1hat, nb, w.y2, w.tmp, st));
    }
    if (upto_stage == 2) return "";
  }
  {
    StageScope s(P, 4, st);
    int err = 0;
    float* part = o.part ? o.part : w.part;
    int n = 0;
    if (P.kd_impl == 1) {
      if (o.joint_only) n += launch_y16_from_y2(P, w.y2, nb, w.y16, w.ys, st);  // given fp32 Y2
      n += launch_kd_tc(P, w.y16, w.ys + (int64_t)nb * P.kd.size(), nb, part, st, &err, o.sel);
    } else {
      n += launch_kd(P, w.y2, nb, part, st, o.sel);
    }
    s.done(n);
    if (err) return "tcgen05 KD: cuTensorMapEncodeTiled failed for the Y2 tensor map";
  }
  if (o.skip_ke) return "";
  KEParams kp{};
  fill_ke_params(P, kp, w.part, w.yphi, out);
  kp.mu = o.mu;
  kp.mu_eps = o.mu_eps;
  { StageScope s(P, 5, st); s.done(launch_ke(P, kp, nb, st)); }
  return "";
}

void fill_ke_params(jtfs::Plan& P, jtfs::KEParams& kp, const float* part, const float* yphi, float* out) {
  using namespace jtfs;
  jtfs_layout_t lay;
  layout_of(P, &lay);
  kp.paths = (const DevPath*)P.d_paths;
  kp.filters = (const DevFilter*)P.d_fr;
  kp.alphas = (const DevAlpha*)P.d_alphas;
  kp.rprime = P.d_rprime;
  kp.W = P.d_W;
  kp.Wrange = (const int2*)P.d_Wrange;
  const int nbeta = (int)P.bf.xi.size();
  kp.hpsi = (const float2*)P.d_hphi;
  kp.hphiF = P.d_hphi + (size_t)2 * nbeta * P.N_fr;
  kp.gT = kp.hphiF + P.N_fr;
  kp.part = part;
  kp.yphi = yphi;
  kp.out = out;
  kp.fps = lay.floats_per_signal;
  kp.off_s2 = lay.off_s2;
  kp.part_stride = P.part_total;
  kp.n1 = P.n1;
  kp.NPT = P.NPT;
  kp.N_fr = P.N_fr;
  kp.lam_out = P.lam_out;
  kp.n_frames = P.n_frames;
  kp.frame0 = P.frame0;
  kp.Mpad = P.Mpad;
  kp.k_phiphi = P.prm.average_fr ? P.log2F : 0;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

extern "C" {

const char* jtfs_status_string(jtfs_status s) {
  switch (s) {
    case JTFS_OK: return "ok";
    case JTFS_ERR_INVALID_ARG: return "invalid argument";
    case JTFS_ERR_UNSUPPORTED: return "unsupported";
    case JTFS_ERR_OOM: return "out of memory";
    case JTFS_ERR_CUDA: return "CUDA error";
    case JTFS_ERR_WORKSPACE: return "workspace too small";
    case JTFS_ERR_NONFINITE: return "non-finite input";
  }
  return "unknown status";
}

const char* jtfs_last_error(void) { return g_err.c_str(); }

jtfs_status jtfs_plan_create(const jtfs_params* params, jtfs_plan_t* out) {
  if (!out) return fail(JTFS_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!params) return fail(JTFS_ERR_INVALID_ARG, "params is NULL");
  jtfs_plan_s* h = new (std::nothrow) jtfs_plan_s();
  if (!h) return fail(JTFS_ERR_OOM, "host allocation failed");
  std::string err;
  try {
    err = jtfs::build_plan(*params, h->P);
  } catch (const std::bad_alloc&) {
    delete h;
    return fail(JTFS_ERR_OOM, "host allocation failed while building the plan");
  } catch (const std::exception& e) {
    err = e.what();
  }
  if (!err.empty()) {
    delete h;
    return fail(JTFS_ERR_INVALID_ARG, err);
  }
  jtfs::Plan& P = h->P;
  if (params->device >= 0) {
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || params->device >= ndev) {
      delete h;
      return e != cudaSuccess ? cuda_fail(e, "cudaGetDeviceCount")
                              : fail(JTFS_ERR_INVALID_ARG, "device ordinal out of range");
    }
    P.device = params->device;
    DeviceGuard g(P.device);
    jtfs_status s = upload_plan(P);
    if (s != JTFS_OK) {
      free_device(P);
      delete h;
      return s;
    }
  }
  *out = h;
  return JTFS_OK;
}

jtfs_status jtfs_plan(int N, int J, int Q, int J_fr, int Q_fr, int T, int F, int flags, jtfs_plan_t* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    if (out) *out = nullptr;
    return cuda_fail(e, "cudaGetDevice");
  }
  jtfs_params p{};
  p.N = N; p.J = J; p.Q = Q; p.Q2 = 1; p.T = T; p.J_fr = J_fr; p.Q_fr = Q_fr; p.F = F;
  p.average_fr = 1; p.pad_mode = JTFS_PAD_REFLECT; p.device = dev; p.flags = (uint32_t)flags;
  return jtfs_plan_create(&p, out);
}

jtfs_status jtfs_plan_destroy(jtfs_plan_t plan) {
  if (!plan) return JTFS_OK;
  free_device(plan->P);
  delete plan;
  return JTFS_OK;
}

jtfs_status jtfs_layout(jtfs_plan_t plan, jtfs_layout_t* out) {
  if (!plan || !out) return fail(JTFS_ERR_INVALID_ARG, "NULL argument");
  layout_of(plan->P, out);
  return JTFS_OK;
}

jtfs_status jtfs_paths(jtfs_plan_t plan, jtfs_path_t* out, int32_t cap) {
  if (!plan || (!out && cap > 0) || cap < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  const int n = std::min<int>(cap, (int)plan->P.paths.size());
  for (int i = 0; i < n; ++i) out[i] = plan->P.paths[i];
  return JTFS_OK;
}

jtfs_status jtfs_lambda_xi(jtfs_plan_t plan, double* out, int32_t cap) {
  if (!plan || (!out && cap > 0) || cap < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  const int n = std::min<int>(cap, plan->P.n1);
  for (int i = 0; i < n; ++i) out[i] = plan->P.b1.xi[i];
  return JTFS_OK;
}

jtfs_status jtfs_workspace_size(jtfs_plan_t plan, int64_t batch, size_t* bytes) {
  if (!plan || !bytes || batch < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  const int64_t mb = std::max<int64_t>(1, std::min<int64_t>(batch, plan->P.mb));
  *bytes = jtfs::ws_layout(plan->P, mb).total;
  return JTFS_OK;
}

static jtfs_status check_forward_args(jtfs_plan_t plan, const void* x, int64_t B, const void* out, void* ws,
                                      size_t ws_bytes) {
  if (!plan) return fail(JTFS_ERR_INVALID_ARG, "plan is NULL");
  if (plan->P.device < 0) return fail(JTFS_ERR_UNSUPPORTED, "host-only plan (device = -1) cannot run forward");
  if (B < 0) return fail(JTFS_ERR_INVALID_ARG, "B < 0");
  if (B == 0) return JTFS_OK;
  if (!x || !out || !ws) return fail(JTFS_ERR_INVALID_ARG, "NULL buffer");
  if (!aligned(x, 16) || !aligned(out, 16)) return fail(JTFS_ERR_INVALID_ARG, "x / out must be 16-byte aligned");
  if (!aligned(ws, 256)) return fail(JTFS_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  size_t need = 0;
  jtfs_workspace_size(plan, B, &need);
  if (ws_bytes < need)
    return fail(JTFS_ERR_WORKSPACE, "workspace " + std::to_string(ws_bytes) + " < required " + std::to_string(need));
  return JTFS_OK;
}

static jtfs_status forward_impl(jtfs_plan_t plan, const float* x, int64_t B, float* out, void* ws,
                                size_t ws_bytes, void* stream, const RunOpts& opts) {
  jtfs_status s = check_forward_args(plan, x, B, out, ws, ws_bytes);
  if (s != JTFS_OK || B == 0) return s;
  jtfs::Plan& P = plan->P;
  DeviceGuard guard(P.device);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t mb = std::min<int64_t>(B, P.mb);
  WsPtrs w = carve(P, ws, mb);
  if (P.prm.flags & JTFS_CHECK_FINITE) {
    cudaMemsetAsync(w.flag, 0, sizeof(int), st);
    jtfs::launch_check_finite(x, B * (int64_t)P.N, w.flag, st);
    int h = 0;
    cudaError_t e = cudaMemcpyAsync(&h, w.flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "finite check");
    if (h) return fail(JTFS_ERR_NONFINITE, "input holds NaN or Inf");
  }
  jtfs_layout_t lay;
  layout_of(P, &lay);
#ifdef JTFS_WS_GUARDS
  // validation build: the trailing guard band of every workspace region is filled with a
  // pattern before and checked after the forward (an overflow of any region is an error)
  std::vector<int64_t> gstart;
  {
    const jtfs::WsLayout L = jtfs::ws_layout(P, mb);
    const size_t sz[13] = {L.xhat, L.tmp, L.tmp2, L.u1, L.u1hat, L.yphi, L.y2, L.y16, L.ys, L.u1max, L.part, L.sel,
                           L.flag};
    int64_t o = 0;
    for (size_t r : sz) {
      o += (int64_t)r;
      gstart.push_back(o - (int64_t)jtfs::kWsGuard);
    }
    for (int64_t g : gstart) cudaMemsetAsync((char*)ws + g, 0xA5, jtfs::kWsGuard, st);
  }
#endif
  for (int64_t b0 = 0; b0 < B; b0 += mb) {
    const int nb = (int)std::min<int64_t>(mb, B - b0);
    const std::string err = run_microbatch(P, x + b0 * P.N, nb, out + b0 * lay.floats_per_signal, w, false, 99, st, opts);
    if (!err.empty()) return fail(JTFS_ERR_CUDA, err);
  }
#ifdef JTFS_WS_GUARDS
  {
    int64_t* d_starts = nullptr;
    int* d_flag = nullptr;
    cudaMalloc(&d_starts, gstart.size() * 8);
    cudaMalloc(&d_flag, 4);
    cudaMemcpy(d_starts, gstart.data(), gstart.size() * 8, cudaMemcpyHostToDevice);
    cudaMemsetAsync(d_flag, 0, 4, st);
    jtfs::launch_guard_check(ws, d_starts, (int)gstart.size(), (int64_t)jtfs::kWsGuard, d_flag, st);
    int h = 0;
    cudaMemcpyAsync(&h, d_flag, 4, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(d_starts);
    cudaFree(d_flag);
    if (h) return fail(JTFS_ERR_CUDA, "workspace guard overwritten (region mask " + std::to_string(h) + ")");
  }
#endif
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return JTFS_OK;
}

jtfs_status jtfs_forward(jtfs_plan_t plan, const float* x, int64_t B, float* out, void* ws, size_t ws_bytes,
                         void* stream) {
  return forward_impl(plan, x, B, out, ws, ws_bytes, stream, RunOpts());
}

jtfs_status jtfs_forward_mulog(jtfs_plan_t plan, const float* x, int64_t B, const float* mu, float eps, float* out,
                               void* ws, size_t ws_bytes, void* stream) {
  if (!(eps > 0.f)) return fail(JTFS_ERR_INVALID_ARG, "eps must be > 0");
  if (B > 0 && !mu) return fail(JTFS_ERR_INVALID_ARG, "mu is NULL");
  RunOpts o;
  o.mu = mu;
  o.mu_eps = eps;
  return forward_impl(plan, x, B, out, ws, ws_bytes, stream, o);
}

jtfs_status jtfs_resynth_loss(jtfs_plan_t plan, const float* Sy, const float* Sx, double* E, float* dout,
                              void* stream) {
  if (!plan || !Sy || !Sx || !E || !dout) return fail(JTFS_ERR_INVALID_ARG, "NULL argument");
  if (plan->P.device < 0) return fail(JTFS_ERR_UNSUPPORTED, "host-only plan");
  DeviceGuard guard(plan->P.device);
  jtfs_layout_t lay;
  layout_of(plan->P, &lay);
  jtfs::launch_resynth_loss(Sy, Sx, lay.floats_per_signal, E, dout, (cudaStream_t)stream);
  cudaError_t e = cudaGetLastError();
  return e != cudaSuccess ? cuda_fail(e, "kernel launch") : JTFS_OK;
}

jtfs_status jtfs_mulog_mu(jtfs_plan_t plan, const float* S, int64_t B, float* mu, void* stream) {
  if (!plan || !S || !mu || B < 1) return fail(JTFS_ERR_INVALID_ARG, "bad argument (B must be >= 1)");
  if (plan->P.device < 0) return fail(JTFS_ERR_UNSUPPORTED, "host-only plan");
  DeviceGuard guard(plan->P.device);
  jtfs::launch_mulog_mu(plan->P, S, B, mu, (cudaStream_t)stream);
  cudaError_t e = cudaGetLastError();
  return e != cudaSuccess ? cuda_fail(e, "kernel launch") : JTFS_OK;
}

jtfs_status jtfs_mulog_apply(jtfs_plan_t plan, const float* S, int64_t B, const float* mu, float eps, float* out,
                             void* stream) {
  if (!plan || B < 0 || !(eps > 0.f)) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  if (plan->P.device < 0) return fail(JTFS_ERR_UNSUPPORTED, "host-only plan");
  if (B == 0) return JTFS_OK;
  if (!S || !mu || !out) return fail(JTFS_ERR_INVALID_ARG, "NULL buffer");
  DeviceGuard guard(plan->P.device);
  jtfs::launch_mulog_apply(plan->P, S, B, mu, eps, out, (cudaStream_t)stream);
  cudaError_t e = cudaGetLastError();
  return e != cudaSuccess ? cuda_fail(e, "kernel launch") : JTFS_OK;
}

static bool u2_shape(const jtfs::Plan& P, int32_t path, int32_t* rows, int32_t* cols) {
  if (path < 0 || path >= (int32_t)P.paths.size()) return false;
  const jtfs_path_t& ph = P.paths[path];
  if (ph.kind != JTFS_PATH_SPIN && ph.kind != JTFS_PATH_PSI_T_PHI_F) return false;
  const jtfs::FrFilter& f = P.fr[P.path_filter[path]];
  int ka = -1;
  for (const auto& d : P.kd)
    if (d.alpha == ph.alpha) ka = d.k_alpha;
  if (ka < 0) return false;
  *rows = (P.n1 + (1 << f.k) - 1) >> f.k;
  *cols = (P.N + (1 << ka) - 1) >> ka;
  return true;
}

jtfs_status jtfs_u2_map_shape(jtfs_plan_t plan, int32_t path, int32_t* rows, int32_t* cols) {
  if (!plan || !rows || !cols) return fail(JTFS_ERR_INVALID_ARG, "NULL argument");
  if (!u2_shape(plan->P, path, rows, cols))
    return fail(JTFS_ERR_INVALID_ARG, "path has no scale-rate map (psi_t paths only) or is out of range");
  return JTFS_OK;
}

jtfs_status jtfs_u2_map(jtfs_plan_t plan, const float* x, int64_t B, int32_t path, float* out, void* ws,
                        size_t ws_bytes, void* stream) {
  jtfs_status s = check_forward_args(plan, x, B, out, ws, ws_bytes);
  if (s != JTFS_OK) return s;
  int32_t rows = 0, cols = 0;
  if (!u2_shape(plan->P, path, &rows, &cols))
    return fail(JTFS_ERR_INVALID_ARG, "path has no scale-rate map (psi_t paths only) or is out of range");
  if (B == 0) return JTFS_OK;
  jtfs::Plan& P = plan->P;
  DeviceGuard guard(P.device);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t mb = std::min<int64_t>(B, P.mb);
  WsPtrs w = carve(P, ws, mb);
  for (int64_t b0 = 0; b0 < B; b0 += mb) {
    const int nb = (int)std::min<int64_t>(mb, B - b0);
    jtfs::launch_pad_fft(P, x + b0 * P.N, nb, w.xhat, w.tmp, st);
    jtfs::launch_first_order(P, w.xhat, nb, w.u1, w.u1hat, w.tmp, false, st, w.tmp2);
    jtfs::launch_second_order(P, w.u1hat, nb, w.y2, w.tmp, st);
    jtfs::launch_u2_map(P, w.y2, nb, path, rows, cols, out + b0 * (int64_t)rows * cols, st);
  }
  cudaError_t e = cudaGetLastError();
  return e != cudaSuccess ? cuda_fail(e, "kernel launch") : JTFS_OK;
}

jtfs_status jtfs_forward_host(jtfs_plan_t plan, const float* x_host, int64_t B, float* out_host, float* x_dev,
                              float* out_dev, void* ws, size_t ws_bytes, void* stream) {
  jtfs_status s = check_forward_args(plan, x_dev, B, out_dev, ws, ws_bytes);
  if (s != JTFS_OK || B == 0) return s;
  if (!x_host || !out_host) return fail(JTFS_ERR_INVALID_ARG, "NULL host buffer");
  jtfs::Plan& P = plan->P;
  DeviceGuard guard(P.device);
  cudaStream_t st = (cudaStream_t)stream;
  jtfs_layout_t lay;
  layout_of(P, &lay);
  const size_t fps = (size_t)lay.floats_per_signal;
  cudaError_t e;
  if (P.prm.flags & JTFS_CHECK_FINITE) {  // the finite check needs the whole batch first
    e = cudaMemcpyAsync(x_dev, x_host, (size_t)B * P.N * 4, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
    s = jtfs_forward(plan, x_dev, B, out_dev, ws, ws_bytes, stream);
    if (s != JTFS_OK) return s;
    e = cudaMemcpyAsync(out_host, out_dev, (size_t)B * fps * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e != cudaSuccess ? cuda_fail(e, "forward_host copies") : JTFS_OK;
  }
  // Copies overlapped with compute per micro-batch: H2D of micro-batch i + 1 on an input
  // copy stream while micro-batch i computes on the caller's stream, D2H of micro-batch i
  // on an output copy stream while i + 1 computes.  x_dev / out_dev hold the whole batch,
  // so no buffer is reused across micro-batches; the workspace is used in stream order.
  const int64_t mb = std::min<int64_t>(B, P.mb);
  const int64_t nmb = (B + mb - 1) / mb;
  cudaStream_t cin = nullptr, cout = nullptr;
  std::vector<cudaEvent_t> evs;
  auto event = [&]() {
    cudaEvent_t ev = nullptr;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    evs.push_back(ev);
    return ev;
  };
  e = cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&cout, cudaStreamNonBlocking);
  std::string err;
  if (e == cudaSuccess) {
    cudaEvent_t start = event();
    cudaEventRecord(start, st);  // the copies follow the caller's earlier work on x_dev / out_dev
    cudaStreamWaitEvent(cin, start, 0);
    cudaStreamWaitEvent(cout, start, 0);
    WsPtrs w = carve(P, ws, mb);
    for (int64_t i = 0; i < nmb && e == cudaSuccess && err.empty(); ++i) {
      const int64_t b0 = i * mb, nb = std::min<int64_t>(mb, B - b0);
      e = cudaMemcpyAsync(x_dev + b0 * P.N, x_host + b0 * P.N, (size_t)nb * P.N * 4, cudaMemcpyHostToDevice, cin);
      cudaEvent_t in_done = event();
      cudaEventRecord(in_done, cin);
      cudaStreamWaitEvent(st, in_done, 0);
      err = run_microbatch(P, x_dev + b0 * P.N, (int)nb, out_dev + b0 * fps, w, false, 99, st);
      cudaEvent_t comp_done = event();
      cudaEventRecord(comp_done, st);
      cudaStreamWaitEvent(cout, comp_done, 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(out_host + b0 * fps, out_dev + b0 * fps, (size_t)nb * fps * 4, cudaMemcpyDeviceToHost,
                            cout);
    }
    cudaEvent_t all_out = event();
    cudaEventRecord(all_out, cout);
    cudaStreamWaitEvent(st, all_out, 0);
    const cudaError_t e2 = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = e2;
  }
  for (cudaEvent_t ev : evs) cudaEventDestroy(ev);
  if (cin) cudaStreamDestroy(cin);
  if (cout) cudaStreamDestroy(cout);
  if (!err.empty()) return fail(JTFS_ERR_CUDA, err);
  if (e != cudaSuccess) return cuda_fail(e, "forward_host");
  e = cudaGetLastError();
  return e != cudaSuccess ? cuda_fail(e, "kernel launch") : JTFS_OK;
}

// ---- backward / VJP (jtfs.h: jtfs_backward_workspace_size / jtfs_backward) ----
namespace {
struct BwdLayoutBytes {
  size_t xhat, tmp, u1, u1hat, yphi, y2, out, dP, dyphi, gy2, G, gu1hat, gu1, wb, gw, gxhat, gxpad, total;
};
BwdLayoutBytes bwd_layout(const jtfs::Plan& P, int64_t nb) {
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const jtfs::WsLayout f = jtfs::ws_layout(P, nb);
  BwdLayoutBytes w{};
  w.xhat = f.xhat;
  w.tmp = f.tmp;
  w.u1 = f.u1;
  w.u1hat = f.u1hat;
  w.yphi = f.yphi;
  w.y2 = f.y2;
  const int64_t fps = (int64_t)P.n_frames * (1 + P.n1) + (int64_t)P.paths.size() * P.lam_out * P.n_frames;
  w.out = al((size_t)nb * fps * 4);
  w.dP = al((size_t)nb * P.kd.size() * P.Mpad * P.n_frames * 4);
  w.dyphi = al((size_t)nb * P.n1 * P.NPT * 4);
  w.gy2 = al((size_t)nb * P.y2_total * 8);
  w.G = al((size_t)nb * P.y2_total * 8);
  w.gu1hat = al((size_t)nb * P.u1_total * 8);
  w.gu1 = al((size_t)nb * P.u1_total * 4);
  w.wb = al((size_t)nb * P.u1_total * 8);
  w.gw = al((size_t)nb * P.u1_total * 8);
  w.gxhat = al((size_t)nb * P.N_pad * 8);
  w.gxpad = al((size_t)nb * P.N_pad * 4);
  w.total = w.xhat + w.tmp + w.u1 + w.u1hat + w.yphi + w.y2 + w.out + w.dP + w.dyphi + w.gy2 + w.G + w.gu1hat +
            w.gu1 + w.wb + w.gw + w.gxhat + w.gxpad;
  return w;
}
int64_t bwd_mb(const jtfs::Plan& P, int64_t B) {
  const size_t per = bwd_layout(P, 1).total;
  const int64_t cap = std::max<int64_t>(1, (int64_t)(((size_t)8 << 30) / std::max<size_t>(per, 1)));
  return std::max<int64_t>(1, std::min<int64_t>(B, cap));
}
jtfs::BwdWs bwd_carve(const jtfs::Plan& P, void* ws, int64_t nb) {
  const BwdLayoutBytes L = bwd_layout(P, nb);
  char* c = (char*)ws;
  jtfs::BwdWs w{};
  w.xhat = (float2*)c; c += L.xhat;
  w.tmp = (float2*)c; c += L.tmp;
  w.u1 = (float*)c; c += L.u1;
  w.u1hat = (float2*)c; c += L.u1hat;
  w.yphi = (float*)c; c += L.yphi;
  w.y2 = (float*)c; c += L.y2;
  w.scratch_out = (float*)c; c += L.out;
  w.dP = (float*)c; c += L.dP;
  w.dyphi = (float*)c; c += L.dyphi;
  w.gy2 = (float*)c; c += L.gy2;
  w.G = (float2*)c; c += L.G;
  w.gu1hat = (float2*)c; c += L.gu1hat;
  w.gu1 = (float*)c; c += L.gu1;
  w.wb = (float2*)c; c += L.wb;
  w.gw = (float2*)c; c += L.gw;
  w.gxhat = (float2*)c; c += L.gxhat;
  w.gxpad = (float*)c; c += L.gxpad;
  return w;
}
}  // namespace

jtfs_status jtfs_backward_workspace_size(jtfs_plan_t plan, int64_t B, size_t* bytes) {
  if (!plan || !bytes || B < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  *bytes = B == 0 ? 0 : bwd_layout(plan->P, bwd_mb(plan->P, B)).total;
  return JTFS_OK;
}

jtfs_status jtfs_backward_regions(jtfs_plan_t plan, int64_t B, int64_t* offsets, int32_t cap) {
  if (!plan || !offsets || B < 1 || cap < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  const BwdLayoutBytes L = bwd_layout(plan->P, bwd_mb(plan->P, B));
  const size_t sz[17] = {L.xhat, L.tmp, L.u1, L.u1hat, L.yphi, L.y2, L.out, L.dP, L.dyphi,
                         L.gy2, L.G, L.gu1hat, L.gu1, L.wb, L.gw, L.gxhat, L.gxpad};
  int64_t o = 0;
  for (int i = 0; i < 18 && i < cap; ++i) {
    offsets[i] = o;
    if (i < 17) o += (int64_t)sz[i];
  }
  return JTFS_OK;
}

jtfs_status jtfs_backward(jtfs_plan_t plan, const float* x, int64_t B, const float* dout, float* dx, void* ws,
                          size_t ws_bytes, void* stream) {
  if (!plan) return fail(JTFS_ERR_INVALID_ARG, "plan is NULL");
  jtfs::Plan& P = plan->P;
  if (P.device < 0) return fail(JTFS_ERR_UNSUPPORTED, "host-only plan (device = -1) cannot run backward");
  if (B < 0) return fail(JTFS_ERR_INVALID_ARG, "B < 0");
  if (B == 0) return JTFS_OK;
  if (!x || !dout || !dx || !ws) return fail(JTFS_ERR_INVALID_ARG, "NULL buffer");
  if (!aligned(x, 16) || !aligned(dout, 16) || !aligned(dx, 16) || !aligned(ws, 256))
    return fail(JTFS_ERR_INVALID_ARG, "misaligned buffer");
  const int64_t mb = bwd_mb(P, B);
  if (ws_bytes < bwd_layout(P, mb).total) return fail(JTFS_ERR_WORKSPACE, "backward workspace too small");
  DeviceGuard guard(P.device);
  cudaStream_t st = (cudaStream_t)stream;
  const jtfs::BwdWs w = bwd_carve(P, ws, mb);
  jtfs_layout_t lay;
  layout_of(P, &lay);
  for (int64_t b0 = 0; b0 < B; b0 += mb) {
    const int nb = (int)std::min<int64_t>(mb, B - b0);
    jtfs::launch_backward(P, x + b0 * P.N, nb, dout + b0 * lay.floats_per_signal, dx + b0 * P.N, w, st);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return JTFS_OK;
}

// ---- second-order time scattering (jtfs.h: jtfs_scat1d_layout / _paths / jtfs_scattering1d) ----
namespace {
void scat1d_layout_of(const jtfs::Plan& P, jtfs_scat1d_layout_t* o) {
  int n2 = 0;
  for (const auto& d : P.kd) n2 += d.K;
  o->n1 = P.n1;
  o->n2 = n2;
  o->n_frames = P.n_frames;
  o->frame0 = P.frame0;
  o->off_s0 = 0;
  o->off_s1 = P.n_frames;
  o->off_s2 = o->off_s1 + (int64_t)P.n1 * P.n_frames;
  o->floats_per_signal = o->off_s2 + (int64_t)n2 * P.n_frames;
}
}  // namespace

jtfs_status jtfs_scat1d_layout(jtfs_plan_t plan, jtfs_scat1d_layout_t* layout) {
  if (!plan || !layout) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  scat1d_layout_of(plan->P, layout);
  return JTFS_OK;
}

jtfs_status jtfs_scat1d_paths(jtfs_plan_t plan, int32_t* pairs, int32_t cap) {
  if (!plan || (cap > 0 && !pairs) || cap < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  int32_t r = 0;
  for (const auto& d : plan->P.kd)
    for (int l = 0; l < d.K; ++l, ++r)
      if (r < cap) {
        pairs[2 * r] = l;
        pairs[2 * r + 1] = d.alpha;
      }
  return JTFS_OK;
}

jtfs_status jtfs_scattering1d(jtfs_plan_t plan, const float* x, int64_t B, float* out, void* ws, size_t ws_bytes,
                              void* stream) {
  jtfs_status s = check_forward_args(plan, x, B, out, ws, ws_bytes);
  if (s != JTFS_OK || B == 0) return s;
  jtfs::Plan& P = plan->P;
  DeviceGuard guard(P.device);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t mb = std::min<int64_t>(B, P.mb);
  WsPtrs w = carve(P, ws, mb);
  jtfs_scat1d_layout_t lay;
  scat1d_layout_of(P, &lay);
  for (int64_t b0 = 0; b0 < B; b0 += mb) {
    const int nb = (int)std::min<int64_t>(mb, B - b0);
    const float* xb = x + b0 * P.N;
    float* ob = out + b0 * lay.floats_per_signal;
    { StageScope sc(P, 0, st); sc.done(jtfs::launch_pad_fft(P, xb, nb, w.xhat, w.tmp, st)); }
    { StageScope sc(P, 1, st); sc.done(jtfs::launch_first_order(P, w.xhat, nb, w.u1, w.u1hat, w.tmp, false, st, w.tmp2)); }
    {
      StageScope sc(P, 2, st);
      sc.done(jtfs::launch_phi_first(P, w.xhat, w.u1hat, nb, w.yphi, ob, lay.floats_per_signal, lay.off_s0,
                                     lay.off_s1, P.d_u1_off, P.d_k1, P.d_band_L1, st));
    }
    { StageScope sc(P, 3, st); sc.done(jtfs::launch_second_order(P, w.u1hat, nb, w.y2, w.tmp, st, true)); }
    {
      StageScope sc(P, 4, st);
      const jtfs::WsLayout L = jtfs::ws_layout(P, mb);
      sc.done(jtfs::launch_time_scat(P, w.y2, nb, ob, lay.floats_per_signal, lay.off_s2, st, w.part,
                                     (L.part - jtfs::kWsGuard) / 4));
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return JTFS_OK;
}

// ---- path sharding (jtfs.h: jtfs_units / jtfs_forward_units / jtfs_reduce_pack) ----
namespace {
// unit table of one signal: alpha-major, chunk-minor
void unit_table(const jtfs::Plan& P, std::vector<jtfs_unit_t>& u) {
  u.clear();
  for (size_t a = 0; a < P.kd.size(); ++a) {
    const auto& d = P.kd[a];
    // modelled cost per time column: tensor work (2 products x 2 columns x K16 per pair
    // row) + epilogue (2 moduli + pooling per pair row)
    const double k16 = (double)((3 * d.K + 15) / 16 * 16);
    const double per_col = (double)P.Mpp * (4.0 * k16 / 8.0 + 48.0);
    for (int c = 0; c < d.nchunks; ++c) {
      jtfs_unit_t x{};
      x.alpha = (int32_t)a;
      x.chunk = c;
      x.col0 = c * d.chunk;
      x.ncols = d.chunk;
      x.cost = per_col * d.chunk;
      u.push_back(x);
    }
  }
}
}  // namespace

jtfs_status jtfs_units(jtfs_plan_t plan, jtfs_unit_t* units, int32_t cap, int32_t* n_units) {
  if (!plan || !n_units || cap < 0 || (cap > 0 && !units)) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  std::vector<jtfs_unit_t> u;
  unit_table(plan->P, u);
  *n_units = (int32_t)u.size();
  for (int32_t i = 0; i < std::min<int32_t>(cap, (int32_t)u.size()); ++i) units[i] = u[i];
  return JTFS_OK;
}

jtfs_status jtfs_partials_size(jtfs_plan_t plan, int64_t* floats_per_signal) {
  if (!plan || !floats_per_signal) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  *floats_per_signal = plan->P.part_total;
  return JTFS_OK;
}

}  // extern "C"

struct jtfs_unitset_s {
  jtfs_plan_t plan = nullptr;
  int device = -1;
  int32_t* d_sel = nullptr;  // per-alpha ascending chunk ids, concatenated (device)
  std::vector<int> off, cnt;
};

namespace {
jtfs_status build_unitset(jtfs_plan_t plan, const int32_t* unit_ids, int32_t n_units, jtfs_unitset_s& set) {
  jtfs::Plan& P = plan->P;
  if (n_units < 0 || (n_units > 0 && !unit_ids)) return fail(JTFS_ERR_INVALID_ARG, "bad unit list");
  std::vector<jtfs_unit_t> table;
  unit_table(P, table);
  // per-alpha chunk lists, in ascending chunk order (the order does not change results)
  std::vector<std::vector<int32_t>> per(P.kd.size());
  std::vector<char> seen(table.size(), 0);
  for (int32_t i = 0; i < n_units; ++i) {
    const int32_t id = unit_ids[i];
    if (id < 0 || id >= (int32_t)table.size()) return fail(JTFS_ERR_INVALID_ARG, "unit id out of range");
    if (seen[id]) return fail(JTFS_ERR_INVALID_ARG, "duplicate unit id");
    seen[id] = 1;
    per[table[id].alpha].push_back(table[id].chunk);
  }
  std::vector<int32_t> flat;
  set.off.clear();
  set.cnt.clear();
  for (auto& v : per) {
    std::sort(v.begin(), v.end());
    set.off.push_back((int)flat.size());
    set.cnt.push_back((int)v.size());
    flat.insert(flat.end(), v.begin(), v.end());
  }
  set.plan = plan;
  set.device = P.device;
  DeviceGuard guard(P.device);
  cudaError_t e = cudaMalloc(&set.d_sel, std::max<size_t>(flat.size(), 1) * 4);
  if (e == cudaSuccess && !flat.empty())
    e = cudaMemcpy(set.d_sel, flat.data(), flat.size() * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (set.d_sel) cudaFree(set.d_sel);
    set.d_sel = nullptr;
    return cuda_fail(e, "unit set upload");
  }
  return JTFS_OK;
}

jtfs_status run_unitset(jtfs_plan_t plan, const float* x, int64_t B, const jtfs_unitset_s& set, float* partials,
                        float* out, void* ws, size_t ws_bytes, void* stream) {
  jtfs_status s = check_forward_args(plan, x, B, out, ws, ws_bytes);
  if (s != JTFS_OK) return s;
  jtfs::Plan& P = plan->P;
  if (set.plan != plan) return fail(JTFS_ERR_INVALID_ARG, "unit set bound to another plan");
  if (B > P.mb) return fail(JTFS_ERR_INVALID_ARG, "forward_units: B exceeds the plan's micro-batch");
  if (!partials || ((uintptr_t)partials & 15)) return fail(JTFS_ERR_INVALID_ARG, "partials NULL or misaligned");
  if (B == 0) return JTFS_OK;
  DeviceGuard guard(P.device);
  cudaStream_t st = (cudaStream_t)stream;
  WsPtrs w = carve(P, ws, B);
  cudaError_t e = cudaMemsetAsync(partials, 0, (size_t)B * P.part_total * 4, st);
  if (e != cudaSuccess) return cuda_fail(e, "forward_units setup");
  jtfs::UnitSel sel;
  sel.d_sel = set.d_sel;
  sel.off = set.off;
  sel.cnt = set.cnt;
  RunOpts o;
  o.sel = &sel;
  o.part = partials;
  o.skip_ke = true;
  const std::string err = run_microbatch(P, x, (int)B, out, w, false, 99, st, o);
  if (!err.empty()) return fail(JTFS_ERR_CUDA, err);
  e = cudaGetLastError();
  return e != cudaSuccess ? cuda_fail(e, "kernel launch") : JTFS_OK;
}
}  // namespace

extern "C" {

jtfs_status jtfs_unitset_create(jtfs_plan_t plan, const int32_t* unit_ids, int32_t n_units, jtfs_unitset_t* out) {
  if (!plan || !out) return fail(JTFS_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  if (plan->P.device < 0) return fail(JTFS_ERR_UNSUPPORTED, "host-only plan");
  jtfs_unitset_s* set = new (std::nothrow) jtfs_unitset_s();
  if (!set) return fail(JTFS_ERR_OOM, "host allocation failed");
  const jtfs_status s = build_unitset(plan, unit_ids, n_units, *set);
  if (s != JTFS_OK) {
    delete set;
    return s;
  }
  *out = set;
  return JTFS_OK;
}

jtfs_status jtfs_unitset_destroy(jtfs_unitset_t set) {
  if (!set) return JTFS_OK;
  if (set->d_sel) {
    DeviceGuard guard(set->device);
    cudaFree(set->d_sel);
  }
  delete set;
  return JTFS_OK;
}

jtfs_status jtfs_forward_unitset(jtfs_plan_t plan, const float* x, int64_t B, jtfs_unitset_t set, float* partials,
                                 float* out, void* ws, size_t ws_bytes, void* stream) {
  if (!set) return fail(JTFS_ERR_INVALID_ARG, "unit set is NULL");
  return run_unitset(plan, x, B, *set, partials, out, ws, ws_bytes, stream);
}

jtfs_status jtfs_forward_units(jtfs_plan_t plan, const float* x, int64_t B, const int32_t* unit_ids,
                               int32_t n_units, float* partials, float* out, void* ws, size_t ws_bytes,
                               void* stream) {
  jtfs_status s = check_forward_args(plan, x, B, out, ws, ws_bytes);
  if (s != JTFS_OK) return s;
  jtfs_unitset_s set;
  s = build_unitset(plan, unit_ids, n_units, set);
  if (s != JTFS_OK) return s;
  s = run_unitset(plan, x, B, set, partials, out, ws, ws_bytes, stream);
  // the temporary device unit list is released after the enqueued work has used it
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  {
    DeviceGuard guard(set.device);
    cudaFree(set.d_sel);
  }
  if (s == JTFS_OK && e != cudaSuccess) return cuda_fail(e, "forward_units");
  return s;
}

jtfs_status jtfs_unit_partials_range(jtfs_plan_t plan, int32_t unit, int64_t* begin, int64_t* end) {
  if (!plan || !begin || !end) return fail(JTFS_ERR_INVALID_ARG, "NULL argument");
  const jtfs::Plan& P = plan->P;
  std::vector<jtfs_unit_t> table;
  unit_table(P, table);
  if (unit < 0 || unit >= (int32_t)table.size()) return fail(JTFS_ERR_INVALID_ARG, "unit id out of range");
  const auto& d = P.kd[table[unit].alpha];
  const int64_t per = (int64_t)(d.nslices / d.nchunks) * P.Mpad * P.n_frames;  // slices of one chunk
  *begin = d.part_off + (int64_t)table[unit].chunk * per;
  *end = *begin + per;
  return JTFS_OK;
}

jtfs_status jtfs_reduce_pack(jtfs_plan_t plan, const float* partials, int64_t B, float* out, void* ws,
                             size_t ws_bytes, void* stream) {
  if (!plan) return fail(JTFS_ERR_INVALID_ARG, "plan is NULL");
  jtfs::Plan& P = plan->P;
  if (P.device < 0) return fail(JTFS_ERR_UNSUPPORTED, "host-only plan");
  if (B < 0 || B > P.mb) return fail(JTFS_ERR_INVALID_ARG, "reduce_pack: B out of range");
  if (!partials || !out || !ws) return fail(JTFS_ERR_INVALID_ARG, "NULL buffer");
  if (ws_bytes < jtfs::ws_layout(P, B).total) return fail(JTFS_ERR_WORKSPACE, "workspace too small");
  if (B == 0) return JTFS_OK;
  DeviceGuard guard(P.device);
  cudaStream_t st = (cudaStream_t)stream;
  WsPtrs w = carve(P, ws, B);
  jtfs::KEParams kp{};
  fill_ke_params(P, kp, partials, w.yphi, out);
  {
    StageScope sc(P, 5, st);
    sc.done(jtfs::launch_ke(P, kp, (int)B, st));
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return JTFS_OK;
}

// ---- NEXT-3: K-NN regression (jtfs.h: jtfs_knn_workspace_size / jtfs_knn_regress) ----
jtfs_status jtfs_knn_workspace_size(int64_t n, size_t* bytes) {
  if (!bytes || n < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  *bytes = jtfs::knn_workspace_bytes(n);
  return JTFS_OK;
}

jtfs_status jtfs_knn_regress(const float* F, int64_t n, int64_t d, int64_t ldf, const double* theta,
                             int32_t n_params, int32_t K, int32_t* nbr, double* theta_hat, double* ratio, void* ws,
                             size_t ws_bytes, void* stream) {
  if (n < 2 || n > 16384) return fail(JTFS_ERR_INVALID_ARG, "need 2 <= n <= 16384");
  if (d < 1 || ldf < d || d > (int64_t)1 << 30) return fail(JTFS_ERR_INVALID_ARG, "need d >= 1 and ldf >= d");
  if (K < 1 || K >= n) return fail(JTFS_ERR_INVALID_ARG, "need 1 <= K < n");
  if (n_params < 0 || (n_params > 0 && !theta)) return fail(JTFS_ERR_INVALID_ARG, "theta is NULL");
  if (!F || !nbr || !ws) return fail(JTFS_ERR_INVALID_ARG, "NULL buffer");
  if (!aligned(ws, 256)) return fail(JTFS_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  if (ws_bytes < jtfs::knn_workspace_bytes(n)) return fail(JTFS_ERR_WORKSPACE, "workspace too small");
  cudaError_t e = jtfs::launch_knn(F, (int)n, (int)d, ldf, theta, n_params, K, nbr, n_params ? theta_hat : nullptr,
                                   n_params ? ratio : nullptr, ws, (cudaStream_t)stream);
  return e != cudaSuccess ? cuda_fail(e, "K-NN kernels") : JTFS_OK;
}

jtfs_status jtfs_isomap_workspace_size(int64_t n, int32_t K, size_t* bytes) {
  if (!bytes || n < 0 || K < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  *bytes = jtfs::isomap_workspace_bytes(n, K);
  return JTFS_OK;
}

jtfs_status jtfs_isomap(const float* F, int64_t n, int64_t d, int64_t ldf, int32_t K, int32_t n_components,
                        double* emb, double* eigvals, void* ws, size_t ws_bytes, void* stream) {
  if (n < 2 || n > 16384) return fail(JTFS_ERR_INVALID_ARG, "need 2 <= n <= 16384");
  if (d < 1 || ldf < d || d > (int64_t)1 << 30) return fail(JTFS_ERR_INVALID_ARG, "need d >= 1 and ldf >= d");
  if (K < 1 || K >= n) return fail(JTFS_ERR_INVALID_ARG, "need 1 <= K < n");
  if (n_components < 1 || n_components > 8 || n_components > n)
    return fail(JTFS_ERR_INVALID_ARG, "need 1 <= n_components <= min(8, n)");
  if (!F || !emb || !eigvals || !ws) return fail(JTFS_ERR_INVALID_ARG, "NULL buffer");
  if (!aligned(ws, 256)) return fail(JTFS_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  if (ws_bytes < jtfs::isomap_workspace_bytes(n, K)) return fail(JTFS_ERR_WORKSPACE, "workspace too small");
  int disc = 0;
  cudaError_t e = jtfs::launch_isomap(F, (int)n, (int)d, ldf, K, n_components, emb, eigvals, ws,
                                      (cudaStream_t)stream, &disc);
  if (e != cudaSuccess) return cuda_fail(e, "Isomap kernels");
  if (disc) return fail(JTFS_ERR_INVALID_ARG, "the K-NN graph is disconnected (infinite geodesic distances)");
  return JTFS_OK;
}

jtfs_status jtfs_debug_tap_size(jtfs_plan_t plan, int32_t tap, int64_t B, int64_t* floats) {
  if (!plan || !floats || B < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  const jtfs::Plan& P = plan->P;
  switch (tap) {
    case 0: *floats = B * (int64_t)P.N_pad * 2; break;
    case 1: *floats = B * P.u1_total; break;
    case 2: *floats = B * P.y2_total * 2; break;
    case 3: *floats = B * (int64_t)P.n1 * P.NPT; break;
    default: return fail(JTFS_ERR_INVALID_ARG, "unknown tap");
  }
  return JTFS_OK;
}

jtfs_status jtfs_debug_tap(jtfs_plan_t plan, int32_t tap, const float* x, int64_t B, float* out,
                           int64_t out_floats, void* ws, size_t ws_bytes, void* stream) {
  int64_t need = 0;
  jtfs_status s = jtfs_debug_tap_size(plan, tap, B, &need);
  if (s != JTFS_OK) return s;
  if (!out || out_floats < need) return fail(JTFS_ERR_INVALID_ARG, "tap output too small");
  if (B > plan->P.mb) return fail(JTFS_ERR_INVALID_ARG, "debug taps take at most one micro-batch");
  jtfs_layout_t lay;
  layout_of(plan->P, &lay);
  s = check_forward_args(plan, x, B, out, ws, ws_bytes);
  if (s != JTFS_OK || B == 0) return s;
  jtfs::Plan& P = plan->P;
  DeviceGuard guard(P.device);
  cudaStream_t st = (cudaStream_t)stream;
  WsPtrs w = carve(P, ws, B);
  float* scratch = nullptr;
  cudaError_t e = cudaMalloc(&scratch, (size_t)B * lay.floats_per_signal * 4);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc scratch");
  const int stage = tap == 0 ? 0 : (tap == 1 || tap == 3) ? 1 : 2;
  const std::string rerr = run_microbatch(P, x, (int)B, scratch, w, true, stage, st);
  if (!rerr.empty()) {
    cudaFree(scratch);
    return fail(JTFS_ERR_CUDA, rerr);
  }
  const void* src = tap == 0 ? (const void*)w.xhat : tap == 1 ? (const void*)w.u1 : tap == 2 ? (const void*)w.y2
                                                                                               : (const void*)w.yphi;
  e = cudaMemcpyAsync(out, src, (size_t)need * 4, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(scratch);
  if (e != cudaSuccess) return cuda_fail(e, "debug tap");
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "debug tap launch");
  return JTFS_OK;
}

jtfs_status jtfs_debug_joint(jtfs_plan_t plan, const float* y2, const float* yphi, int64_t B, float* out, void* ws,
                             size_t ws_bytes, void* stream) {
  jtfs_status s = check_forward_args(plan, y2, B, out, ws, ws_bytes);
  if (s != JTFS_OK || B == 0) return s;
  jtfs::Plan& P = plan->P;
  if (B > P.mb) return fail(JTFS_ERR_INVALID_ARG, "debug_joint takes at most one micro-batch");
  if (!yphi || !aligned(yphi, 16)) return fail(JTFS_ERR_INVALID_ARG, "yphi NULL or misaligned");
  DeviceGuard guard(P.device);
  cudaStream_t st = (cudaStream_t)stream;
  WsPtrs w = carve(P, ws, B);
  jtfs_layout_t lay;
  layout_of(P, &lay);
  cudaError_t e = cudaMemcpyAsync(w.y2, y2, (size_t)B * P.y2_total * 8, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(w.yphi, yphi, (size_t)B * P.n1 * P.NPT * 4, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(out, 0, (size_t)B * lay.floats_per_signal * 4, st);
  if (e != cudaSuccess) return cuda_fail(e, "debug_joint copies");
  RunOpts o;
  o.joint_only = true;
  const std::string err = run_microbatch(P, nullptr, (int)B, out, w, false, 99, st, o);
  if (!err.empty()) return fail(JTFS_ERR_CUDA, err);
  e = cudaGetLastError();
  return e != cudaSuccess ? cuda_fail(e, "kernel launch") : JTFS_OK;
}

jtfs_status jtfs_debug_kd_tiling(jtfs_plan_t plan, int32_t* out, int32_t cap) {
  if (!plan || !out || cap < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  const auto& P = plan->P;
  if ((size_t)cap < 10 * P.kd.size()) return fail(JTFS_ERR_INVALID_ARG, "cap < 10 x n_alpha");
  int32_t* o = out;
  for (const auto& d : P.kd) {
    const int32_t v[10] = {P.kd_impl, d.tc_pair, d.tc_stat, d.tc_Nt, d.tc_mpart, d.tc_mblk,
                           d.tc_NBB, d.tc_S, d.tc_nkc, d.pool_mode};
    for (int i = 0; i < 10; ++i) *o++ = v[i];
  }
  return JTFS_OK;
}

jtfs_status jtfs_debug_a16_density(jtfs_plan_t plan, double thr, int64_t* out, int32_t cap) {
  if (!plan || !out || cap < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  std::vector<int64_t> v;
  jtfs::a16_density(plan->P, thr, v);
  if ((size_t)cap < v.size()) return fail(JTFS_ERR_INVALID_ARG, "cap < 6 x n_alpha");
  std::copy(v.begin(), v.end(), out);
  return JTFS_OK;
}

jtfs_status jtfs_debug_fft(jtfs_plan_t plan, int32_t log2L, int32_t dir, int32_t fp64, const void* in, void* out,
                           int64_t rows, void* tmp, size_t tmp_bytes, void* stream) {
  if (!plan) return fail(JTFS_ERR_INVALID_ARG, "plan is NULL");
  jtfs::Plan& P = plan->P;
  if (P.device < 0) return fail(JTFS_ERR_UNSUPPORTED, "host-only plan");
  if (log2L < 1 || (1LL << log2L) > P.N_tw) return fail(JTFS_ERR_INVALID_ARG, "need 2 <= 2^log2L <= N_pad");
  if (dir != -1 && dir != 1) return fail(JTFS_ERR_INVALID_ARG, "dir must be -1 or +1");
  if (fp64 && dir != -1) return fail(JTFS_ERR_UNSUPPORTED, "the fp64 engine is forward only (KA)");
  if (rows < 0 || rows > (1 << 30)) return fail(JTFS_ERR_INVALID_ARG, "bad row count");
  if (rows == 0) return JTFS_OK;
  if (!in || !out || !aligned(in, 16) || !aligned(out, 16)) return fail(JTFS_ERR_INVALID_ARG, "NULL or misaligned");
  const size_t need = (size_t)rows * ((size_t)1 << log2L) * (fp64 ? 16 : 8);
  if (!tmp || tmp_bytes < need) return fail(JTFS_ERR_WORKSPACE, "tmp must hold rows x L complex");
  DeviceGuard guard(P.device);
  jtfs::launch_debug_fft(P, log2L, dir, fp64 != 0, in, out, (int)rows, tmp, (cudaStream_t)stream);
  cudaError_t e = cudaGetLastError();
  return e != cudaSuccess ? cuda_fail(e, "kernel launch") : JTFS_OK;
}

jtfs_status jtfs_measure_fp32_peak(int32_t device, double* tflops_ffma, double* tflops_ffma2) {
  if (!tflops_ffma || !tflops_ffma2 || device < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  DeviceGuard guard(device);
  cudaError_t e = jtfs::measure_fp32_peak(tflops_ffma, tflops_ffma2);
  return e != cudaSuccess ? cuda_fail(e, "fp32 peak probe") : JTFS_OK;
}

jtfs_status jtfs_cost(jtfs_plan_t plan, double* flops, double* bytes, int32_t cap) {
  if (!plan || cap < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  double f[7], b[7];
  jtfs::stage_cost(plan->P, f, b);
  // executed tensor work of the tcgen05 KD (fp16 split: 3 products, re and im
  // accumulators, K' padded to 16) and the bytes it stages through shared memory
  const jtfs::Plan& P = plan->P;
  f[6] = 0;
  b[6] = 0;
  for (const auto& d : P.kd) {
    // per (M-block of 128 pair rows, Nt-column tile): 2 MMAs (Re / Im A'') per 16-wide chunk
    // of the packed K' = 3K, each 128 x 2 Nt x 16 MACs
    const double K16 = d.tc_K16, L = d.L, M = P.Mpp;
    f[6] += 8.0 * M * K16 * L;
    const double tiles = L / std::max(d.tc_Nt, 1);
    // A stationary: A loaded once per CTA (negligible per signal); else streamed per tile
    b[6] += tiles * d.tc_mpart * ((d.tc_stat ? 0.0 : d.tc_mblk * (double)d.tc_nkc * 8192.0) + 4.0 * d.tc_K16 * d.tc_Nt);
  }
  for (int i = 0; i < std::min(cap, 7); ++i) {
    if (flops) flops[i] = f[i];
    if (bytes) bytes[i] = b[i];
  }
  return JTFS_OK;
}

jtfs_status jtfs_profile_enable(jtfs_plan_t plan, int32_t enable) {
  if (!plan) return fail(JTFS_ERR_INVALID_ARG, "plan is NULL");
  plan->P.prof = enable != 0;
  return JTFS_OK;
}

jtfs_status jtfs_profile_read(jtfs_plan_t plan, double* stage_ms, int64_t* stage_launches, int32_t cap,
                              int32_t reset) {
  if (!plan || cap < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  jtfs::Plan& P = plan->P;
  for (int s = 0; s < JTFS_N_STAGES; ++s) {
    double ms = 0;
    for (auto& pr : P.prof_events[s]) {
      float t = 0;
      cudaError_t e = cudaEventSynchronize((cudaEvent_t)pr.second);
      if (e == cudaSuccess) e = cudaEventElapsedTime(&t, (cudaEvent_t)pr.first, (cudaEvent_t)pr.second);
      if (e != cudaSuccess) return cuda_fail(e, "profile events");
      ms += t;
    }
    if (s < cap) {
      if (stage_ms) stage_ms[s] = ms;
      if (stage_launches) stage_launches[s] = P.launches[s];
    }
    if (reset) {
      for (auto& pr : P.prof_events[s]) {
        cudaEventDestroy((cudaEvent_t)pr.first);
        cudaEventDestroy((cudaEvent_t)pr.second);
      }
      P.prof_events[s].clear();
      P.launches[s] = 0;
    }
  }
  return JTFS_OK;
}

jtfs_status jtfs_profile_read_kd(jtfs_plan_t plan, double* ms, int32_t cap, int32_t reset) {
  if (!plan || cap < 0) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  jtfs::Plan& P = plan->P;
  for (size_t a = 0; a < P.kd.size(); ++a) {
    double t = 0;
    if (a < P.prof_kd.size())
      for (auto& pr : P.prof_kd[a]) {
        float x = 0;
        cudaError_t e = cudaEventSynchronize((cudaEvent_t)pr.second);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&x, (cudaEvent_t)pr.first, (cudaEvent_t)pr.second);
        if (e != cudaSuccess) return cuda_fail(e, "profile events");
        t += x;
      }
    if ((int)a < cap && ms) ms[a] = t;
  }
  if (reset) {
    for (auto& v : P.prof_kd)
      for (auto& pr : v) {
        cudaEventDestroy((cudaEvent_t)pr.first);
        cudaEventDestroy((cudaEvent_t)pr.second);
      }
    P.prof_kd.clear();
  }
  return JTFS_OK;
}

jtfs_status jtfs_debug_filter(jtfs_plan_t plan, int32_t bank, int32_t idx, int32_t L, int32_t n_grid,
                              double* out) {
  if (!plan || !out || L < 1 || n_grid < 1) return fail(JTFS_ERR_INVALID_ARG, "bad argument");
  const jtfs::Plan& P = plan->P;
  const jtfs::Bank* b = bank == 1 ? &P.b1 : bank == 2 ? &P.b2 : bank == 3 ? &P.bf : nullptr;
  if (b) {
    if (idx < 0 || idx >= (int)b->xi.size()) return fail(JTFS_ERR_INVALID_ARG, "filter index out of range");
    jtfs::morlet_hat(b->xi[idx], b->sigma[idx], L, n_grid, out);
    return JTFS_OK;
  }
  if (bank == 4) { jtfs::gauss_hat(0.1 / P.T, L, n_grid, out); return JTFS_OK; }
  if (bank == 5) { jtfs::gauss_hat(0.1 / P.F, L, n_grid, out); return JTFS_OK; }
  return fail(JTFS_ERR_INVALID_ARG, "unknown bank");
}

}  // extern "C"
