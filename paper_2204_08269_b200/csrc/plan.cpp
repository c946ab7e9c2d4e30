// Host-side plan generator (fp64 -> fp32 device tables) for the B200 JTFS path.
//
// Written from PAPER.md Sec. 2 and the readings of DESIGN.md §3
// (SURVEY.md §8(c)); it shares no code with oracle/ (checked against it only
// in tests, through jtfs_debug_filter and the forward output).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <complex>
#include <map>
#include <stdexcept>

#include "jtfs_internal.h"

namespace jtfs {

namespace {
// IEEE binary16 round-to-nearest-even of a double (host side, for the A'' tables)
uint16_t half_rn(double v) {
  const uint16_t sign = std::signbit(v) ? 0x8000 : 0;
  double a = std::fabs(v);
  if (a == 0) return sign;
  if (a >= 65520.0) return sign | 0x7C00;  // overflow -> inf (never reached: |v| < 2^14)
  int e = std::ilogb(a);
  if (e < -14) {  // subnormal: units of 2^-24
    const double q = std::nearbyint(a * 16777216.0);  // ties-to-even in the default mode
    return sign | (uint16_t)q;                         // q == 1024 rolls into the first normal
  }
  double m = std::ldexp(a, -e) * 1024.0;  // [1024, 2048)
  double q = std::nearbyint(m);
  if (q == 2048.0) {
    q = 1024.0;
    ++e;
  }
  if (e > 15) return sign | 0x7C00;
  return sign | (uint16_t)((e + 15) << 10) | (uint16_t)((int)q - 1024);
}
double half_to_double(uint16_t h) {
  const int e = (h >> 10) & 31, f = h & 1023;
  const double v = e == 0 ? std::ldexp((double)f, -24) : std::ldexp((double)(f + 1024), e - 25);
  return (h & 0x8000) ? -v : v;
}
}  // namespace


namespace {
constexpr double kSigma0 = 0.1;             // sigma_phi = 0.1 / T        (R4)
constexpr double kAlphaC = 5.0;             // critical-rate support rule (R5)
constexpr double kEpsBand = 1e-9;           // spectral band truncation (relative to peak)
constexpr double kEpsPool = 1e-9;           // lambda-pooling row truncation (relative)
constexpr double kTwoPi = 6.283185307179586476925286766559;

double xi_max(int Q) { return std::max(1.0 / (1.0 + std::pow(2.0, 3.0 / Q)), 0.35); }

double sigma_ratio(int Q) {
  const double q = std::pow(2.0, -1.0 / Q);
  const double r = 1.0 / std::sqrt(2.0);  // neighbours cross at ~ -3 dB (R2)
  return (1.0 - q) / (1.0 + q) / std::sqrt(2.0 * std::log(1.0 / r));
}

int dyadic_j(double xi, double sigma) {
  const int j = (int)std::floor(-std::log2(std::min(xi + kAlphaC * sigma, 0.5))) - 1;
  return std::max(j, 0);
}

// cos/sin of 2 pi a / b with exact integer range reduction
std::complex<double> unit_root(int64_t a, int64_t b) {
  a %= b;
  if (a < 0) a += b;
  const double th = kTwoPi * (double)a / (double)b;
  return {std::cos(th), std::sin(th)};
}

// inverse DFT (with 1/L) of a length-L spectrum, direct O(L * nnz)
std::vector<std::complex<double>> idft(const std::vector<std::complex<double>>& X) {
  const int64_t L = (int64_t)X.size();
  std::vector<std::complex<double>> x(L);
  std::vector<int64_t> nz;
  double mx = 0;
  for (int64_t m = 0; m < L; ++m) mx = std::max(mx, std::abs(X[m]));
  for (int64_t m = 0; m < L; ++m)
    if (std::abs(X[m]) > 1e-300 && std::abs(X[m]) >= 1e-30 * mx) nz.push_back(m);
  for (int64_t n = 0; n < L; ++n) {
    std::complex<double> acc = 0;
    for (int64_t m : nz) acc += X[m] * unit_root(m * n, L);
    x[n] = acc / (double)L;
  }
  return x;
}

Band add_band(std::vector<float>& vals, const std::vector<double>& f) {
  // minimal circular arc holding every bin with |f| >= eps * max|f|
  const int L = (int)f.size();
  double mx = 0;
  for (double v : f) mx = std::max(mx, std::fabs(v));
  std::vector<int> on;
  for (int m = 0; m < L; ++m)
    if (mx > 0 && std::fabs(f[m]) >= kEpsBand * mx) on.push_back(m);
  Band b;
  b.off = (int64_t)vals.size();
  if (on.empty()) { b.m0 = 0; b.len = 0; return b; }
  // largest circular gap between consecutive "on" bins
  int best_gap = -1, best_after = 0;
  for (size_t i = 0; i < on.size(); ++i) {
    const int a = on[i], nxt = on[(i + 1) % on.size()];
    const int gap = (i + 1 < on.size()) ? (nxt - a - 1) : (nxt + L - a - 1);
    if (gap > best_gap) { best_gap = gap; best_after = (int)((i + 1) % on.size()); }
  }
  b.m0 = on[best_after];
  b.len = L - best_gap;
  if (b.len > L) b.len = L;
  for (int t = 0; t < b.len; ++t) vals.push_back((float)f[(b.m0 + t) % L]);
  return b;
}
}  // namespace

int ilog2_exact(int64_t v) {
  if (v < 1 || (v & (v - 1))) return -1;
  int r = 0;
  while ((1LL << r) < v) ++r;
  return r;
}

Bank morlet_bank(int J, int Q) {
  // G(J,Q) (R2): constant-Q ladder xi_i = xi_max 2^{-i/Q}, sigma_i = c xi_i while
  // sigma_i > sigma0 / 2^J, then Q-1 linearly spaced tail filters at sigma_min.
  Bank b;
  const double xm = xi_max(Q), c = sigma_ratio(Q), smin = kSigma0 / std::pow(2.0, J);
  for (int i = 0;; ++i) {
    const double xi = xm * std::pow(2.0, -(double)i / Q);
    const double s = c * xi;
    if (!(s > smin)) break;
    b.xi.push_back(xi);
    b.sigma.push_back(s);
  }
  if (b.xi.empty()) throw std::runtime_error("filter bank has no constant-Q filter");
  const double xl = b.xi.back();
  for (int q = 1; q < Q; ++q) {
    b.xi.push_back((double)(Q - q) / Q * xl);
    b.sigma.push_back(smin);
  }
  for (size_t i = 0; i < b.xi.size(); ++i) b.j.push_back(dyadic_j(b.xi[i], b.sigma[i]));
  return b;
}

void morlet_hat(double xi, double sigma, int L, int n_grid, double* out) {
  // R1 + R8: Gabor on the one-sided grid w+ = m / n_grid minus kappa * Gaussian
  // on the two-sided grid (fftfreq), kappa making psi_hat[0] exactly 0.
  const double two_s2 = 2.0 * sigma * sigma;
  const double kappa = std::exp(-(xi * xi) / two_s2);
  for (int m = 0; m < L; ++m) {
    const double wp = (double)m / n_grid;
    const double wpm = (m < L / 2 ? (double)m : (double)(m - L)) / n_grid;
    const double gab = (m == 0) ? kappa : std::exp(-((wp - xi) * (wp - xi)) / two_s2);
    out[m] = gab - kappa * std::exp(-(wpm * wpm) / two_s2);
  }
}

void gauss_hat(double sigma, int L, int n_grid, double* out) {
  const double two_s2 = 2.0 * sigma * sigma;
  for (int m = 0; m < L; ++m) {
    const double wpm = (m < L / 2 ? (double)m : (double)(m - L)) / n_grid;
    out[m] = std::exp(-(wpm * wpm) / two_s2);
  }
}

static std::vector<double> morlet_vec(double xi, double s, int L, int n) {
  std::vector<double> v(L);
  morlet_hat(xi, s, L, n, v.data());
  return v;
}
static std::vector<double> gauss_vec(double s, int L, int n) {
  std::vector<double> v(L);
  gauss_hat(s, L, n, v.data());
  return v;
}

// phi_T pooling weight of time column t for retained frame m of alpha's grid
static double pool_tap(const Plan& P, const AlphaKD& d, int m, int64_t t) {
  if (m >= P.n_frames) return 0.0;
  int64_t i = ((int64_t)(P.frame0 + m) * d.D - t) % d.L;
  if (i < 0) i += d.L;
  return (double)P.g[d.g_off + i];
}

// Density of the tensor-core operand A''_alpha (measurement, jtfs_debug_a16_density): per
// alpha, the 8 KiB records (128 pair rows x 16 packed K-columns x {Re, Im}) and how many hold
// an entry above thr relative to its row's scale (rows are scaled to a maximum in [2^13,
// 2^14), so |fp16| > thr 2^13 is "above thr of the row's largest coefficient").
void a16_density(const Plan& P, double thr, std::vector<int64_t>& out) {
  out.clear();
  for (const auto& d : P.kd) {
    const int nkc = (3 * d.K + 15) / 16, nblk = P.Mpp / 128;
    int64_t live = 0, band = 0;
    for (int mb = 0; mb < nblk; ++mb) {
      int lo = nkc, hi = -1;
      for (int kc = 0; kc < nkc; ++kc) {
        const uint16_t* r = P.A16.data() + d.tc_a16_off + ((size_t)mb * nkc + kc) * 4096;
        double mx = 0;
        for (int i = 0; i < 4096; ++i) mx = std::max(mx, std::abs(half_to_double(r[i])));
        if (mx > thr * 8192.0) {
          ++live;
          lo = std::min(lo, kc);
          hi = kc;
        }
      }
      if (hi >= lo) band += hi - lo + 1;
    }
    // entry level: coefficients A_alpha[p][lambda] (the hi copy, packed columns 0..K-1) above thr
    int64_t ent = 0;
    for (int m = 0; m < P.Mpp; ++m)
      for (int lam = 0; lam < d.K; ++lam) {
        const int mb = m / 128, r = m % 128, kc = lam / 16, kk = lam % 16;
        const uint32_t o = (uint32_t)((r / 8) * 256 + (r % 8) * 32 + kk * 2);
        const uint32_t sw = o ^ (((o >> 7) & 1u) << 4);
        const uint16_t* rec = P.A16.data() + d.tc_a16_off + ((size_t)mb * nkc + kc) * 4096;
        const double a = std::max(std::abs(half_to_double(rec[sw / 2])), std::abs(half_to_double(rec[2048 + sw / 2])));
        if (a > thr * 8192.0) ++ent;
      }
    out.push_back((int64_t)nblk * nkc);
    out.push_back(live);
    out.push_back(band);
    out.push_back(nkc);
    out.push_back(ent);
    out.push_back((int64_t)P.Mpp_rows * d.K);
  }
}

std::string build_plan(const jtfs_params& p, Plan& P) {
  P.prm = p;
  std::vector<std::vector<float>> mom_tabs;  // per alpha: moment-form pooling table (if eligible)
  // ---- validation ----
  const int log2N = ilog2_exact(p.N);
  if (log2N < 4) return "N must be a power of two >= 16";
  if (ilog2_exact(p.T) < 0 || p.T > p.N) return "T must be a power of two with T <= N";
  if (p.J < 1 || (1LL << p.J) > p.N) return "J must satisfy 1 <= J and 2^J <= N";
  if (p.Q < 1 || p.Q2 < 1 || p.Q_fr < 1) return "Q, Q2, Q_fr must be >= 1";
  if (p.J_fr < 1) return "J_fr must be >= 1";
  if (p.pad_mode != JTFS_PAD_REFLECT && p.pad_mode != JTFS_PAD_PERIODIC) return "bad pad_mode";
  if (p.average_fr != 0 && p.average_fr != 1) return "average_fr must be 0 or 1";
  if (p.Q > 64 || p.J > 24 || p.J_fr > 12) return "J / Q / J_fr out of supported range";
  P.N = p.N;
  P.T = p.T;
  P.log2T = ilog2_exact(p.T);
  P.F = p.F ? p.F : (1 << p.J_fr);
  P.log2F = ilog2_exact(P.F);
  if (P.log2F < 0) return "F must be a power of two";
  if (p.pad_mode == JTFS_PAD_REFLECT) { P.N_pad = 2 * p.N; P.pad_left = p.N / 2; }
  else { P.N_pad = p.N; P.pad_left = 0; }
  if (P.N_pad > (1 << 18)) return "N_pad > 2^18 is not supported";
  P.NPT = P.N_pad / P.T;
  try {
    P.b1 = morlet_bank(p.J, p.Q);
    P.b2 = morlet_bank(p.J, p.Q2);
    P.bf = morlet_bank(p.J_fr, p.Q_fr);
  } catch (const std::exception& e) {
    return e.what();
  }
  P.n1 = (int)P.b1.xi.size();
  if (P.n1 < 4) return "fewer than 4 first-order filters (n1 < 4)";
  {
    int c = 0;
    while ((1 << c) < P.n1) ++c;
    P.N_fr = 1 << (c + 1);                       // 2^(ceil(log2 n1) + 1)   (R9)
  }
  if (P.F > P.N_fr) return "F larger than the frequential grid N_fr";
  P.frame0 = (P.pad_left + P.T - 1) / P.T;       // U(log2 T)
  P.n_frames = (P.N + P.T - 1) / P.T;
  P.lam_out = p.average_fr ? (P.n1 + P.F - 1) / P.F : P.n1;
  if (P.n_frames > 32) return "more than 32 output frames (N/T > 32) is not supported";

  // ---- first order ----
  P.k1.resize(P.n1);
  P.L1.resize(P.n1);
  P.u1_off.resize(P.n1);
  P.u1_total = 0;
  for (int l = 0; l < P.n1; ++l) {
    P.k1[l] = std::min(P.b1.j[l], P.log2T);
    P.L1[l] = P.N_pad >> P.k1[l];
    P.u1_off[l] = P.u1_total;
    P.u1_total += P.L1[l];
    if (l > 0 && P.b1.j[l] < P.b1.j[l - 1]) return "internal: j1 not monotone";
  }
  auto& bv = P.bandvals;
  bv.clear();
  P.band_psi1.resize(P.n1);
  for (int l = 0; l < P.n1; ++l)
    P.band_psi1[l] = add_band(bv, morlet_vec(P.b1.xi[l], P.b1.sigma[l], P.N_pad, P.N_pad));
  const double sigT = kSigma0 / P.T, sigF = kSigma0 / P.F;
  P.band_phiT_pad = add_band(bv, gauss_vec(sigT, P.N_pad, P.N_pad));
  P.band_phiT_L1.resize(P.log2T + 1);
  for (int k = 0; k <= P.log2T; ++k)
    P.band_phiT_L1[k] = add_band(bv, gauss_vec(sigT, P.N_pad >> k, P.N_pad));

  // U1 groups by L1
  P.u1_groups.clear();
  for (int l = 0; l < P.n1; ++l) {
    const int lg = ilog2_exact(P.L1[l]);
    if (P.u1_groups.empty() || P.u1_groups.back().log2L != lg) {
      P.u1_groups.push_back(FoldGroup{});
      P.u1_groups.back().log2L = lg;
    }
    FoldRow r{};
    r.src_off = 0;
    r.Lsrc = P.N_pad;
    r.m0 = P.band_psi1[l].m0;
    r.len = P.band_psi1[l].len;
    r.band_off = P.band_psi1[l].off;
    r.dst_off = P.u1_off[l];
    r.scale = (float)(1.0 / P.N_pad);
    r.pad = l;  // lambda (KB's per-row max |U1|)
    P.u1_groups.back().rows.push_back(r);
  }

  // ---- second order in time: active alphas, admissibility j1 < j2 (R7) ----
  P.kd.clear();
  P.y2_total = 0;
  std::map<std::pair<int, int>, Band> band2;
  for (int a = 0; a < (int)P.b2.xi.size(); ++a) {
    int K = 0;
    while (K < P.n1 && P.b1.j[K] < P.b2.j[a]) ++K;
    for (int l = K; l < P.n1; ++l)
      if (P.b1.j[l] < P.b2.j[a]) return "internal: admissible set not a prefix";
    if (K == 0) continue;
    AlphaKD d{};
    d.alpha = a;
    d.K = K;
    d.k_alpha = std::min(P.b2.j[a], P.log2T);
    d.L = P.N_pad >> d.k_alpha;
    d.D = 1 << (P.log2T - d.k_alpha);
    d.y2_off = P.y2_total;
    P.y2_total += (int64_t)K * d.L;
    for (int l = 0; l < K; ++l) {
      auto key = std::make_pair(a, P.k1[l]);
      if (!band2.count(key))
        band2[key] = add_band(bv, morlet_vec(P.b2.xi[a], P.b2.sigma[a], P.L1[l], P.N_pad));
    }
    P.kd.push_back(d);
  }
  if (P.kd.empty()) return "no admissible second-order path";
  // Y2 groups by L_alpha (descending)
  P.y2_groups.clear();
  for (const auto& d : P.kd) {
    const int lg = ilog2_exact(d.L);
    FoldGroup* G = nullptr;
    for (auto& g : P.y2_groups)
      if (g.log2L == lg) G = &g;
    if (!G) {
      P.y2_groups.push_back(FoldGroup{});
      G = &P.y2_groups.back();
      G->log2L = lg;
    }
    for (int l = 0; l < d.K; ++l) {
      const Band& b = band2[std::make_pair(d.alpha, P.k1[l])];
      FoldRow r{};
      r.src_off = P.u1_off[l];
      r.Lsrc = P.L1[l];
      r.m0 = b.m0;
      r.len = b.len;
      r.band_off = b.off;
      r.dst_off = 2 * d.y2_off + (int64_t)(2 * l) * d.L;  // planar: re row, then im row
      r.scale = (float)(1.0 / P.L1[l]);
      G->rows.push_back(r);
    }
  }

  // ---- fp16 destinations of the Y2 rows (KC writes the KD's packed B rows directly) and
  // the Cauchy-Schwarz bound sqrt(sum_m psi_hat_alpha[m]^2) of each (alpha, lambda) band:
  // |Y2_alpha[lambda](n)| = |sum_t psi(t) U1_lambda(n - t)| <= ||psi||_1 max|U1_lambda|
  // <= sqrt(L) ||psi||_2 max|U1_lambda| = sqrt(sum_m |psi_hat[m]|^2) max|U1_lambda|
  // (Parseval; psi = IDFT_L of the band values KC multiplies) ----
  {
    std::vector<int64_t> y16_off_of(P.kd.size());
    int64_t acc = 0;
    for (size_t a = 0; a < P.kd.size(); ++a) {
      y16_off_of[a] = acc;
      const int K48 = (3 * P.kd[a].K + 15) / 16 * 16;
      acc += (int64_t)K48 * 2 * P.kd[a].L;
    }
    for (auto& G : P.y2_groups) G.y16rows.clear();
    for (size_t a = 0; a < P.kd.size(); ++a) {
      const auto& d = P.kd[a];
      FoldGroup* G = nullptr;
      for (auto& g : P.y2_groups)
        if (g.log2L == ilog2_exact(d.L)) G = &g;
      for (int l = 0; l < d.K; ++l)
        G->y16rows.push_back(Y16Row{y16_off_of[a] + (int64_t)l * 2 * d.L, (int64_t)d.K * 2 * d.L, (int32_t)a, 0});
    }
    P.ybound.assign(P.kd.size() * (size_t)P.n1, 0.f);
    for (size_t a = 0; a < P.kd.size(); ++a)
      for (int l = 0; l < P.kd[a].K; ++l) {
        const Band& bd = band2[std::make_pair(P.kd[a].alpha, P.k1[l])];
        double e = 0;
        for (int t = 0; t < bd.len; ++t) e += (double)bv[bd.off + t] * (double)bv[bd.off + t];
        P.ybound[a * P.n1 + l] = (float)(std::sqrt(e) * (1.0 + 1e-6));
      }
  }

  // ---- frequential filters and the joint-stage row set (R9, R10, R11) ----
  const int nb = (int)P.bf.xi.size();
  P.fr.clear();
  auto make_filter = [&](int kind, int theta, int beta) {
    FrFilter f{};
    f.kind = kind;
    f.theta = theta;
    f.beta = beta;
    if (kind == 0) f.k = p.average_fr ? std::min(P.bf.j[beta], P.log2F) : 0;
    else f.k = p.average_fr ? P.log2F : 0;
    f.R = P.N_fr >> f.k;
    return f;
  };
  for (int th : {-1, +1})
    for (int b = 0; b < nb; ++b) P.fr.push_back(make_filter(0, th, b));
  P.fr.push_back(make_filter(1, 0, -1));
  // retained rows and lambda-pooling matrices
  P.W.clear();
  P.M = 0;
  for (auto& f : P.fr) {
    f.rprime.clear();
    if (p.average_fr) {
      std::vector<std::complex<double>> ph(f.R);
      {
        auto gv = gauss_vec(sigF, f.R, P.N_fr);
        for (int m = 0; m < f.R; ++m) ph[m] = gv[m];
      }
      auto gF = idft(ph);
      double mx = 0;
      for (auto& v : gF) mx = std::max(mx, std::abs(v.real()));
      const int step = 1 << (P.log2F - f.k);
      for (int r = 0; r < f.R; ++r) {
        bool need = false;
        for (int q = 0; q < P.lam_out && !need; ++q) {
          const int d = ((q * step - r) % f.R + f.R) % f.R;
          need = std::fabs(gF[d].real()) >= kEpsPool * mx;
        }
        if (need) f.rprime.push_back(r);
      }
      f.nrows = (int)f.rprime.size();
      f.w_off = (int64_t)P.W.size();
      for (int q = 0; q < P.lam_out; ++q)
        for (int i = 0; i < f.nrows; ++i) {
          const int d = ((q * step - f.rprime[i]) % f.R + f.R) % f.R;
          P.W.push_back((float)gF[d].real());
        }
    } else {
      for (int r = 0; r < P.n1; ++r) f.rprime.push_back(r);
      f.nrows = P.n1;
      f.w_off = (int64_t)P.W.size();
      for (int q = 0; q < P.lam_out; ++q)
        for (int i = 0; i < f.nrows; ++i) P.W.push_back(q == f.rprime[i] ? 1.f : 0.f);
    }
    // per output row q: the band [first, last] of rows with |W| >= kEpsPool of the
    // filter's largest weight (the same cut that selects the retained rows)
    {
      double wmax = 0;
      for (int64_t i = f.w_off; i < (int64_t)P.W.size(); ++i) wmax = std::max(wmax, (double)std::fabs(P.W[i]));
      f.wr_off = (int64_t)P.Wrange.size() / 2;
      for (int q = 0; q < P.lam_out; ++q) {
        int lo = f.nrows, hi = -1;
        for (int i = 0; i < f.nrows; ++i)
          if (std::fabs((double)P.W[f.w_off + (int64_t)q * f.nrows + i]) >= kEpsPool * wmax) {
            lo = std::min(lo, i);
            hi = std::max(hi, i);
          }
        P.Wrange.push_back(lo);
        P.Wrange.push_back(hi + 1);
      }
    }
    P.M += f.nrows;
  }
  {
    // Spin pairs (kernels_tc.cu, KD): the theta = -1 and theta = +1 wavelets of one beta
    // share their decimation k, hence their retained rows, and h_{beta,+1} = conj h_{beta,-1}
    // (psi_hat real, R10).  Pair row p holds one retained row r' of beta (and, after the
    // wavelets, the phi_F rows, whose taps are real); KD computes both spins of a pair from
    // the same four real products.  Pair rows are laid out beta-major: [beta 0 rows, ...,
    // beta nb-1 rows, phi_F rows], padded to whole 128-row M-blocks; the "full" rows of the
    // partials / KE / SIMT layout are spin-major: theta = -1 (and phi_F) rows at p,
    // theta = +1 rows at Mpp + p.
    int prow = 0;
    std::vector<int> prow0(nb + 1, 0);
    for (int b = 0; b < nb; ++b) {
      const FrFilter& fm = P.fr[b];
      const FrFilter& fp = P.fr[nb + b];
      if (fm.k != fp.k || fm.rprime != fp.rprime) return "internal: spin-pair rows differ";
      prow0[b] = prow;
      prow += fm.nrows;
    }
    prow0[nb] = prow;
    prow += P.fr[2 * nb].nrows;
    P.Mpp_rows = prow;
    // M-blocks of 128 pair rows (one TMEM lane each), split into M-parts so that one part's
    // pooled accumulators (2 spins x NF frames per block) stay in the epilogue's registers:
    // <= MAXSLOT M-blocks per part (kernels_tc.cu: NF 8: 5, 16: 2, 32: 1)
    const int n_frames_pad = P.n_frames <= 8 ? 8 : P.n_frames <= 16 ? 16 : 32;
    const int max_mblk = n_frames_pad == 8 ? 5 : n_frames_pad == 16 ? 2 : 1;
    const int mblocks = (prow + 127) / 128;
    P.tc_n_mpart = (mblocks + max_mblk - 1) / max_mblk;
    P.tc_n_mblk = (mblocks + P.tc_n_mpart - 1) / P.tc_n_mpart;
    P.Mpp = P.tc_n_mblk * P.tc_n_mpart * 128;
    P.Mpad = 2 * P.Mpp;
    for (int b = 0; b < nb; ++b) {
      P.fr[b].row0 = prow0[b];
      P.fr[nb + b].row0 = P.Mpp + prow0[b];
    }
    P.fr[2 * nb].row0 = prow0[nb];
    P.kd_impl = (p.flags & JTFS_KD_SIMT) ? 0 : 1;  // SIMT KD only on explicit request (validation)
  }
  // frequential taps h_f = IDFT_{N_fr}(f_hat) (fp64)
  std::vector<std::vector<std::complex<double>>> htap(P.fr.size());
  for (size_t i = 0; i < P.fr.size(); ++i) {
    const auto& f = P.fr[i];
    std::vector<std::complex<double>> fh(P.N_fr);
    if (f.kind == 0) {
      auto v = morlet_vec(P.bf.xi[f.beta], P.bf.sigma[f.beta], P.N_fr, P.N_fr);
      for (int m = 0; m < P.N_fr; ++m)  // theta=-1: psi_hat[m]; theta=+1: psi_hat[-m] (R10)
        fh[m] = (f.theta == -1) ? v[m] : v[(P.N_fr - m) % P.N_fr];
    } else {
      auto v = gauss_vec(sigF, P.N_fr, P.N_fr);
      for (int m = 0; m < P.N_fr; ++m) fh[m] = v[m];
    }
    htap[i] = idft(fh);
  }
  // A_alpha^T [Kpad][Mpad] complex: A[row][lam] = h_f[(r' 2^k - lam) mod N_fr]
  P.A.clear();
  for (auto& d : P.kd) {
    d.Kpad = (d.K + 7) / 8 * 8;
    d.a_off = (int64_t)P.A.size() / 2;
    const size_t base = P.A.size();
    P.A.resize(base + (size_t)d.Kpad * P.Mpad * 2, 0.f);
    for (size_t fi = 0; fi < P.fr.size(); ++fi) {
      const auto& f = P.fr[fi];
      for (int i = 0; i < f.nrows; ++i) {
        const int row = f.row0 + i;
        for (int l = 0; l < d.K; ++l) {
          const int idx = (((f.rprime[i] << f.k) - l) % P.N_fr + P.N_fr) % P.N_fr;
          const auto v = htap[fi][idx];
          P.A[base + ((size_t)l * P.Mpad + row) * 2 + 0] = (float)v.real();
          P.A[base + ((size_t)l * P.Mpad + row) * 2 + 1] = (float)v.imag();
        }
      }
    }
  }
  // A''_alpha for the tensor cores (kernels_tc.cu): per pair row p (filter theta = -1 of
  // its beta, or phi_F) the real and imaginary parts of A_alpha[p][lambda], scaled by a
  // power of two s_p (max(|Re|, |Im|) s_p in [2^13, 2^14)) and split into fp16
  // hi = rn(a s_p), lo = rn(a s_p - hi), packed along K as [hi | hi | lo] (3K columns,
  // padded to 16) against KY's B rows [Y_hi; Y_lo; Y_hi]: one MMA chain then sums
  // A_hi Y_hi + A_hi Y_lo + A_lo Y_hi.  Stored pre-tiled for cp.async.bulk: per (128-row
  // M-block, 16-wide K chunk) one 8 KiB record [Re | Im], each a 4 KiB UMMA K-major
  // SWIZZLE_32B image (8-row x 32 B atoms, 16 B chunk index ^= row bit 2).  Ainv = 1 / s_p.
  P.A16.clear();
  P.Ainv.clear();
  for (auto& d : P.kd) {
    const int K3 = 3 * d.K;
    const int nkc = (K3 + 15) / 16;
    const int nblk = P.Mpp / 128;
    d.tc_a16_off = (int64_t)P.A16.size();
    d.tc_ainv_off = (int64_t)P.Ainv.size();
    const size_t base = P.A16.size();
    P.A16.resize(base + (size_t)nblk * nkc * 4096, 0);
    P.Ainv.resize(P.Ainv.size() + P.Mpp, 1.f);
    std::vector<int> row_f(P.Mpp, -1), row_i(P.Mpp, 0);
    for (int fi = 0; fi < nb; ++fi)
      for (int i = 0; i < P.fr[fi].nrows; ++i) {
        row_f[P.fr[fi].row0 + i] = fi;
        row_i[P.fr[fi].row0 + i] = i;
      }
    for (int i = 0; i < P.fr[2 * nb].nrows; ++i) {
      row_f[P.fr[2 * nb].row0 + i] = 2 * nb;
      row_i[P.fr[2 * nb].row0 + i] = i;
    }
    auto put = [&](int m, int img, int col, uint16_t h) {
      const int mb = m / 128, r = m % 128, kc = col / 16, kk = col % 16;
      const uint32_t o = (uint32_t)((r / 8) * 256 + (r % 8) * 32 + kk * 2);
      const uint32_t sw = o ^ (((o >> 7) & 1u) << 4);
      P.A16[base + ((size_t)mb * nkc + kc) * 4096 + (size_t)img * 2048 + sw / 2] = h;
    };
    std::vector<std::complex<double>> arow(d.K);
    for (int m = 0; m < P.Mpp; ++m) {
      if (row_f[m] < 0) continue;
      const int fi = row_f[m];
      const auto& f = P.fr[fi];
      const int rp = f.rprime[row_i[m]];
      const bool real_taps = f.kind == 1;  // phi_F: real, even spectrum -> real taps
      double amax = 0;
      for (int lam = 0; lam < d.K; ++lam) {
        const int idx = (((rp << f.k) - lam) % P.N_fr + P.N_fr) % P.N_fr;
        arow[lam] = real_taps ? std::complex<double>(htap[fi][idx].real(), 0.0) : htap[fi][idx];
        amax = std::max(amax, std::max(std::abs(arow[lam].real()), std::abs(arow[lam].imag())));
      }
      if (amax == 0) continue;
      const int E = std::ilogb(amax);            // amax in [2^E, 2^(E+1))
      const double sc = std::ldexp(1.0, 13 - E);  // amax * sc in [2^13, 2^14)
      P.Ainv[d.tc_ainv_off + m] = (float)std::ldexp(1.0, E - 13);
      for (int lam = 0; lam < d.K; ++lam) {
        const double v[2] = {arow[lam].real() * sc, arow[lam].imag() * sc};
        for (int c = 0; c < 2; ++c) {  // image 0: Re A, image 1: Im A
          const uint16_t h = half_rn(v[c]);
          const uint16_t l = half_rn(v[c] - half_to_double(h));
          put(m, c, lam, h);
          put(m, c, d.K + lam, h);
          put(m, c, 2 * d.K + lam, l);
        }
      }
    }
  }
  // time pooling taps g_alpha = IDFT_L(phi_T_hat^(L)) (real, even)
  P.g.clear();
  for (auto& d : P.kd) {
    d.g_off = (int64_t)P.g.size();
    auto ph = gauss_vec(sigT, d.L, P.N_pad);
    // band-limited real-even inverse DFT
    std::vector<int> nz;
    for (int m = 0; m < d.L; ++m)
      if (ph[m] > 1e-30) nz.push_back(m);
    for (int t = 0; t < d.L; ++t) {
      double acc = 0;
      for (int m : nz) acc += ph[m] * unit_root((int64_t)m * t, d.L).real();
      P.g.push_back((float)(acc / d.L));
    }
    d.chunk = std::min(d.L, 4096);   // refined by plan_tc (work units per launch)
    d.nchunks = d.L / d.chunk;
  }
  // KY output (fp16 hi/lo planes, rows padded to 16), per-tile scale slots (tiles
  // of >= 32 columns) and the phi_T pooling tables of the tensor-core KD (built after
  // plan_tc, which decides the tile width the moment form needs)
  {
    const int NF = P.n_frames <= 8 ? 8 : P.n_frames <= 16 ? 16 : 32;
    P.y16_total = 0;
    P.ys_total = 0;
    P.wtab.clear();
    mom_tabs.assign(P.kd.size(), {});
    for (size_t ai = 0; ai < P.kd.size(); ++ai) {
      auto& d = P.kd[ai];
      const int K48 = (3 * d.K + 15) / 16 * 16;
      d.y16_off = P.y16_total;
      P.y16_total += (int64_t)K48 * 2 * d.L;  // [Y_hi; Y_lo; Y_hi][2L] rows, (re, im) interleaved (KY)
      d.ys_off = P.ys_total;
      P.ys_total += 1;  // one scale per (signal, alpha): KC's fp16 store and KD share it
      const float* g = P.g.data() + d.g_off;
      auto tap = [&](int m, int64_t t) -> double { return pool_tap(P, d, m, t); };
      // phi_T pooling in moment form where it is exact to fp32 (kernels_tc.cu,
      // DESIGN.md §6): over each 32-column block, every frame's tap sequence is
      // replaced by its least-squares cubic in u_j = (j - 15.5) / 16 (coefficients
      // rounded to fp32).  The mode is used only if, on every block and frame,
      // the evaluated cubic deviates from the fp32 taps by <= 2^-22 of that block's
      // largest tap (the taps' own fp32 rounding is 2^-24), plus 2^-40 max |g|.
      d.pool_mode = 0;
      if (d.L % 32 == 0 && !(p.flags & JTFS_POOL_EXACT)) {  // flag: validation of the moment form
        double gmax = 0;
        for (int t = 0; t < d.L; ++t) gmax = std::max(gmax, std::abs((double)g[t]));
        // normal equations of the cubic fit (same for every block)
        double Mn[4][4] = {}, U[32][4];
        for (int j = 0; j < 32; ++j) {
          const double u = (j - 15.5) / 16.0;
          U[j][0] = 1;
          U[j][1] = u;
          U[j][2] = u * u;
          U[j][3] = u * u * u;
          for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) Mn[r][c] += U[j][r] * U[j][c];
        }
        // invert the 4x4 (Gauss-Jordan, fp64)
        double Inv[4][8];
        for (int r = 0; r < 4; ++r)
          for (int c = 0; c < 8; ++c) Inv[r][c] = c < 4 ? Mn[r][c] : (c - 4 == r ? 1.0 : 0.0);
        for (int c = 0; c < 4; ++c) {
          int piv = c;
          for (int r = c + 1; r < 4; ++r)
            if (std::abs(Inv[r][c]) > std::abs(Inv[piv][c])) piv = r;
          for (int k = 0; k < 8; ++k) std::swap(Inv[c][k], Inv[piv][k]);
          const double dv = Inv[c][c];
          for (int k = 0; k < 8; ++k) Inv[c][k] /= dv;
          for (int r = 0; r < 4; ++r)
            if (r != c) {
              const double f = Inv[r][c];
              for (int k = 0; k < 8; ++k) Inv[r][k] -= f * Inv[c][k];
            }
        }
        std::vector<float> tab;
        tab.reserve((size_t)d.L / 32 * 4 * NF);
        bool ok = true;
        for (int blk = 0; blk < d.L / 32 && ok; ++blk) {
          double G[4][32] = {};  // [k][m]
          for (int m = 0; m < NF; ++m) {
            double rhs[4] = {0, 0, 0, 0}, w[32], wmax = 0;
            for (int j = 0; j < 32; ++j) {
              w[j] = tap(m, (int64_t)blk * 32 + j);
              wmax = std::max(wmax, std::abs(w[j]));
              for (int r = 0; r < 4; ++r) rhs[r] += U[j][r] * w[j];
            }
            double c[4];
            for (int r = 0; r < 4; ++r) {
              c[r] = 0;
              for (int k = 0; k < 4; ++k) c[r] += Inv[r][4 + k] * rhs[k];
            }
            double worst = 0;
            for (int j = 0; j < 32; ++j) {
              double f = 0;
              for (int k = 0; k < 4; ++k) f += (double)(float)c[k] * U[j][k];
              worst = std::max(worst, std::abs(f - w[j]));
            }
            if (worst > std::ldexp(wmax, -22) + std::ldexp(gmax, -40)) ok = false;
            for (int k = 0; k < 4; ++k) G[k][m] = c[k];
          }
          for (int k = 0; k < 4; ++k)
            for (int m = 0; m < NF; ++m) tab.push_back((float)G[k][m]);
        }
        if (ok) {
          d.pool_mode = 1;
          mom_tabs[ai] = std::move(tab);
        }
      }
    }
  }
  // micro-batch: <= 128 signals and one micro-batch's workspace <= 40 GiB (HBM is 180 GB;
  // larger micro-batches mean fewer launches and better-balanced KD grids: measured on c3,
  // 64 -> 128 signals per micro-batch = +1.3 %, KE 2.0 -> 1.4 ms).  The KD
  // partials depend on the chunking plan_tc picks for this micro-batch; they are
  // small next to Y2, so size first without them and shrink if needed.
#ifndef JTFS_WS_GIB
#define JTFS_WS_GIB 40
#endif
#ifndef JTFS_MB_CAP
#define JTFS_MB_CAP 128
#endif
  const size_t ws_budget = (size_t)JTFS_WS_GIB << 30;
  P.part_total = 0;
  {
    const size_t per = ws_layout(P, 1).total;
    P.mb = (int)std::max<size_t>(1, std::min<size_t>(JTFS_MB_CAP, ws_budget / std::max<size_t>(per, 1)));
  }
  if (P.kd_impl == 1) {
    const std::string e = plan_tc(P);
    if (!e.empty()) return e + " (JTFS_KD_SIMT selects the SIMT validation KD)";
  }
  // phi_T pooling tables per alpha: cubic-moment coefficients where plan_tc kept the
  // moment form, else the exact taps [L][NF]
  {
    const int NF = P.n_frames <= 8 ? 8 : P.n_frames <= 16 ? 16 : 32;
    for (size_t ai = 0; ai < P.kd.size(); ++ai) {
      auto& d = P.kd[ai];
      d.wtab_off = (int64_t)P.wtab.size();
      if (d.pool_mode == 1 && P.kd_impl == 1) {
        P.wtab.insert(P.wtab.end(), mom_tabs[ai].begin(), mom_tabs[ai].end());
      } else {
        d.pool_mode = 0;
        for (int t = 0; t < d.L; ++t)
          for (int m = 0; m < NF; ++m) P.wtab.push_back((float)pool_tap(P, d, m, t));
      }
    }
  }
  P.part_total = 0;
  for (auto& d : P.kd) {
    d.nslices = d.nchunks * (P.kd_impl == 1 ? 2 : 1);  // tcgen05 KD: one slice per epilogue set
    d.part_off = P.part_total;
    P.part_total += (int64_t)d.nslices * P.Mpad * P.n_frames;
  }
  while (P.mb > 1 && ws_layout(P, P.mb).total > ws_budget) --P.mb;

  // phi_t paths: psi_{beta,+1} taps (complex), phi_F taps (real), phi_T taps at rate T (real)
  P.hphi.clear();
  for (int b = 0; b < nb; ++b)
    for (int m = 0; m < P.N_fr; ++m) {
      const auto v = htap[nb + b][m];
      P.hphi.push_back((float)v.real());
      P.hphi.push_back((float)v.imag());
    }
  for (int m = 0; m < P.N_fr; ++m) P.hphi.push_back((float)htap[2 * nb][m].real());
  {
    std::vector<std::complex<double>> ph(P.NPT);
    auto gv = gauss_vec(sigT, P.NPT, P.N_pad);
    for (int m = 0; m < P.NPT; ++m) ph[m] = gv[m];
    auto gt = idft(ph);
    for (int m = 0; m < P.NPT; ++m) P.hphi.push_back((float)gt[m].real());
  }

  // ---- paths (R-O11) ----
  P.paths.clear();
  P.path_filter.clear();
  for (int th : {-1, +1})
    for (const auto& d : P.kd)
      for (int b = 0; b < nb; ++b) {
        P.paths.push_back({JTFS_PATH_SPIN, th, d.alpha, b, P.b2.xi[d.alpha], P.bf.xi[b]});
        P.path_filter.push_back(th == -1 ? b : nb + b);
      }
  for (const auto& d : P.kd) {
    P.paths.push_back({JTFS_PATH_PSI_T_PHI_F, 0, d.alpha, -1, P.b2.xi[d.alpha], 0.0});
    P.path_filter.push_back(2 * nb);
  }
  for (int b = 0; b < nb; ++b) {
    P.paths.push_back({JTFS_PATH_PHI_T_PSI_F, 0, -1, b, 0.0, P.bf.xi[b]});
    P.path_filter.push_back(nb + b);
  }
  P.paths.push_back({JTFS_PATH_PHI_T_PHI_F, 0, -1, -1, 0.0, 0.0});
  P.path_filter.push_back(-1);

  // ---- twiddles exp(-2 pi i t / N_tw) ----
  // per-length twiddle tables exp(-2 pi i t / L), t < L, for L = 2, 4, ..., N_pad,
  // stored back to back (offset(L) = L - 2); plus the full-length table at the end
  // for the scattered-index users (KS inverse DFT of NPT bins)
  P.N_tw = P.N_pad;
  const int lgN = ilog2_exact(P.N_tw);
  const size_t nper = (size_t)2 * P.N_tw - 2;
  P.twiddle.assign(2 * nper, 0.f);
  P.twiddle64.assign(2 * nper, 0.0);
  for (int lg = 1; lg <= lgN; ++lg) {
    const int L = 1 << lg;
    for (int t = 0; t < L; ++t) {
      const auto w = unit_root(-(int64_t)t, L);
      const size_t o = (size_t)(L - 2 + t);
      P.twiddle[2 * o] = (float)w.real();
      P.twiddle[2 * o + 1] = (float)w.imag();
      P.twiddle64[2 * o] = w.real();
      P.twiddle64[2 * o + 1] = w.imag();
    }
  }
  return "";
}

WsLayout ws_layout(const Plan& p, int64_t mb) {
  // (JTFS_WS_GUARDS validation builds: every region carries a trailing guard band that the
  // forward fills with a pattern and checks afterwards -- abi.cu)
  auto al = [](size_t b) { return (b + 255) / 256 * 256 + kWsGuard; };
  WsLayout w{};
  w.xhat = al((size_t)mb * p.N_pad * 8);
  // four-step intermediate: largest group (rows x L) among U1 / Y2 / KA
  size_t tmp = (size_t)p.N_pad * 16;  // fp64 KA intermediate
  for (const auto& g : p.u1_groups)
    if (g.log2L > 12) tmp = std::max(tmp, g.rows.size() * ((size_t)8 << g.log2L));
  for (const auto& g : p.y2_groups)
    if (g.log2L > 12) tmp = std::max(tmp, g.rows.size() * ((size_t)8 << g.log2L));
  w.tmp = al((size_t)mb * tmp);
  // second four-step intermediate of the fused first-order middle stage (k_fft4_mid)
  {
    size_t t2 = 0;
    for (const auto& g : p.u1_groups)
      if (g.log2L > 12) t2 = std::max(t2, g.rows.size() * ((size_t)8 << g.log2L));
    w.tmp2 = al((size_t)mb * t2);
  }
  w.u1 = al((size_t)mb * p.u1_total * 4);
  w.u1hat = al((size_t)mb * p.u1_total * 8);
  w.yphi = al((size_t)mb * p.n1 * p.NPT * 4);
  w.y2 = al((size_t)mb * p.y2_total * 8);
  w.y16 = al((size_t)mb * p.y16_total * 2);
  w.ys = al((size_t)mb * p.ys_total * 8);        // [mb][n_alpha] scales, then [mb][n_alpha] inverses
  w.u1max = al((size_t)mb * p.n1 * 4);         // per (signal, lambda) max |U1| (KB)
  w.part = al((size_t)mb * p.part_total * 4);
  {
    size_t nsel = 0;  // jtfs_forward_units' chunk lists (at most one id per chunk)
    for (const auto& d : p.kd) nsel += (size_t)std::max(1, d.L / 32);  // chunks >= 32 columns
    w.sel = al(nsel * 4);
  }
  w.flag = 256 + kWsGuard;
  w.total = w.xhat + w.tmp + w.tmp2 + w.u1 + w.u1hat + w.yphi + w.y2 + w.y16 + w.ys + w.u1max + w.part + w.sel +
            w.flag;
  return w;
}

void stage_cost(const Plan& p, double fl[6], double by[6]) {
  auto lg = [](double L) { return std::log2(L); };
  for (int i = 0; i < 6; ++i) fl[i] = by[i] = 0;
  // KA: real DFT of the padded signal; reads x
  fl[0] = 2.5 * p.N_pad * lg(p.N_pad);
  by[0] = 4.0 * p.N;
  // KB: per lambda band multiply, complex IDFT_L1, modulus, real DFT_L1
  for (int l = 0; l < p.n1; ++l) {
    const double L1 = p.L1[l];
    fl[1] += 2.0 * p.band_psi1[l].len + 5.0 * L1 * lg(L1) + 5.0 * L1 + 2.5 * L1 * lg(L1);
  }
  // KS: phi_T folds + NPT-point inverse DFTs (S0, S1, Y_phi); writes S0 + S1
  fl[2] = (double)(p.n1 + 1) * (2.0 * 12 * p.NPT + 5.0 * p.NPT * lg(std::max(p.NPT, 2)));
  by[2] = 4.0 * p.n_frames * (1 + p.n1);
  // KC: per admissible (alpha, lambda): band multiply + complex IDFT_{L_alpha}
  for (const auto& g : p.y2_groups)
    for (const auto& r : g.rows) {
      const double L = (double)(1 << g.log2L);
      fl[3] += 2.0 * r.len + 5.0 * L * lg(L);
    }
  // KD: per alpha and time column: DFT_{N_fr} along lambda, per filter multiply + IDFT_R,
  //     then modulus + pooling on the M retained rows
  for (const auto& d : p.kd) {
    double col = 5.0 * p.N_fr * lg(p.N_fr);
    for (const auto& f : p.fr) col += 2.0 * p.N_fr + 5.0 * f.R * lg(std::max(f.R, 2));
    fl[4] += (double)d.L * col + (double)p.M * d.L * (5.0 + 2.0 * p.n_frames);
  }
  // KE: lambda pooling matrices + phi paths; writes S2
  for (size_t i = 0; i < p.paths.size(); ++i) {
    const int fi = p.path_filter[i];
    const double rows = fi >= 0 ? p.fr[fi].nrows : p.n1;
    fl[5] += 2.0 * p.lam_out * rows * p.n_frames;
    if (p.paths[i].kind == JTFS_PATH_PHI_T_PSI_F) fl[5] += rows * p.NPT * (8.0 * p.n1 + 5.0 + 2.0 * p.n_frames);
  }
  by[5] = 4.0 * (double)p.paths.size() * p.lam_out * p.n_frames;
}

}  // namespace jtfs
