/*
 * jtfs.h -- C ABI of the B200-native forward Joint Time-Frequency Scattering.
 *
 * Operator: PAPER.md (arXiv 2204.08269, DAFx-22), Sec. 2:
 *   scalogram  X(t,lambda) = |x * psi_lambda|(t)
 *   Eq. (1)    psi_alpha(t) = 2^a psi(2^a t),
 *              psi_{beta,theta}(lambda) = 2^b psi(theta 2^b lambda)
 *   Eq. (2)    Psi_{alpha,beta,theta} = psi_alpha(t) psi_{beta,theta}(lambda)
 *   Eq. (3)    S2 = | X *_{t,lambda} Psi | *_{t,lambda} Phi_{T,F}
 *   Eq. (4)    S2 = | X *_{t,lambda} Psi | *_t Phi_T
 *   first order S1 = U1 * phi_T (no Phi_F), out_3D layout,
 * with the readings of DESIGN.md §3 for everything the paper
 * leaves unstated (filter constants, critical subsampling, padding,
 * admissibility, lambda-axis boundary, spin orientation, path order).
 *
 * Conventions for every function:
 *   - extern "C", returns jtfs_status (0 = JTFS_OK); no C++ exception crosses the ABI;
 *   - on error a thread-local message is available from jtfs_last_error();
 *   - "device" pointers are CUDA global-memory pointers on the plan's device,
 *     "host" pointers are ordinary CPU memory;
 *   - the caller owns every buffer it passes; the plan owns its device tables
 *     and frees them in jtfs_plan_destroy.
 */
#ifndef JTFS_H_
#define JTFS_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define JTFS_API __attribute__((visibility("default")))
#else
#define JTFS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  JTFS_OK = 0,
  JTFS_ERR_INVALID_ARG = 1,  /* bad parameter / null or misaligned pointer / bad size */
  JTFS_ERR_UNSUPPORTED = 2,  /* valid but not supported (e.g. forward on a host-only plan) */
  JTFS_ERR_OOM = 3,          /* device or host allocation failed */
  JTFS_ERR_CUDA = 4,         /* a CUDA runtime call or kernel launch failed */
  JTFS_ERR_WORKSPACE = 5,    /* workspace smaller than jtfs_workspace_size() */
  JTFS_ERR_NONFINITE = 6     /* JTFS_CHECK_FINITE set and the input holds NaN/Inf */
} jtfs_status;

/* flags */
#define JTFS_CHECK_FINITE 1u   /* forward scans x for NaN/Inf first (one device sync) */
#define JTFS_LATENCY 2u        /* size KD work units for one signal per forward (c4, path sharding) */
/* validation / measurement flags (never needed for production use; every output byte
 * is a function of (params incl. flags, x) -- the library reads no environment): */
#define JTFS_KD_SIMT 4u        /* KD on the FP32 SIMT validation kernel instead of tcgen05 */
#define JTFS_POOL_EXACT 8u     /* KD epilogue with the exact phi_T taps (no cubic-moment form) */
#define JTFS_KD_PROF 16u       /* instrumented KD: per-role wait cycles to stderr (syncs per launch) */
#define JTFS_KD_NOPAIR 32u     /* tcgen05 KD on single CTAs only (no cta_group::2 CTA pairs) */

/* pad modes (reading R6) */
#define JTFS_PAD_REFLECT 0     /* numpy 'reflect' to N_pad = 2N, centred */
#define JTFS_PAD_PERIODIC 1    /* N_pad = N, circular (exact-invariant tests) */

typedef struct jtfs_plan_s* jtfs_plan_t;  /* opaque; immutable after creation */

/* Operator parameters (Sec. 4.2, Sec. 3.3).
 *   N      signal length, power of two
 *   J      octaves of the temporal banks (2^J <= N)
 *   Q      first-order wavelets per octave (>= 1)
 *   Q2     second-order wavelets per octave (paper: 1)
 *   T      temporal lowpass support, power of two, T <= N
 *   J_fr   octaves of the frequential bank (>= 1)
 *   Q_fr   frequential wavelets per octave (paper: 1)
 *   F      frequential lowpass support, power of two (0 -> 2^J_fr)
 *   average_fr  1: Eq. (3) (Phi_{T,F}); 0: Eq. (4) (Phi_T only)
 *   pad_mode    JTFS_PAD_REFLECT or JTFS_PAD_PERIODIC
 *   device      CUDA device ordinal; -1 = host-only plan (queries only, no forward)
 *   flags       JTFS_CHECK_FINITE | JTFS_LATENCY (| validation flags above)
 */
typedef struct {
  int32_t N, J, Q, Q2, T, J_fr, Q_fr, F;
  int32_t average_fr, pad_mode, device;
  uint32_t flags;
} jtfs_params;

/* Packed out_3D record of one signal (DESIGN.md §3 R-O11/O12), fp32:
 *   [ S0 : n_frames ][ S1 : n1 x n_frames ][ S2 : n_paths x lambda_out x n_frames ]
 * all row-major; S1 rows in descending centre frequency; frames are the
 * un-padded time frames m in [frame0, frame0 + n_frames) at rate T. */
typedef struct {
  int32_t n1;            /* first-order filters (lambda rows) */
  int32_t n_frames;      /* time frames per coefficient = ceil(N / T) */
  int32_t frame0;        /* first retained frame index on the padded grid */
  int32_t lambda_out;    /* S2 log-frequency rows: ceil(n1/F) (Eq. 3) or n1 (Eq. 4) */
  int32_t n_paths;       /* S2 paths lambda2 = (alpha, beta, theta) incl. phi-only paths */
  int32_t n_alpha;       /* active second-order temporal wavelets */
  int32_t n_beta;        /* frequential wavelets per spin */
  int32_t N_pad;         /* padded length */
  int32_t N_fr;          /* frequential (lambda) grid length */
  int32_t reserved;
  int64_t off_s0, off_s1, off_s2;  /* float offsets inside one record */
  int64_t floats_per_signal;
} jtfs_layout_t;

/* Path kinds, in output order (DESIGN.md R-O11). */
#define JTFS_PATH_SPIN 0        /* psi_alpha (x) psi_{beta,theta} */
#define JTFS_PATH_PSI_T_PHI_F 1 /* psi_alpha (x) phi_F */
#define JTFS_PATH_PHI_T_PSI_F 2 /* phi_T (x) psi_beta (one spin, real input) */
#define JTFS_PATH_PHI_T_PHI_F 3 /* phi_T (x) phi_F (no modulus) */

typedef struct {
  int32_t kind;     /* JTFS_PATH_* */
  int32_t theta;    /* -1 / +1 for spinned paths, 0 otherwise */
  int32_t alpha;    /* index into the second-order bank G(J,Q2) (0 = highest xi), -1 if none */
  int32_t beta;     /* index into the frequential bank G(J_fr,Q_fr), -1 if none */
  double xi_alpha;  /* centre frequency of psi_alpha, cycles/sample (0 if none) */
  double xi_beta;   /* centre frequency of psi_beta, cycles/bin (0 if none) */
} jtfs_path_t;

/* North-star form (north_star's jtfs_plan(N,J,Q,J_fr,Q_fr,T,F,...)): equivalent
 * to jtfs_plan_create with Q2 = 1, average_fr = 1 (Eq. (3)), reflect
 * padding, device = current CUDA device, flags as given. */
JTFS_API jtfs_status jtfs_plan(int N, int J, int Q, int J_fr, int Q_fr, int T, int F, int flags,
                      jtfs_plan_t* out);

/* Build a plan: validates every constraint of DESIGN.md §3 (pow2 N, T, F;
 * 2^J <= N; T <= N; n1 >= 4; F <= N_fr), generates the filter banks in fp64,
 * derives the schedule, and (device >= 0) uploads fp32 tables to the device.
 * *out receives the handle (NULL on error). */
JTFS_API jtfs_status jtfs_plan_create(const jtfs_params* params, jtfs_plan_t* out);

/* Frees the plan's device tables.  NULL-safe.  Must not race a forward on it. */
JTFS_API jtfs_status jtfs_plan_destroy(jtfs_plan_t plan);

/* Output layout of one signal (host query, valid for host-only plans). */
JTFS_API jtfs_status jtfs_layout(jtfs_plan_t plan, jtfs_layout_t* out);

/* Path metadata in output order; writes min(cap, n_paths) entries to out (host). */
JTFS_API jtfs_status jtfs_paths(jtfs_plan_t plan, jtfs_path_t* out, int32_t cap);

/* First-order centre frequencies xi_lambda (cycles/sample), descending; host. */
JTFS_API jtfs_status jtfs_lambda_xi(jtfs_plan_t plan, double* out, int32_t cap);

/* Device workspace bytes jtfs_forward needs for a batch of `batch` signals. */
JTFS_API jtfs_status jtfs_workspace_size(jtfs_plan_t plan, int64_t batch, size_t* bytes);

/* Forward JTFS of a batch.
 *   x      device, fp32 [B][N] row-major, 16-byte aligned
 *   B      number of signals (>= 0; B = 0 is a no-op)
 *   out    device, fp32 [B][floats_per_signal], 16-byte aligned
 *   ws     device workspace of ws_bytes >= jtfs_workspace_size(plan, B), 256-byte aligned
 *   stream cudaStream_t (NULL = legacy default stream)
 * Asynchronous: enqueues kernels on `stream` and returns; asynchronous faults
 * surface at the caller's next synchronisation.  Output bytes are a
 * deterministic function of (plan, x) independent of B and of the GPU count. */
JTFS_API jtfs_status jtfs_forward(jtfs_plan_t plan, const float* x, int64_t B, float* out,
                         void* ws, size_t ws_bytes, void* stream);

/* End-to-end variant with HOST buffers: copies x_host (fp32 [B][N]) to the
 * device, runs jtfs_forward, copies the result to out_host (fp32
 * [B][floats_per_signal]) and synchronises `stream`.  x_dev / out_dev are
 * caller-owned device staging buffers of the same shapes.  Host buffers should
 * be pinned for full copy bandwidth.  The copies are pipelined per micro-batch on two
 * internal copy streams (H2D of micro-batch i+1 and D2H of i-1 overlap the compute of
 * i on `stream`); the result bytes equal jtfs_forward's. */
JTFS_API jtfs_status jtfs_forward_host(jtfs_plan_t plan, const float* x_host, int64_t B,
                              float* out_host, float* x_dev, float* out_dev,
                              void* ws, size_t ws_bytes, void* stream);

/* ---- Path sharding of one forward over several GPUs (
 * DESIGN.md §7).  The joint stage's frequential contraction + modulus + phi_T
 * pooling (Eq. (3)) is a sum over time of per-(alpha, time chunk)
 * contributions, so KD's work splits into units (alpha, time chunk) whose
 * pooled partial slices are additive and disjoint.  A rank runs the replicated
 * first stages (Eqs. (1)-(2): KA..KC, and S0/S1) plus KD for its own units;
 * the ranks' partial buffers are summed (each slice is nonzero on exactly one
 * rank, so the sum is exact), and one rank finishes Eq. (3)'s phi_F pooling and
 * packing with jtfs_reduce_pack.  The result is byte-identical to jtfs_forward. */

typedef struct {
  int32_t alpha;   /* index of the active alpha (KD order = path order of jtfs_paths) */
  int32_t chunk;   /* time chunk of that alpha */
  int32_t col0;    /* first time column of the chunk on the alpha's grid */
  int32_t ncols;   /* columns in the chunk */
  double cost;     /* modelled relative cost (tensor + epilogue work), for load balancing */
} jtfs_unit_t;

/* The KD work units of one signal, alpha-major then chunk (unit id = position).
 * Writes min(cap, n) units; *n_units = total.  Host query.  Plans created with
 * JTFS_LATENCY use small chunks (many units for one signal). */
JTFS_API jtfs_status jtfs_units(jtfs_plan_t plan, jtfs_unit_t* units, int32_t cap, int32_t* n_units);

/* Floats of KD partials per signal (the buffer of jtfs_forward_units). */
JTFS_API jtfs_status jtfs_partials_size(jtfs_plan_t plan, int64_t* floats_per_signal);

/* Forward restricted to KD units unit_ids[0..n_units) (host array of unit ids,
 * any order, no duplicates).  x: device fp32 [B][N]; partials: device fp32
 * [B][partials_size], fully overwritten (slices of other units are zeroed);
 * out: device fp32 [B][floats_per_signal] -- receives S0 and S1 only.  ws must
 * be kept untouched until jtfs_reduce_pack (it holds the phi_T-averaged first
 * order Y_phi).  B must not exceed the plan's micro-batch (JTFS_ERR_INVALID_ARG
 * otherwise; c4 uses B = 1).  Synchronises `stream` once (it uploads the unit list
 * per call); jtfs_forward_unitset is the asynchronous, capturable form. */
JTFS_API jtfs_status jtfs_forward_units(jtfs_plan_t plan, const float* x, int64_t B,
                                        const int32_t* unit_ids, int32_t n_units, float* partials,
                                        float* out, void* ws, size_t ws_bytes, void* stream);

/* A unit set bound once to device tables (host list -> device, synchronous at creation),
 * so the sharded forward below never synchronises and can be captured in a CUDA graph.
 * The set belongs to `plan` (destroy it before the plan); NULL-safe destroy. */
typedef struct jtfs_unitset_s* jtfs_unitset_t;
JTFS_API jtfs_status jtfs_unitset_create(jtfs_plan_t plan, const int32_t* unit_ids, int32_t n_units,
                                         jtfs_unitset_t* out);
JTFS_API jtfs_status jtfs_unitset_destroy(jtfs_unitset_t set);

/* jtfs_forward_units with a bound unit set: same arguments and results, asynchronous on
 * `stream` with no host synchronisation (graph-capturable).  (jtfs_forward_units binds a
 * temporary set per call and synchronises `stream` before releasing it.) */
JTFS_API jtfs_status jtfs_forward_unitset(jtfs_plan_t plan, const float* x, int64_t B, jtfs_unitset_t set,
                                          float* partials, float* out, void* ws, size_t ws_bytes,
                                          void* stream);

/* Float range [begin, end) of one signal's partials buffer that unit `unit` writes (its
 * chunk's slices; every other unit's range is disjoint).  Unit ids are ordered like the
 * buffer: a contiguous id range owns one contiguous float range, which is what a sharded
 * forward exchanges.  Host query. */
JTFS_API jtfs_status jtfs_unit_partials_range(jtfs_plan_t plan, int32_t unit, int64_t* begin, int64_t* end);

/* Eq. (3)/(4) completion from summed partials (device fp32 [B][partials_size])
 * and the Y_phi left in ws by jtfs_forward_units on the same plan: phi_F pooling,
 * phi-only paths and packing of S2 into out (S0/S1 already there).  Asynchronous. */
JTFS_API jtfs_status jtfs_reduce_pack(jtfs_plan_t plan, const float* partials, int64_t B, float* out,
                                      void* ws, size_t ws_bytes, void* stream);

/* ---- Second-order time scattering (Scattering1D):
 * "applying only a 1-D temporal wavelet filterbank to the first-order
 * scalogram": S2_t[lambda, alpha] = (|U1_lambda * psi_alpha| * phi_T) at the
 * retained frames, over the plan's admissible pairs j1(lambda) < j2(alpha)
 * (DESIGN.md §3 R7) -- the JTFS's Y2 without the lambda convolution.  Shares
 * every first stage of jtfs_forward (KA..KC); the frequential filters of the
 * plan are unused.  Record of one signal, fp32:
 *   [ S0 : n_frames ][ S1 : n1 x n_frames ][ S2_t : n2 x n_frames ],
 * S2_t rows alpha-major (active alphas in jtfs_paths order), then lambda. */
typedef struct {
  int32_t n1, n2, n_frames, frame0;
  int64_t off_s0, off_s1, off_s2, floats_per_signal;
} jtfs_scat1d_layout_t;

JTFS_API jtfs_status jtfs_scat1d_layout(jtfs_plan_t plan, jtfs_scat1d_layout_t* layout);

/* (lambda, alpha) of every S2_t row: pairs[2 r] = lambda (first-order filter
 * index), pairs[2 r + 1] = alpha (second-order bank index); writes min(cap, n2) rows. */
JTFS_API jtfs_status jtfs_scat1d_paths(jtfs_plan_t plan, int32_t* pairs, int32_t cap);

/* Time scattering of x (device fp32 [B][N]) into out (device fp32
 * [B][floats_per_signal of jtfs_scat1d_layout]); same workspace, stream and
 * error rules as jtfs_forward. */
JTFS_API jtfs_status jtfs_scattering1d(jtfs_plan_t plan, const float* x, int64_t B, float* out,
                                       void* ws, size_t ws_bytes, void* stream);

/* ---- Backward: vector-Jacobian product of jtfs_forward for
 * texture resynthesis by gradient descent (the gradient "is
 * computed via reverse-ordered Hermitian adjoints of the forward scattering
 * operations").  dx = d<dout, jtfs_forward(x)>/dx, every stage the exact
 * adjoint of the forward kernels; the subgradient of |z| at z = 0 is 0.
 *   x     device fp32 [B][N] (the point of linearisation; the forward intermediates
 *         are recomputed)
 *   dout  device fp32 [B][floats_per_signal] (gradient of the loss w.r.t. the record)
 *   dx    device fp32 [B][N] (output)
 * Workspace: jtfs_backward_workspace_size (separate from the forward's); same
 * stream / error rules as jtfs_forward. */
JTFS_API jtfs_status jtfs_backward_workspace_size(jtfs_plan_t plan, int64_t B, size_t* bytes);
JTFS_API jtfs_status jtfs_backward(jtfs_plan_t plan, const float* x, int64_t B, const float* dout, float* dx,
                                   void* ws, size_t ws_bytes, void* stream);

/* Texture-resynthesis loss of one record: E = ||Sy - Sx||_2 / ||Sx||_2 and
 * dE/dSy = (Sy - Sx) / (||Sy - Sx|| ||Sx||) (0 where Sy = Sx), fp64 fixed-order sums.
 *   Sy, Sx  device fp32 [floats_per_signal];  E  device fp64 scalar;  dout  device fp32
 *   [floats_per_signal] (the jtfs_backward input).  Asynchronous on `stream`. */
JTFS_API jtfs_status jtfs_resynth_loss(jtfs_plan_t plan, const float* Sy, const float* Sx, double* E,
                                       float* dout, void* stream);

/* Debug/test query: byte offsets inside the backward workspace (for B signals)
 * of its regions, in this order: 0 X_hat, 1 tmp, 2 U1, 3 U1hat, 4 Y_phi, 5 Y2,
 * 6 scratch out, 7 dP, 8 dY_phi, 9 dY2, 10 DFT(dY2), 11 dU1hat, 12 dU1, 13 W,
 * 14 DFT(dU1 W/|W|), 15 dX_hat, 16 dx_pad; offsets[17] = total.  Host query. */
JTFS_API jtfs_status jtfs_backward_regions(jtfs_plan_t plan, int64_t B, int64_t* offsets, int32_t cap);

/* ---- NEXT-4: mu-log compression and the scale-rate map ---- */

/* mu(lambda_2) of Eq. (adalog:mu) over a batch of jtfs_forward records:
 *   mu[p] = (1/B) sum_b sum_{lambda, t} S2_b[p][lambda][t]   for every S2 path p
 * (jtfs_paths order; the double integral over the sampled grid is the map's sum),
 * accumulated in fp64 in a fixed order (bit-stable), rounded to fp32.
 *   S   device fp32 [B][floats_per_signal], B >= 1
 *   mu  device fp32 [n_paths] (output)
 * Asynchronous on `stream`.  For a set larger than one batch, average the per-batch
 * mu weighted by the batch sizes. */
JTFS_API jtfs_status jtfs_mulog_mu(jtfs_plan_t plan, const float* S, int64_t B, float* mu, void* stream);

/* Eq. (adalog): out = S with every S2 value of path p replaced by
 *   log(1 + S / (eps mu[p]))        (eps = 0.1 in the paper),
 * S0 and S1 copied unchanged (reading R22: the transform is per second-order path
 * lambda_2).  A path with eps * mu[p] <= 0 maps to 0.  out may alias S.
 *   S, out  device fp32 [B][floats_per_signal];  mu device fp32 [n_paths];  eps > 0.
 * Asynchronous on `stream`. */
JTFS_API jtfs_status jtfs_mulog_apply(jtfs_plan_t plan, const float* S, int64_t B, const float* mu, float eps,
                                      float* out, void* stream);

/* jtfs_forward with the mu-log of Eq. (adalog) fused into the phi_F pooling /
 * packing kernel (KE): out = [S0][S1][log(1 + S2 / (eps mu))] in one pass, bit-identical
 * to jtfs_forward followed by jtfs_mulog_apply.  Arguments and rules as jtfs_forward,
 * plus mu (device fp32 [n_paths], e.g. from jtfs_mulog_mu over a training set) and eps > 0. */
JTFS_API jtfs_status jtfs_forward_mulog(jtfs_plan_t plan, const float* x, int64_t B, const float* mu, float eps,
                                        float* out, void* ws, size_t ws_bytes, void* stream);

/* Shape of the scale-rate map of S2 path `path` (reading R21): rows = ceil(n1 / 2^k),
 * k = the path's lambda decimation (k_f(beta) for a spinned path in Eq. (3) mode,
 * log2 F for psi_t x phi_f, 0 in Eq. (4) mode); cols = ceil(N / 2^k_alpha).  Only the
 * psi_t paths (kinds SPIN, PSI_T_PHI_F) have one; other kinds or an out-of-range path
 * return JTFS_ERR_INVALID_ARG.  Host query. */
JTFS_API jtfs_status jtfs_u2_map_shape(jtfs_plan_t plan, int32_t path, int32_t* rows, int32_t* cols);

/* Scale-rate visualisation of Fig. 1: |X * Psi_{alpha,beta,theta}|, the joint
 * wavelet modulus BEFORE the lowpass Phi of Eq. (3), on the whole log-frequency and time
 * axes: out[b][r][c] = |sum_lambda h_f[(r 2^k - lambda) mod N_fr] Y2_alpha[lambda][c0 + c]|,
 * r' = r over the scalogram rows, c0 = ceil(pad_left / 2^k_alpha) (the unpadded signal).
 *   x    device fp32 [B][N];  out device fp32 [B][rows][cols] (jtfs_u2_map_shape)
 *   ws   the forward workspace (jtfs_workspace_size(plan, B)); asynchronous on `stream`. */
JTFS_API jtfs_status jtfs_u2_map(jtfs_plan_t plan, const float* x, int64_t B, int32_t path, float* out,
                                 void* ws, size_t ws_bytes, void* stream);

/* ---- NEXT-3: K-nearest-neighbour parameter regression ----
 * For every example i of a feature set F (e.g. JTFS records of the 16^3 AM/FM chirp grid,
 * P:139-140), the K examples j != i at the smallest Euclidean distance ||F_j - F_i||_2 --
 * the greedy argmin recursion of P:201-209, ties to the smaller index (reading R23) --
 * and theta~_i = (1/K) sum_{j in N_K(i)} theta_j, ratio theta~_i / theta_i
 * (P:210).  Distances are sums of squared differences in fp64 over the fp32 features.
 * Plan-independent. */

/* Workspace bytes for n examples (the n x n fp64 distance matrix).  Host query. */
JTFS_API jtfs_status jtfs_knn_workspace_size(int64_t n, size_t* bytes);

/*   F          device fp32, example i's features at F[i * ldf + 0 .. d)   (ldf >= d)
 *   n, d       2 <= n <= 16384 examples, d >= 1 features
 *   theta      device fp64 [n][n_params] parameters (may be NULL when n_params = 0)
 *   K          1 <= K < n  (the paper uses K = 40)
 *   nbr        device int32 [n][K] neighbour indices in the recursion's order (output)
 *   theta_hat  device fp64 [n][n_params] or NULL;  ratio device fp64 [n][n_params] or NULL
 *   ws         device, >= jtfs_knn_workspace_size(n) bytes, 256-byte aligned
 * Asynchronous on `stream`; deterministic (fixed-order sums, total order on keys).
 * JTFS_ERR_INVALID_ARG for sizes out of range / NULL buffers, JTFS_ERR_WORKSPACE. */
JTFS_API jtfs_status jtfs_knn_regress(const float* F, int64_t n, int64_t d, int64_t ldf, const double* theta,
                                      int32_t n_params, int32_t K, int32_t* nbr, double* theta_hat,
                                      double* ratio, void* ws, size_t ws_bytes, void* stream);

/* Isomap of the same feature set (Fig. 3; Tenenbaum et al. 2000, cited at
 * P:157) on the K-NN graph above: edges (i, j) of length ||F_i - F_j|| for j in N_K(i)
 * or i in N_K(j); geodesic distances = all-pairs shortest paths (blocked Floyd-Warshall,
 * fp64); classical MDS B = -1/2 H (G o G) H; the top n_components eigenpairs of B by a
 * fixed-length subspace iteration with Rayleigh-Ritz (reading R25).  Each eigenvector's
 * sign is fixed so that its entry of largest magnitude is positive.
 *   F, n, d, ldf, K  as jtfs_knn_regress (2 <= n <= 16384, 1 <= K < n)
 *   n_components     1 .. 8 (the paper uses 3)
 *   emb              device fp64 [n][n_components]: eigenvector * sqrt(max(eigenvalue, 0))
 *   eigvals          device fp64 [n_components], descending
 *   ws               device, >= jtfs_isomap_workspace_size(n, K) bytes, 256-byte aligned
 * SYNCHRONOUS (reads back a connectivity flag): JTFS_ERR_INVALID_ARG if the neighbour
 * graph is disconnected (outputs then undefined). */
JTFS_API jtfs_status jtfs_isomap_workspace_size(int64_t n, int32_t K, size_t* bytes);
JTFS_API jtfs_status jtfs_isomap(const float* F, int64_t n, int64_t d, int64_t ldf, int32_t K,
                                 int32_t n_components, double* emb, double* eigvals, void* ws, size_t ws_bytes,
                                 void* stream);

/* Debug taps for kernel-level tests (device outputs, synchronous).
 *   tap 0: X_hat   -> out complex (float2) [B][N_pad]
 *   tap 1: U1      -> out fp32 [B][sum_lambda L1(lambda)]   (rows in lambda order)
 *   tap 2: Y2      -> out fp32 [B][sum_alpha 2 K_alpha L_alpha]: per alpha a planar [2 K_alpha][L_alpha]
 *                     block, row 2*lambda = Re Y2_alpha[lambda], row 2*lambda+1 = Im
 *   tap 3: Yphi    -> out fp32 [B][n1][N_pad/T]
 * `out_floats` is the capacity of out in floats. */
JTFS_API jtfs_status jtfs_debug_tap(jtfs_plan_t plan, int32_t tap, const float* x, int64_t B,
                           float* out, int64_t out_floats, void* ws, size_t ws_bytes,
                           void* stream);

/* Size in floats of a debug tap for B signals. */
JTFS_API jtfs_status jtfs_debug_tap_size(jtfs_plan_t plan, int32_t tap, int64_t B, int64_t* floats);

/* Joint stage alone (validation of KD + KE, SURVEY §4 T4 invariants and stage parity):
 * Eqs. (1)-(3) / (4) from a given Y2 and Y_phi instead of from x.
 *   y2    device fp32 [B][...] in the layout of debug tap 2 (per alpha a (2K) x L_alpha
 *         planar block, rows 2 lambda / 2 lambda + 1 = Re / Im Y2_alpha[lambda])
 *   yphi  device fp32 [B][n1][N_pad/T] in the layout of debug tap 3
 *   out   device fp32 [B][floats_per_signal]: S0 / S1 zero, S2 = the joint stage
 * B <= one micro-batch; workspace as for jtfs_forward; asynchronous on `stream`. */
JTFS_API jtfs_status jtfs_debug_joint(jtfs_plan_t plan, const float* y2, const float* yphi, int64_t B,
                             float* out, void* ws, size_t ws_bytes, void* stream);

/* The FFT engine alone on contiguous complex rows: out[r] = DFT of in[r]
 * (dir -1: sum_n x[n] e^{-2 pi i n k / L}) or the unnormalised inverse (dir +1), L = 2^log2L.
 *   fp64 = 0: float2 rows (the fp32 engine of KB / KC, both directions, L <= N_pad);
 *   fp64 = 1: double2 rows (the fp64 engine of KA, forward only).
 * in / out device, 16-B aligned, rows x L elements; tmp: device scratch of rows x L
 * elements (the four-step intermediate).  Asynchronous on `stream`. */
JTFS_API jtfs_status jtfs_debug_fft(jtfs_plan_t plan, int32_t log2L, int32_t dir, int32_t fp64,
                           const void* in, void* out, int64_t rows, void* tmp, size_t tmp_bytes,
                           void* stream);

/* The KD tiling the plan chose (plan_tc, kernels_tc.cu; host plans too): per active alpha
 * a, out[10a..10a+9] = { kd_impl (1 tcgen05, 0 SIMT validation), CTA pairs (cta_group::2),
 * A stationary, Nt, M-parts, M-blocks per part (pairs: per CTA), B buffers, A ring stages,
 * K-chunks, pooling form (0 taps, 1 cubic moments) }.  cap >= 10 x n_alpha. */
JTFS_API jtfs_status jtfs_debug_kd_tiling(jtfs_plan_t plan, int32_t* out, int32_t cap);

/* Density of the KD's tensor-core operand A''_alpha (VERDICT r1 "measure A's
 * density"): per active alpha a, { records (128 pair rows x 16 packed
 * K-columns), records holding an entry > thr x its row's largest coefficient, records in
 * the per-M-block band [first, last] such record, K-chunks per M-block, coefficients
 * A_alpha[p][lambda] > thr x row max, coefficients (pair rows x K) }: out[6a..6a+5].
 * Host only (works on a host plan, device < 0); cap >= 6 x n_alpha. */
JTFS_API jtfs_status jtfs_debug_a16_density(jtfs_plan_t plan, double thr, int64_t* out, int32_t cap);

/* Host copy of a sampled filter spectrum as the plan generated it (fp64), for
 * cross-checking the plan generator against the oracle's independent one.
 *   bank 1: psi_lambda, 2: psi_alpha, 3: psi_beta (theta=-1), 4: phi_T, 5: phi_F
 *   idx   filter index in its bank (ignored for lowpass)
 *   L, n_grid  grid length and physical spacing 1/n_grid (R8)
 * out: L doubles. */
JTFS_API jtfs_status jtfs_debug_filter(jtfs_plan_t plan, int32_t bank, int32_t idx, int32_t L,
                              int32_t n_grid, double* out);

/* FP32 SIMT peak probe (the ALU roofline must be measured with an FFMA
 * loop): runs FFMA and packed FFMA2 (fma.rn.f32x2) loops on every SM of `device` for a few
 * ms each and returns the achieved TFLOP/s (FMA = 2 flops) of the better of 3 timed runs.
 * Synchronous (blocks until done); at the clock the GPU runs at during the call. */
JTFS_API jtfs_status jtfs_measure_fp32_peak(int32_t device, double* tflops_ffma, double* tflops_ffma2);

/* Algorithmic cost of one signal per stage (same stage numbering as profiling),
 * for roofline reporting; cost model of DESIGN.md §5 (SURVEY App. B conventions:
 * complex FFT 5 L log2 L, real FFT 2.5 L log2 L, complex modulus 5, pooling
 * 2 per frame per element).  flops[s]: the cheapest exact formulation of the
 * stage's arithmetic (for KD the FFT-along-lambda form); bytes[s]: the stage's
 * unavoidable HBM traffic (input + output of the whole path are charged to
 * KA / KS / KE).  With cap >= 7, flops[6] is the tensor-core work KD actually
 * executes per signal (spin-pair contraction, fp16 two-term split packed along K:
 * 8 Mpp K16 L flops summed over alpha, Mpp = pair rows, K16 = 3K rounded up to 16)
 * and bytes[6] the A''/Y'' bytes KD stages
 * into shared memory per signal.  Host query. */
JTFS_API jtfs_status jtfs_cost(jtfs_plan_t plan, double* flops, double* bytes, int32_t cap);

/* Stage profiling (tracing).  When enabled, jtfs_forward records a CUDA event
 * pair on the caller's stream around each stage of every micro-batch:
 *   0 KA pad+DFT, 1 KB first order (U1, U1hat), 2 KS phi_T averaging (S0, S1, Y_phi),
 *   3 KC second order in time (Y2), 4 KD frequential contraction + modulus +
 *   phi_T pooling, 5 KE phi_F pooling + phi paths + packing.
 * jtfs_profile_read synchronises on the recorded events, writes the summed
 * milliseconds per stage into stage_ms[cap] and the number of kernel launches
 * per stage (counted whether or not profiling is enabled) into
 * stage_launches[cap], and (reset != 0) clears both.  Profiling state is the
 * only mutable part of a plan: do not profile one plan from two threads. */
#define JTFS_N_STAGES 6
JTFS_API jtfs_status jtfs_profile_enable(jtfs_plan_t plan, int32_t enable);
JTFS_API jtfs_status jtfs_profile_read(jtfs_plan_t plan, double* stage_ms, int64_t* stage_launches,
                                       int32_t cap, int32_t reset);
/* Per-alpha breakdown of stage 4 (KD) recorded while profiling is enabled:
 * ms[i] = summed milliseconds of the KD launches of the i-th active alpha
 * (layout.n_alpha entries).  Synchronises; reset != 0 clears. */
JTFS_API jtfs_status jtfs_profile_read_kd(jtfs_plan_t plan, double* ms, int32_t cap, int32_t reset);

JTFS_API const char* jtfs_status_string(jtfs_status s);
JTFS_API const char* jtfs_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* JTFS_H_ */
