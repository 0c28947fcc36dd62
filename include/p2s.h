/*
 * p2s.h -- C ABI of the B200-native DF-P2S dense-field turbulence simulator.
 *
 * Method: Chimitt, Zhang, Mao, Chan, "Real-Time Dense Field Phase-to-Space
 * Simulation of Imaging through Atmospheric Turbulence", arXiv 2210.06713.
 * Citations "P:<line>" refer to the paper's text; "Q<n>" to the
 * readings of SURVEY.md Sec. 8(c) that DESIGN.md lists where the paper is
 * silent.
 *
 * Per frame the library runs five steps on the GPU:
 *   1. Fourier sampling of per-pixel Zernike coefficient fields: per-mode PSDs of
 *      the homogeneous auto-correlation slices A_jj filter seeded
 *      Hermitian white noise, a 2-D inverse DFT yields two real unit-variance
 *      fields per complex transform, point-wise Noll mixing
 *      a = L f with L L^T = A_0 (Eq.10).
 *   2. Tilt warp from a_2, a_3 (bilinear gather, clamp-to-edge; Q12).
 *   3. The P2S network mapping each pixel's higher-order Zernike vector a_4..a_Z
 *      to K basis weights (shape Q13).
 *   4. The spatially varying blur out_c(x) = sum_k w_k(x) (h_k (*) Iw_c)(x)
 *      (Eq.9; true convolution, centre tap, mirror boundary Q14).
 *   5. Optional PSF-sum normalisation, additive Gaussian noise, clamp (Q16).
 *
 * Conventions for every entry point:
 *   - Functions never throw or abort; they return a p2s_status and store a
 *     thread-local message retrievable with p2s_last_error().
 *   - Argument checks are synchronous and happen before any launch
 *     (P2S_ERR_INVALID_ARGUMENT).  Launch/driver failures -> P2S_ERR_CUDA.
 *   - "dev" pointers are CUDA device pointers on the plan's device, "host"
 *     pointers are ordinary host memory.  All arrays are dense, C order.
 *   - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Work is enqueued on it and the call returns without synchronising,
 *     except the *_host entry point, which synchronises before returning.
 *   - Ownership: the plan owns its device tables and workspace (allocated in
 *     p2s_plan_create, freed in p2s_plan_destroy).  The caller owns every buffer
 *     it passes and must keep it alive until the enqueued work completes.  Host
 *     arrays given to p2s_plan_create are copied.  No caller pointer is kept.
 *   - Concurrency: a plan serialises its own calls (shared workspace); use one
 *     plan per device/stream.  Plans on different devices are independent.
 *   - Noise is counter-based (Philox4x32-10 keyed by the 64-bit seed, counter by
 *     global frame index and spectral bin), so any frame range, batch split or
 *     GPU partition reproduces the same bits.
 *   - Kernel watchdog: the tensor-core kernels (MLP, blur) wait on mbarriers; a wait that
 *     has not completed after 4 s (a pipeline deadlock -- a library or hardware fault,
 *     never an input condition: every input is validated before launch) executes a trap
 *     rather than hanging the GPU.  A trap is a sticky CUDA error: the calling process's
 *     CUDA context is unusable afterwards (every later call, ours or the caller's,
 *     returns cudaErrorLaunchFailure / P2S_ERR_CUDA) and must be torn down.
 *   - The library reads no environment variables; kernel variants are chosen at plan
 *     creation (p2s_options.force pins them for tests and A/B runs).
 */
#ifndef P2S_H
#define P2S_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  P2S_OK = 0,
  P2S_ERR_INVALID_ARGUMENT = 1,
  P2S_ERR_NUMERIC = 2,       /* Cholesky of A_0 failed after regularisation */
  P2S_ERR_CUDA = 3,          /* launch / driver error */
  P2S_ERR_OUT_OF_MEMORY = 4, /* device or host allocation failed */
  P2S_ERR_UNSUPPORTED = 5    /* e.g. forced FFT grid that is not 5-smooth */
} p2s_status;

typedef struct p2s_plan_s* p2s_plan;

/* Optional settings; a zero-initialised struct (or NULL) selects defaults,
 * except `taps`, which is required (the basis is K x T x T). */
typedef struct {
  int    taps;              /* T: odd, 3 <= T <= 63, T/2 <= min(H,W)-1 (Q22)        */
  double aperture_m;        /* D in metres, default 0.1                              */
  double wavelength_m;      /* lambda, default 525e-9                                */
  double s_per_px;          /* lag per pixel in units of D; >0 overrides L*lambda/(2 D^2) (Q5) */
  double tilt_px_per_rad;   /* kappa_t pixels per unit a_2; >0 overrides 4/pi (Q12)  */
  int    pad;               /* FFT grid P x Q = next 5-smooth >= pad*(H,W); default 1 (Q6) */
  int    mlp_hidden[2];     /* hidden widths, default {100, 100}; each <= 256, and the
                               bf16 weight images must fit shared memory next to one
                               128-pixel tile (UNSUPPORTED otherwise; <= 128 always fits) */
  int    max_batch;         /* frames per internal chunk (workspace sizing); 0 = auto */
  float  ar_alpha;          /* AR(1) coefficient on the spectral noise in [0,1), default 0 (Q18) */
  float  noise_sigma;       /* step 5 additive Gaussian noise sigma, default 0       */
  int    normalize_psf_sum; /* step 5: divide by sum_k w_k sum_u h_k, default 0      */
  int    clamp01;           /* step 5: clamp output to [0,1], default 0             */
  int    device;            /* CUDA ordinal the plan is bound to; 0 = current device */
  float  flow_px_per_frame[2]; /* frozen flow: (vx, vy) pixels per
                              * frame; nonzero selects it: the fields of frame t are those of
                              * frame 0 of the sequence translated by t (vx, vy) on the periodic
                              * grid (exact sub-pixel shift in the spectral domain, Q23).
                              * The translation is periodic on the P x Q grid: frame
                              * t + P/|vy| (t + Q/|vx|) repeats frame t along that axis
                              * (512 px at 0.5 px/frame: every 1024 frames); use pad > 1 or
                              * shorter sequences for longer non-repeating flows.
                              * Exclusive with ar_alpha.  Default (0, 0). */
  int    slab_count;        /* G >= 2: the plan is rank slab_rank's share of ONE frame sharded
                               over G ranks (single-frame latency mode; see
                               p2s_slab_*).  0 or 1: a normal plan. */
  int    slab_rank;         /* 0 <= slab_rank < slab_count */
  unsigned int force;       /* kernel-selection overrides, P2S_FORCE_* bits; 0 = the production
                               dispatch.  For parity tests that pin one kernel variant against
                               another and for A/B measurements: every variant computes the
                               same result (up to rounding).  Read once, by p2s_plan_create; the
                               library reads no environment variables. */
} p2s_options;

/* p2s_options.force bits */
#define P2S_FORCE_FFT_GENERIC     0x001u /* generic shared-memory Stockham even at 512 points  */
#define P2S_FORCE_FFT_SMALL_RADIX 0x002u /* radices <= 8 only (no composite 9..16 butterflies) */
#define P2S_FORCE_AR_ROW_KERNEL   0x004u /* AR(1): one CTA per spectral row (k_rows_ar)        */
#define P2S_FORCE_AR_PAIR_KERNEL  0x008u /* AR(1): Hermitian row-pair CTAs (k_rows_ar_pair)    */
#define P2S_FORCE_ROWS_PINGPONG   0x010u /* long rows: ping-pong buffers, not in place         */
#define P2S_FORCE_COLS_PER_BLOCK  0x020u /* long columns: one CTA per block, not persistent    */
#define P2S_FORCE_X_PLANES        0x040u /* MLP inputs as [F][slot][H*W] planes                */
#define P2S_FORCE_X_TILES         0x080u /* MLP inputs tile-major [F][H][ntx][slot][128]       */
#define P2S_FORCE_WARP_FUSION     0x100u /* step 2 inside the 512-point column kernel          */
#define P2S_FORCE_BLUR_SINGLE     0x200u /* blur on single CTAs (cta_group::1), not CTA pairs  */
#define P2S_FORCE_COLS_PERSISTENT 0x400u /* long columns: persistent one-CTA-per-SM kernel     */
#define P2S_FORCE_WARP_GATHER     0x800u /* step 2 gathering from global memory, no TMA window  */
#define P2S_FORCE_X_OCTETS        0x1000u /* MLP inputs [F][H][ntx][slot/2][16][2][8 px]       */
#define P2S_FORCE_MLP_A1_THREADS  0x2000u /* MLP inputs loaded by per-thread copies, no TMA box */

/* Build a plan (P:312-330 generation setup; runs once, off the per-frame clock).
 *   H, W        image size in pixels (>= T, <= 8192)
 *   C           channels, 1..4 (channels share field, warp and weights, Q17)
 *   d_over_r0   D/r0 >= 0 (0 = diffraction limited: A_0 = 0, L = 0)
 *   L_m         propagation path length in metres (> 0), sets s_px (Q5)
 *   Z           number of Noll modes N ("we set N = 36"); 4 <= Z <= 66
 *   K           number of PSF basis functions M; 1 <= K <= 128
 *   basis       host float [K][T][T], h_k on the tap grid, centre tap T/2 (copied)
 *   mlp_weights host float, packed row-major [out][in]:
 *                 W1[h1][Z-3], b1[h1], W2[h2][h1], b2[h2], W3[K][h2], b3[K]  (copied)
 *   opt         nullable; see p2s_options.
 * Computes A_0 (Noll's closed form), L = chol(A_0[2..Z]) in fp64, the
 * auto-correlation kernels c_j on the periodic lag grid, S_j = DFT(c_j) clamped
 * at 0 and renormalised to sum S_j = PQ (Q7), sqrt(S_j), and the packed bf16
 * tensor-core images of the MLP (with L folded into layer 1) and of the basis.
 * Errors: INVALID_ARGUMENT, NUMERIC, CUDA, OUT_OF_MEMORY, UNSUPPORTED. */
p2s_status p2s_plan_create(p2s_plan* out, int H, int W, int C, double d_over_r0, double L_m,
                           int Z, int K, const float* basis, const float* mlp_weights,
                           const p2s_options* opt);

/* Free every device and host resource of the plan (synchronises its device). */
p2s_status p2s_plan_destroy(p2s_plan p);

/* Step 1: zern (dev float [nframes][Z][H][W]) <- a for frames frame0..frame0+nframes-1 of
 * sequence `seed`.  Plane 0 (piston) is 0; plane j-1 holds Noll mode j.
 * With ar_alpha != 0 the spectral noise follows eta_t = alpha eta_{t-1} +
 * sqrt(1-alpha^2) xi_t from t = 0 (replayed on the device when frame0 does not
 * continue the previous call).  With frozen flow, frame t is the translation of frame 0
 * (stateless: any frame range, any batch split). */
p2s_status p2s_sample_zernike(p2s_plan p, uint64_t seed, int64_t frame0, int nframes,
                              float* zern, void* stream);

/* Step 1 from caller-supplied spectral noise (parity entry: identical host-generated noise
 * on both sides, BASELINE north_star).  eta: device complex64 (float2) [nframes][Z-1][P][Q]
 * (P x Q = the plan's FFT grid, p2s_plan_info), mode slot m <-> Noll j = m + 2: the
 * Hermitian spectral noise of reading Q8 (canonical bin sqrt(PQ/2)(g1 + i g2), mirror bin
 * its conjugate, self-conjugate bins sqrt(PQ) g1).  Runs Y = sqrt(S_a) eta_a + i sqrt(S_b)
 * eta_b, the 2-D inverse DFT, the crop and the mixing a = L f exactly like
 * p2s_sample_zernike (each bin read as stored; no AR state, no frozen flow) into
 * zern (device float [nframes][Z][H][W]).  Spectra that are not Hermitian are not rejected
 * (checking would cost a pass): the result is then still f_a = Re y, f_b = Im y of the same
 * inverse DFT, mixed -- well defined, but no longer two independent real fields. */
p2s_status p2s_sample_zernike_from_noise(p2s_plan p, const float* eta, int nframes, float* zern, void* stream);

/* Step 2: warped (dev float [nframes][C][H][W]) <- bilinear(img, x + kappa (a_2, a_3)).
 *   img              dev float [..][C][H][W]; frame i uses img + i*img_frame_stride
 *                    (in floats; 0 = one image broadcast to all frames)
 *   zern             dev float [nframes][Z][H][W] as written by p2s_sample_zernike */
p2s_status p2s_warp(p2s_plan p, const float* img, int64_t img_frame_stride, const float* zern,
                    float* warped, int nframes, void* stream);

/* Steps 3-5: out (dev float [nframes][C][H][W]) <- step5(sum_k w_k(x) (h_k (*) warped_c)(x)),
 * w = MLP(a_4..a_Z) from zern (dev float [nframes][Z][H][W]).  seed/frame0 key the
 * step-5 noise (Philox stream 1). */
p2s_status p2s_blur(p2s_plan p, const float* warped, const float* zern, uint64_t seed,
                    int64_t frame0, float* out, int nframes, void* stream);

/* Steps 4-5 with caller-supplied basis weights instead of the MLP (e.g. the exact
 * projection of each pixel's PSF on the basis, NEXT-1):
 *   out (dev float [nframes][C][H][W]) <- step5(sum_k weights_k(x) (h_k (*) warped_c)(x)).
 *   weights: dev float [nframes][K][H][W] (the plan's K). */
p2s_status p2s_blur_weights(p2s_plan p, const float* warped, const float* weights, uint64_t seed,
                            int64_t frame0, float* out, int nframes, void* stream);

/* Steps 1-5 fused: out (dev float [nframes][C][H][W]) for frames frame0.. of sequence seed.
 * img as in p2s_warp.  Equivalent to sample_zernike -> warp -> blur up to rounding
 * (L is folded into the MLP's first layer; tensor-core stages run in bf16 with
 * fp32 accumulation). */
p2s_status p2s_simulate_frames(p2s_plan p, const float* img, int64_t img_frame_stride, uint64_t seed,
                               int64_t frame0, int nframes, float* out, void* stream);

/* Same as p2s_simulate_frames with HOST buffers: img_host [..][C][H][W] (stride as above),
 * out_host [nframes][C][H][W].  Copies in, runs, copies out, synchronises.  Internally the
 * frames run as tapered sub-batches on `stream` while a second (plan-owned) stream uploads
 * the images and downloads each finished sub-batch; pinned host memory gives full PCIe
 * overlap.  The image upload overlaps step 1 (only the warp waits for it), and a one-frame
 * last sub-batch runs its blur in two row-band halves so the top half's download overlaps
 * the bottom half.  Results are bit-identical to p2s_simulate_frames. */
p2s_status p2s_simulate_frames_host(p2s_plan p, const float* img_host, int64_t img_frame_stride,
                                    uint64_t seed, int64_t frame0, int nframes, float* out_host,
                                    void* stream);

/* Thread-local message describing the last failure on this thread ("" if none). */
const char* p2s_last_error(void);

/* ---- introspection / test support (not on the hot path) ---- */

/* FFT grid P x Q, workspace bytes for max_batch frames, max clamped-PSD fraction over modes.
 * Any output pointer may be NULL. */
p2s_status p2s_plan_info(p2s_plan p, int* P, int* Q, size_t* workspace_bytes,
                         double* clamped_psd_fraction, int* max_batch);

/* Copy plan tables to host (each pointer nullable):
 *   A0    double [Z][Z]    Noll matrix (piston row/col 0)
 *   chol  double [Z][Z]    lower-triangular L, L L^T = A0
 *   sqrtS float  [Z-1][P][Q] sqrt(S_j) for j = 2..Z (sum S_j = P*Q) */
p2s_status p2s_plan_export_tables(p2s_plan p, double* A0, double* chol, float* sqrtS);

/* Per-stage device timing of the fused path (measurement support).
 * p2s_plan_stage_timing(p, 1) starts recording a CUDA event pair around every kernel
 * launch that p2s_simulate_frames enqueues (on the caller's stream) and clears the
 * accumulators; 0 stops.  p2s_plan_stage_times synchronises on the recorded events and
 * returns, per stage, the summed kernel time in ms and the number of launches:
 * index 0 k_rows (noise+PSD+row IDFT), 1 k_cols (column IDFT), 2 k_warp, 3 k_mlp,
 * 4 k_blur.  ms and launches are arrays of length 5 (nullable). */
p2s_status p2s_plan_stage_timing(p2s_plan p, int enable);
p2s_status p2s_plan_stage_times(p2s_plan p, double* ms, int64_t* launches);

/* Replace the plan's sqrt(S_j) (host float [Z-1][P][Q], same layout as export). */
p2s_status p2s_plan_import_sqrtS(p2s_plan p, const float* sqrtS);

/* Validation battery: empirical spatial auto-correlation of sampled
 * Zernike coefficient fields, the statistic the sampler is built to reproduce (homogeneous
 * A_jj(s); mixed model E[a_j(x) a_j(x+s)] = sum_k L_jk^2 c_k(s), Eq.10
 * P:318-330; tilt j = 2, 3 and the differential tilt variance 2(A_22(0) - A_22(s)),
 * P:523-532).
 *   zern  : device float [nframes][Z][H][W] (the p2s_sample_zernike layout of this plan).
 *   out   : device double [Z][2][max_lag]; out[j][0][l] = mean a_j(y,x) a_j(y,(x+l) mod W),
 *           out[j][1][l] = mean a_j(y,x) a_j((y+l) mod H,x), over all frames and pixels
 *           (periodic lags: the fields are periodic when the FFT grid equals the image).
 *   max_lag in [1, 64].  Stream-ordered; a temporary partial-sum buffer is allocated and
 *   freed on the stream.  Errors: P2S_ERR_INVALID_ARGUMENT for bad sizes / NULL. */
p2s_status p2s_field_autocorr(p2s_plan p, const float* zern, int nframes, int max_lag, double* out, void* stream);

/* Validation battery: aperture statistics of the sampled Zernike
 * vectors -- the phase structure function (Fig. struct_fun, against Eq.4) and the
 * long/short-exposure OTFs H_LE = E[H], H_SE = E[H] of the tilt-corrected phase, H the
 * pupil autocorrelation.  Pupil: the 32-sample disc of reading Q24.  Every
 * (frame, pixel) pair is one sample: phi = sum_j a_j Z_j, its residual after the
 * least-squares plane over the disc, and per lag xi = (dy, dx), dy in [0, 32),
 * dx in [-31, 31], Delta = phi(x) - phi(x + xi), M the disc mask:
 *   out[0][dy][dx+31] = mean over samples of sum_x M M' Delta^2 / sum_x M M'  (0 if no overlap)
 *   out[1][dy][dx+31] = mean of sum_x M M' cos(Delta) / sum_x M         (Re H / H(0), LE)
 *   out[2][dy][dx+31] = the same for the plane residual                  (SE)
 *   zern   : device float [nframes][Z][H][W] (the p2s_sample_zernike layout), Z <= 72.
 *   pixels : device int32 [npix] pixel indices y*W + x used in every frame.
 *   out    : device double [3][32][63].
 * Stream-ordered; a temporary partial-sum buffer is allocated and freed on the stream.
 * Per-sample sums in fp32, across samples in fp64, deterministic.  Errors:
 * P2S_ERR_INVALID_ARGUMENT for NULL / nframes < 1 / npix < 1. */
p2s_status p2s_aperture_stats(p2s_plan p, const float* zern, int nframes, const int32_t* pixels, int npix,
                              double* out, void* stream);

/* Exact-PSF path: the slow per-pixel reference that P2S
 * replaces.  Eq.2: h_x(u) = |F{P e^{-j phi_x}}|^2 with phi_x = sum_j a_j(x) Z_j on
 * a 32-sample pupil zero-padded to a 64-point FFT (PSF pixel = lambda/(2D): a pure tilt moves
 * the PSF by 4 a_2/pi px, reading Q24), T x T window (the plan's taps), unit sum.
 *   zern   : device float [Z][H][W], ONE frame in the p2s_sample_zernike layout.
 *   pixels : device int32 [n] pixel indices y*W + x.
 *   include_tilt: 0 drops a_2, a_3 from the phase (the higher-order PSF that P2S maps).
 *   out    : device float [n][T][T], tap (T/2 + uy, T/2 + ux) = h(uy, ux).
 * Errors: INVALID_ARGUMENT (NULL, n < 1), CUDA. */
p2s_status p2s_exact_psf(p2s_plan p, const float* zern, const int32_t* pixels, int n, int include_tilt,
                         float* out, void* stream);

/* Eq.1 gather render of one frame with the exact per-pixel PSFs:
 * out_c(x) = sum_u h_x(u) img_c(x - u) (true convolution, whole-sample mirror boundary).
 *   img: device float [C][H][W]; zern: device float [Z][H][W]; out: device float [C][H][W]. */
p2s_status p2s_render_exact(p2s_plan p, const float* img, const float* zern, int include_tilt, float* out,
                            void* stream);

/* Host-only: PSF basis by principal components (Eq.7; NEXT-1 part).
 *   psfs  : host float [n][T*T] PSF database (e.g. p2s_exact_psf at sampled pixels).
 *   basis : host float [M+1][T*T] out: row 0 the mean PSF, rows 1..M the M leading principal
 *           components (unit L2 norm, ordered by variance, largest entry positive).
 *   residual: optional out, fraction of the centred database energy the M components miss.
 * fp64 covariance, block iteration + Rayleigh-Ritz.  Errors: INVALID_ARGUMENT. */
p2s_status p2s_fit_basis(const float* psfs, int n, int T, int M, float* basis, double* residual);

/* Host-only: fit the output layer of the P2S network (NEXT-1 readout training).  Keeps W1,
 * b1, W2, b2 of the packed MLP `mlp_in` (p2s_plan_create layout, input n_in, hidden h1, h2,
 * output K) and solves (W3, b3) by ridge regression (lambda on W3 only) from the second
 * hidden layer's activations at the inputs a (host float [n][n_in], Zernike a_4..a_Z) to the
 * target basis weights beta (host float [n][K], e.g. projections of exact PSFs on the basis).
 *   mlp_out: host float, packed like mlp_in.  rel_residual: optional ||X Theta - beta||/||beta||.
 * Errors: INVALID_ARGUMENT, NUMERIC (singular normal equations). */
p2s_status p2s_fit_readout(const float* mlp_in, int n_in, int h1, int h2, int K, const float* a,
                           const float* beta, int n, double lambda, float* mlp_out, double* rel_residual);

/* P2S network training ("train a small neural network to convert
 * the Zernike coefficients ... to the PSF coefficients"), host fp64.  Reading Q26: loss
 * L = 1/(B K) sum_i sum_k (y_ik - beta_ik)^2 over each mini-batch, Adam (beta1 = 0.9,
 * beta2 = 0.999, eps = 1e-8, bias-corrected), one update per mini-batch; relu'(0) = 0.
 *   mlp_in  : host float packed [W1 (h1 x n_in), b1, W2 (h2 x h1), b2, W3 (K x h2), b3]
 *             (the initial weights, e.g. after p2s_fit_readout).
 *   a, beta : host float [n][n_in] inputs, [n][K] targets.
 *   order   : host int32 [epochs][n] sample order of each epoch; mini-batches are its
 *             consecutive chunks of `batch` samples (the last may be shorter).
 *   mlp_out : host float, same layout (may alias nothing; caller-owned).
 *   loss_curve: host double [epochs] (nullable): per epoch, the sample-weighted mean of the
 *             batch losses evaluated before each update.
 * Errors: P2S_ERR_INVALID_ARGUMENT for sizes < 1, lr <= 0, NULL or out-of-range order. */
p2s_status p2s_train_mlp(const float* mlp_in, int n_in, int h1, int h2, int K, const float* a,
                         const float* beta, int n, const int32_t* order, int epochs, int batch, double lr,
                         float* mlp_out, double* loss_curve);

/* Validation battery: approximation energies of P:369-397, host fp64.
 * A_ij(s, phi) = E[a_i(x) a_j(x+s)] of the single-screen model (Hankel form of P:234-238
 * generalised to i != j), A~ = L diag(c_k) L^T the block-diagonal model of Eq.10 with
 * c_k = A_kk / A_kk(0).  On the grid s_i = s_max i / ns, ns = max(2, round(n_per_unit s_max)):
 *   E[i]  = Int_0^{s_i} Int_0^{2pi} tr(A^T A) s' dphi ds'      (modes mode_lo..Z)
 *   Et[i] = the same with A~,   Em[i] = the same with |tr(A^T A - A~^T A~)|,
 * radial integral by the cumulative trapezoid.  angle_mean = 0: the printed formulas (the
 * angular integral as the exact mean over 32 uniform angles); 1: reading Q25 (functions
 * averaged over the angle before squaring).  s in units of D; D/r0 sets the scale.
 * Outputs: s_out, E, Et, Em host double [ns+1] (caller-owned).  Errors:
 * P2S_ERR_INVALID_ARGUMENT for Z outside [4, 66], mode_lo outside [2, Z], s_max <= 0,
 * n_per_unit < 1 or NULL outputs. */
p2s_status p2s_correlation_energies(int Z, double d_over_r0, double s_max, int n_per_unit, int angle_mean,
                                    int mode_lo, double* s_out, double* E, double* Et, double* Em);

/* Device Philox4x32-10 test fill: out (dev uint32 [n][4]) <- philox(counter =
 * (i, c1, c2, c3), key = (k0, k1)) for i = 0..n-1. */
p2s_status p2s_philox_fill(uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1,
                           int64_t n, uint32_t* out, void* stream);

/* Host-only (no GPU needed): plan tables for the given geometry, for CPU tests.
 *   A0, chol: double [Z][Z]; sqrtS: double [Z-1][P][Q] with P, Q from p2s_grid_size;
 *   clamped: double [Z-1] negative-PSD mass fraction per mode. Any output nullable. */
p2s_status p2s_host_tables(int P, int Q, double s_per_px, double d_over_r0, int Z,
                           double* A0, double* chol, double* sqrtS, double* clamped);

/* Smallest 5-smooth n >= x (the FFT grid rule of p2s_plan_create). */
int p2s_grid_size(int x);

/* ---------------------------------------------------------------------------------------
 * Single-frame latency mode: one frame sharded over G ranks -- for
 * the large-frame case where one frame's latency matters (the paper's 3840x2160 frame,
 * "about 60 seconds per frame" with split-step).
 * Step 1's first pass (noise + PSD + row IDFT) is split by Hermitian spectral
 * row pairs {ky, P-ky}: rank r transforms pairs kp in [kp0, kp1).  The second pass needs
 * whole columns, so the row-transformed spectrum is transposed across ranks by one
 * all-to-all (the caller's collective, e.g. NCCL all_to_all_single): rank r then owns the
 * output column strip [x0, x1) of the frame plus a halo of T/2 columns each side (clipped
 * at the frame edges), runs the column pass, the warp, the MLP and the blur on that strip
 * and returns the strip [x0, x1).  The strips of all ranks tile the frame and are
 * bit-identical to p2s_simulate_frames of the unsharded frame (same kernels, same
 * per-pixel and per-bin arithmetic; the halo makes the mirror boundary exact).
 * The plan is created with opt->slab_count = G >= 2, opt->slab_rank = r and the GLOBAL
 * H, W; max_batch is 1.  White noise, frozen flow and AR(1) sequences (each rank keeps
 * the AR state of its own spectral rows; a frame that does not continue the rank's previous
 * call is replayed from frame 0, as in p2s_sample_zernike).
 *
 * Exchange buffers (dev float, complex values as interleaved pairs):
 *   send [G dest][rows_r][npairs][Ws(dest)] x 2 floats, recv [G src][rows_src][npairs][Ws(r)]
 *   x 2 floats, rows_r = spectral rows of rank r, Ws(d) = x-halo strip width of rank d,
 *   npairs = (Z-1+1)/2.  p2s_slab_counts gives the per-peer float counts (the split sizes
 *   of an all_to_all_single). */

/* Geometry of rank `rank` of G for a frame H x W with T taps (host only, no GPU):
 * info[0..8] = x0, x1, hx0, hx1, kp0, kp1, rows, P, Q. */
p2s_status p2s_slab_geometry(int H, int W, int T, int pad, int G, int rank, int64_t* info);

/* Per-peer float counts of this plan's rank: send_counts[d] (to rank d), recv_counts[s]
 * (from rank s); either pointer nullable.  Host arrays of G int64. */
p2s_status p2s_slab_counts(p2s_plan p, int64_t* send_counts, int64_t* recv_counts);

/* Phase 1 (rank r): spectral noise, PSD and the row IDFT of this rank's row pairs for frame
 * `frame` of sequence `seed`, packed into send (see above).  Enqueued on stream. */
p2s_status p2s_slab_rows(p2s_plan p, uint64_t seed, int64_t frame, float* send, void* stream);

/* Phase 2 (rank r), after the all-to-all delivered recv: column IDFT of the halo strip,
 * warp (gathering from the whole image img, dev float [C][H][W]), MLP, Eq.9 blur and step 5;
 * out_strip (dev float [C][H][x1-x0]) <- the rank's output columns [x0, x1). */
p2s_status p2s_slab_finish(p2s_plan p, const float* recv, const float* img, uint64_t seed, int64_t frame,
                           float* out_strip, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* P2S_H */
