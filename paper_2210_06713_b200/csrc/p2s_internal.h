// p2s_internal.h -- private declarations shared by the host plan code and the kernels.
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "../../include/p2s.h"

#include <cuda.h>
#include <cuda_runtime.h>

namespace p2s {

p2s_status set_error(p2s_status st, const std::string& msg);

// ---- plan math (plan_math.cpp, host fp64) ----
double kolmogorov_cd();
double kolmogorov_cw();
double noll_constant();
void noll_nm(int j, int* n, int* m, int* kind);
void noll_matrix(int Z, double d_over_r0, std::vector<double>& A);
bool noll_cholesky(int Z, const std::vector<double>& A, std::vector<double>& L);
void bessel_j_all(double x, int nmax, double* J);
void psd_tables(int P, int Q, double s_px, int Z, std::vector<double>& sqrtS, std::vector<double>& clamped);
int grid_size(int x);
double zernike_value(int j, double rho, double theta);

constexpr int kMaxRadix = 24;

// Inverse-DFT plan for one axis: radix list and e^{+2 pi i k/N} table (device).
struct AxisFFT {
  int N = 0;
  int nrad = 0;
  int rad[kMaxRadix] = {0};
  float2* tw = nullptr;  // device [N]
};

// MLP geometry (all padded sizes are multiples of 16).
struct MlpGeom {
  int nin = 0;   // real inputs
  int k1 = 0;    // padded layer-1 K
  int n1 = 0, n2 = 0, n3 = 0;  // padded widths (n3 = padded K bases)
  int kout = 0;  // real K
  bool bias_folded = false;  // biases carried by a constant-1 unit inside the GEMMs
  size_t blob_bytes = 0;  // W1img | W2img | W3img | b1 | b2 | b3
  size_t off_w2 = 0, off_w3 = 0, off_b1 = 0, off_b2 = 0, off_b3 = 0;
};

// Blur geometry: K-step schedule of the tap-row groups (see k_blur.cu).
// K-steps (B tiles) moved per blur ring stage (the pair-mode B tensor-map box spans one stage).
#ifndef P2S_KSPS
#define P2S_KSPS 7
#endif
constexpr int kBlurStepsPerStage = P2S_KSPS;
// Height (in 16-byte rows) of one chunk column of the blur's source tile: RS rounded up to
// odd, so that the 16-byte stores of consecutive chunk columns fall in different banks.
#ifdef __CUDACC__
__host__ __device__
#endif
inline constexpr int blur_rs_pad(int RS) { return RS | 1; }
// bytes of one channel's column-ordered source tile (NC chunk columns x padded RS rows)
#ifdef __CUDACC__
__host__ __device__
#endif
inline constexpr uint32_t blur_main_bytes(int NC, int RS) { return ((uint32_t)NC * blur_rs_pad(RS) * 16 + 127) & ~127u; }
constexpr int kBlurTSlots = 2;  // ring of transposed-row slots (leftover tap rows)
// Tap-row grouping of the blur: g8 groups of 8 tap rows per tap column and lr leftover tap
// rows run along the tap columns on transposed source rows (lr = T % 8 when it is at most
// 3; with more leftover rows the transposed copies cost more shared memory than the
// padded 8-row group they replace, so the last group is padded instead: lr = 0).
inline void blur_tap_split(int T, int* g8, int* lr) {
  if (T % 8 <= 3) {
    *g8 = T / 8;
    *lr = T % 8;
  } else {
    *g8 = (T + 7) / 8;
    *lr = 0;
  }
}
// Source rows a tile needs for RB output rows.
inline int blur_tile_rows(int RB, int T, int g8, int lr) { return lr ? RB + T - 1 : RB + 8 * g8; }

struct BlurGeom {
  int T = 0, c = 0;        // taps, centre
  int NC = 0;              // source chunks = T + 15
  int RB = 32;             // output rows per CTA
  int racc = 4;            // output rows per accumulator group (C * racc <= 4 accumulators)
  bool pair = false;       // CTA pairs with tcgen05 cta_group::2 (M = 256)
  int stages = 8;          // B ring depth (stages of 2 K-steps)
  int RS = 0;              // source rows held in smem
  int nks = 0;             // number of K-steps
  int nks_main = 0;        // K-steps over 8-row tap groups (the rest run along transposed rows)
  int g8 = 0;              // full 8-row tap groups per tap column (T / 8)
  int lr = 0;              // leftover tap rows (T % 8), run along the tap columns
  int nct = 0;             // chunks per transposed row (>= NC)
  int np = 0;              // padded N (= MlpGeom.n3)
  uint32_t* koff = nullptr;  // device [nks]: byte offset of group a relative to (src + yl*16)
  uint32_t* klbo = nullptr;  // device [nks]: LBO (group b - group a) in bytes
  uint8_t* bimg = nullptr;   // device [nks][np*32 bytes] B tiles (K-major, no swizzle)
  uint8_t* bimg2 = nullptr;  // device [2 halves][nks][np*16 bytes] (pair mode)
  float* hsum = nullptr;     // device [np] per-basis tap sum (normalisation)
  uint64_t* adesc = nullptr;  // device [nks]: A descriptor per K-step relative to tile base 0
  int brep = 1;              // copies of the B image in HBM (spreads the L2 hot spot)
  size_t bstride = 0;        // bytes between copies of bimg
  int brows = 0;             // 256-byte rows between copies of bimg2 (tmap_b coordinate)
};

}  // namespace p2s

struct p2s_plan_s {
  int H = 0, W = 0, C = 0, Z = 0, K = 0, T = 0, P = 0, Q = 0;
  int nslots = 0, npairs = 0, h1 = 0, h2 = 0;
  double d_over_r0 = 0, L_m = 0, s_px = 0, kappa = 0;
  float ar_alpha = 0, noise_sigma = 0;
  double flow_vx = 0, flow_vy = 0;  // frozen flow, pixels per frame (0 = off)
  int normalize = 0, clamp01 = 0, device = 0, max_batch = 0;
  unsigned force = 0;           // p2s_options.force (P2S_FORCE_* bits), fixed at plan creation
  // single-frame slab mode (NEXT-4; slab_G > 1): this rank's geometry.  W above is then the
  // rank's x-halo strip width (steps 1b-5 run on the strip), W_glob the frame's width.
  int slab_G = 1, slab_r = 0, W_glob = 0;
  int slab_x0 = 0, slab_x1 = 0, slab_hx0 = 0, slab_kp0 = 0, slab_kp1 = 0, slab_rows = 0;
  int* d_slab_ky = nullptr;     // device: [rows_r] this rank's rows (pack) | [P] rows in recv order (unpack)
  int* d_slab_dest = nullptr;   // device: [G][3] per destination: hx0, width, float2 offset of its block
  std::vector<int64_t> slab_send, slab_recv;  // per-peer float counts
  int xtile = 0;                // MLP input layout, fixed at plan creation (1: tile-major, x_index)
  double clamped_max = 0;
  std::vector<double> A0, Lc;      // Z x Z
  std::vector<float> sqrtS_host;   // [nslots][P][Q]
  std::vector<float> basis_host;   // [K][T][T]
  std::vector<float> mlp_host;     // packed
  // device tables
  float2* d_sqrtS = nullptr;    // [npairs][P][Q] scaled (sa, sb)
  float4* d_ar = nullptr;       // [npairs][P][Q] AR(1) state (zeta_a, zeta_b)
  float* d_ztab = nullptr;      // exact-PSF pupil table [Z][32*32] (lazy, NEXT-1)
  float* d_L = nullptr;         // [(Z-1)*(Z-1)] float L[2..Z][2..Z]
  uint8_t* d_mlp_fold = nullptr;   // L folded into layer 1 (inputs f_2..f_Z)
  uint8_t* d_mlp_plain = nullptr;  // plain layer 1 (inputs a_4..a_Z)
  p2s::MlpGeom mg_fold, mg_plain;
  p2s::BlurGeom bg;
  p2s::AxisFFT fq, fp;
  // workspace (max_batch frames)
  void* d_ws = nullptr;
  size_t ws_bytes = 0;
  float2* d_Z = nullptr;        // [mb][npairs][P][Q]
  uint16_t* d_X = nullptr;      // bf16 MLP inputs, nin = nslots (simulate) or Z-3 (blur API) values per
                                // pixel: planes [mb][nin][H*W], or (xtile) tile-major
                                // [mb][H][ntx][nin][128 px] (x_index in p2s_dev.cuh)
  float* d_tilt = nullptr;      // [mb][2][H*W]
  uint16_t* d_Iw = nullptr;     // bf16 [mb][C][H][W]
  uint16_t* d_w = nullptr;      // bf16 [mb][H][ntx][n3/8][128 px][8]: per 128-pixel row tile, 8-basis chunks
  int ntx = 0;                  // 128-pixel tiles per image row
  int nsm = 148;                // SMs of the plan's device (blur wave accounting)
  std::map<int, std::vector<int>> host_sched;  // p2s_simulate_frames_host sub-batch plan per batch size
  CUtensorMap tmap_b;           // 2-D TMA view of bg.bimg2: rows of 256 B, box 2 K-steps of one half
  float* d_img = nullptr;       // staging for the host entry point [mb][C][H][W]
  float* d_out = nullptr;       // staging for the host entry point [mb][C][H][W]
  // per-stage timing (p2s_plan_stage_timing)
  bool timing = false;
  std::vector<int> t_stage;
  std::vector<cudaEvent_t> t_ev;  // pairs
  cudaStream_t copy_stream = nullptr;  // host entry: device->host copies overlapped with compute
  cudaEvent_t ev_sub = nullptr, ev_copied = nullptr, ev_img = nullptr, ev_half = nullptr;
  // AR bookkeeping
  bool ar_valid = false;
  uint64_t ar_seed = 0;
  int64_t ar_next = 0;
  int num_sms = 148;
};

// Dynamic shared memory above the default 48 KB needs an opt-in per kernel; its failure
// (a request above the 227 KB per-CTA limit) is returned, never ignored.
#define P2S_SMEM_OPTIN(kern, bytes)                                                               \
  do {                                                                                          \
    cudaError_t e_ = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes)); \
    if (e_ != cudaSuccess) return (int)e_;                                                      \
  } while (0)

namespace p2s {
// ---- kernel launchers (k_*.cu); all return cudaGetLastError() as int ----
int launch_rows(const p2s_plan_s* p, uint64_t seed, int64_t frame0, int F, bool ar, int ar_mode,
                int64_t replay_from, cudaStream_t s, const float2* eta = nullptr);
int launch_cols(const p2s_plan_s* p, int F, int mode, float* zern, cudaStream_t s, const float* img = nullptr,
                int64_t img_stride = 0, bool* warp_fused = nullptr);
int launch_mix(const p2s_plan_s* p, int F, float* zern, cudaStream_t s);
int launch_zern_to_x(const p2s_plan_s* p, int F, const float* zern, cudaStream_t s);
int launch_warp_f32(const p2s_plan_s* p, int F, const float* img, int64_t stride, const float* zern, float* out,
                    cudaStream_t s);
int launch_warp_sim(const p2s_plan_s* p, int F, const float* img, int64_t stride, cudaStream_t s);
int launch_slab_pack(const p2s_plan_s* p, float2* send, cudaStream_t s);
int launch_slab_unpack(const p2s_plan_s* p, const float2* recv, cudaStream_t s);
struct SlabGeom {
  int x0, x1, hx0, hx1, kp0, kp1, rows;
};
SlabGeom slab_geometry(int W, int T, int P, int G, int r);
int launch_mlp(const p2s_plan_s* p, int F, bool folded, cudaStream_t s);
size_t rows_smem_bytes(const p2s_plan_s* p, bool ar, bool given_noise);  // row pass dynamic smem
int x_tile_layout(const p2s_plan_s* p);  // decided at plan creation; 1: MLP input X tile-major (x_index)
int launch_pack_weights(const p2s_plan_s* p, int F, const float* wts, cudaStream_t s);
int launch_blur(const p2s_plan_s* p, int F, const void* src, bool src_f32, uint64_t seed, int64_t frame0,
                float* out, cudaStream_t s, int band0 = 0, int nbands = -1);  // row bands [band0, band0 + nbands)
bool cols_fuse_warp(const p2s_plan_s* p);  // step 2 runs inside the simulate path's column kernel
int blur_rows_per_cta(int C, int T, int np, int racc, int H, int W, bool pair, int stages, int F, int nsm);
int blur_waves(const p2s_plan_s* p, int F);
size_t acorr_partial_bytes(int F, int Z, int W, int L);
int launch_acorr(const float* zern, int F, int Z, int H, int W, int L, double* partial, double* out, cudaStream_t s);
int ensure_pupil_table(p2s_plan_s* p);
size_t aperture_partial_bytes(int64_t nsamples);
int launch_aperture(const p2s_plan_s* p, const float* zern, int nframes, const int* pix, int npix, double* partial,
                    double* out, cudaStream_t s);
int launch_exact_psf(const p2s_plan_s* p, const float* zern, const int* pix, int n, int include_tilt, float* out,
                     cudaStream_t s);
int launch_render_exact(const p2s_plan_s* p, const float* img, const float* zern, int include_tilt, float* out,
                        cudaStream_t s);
int launch_philox_fill(uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1, int64_t n, uint32_t* out,
                       cudaStream_t s);
}  // namespace p2s
