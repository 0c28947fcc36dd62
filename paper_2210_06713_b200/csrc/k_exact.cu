// k_exact.cu -- exact-PSF path (partial): Eq.2 PSF synthesis and the
// Eq.1 gather render, the slow per-pixel reference the P2S approximation replaces.
//
// Eq.2: h_x(u) = |F{P(xi) e^{-j phi_x(xi)}}|^2, phi_x = sum_j a_j(x) Z_j(xi).
// Reading Q24 (the paper withholds the sampling constants): 32 pupil samples across the
// aperture, zero-padded to a 64-point FFT (padding 2: one PSF pixel = lambda/(2D), the
// image's Nyquist IFOV of reading Q5, so a pure tilt moves the PSF by 4 a_2 / pi pixels, the
// warp constant of Q12), T x T displacement window, unit sum.  Eq.1: each output
// pixel is the true convolution of its own PSF with the input neighbourhood (whole-sample
// mirror boundary, as the blur).
//
// One 512-thread CTA per pixel: the pupil phase from a Zernike table (sum over modes), the
// field e^{-j phi} on the disk into a padded 64 x 64 shared-memory grid, 64-point radix-8
// Stockham passes along rows then columns (one butterfly per thread per pass), |.|^2 over
// the T x T window, block reduction for the normalisation; the render CTA then forms the
// C dot products of the window with the image.
#include "p2s_dev.cuh"
#include "p2s_internal.h"

#include <cmath>

namespace p2s {

constexpr int kPupD = 32;     // pupil samples across the aperture diameter
constexpr int kPsfN = 64;     // FFT size (padding 2)
constexpr int kPsfLd = 65;    // padded row pitch of the shared-memory grid (float2)

// 8-point inverse DFT (e^{+2 pi i}); the forward transform of Eq.2 is recovered by reading
// the result at -k (|F(-k)|^2 of the inverse equals |F(k)|^2 of the forward transform).
__device__ __forceinline__ void idft8(float2* v) {
  float2 e[4] = {v[0], v[2], v[4], v[6]};
  float2 o[4] = {v[1], v[3], v[5], v[7]};
  auto dft4 = [](float2* q) {
    float2 a = q[0], b = q[1], c = q[2], d = q[3];
    float2 s0 = make_float2(a.x + c.x, a.y + c.y), s1 = make_float2(a.x - c.x, a.y - c.y);
    float2 s2 = make_float2(b.x + d.x, b.y + d.y), s3 = make_float2(b.x - d.x, b.y - d.y);
    q[0] = make_float2(s0.x + s2.x, s0.y + s2.y);
    q[2] = make_float2(s0.x - s2.x, s0.y - s2.y);
    q[1] = make_float2(s1.x - s3.y, s1.y + s3.x);
    q[3] = make_float2(s1.x + s3.y, s1.y - s3.x);
  };
  dft4(e);
  dft4(o);
  const float r = 0.70710678118654752f;
  float2 w1 = make_float2(r * (o[1].x - o[1].y), r * (o[1].x + o[1].y));
  float2 w2 = make_float2(-o[2].y, o[2].x);
  float2 w3 = make_float2(-r * (o[3].x + o[3].y), r * (o[3].x - o[3].y));
  v[0] = make_float2(e[0].x + o[0].x, e[0].y + o[0].y);
  v[4] = make_float2(e[0].x - o[0].x, e[0].y - o[0].y);
  v[1] = make_float2(e[1].x + w1.x, e[1].y + w1.y);
  v[5] = make_float2(e[1].x - w1.x, e[1].y - w1.y);
  v[2] = make_float2(e[2].x + w2.x, e[2].y + w2.y);
  v[6] = make_float2(e[2].x - w2.x, e[2].y - w2.y);
  v[3] = make_float2(e[3].x + w3.x, e[3].y + w3.y);
  v[7] = make_float2(e[3].x - w3.x, e[3].y - w3.y);
}

// 64-point inverse DFTs of the 64 lines of the grid (rows when ROWS, else columns), in
// place: Stockham 8 x 8, thread t -> line t / 8, butterfly t % 8.
template <bool ROWS>
__device__ __forceinline__ void fft64_lines(float2* g, const float2* tw64) {
  const int t = threadIdx.x, line = t >> 3, j = t & 7;
  auto at = [&](int i) -> float2& { return ROWS ? g[line * kPsfLd + i] : g[i * kPsfLd + line]; };
  float2 v[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) v[m] = at(j + 8 * m);
  idft8(v);
  __syncthreads();
#pragma unroll
  for (int m = 0; m < 8; ++m) at(8 * j + m) = v[m];  // pass 1 (span 1): y[8 j + m]
  __syncthreads();
#pragma unroll
  for (int m = 0; m < 8; ++m) v[m] = at(j + 8 * m);
#pragma unroll
  for (int m = 1; m < 8; ++m) v[m] = cmul(v[m], tw64[(m * j) & 63]);  // pass 2 (span 8), k = j
  idft8(v);
  __syncthreads();
#pragma unroll
  for (int m = 0; m < 8; ++m) at(j + 8 * m) = v[m];  // natural order
  __syncthreads();
}

struct ExactArgs {
  const float* zern;  // [Z][H][W] (one frame, the p2s_sample_zernike layout)
  const float* ztab;  // [Z][32*32] Noll Z_j at the pupil samples; Z_1 = 1 inside the disk, 0 outside
  const float* img;   // [C][H][W] (render) or null
  float* out;         // psf: [n][T][T]; render: [C][H][W]
  const int* pix;     // psf: pixel indices y*W + x
  int n, Z, H, W, C, T, include_tilt;
};

__device__ __forceinline__ float block_sum512(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int w = 0; w < 16; ++w) s += red[w];
  __syncthreads();
  return s;
}

// PSF of pixel `p` into psf[T*T] (unit sum); smem grid g, twiddles tw64, scratch coef/red.
__device__ void exact_psf_cta(const ExactArgs& a, int p, float2* g, const float2* tw64, float* coef, float* red,
                              float* psf) {
  const int t = threadIdx.x;
  const size_t HW = (size_t)a.H * a.W;
  for (int j = t; j < a.Z; j += 512) {
    float v = __ldg(&a.zern[(size_t)j * HW + p]);
    if (j == 0 || (!a.include_tilt && (j == 1 || j == 2))) v = 0.f;  // piston; tilt optional
    coef[j] = v;
  }
  for (int i = t; i < kPsfN * kPsfLd; i += 512) g[i] = make_float2(0.f, 0.f);
  __syncthreads();
  for (int s = t; s < kPupD * kPupD; s += 512) {
    float phi = 0.f;
    for (int j = 1; j < a.Z; ++j) phi = fmaf(coef[j], __ldg(&a.ztab[(size_t)j * kPupD * kPupD + s]), phi);
    const float inside = __ldg(&a.ztab[s]);  // Z_1: 1 inside the disk
    float sn, cs;
    sincosf(phi, &sn, &cs);
    g[(s / kPupD) * kPsfLd + (s % kPupD)] = make_float2(inside * cs, -inside * sn);  // P e^{-j phi}
  }
  __syncthreads();
  fft64_lines<true>(g, tw64);
  fft64_lines<false>(g, tw64);
  const int c = a.T / 2, TT = a.T * a.T;
  float part = 0.f;
  for (int i = t; i < TT; i += 512) {
    const int uy = i / a.T - c, ux = i % a.T - c;
    // forward-transform bin u = inverse-transform bin -u
    const float2 f = g[((kPsfN - uy) & (kPsfN - 1)) * kPsfLd + ((kPsfN - ux) & (kPsfN - 1))];
    const float v = f.x * f.x + f.y * f.y;
    psf[i] = v;
    part += v;
  }
  const float total = block_sum512(part, red);
  const float inv = 1.f / total;
  for (int i = t; i < TT; i += 512) psf[i] *= inv;
  __syncthreads();
}

__global__ void __launch_bounds__(512) k_exact_psf(ExactArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  float2* g = reinterpret_cast<float2*>(smem);          // [64][65]
  float2* tw64 = g + kPsfN * kPsfLd;                     // [64]
  float* coef = reinterpret_cast<float*>(tw64 + kPsfN);  // [Z]
  float* red = coef + 72;                                // [16]
  float* psf = red + 16;                                 // [T*T]
  if (threadIdx.x < kPsfN) {
    float sn, cs;
    sincospif(2.f * threadIdx.x / kPsfN, &sn, &cs);  // e^{+2 pi i k / 64}
    tw64[threadIdx.x] = make_float2(cs, sn);
  }
  const int q = blockIdx.x;
  exact_psf_cta(a, __ldg(&a.pix[q]), g, tw64, coef, red, psf);
  const int TT = a.T * a.T;
  for (int i = threadIdx.x; i < TT; i += 512) a.out[(size_t)q * TT + i] = psf[i];
}

__device__ __forceinline__ int reflect_px(int i, int n) {
  if (i < 0) i = -i;
  if (i >= n) i = 2 * n - 2 - i;
  return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

__global__ void __launch_bounds__(512) k_render_exact(ExactArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  float2* g = reinterpret_cast<float2*>(smem);
  float2* tw64 = g + kPsfN * kPsfLd;
  float* coef = reinterpret_cast<float*>(tw64 + kPsfN);
  float* red = coef + 72;
  float* psf = red + 16;
  if (threadIdx.x < kPsfN) {
    float sn, cs;
    sincospif(2.f * threadIdx.x / kPsfN, &sn, &cs);
    tw64[threadIdx.x] = make_float2(cs, sn);
  }
  const int p = blockIdx.x;
  const int y = p / a.W, x = p - y * a.W;
  exact_psf_cta(a, p, g, tw64, coef, red, psf);
  const int c = a.T / 2, TT = a.T * a.T;
  const size_t HW = (size_t)a.H * a.W;
  for (int ch = 0; ch < a.C; ++ch) {
    float part = 0.f;
    for (int i = threadIdx.x; i < TT; i += 512) {
      const int uy = i / a.T - c, ux = i % a.T - c;
      part = fmaf(psf[i], __ldg(&a.img[(size_t)ch * HW + (size_t)reflect_px(y - uy, a.H) * a.W + reflect_px(x - ux, a.W)]),
                  part);
    }
    const float s = block_sum512(part, red);
    if (threadIdx.x == 0) a.out[(size_t)ch * HW + p] = s;
  }
}

static size_t exact_smem(int T) {
  return (size_t)kPsfN * kPsfLd * sizeof(float2) + kPsfN * sizeof(float2) + (72 + 16 + T * T) * sizeof(float);
}

// Host table of Z_j at the pupil sample centres (rho in radius units, theta from x).
static void pupil_table(int Z, std::vector<float>& tab) {
  tab.assign((size_t)Z * kPupD * kPupD, 0.f);
  for (int py = 0; py < kPupD; ++py)
    for (int px = 0; px < kPupD; ++px) {
      const double yy = (py + 0.5 - kPupD / 2.0) / (kPupD / 2.0), xx = (px + 0.5 - kPupD / 2.0) / (kPupD / 2.0);
      const double rho = std::hypot(xx, yy), th = std::atan2(yy, xx);
      if (rho > 1.0) continue;
      for (int j = 1; j <= Z; ++j) tab[(size_t)(j - 1) * kPupD * kPupD + py * kPupD + px] = (float)zernike_value(j, rho, th);
    }
}

int ensure_pupil_table(p2s_plan_s* p) {
  if (p->d_ztab) return 0;
  std::vector<float> tab;
  pupil_table(p->Z, tab);
  cudaError_t e = cudaMalloc(&p->d_ztab, tab.size() * sizeof(float));
  if (e != cudaSuccess) return (int)e;
  return (int)cudaMemcpy(p->d_ztab, tab.data(), tab.size() * sizeof(float), cudaMemcpyHostToDevice);
}

int launch_exact_psf(const p2s_plan_s* p, const float* zern, const int* pix, int n, int include_tilt, float* out,
                     cudaStream_t s) {
  ExactArgs a{zern, p->d_ztab, nullptr, out, pix, n, p->Z, p->H, p->W, p->C, p->T, include_tilt};
  const size_t sm = exact_smem(p->T);
  P2S_SMEM_OPTIN(k_exact_psf, sm);
  k_exact_psf<<<n, 512, sm, s>>>(a);
  return (int)cudaGetLastError();
}

int launch_render_exact(const p2s_plan_s* p, const float* img, const float* zern, int include_tilt, float* out,
                        cudaStream_t s) {
  ExactArgs a{zern, p->d_ztab, img, out, nullptr, p->H * p->W, p->Z, p->H, p->W, p->C, p->T, include_tilt};
  const size_t sm = exact_smem(p->T);
  P2S_SMEM_OPTIN(k_render_exact, sm);
  k_render_exact<<<p->H * p->W, 512, sm, s>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace p2s
