// k_aperture.cu -- aperture statistics of the validation battery (SURVEY 8(f) NEXT-2,
// P:477-500): the phase structure function and the long/short-exposure OTFs of the
// sampled Zernike vectors, accumulated over every (frame, pixel) sample.
//
// Per sample the pupil phase phi = sum_j a_j Z_j on the 32-sample pupil of reading Q24
// (the table the exact-PSF path uses), its tilt-corrected residual phi - (c + alpha^T xi)
// (least-squares plane over the disc: the disc is symmetric, so 1, X, Y are orthogonal on
// it and each coefficient is one ratio of sums), and for every lag xi = (dy, dx),
// dy in [0, 32), dx in [-31, 31], with Delta = phi(x) - phi(x + xi):
//   sum_x M M' Delta^2,  sum_x M M' cos(Delta),  sum_x M M' cos(Delta_residual).
// Layout: the phase grids sit in shared memory with a zero/mask-0 margin (64 rows x 96
// columns, pupil at rows 0-31, columns 32-63), so every lag reads x + xi without bounds
// tests; the loop runs over the ~800 disc samples only (a compacted list) and each thread
// owns 4 lags: one warp = 32 consecutive dx of one dy, so the shifted reads are
// consecutive words (conflict-free) and the unshifted ones broadcasts.  Per-sample sums in
// fp32 (<= 804 terms), across samples in fp64; per-CTA partials are reduced in a fixed
// order by a second kernel (deterministic).
#include "p2s_dev.cuh"
#include "p2s_internal.h"

#include <algorithm>

namespace p2s {

namespace {

constexpr int kPD = 32;           // pupil samples across the diameter (reading Q24)
constexpr int kGW = 96;           // padded grid width
constexpr int kGH = 64;           // padded grid height
constexpr int kSlots = 2048;      // 32 dy x 64 dx slots (dx slot 63 unused)
constexpr int kThreads = 512;
constexpr int kPerThread = kSlots / kThreads;

struct ApArgs {
  const float* zern;  // [F][Z][H][W]
  const float* ztab;  // [Z][32*32]; plane 0 = 1 inside the disc
  const int* pix;     // [npix]
  double* partial;    // [grid][4][kSlots]: sf, le, se, cnt
  int64_t nsamples;
  int npix, Z;
  int64_t HW;
};

__device__ __forceinline__ float cos_red(float d) {
  // cos after reduction to [-pi, pi] (two-term 2 pi), then the SFU cosine
  const float k = rintf(d * 0.159154943f);
  float r = fmaf(-k, 6.28318548f, d);
  r = fmaf(-k, -1.74845553e-7f, r);
  return __cosf(r);
}

__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) s += red[w];
  __syncthreads();
  return s;
}

__global__ void __launch_bounds__(kThreads, 2) k_aperture(ApArgs a) {
  extern __shared__ __align__(16) float sm[];
  float* phi = sm;                  // [64][96]
  float* vph = phi + kGH * kGW;     // [64][96] plane residual
  float* msk = vph + kGH * kGW;     // [64][96]
  int* pos = reinterpret_cast<int*>(msk + kGH * kGW);  // [1024] disc samples (grid index)
  float* coef = reinterpret_cast<float*>(pos + kPD * kPD);  // [72]
  float* red = coef + 72;           // [16]
  int* wcnt = reinterpret_cast<int*>(red + 16);  // [17]
  const int t = threadIdx.x;
  for (int i = t; i < 3 * kGH * kGW; i += kThreads) sm[i] = 0.f;
  __syncthreads();
  // disc mask and the compacted list of its samples (row-major order)
  int npos;
  {
    bool in[2];
    int c = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int s = 2 * t + h;  // warp w covers samples [64 w, 64 w + 64)
      in[h] = __ldg(&a.ztab[s]) > 0.5f;
      c += in[h];
      msk[(s / kPD) * kGW + kGW / 3 + (s % kPD)] = in[h] ? 1.f : 0.f;
    }
    const int lane = t & 31, w = t >> 5;
    int incl = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wcnt[w] = incl;
    __syncthreads();
    if (t == 0) {
      int acc = 0;
      for (int i = 0; i < kThreads / 32; ++i) {
        const int v = wcnt[i];
        wcnt[i] = acc;
        acc += v;
      }
      wcnt[16] = acc;
    }
    __syncthreads();
    int o = wcnt[w] + incl - c;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int s = 2 * t + h;
      if (in[h]) pos[o++] = (s / kPD) * kGW + kGW / 3 + (s % kPD);
    }
    __syncthreads();
    npos = wcnt[16];
  }
  // plane-fit denominators sum M, sum M X^2, sum M Y^2 (X, Y in radius units)
  float x2 = 0.f, y2 = 0.f;
  for (int s = t; s < kPD * kPD; s += kThreads) {
    const float X = (s % kPD + 0.5f - kPD / 2.f) / (kPD / 2.f), Y = (s / kPD + 0.5f - kPD / 2.f) / (kPD / 2.f);
    const float m = __ldg(&a.ztab[s]) > 0.5f ? 1.f : 0.f;
    x2 += m * X * X;
    y2 += m * Y * Y;
  }
  const float sX2 = block_sum(x2, red), sY2 = block_sum(y2, red);
  const float sM = (float)npos;

  int off[kPerThread];
  bool live[kPerThread];
#pragma unroll
  for (int r = 0; r < kPerThread; ++r) {
    const int slot = t + r * kThreads, dy = slot >> 6, dx = (slot & 63) - (kPD - 1);
    live[r] = (slot & 63) < 2 * kPD - 1;
    off[r] = live[r] ? dy * kGW + dx : 0;
  }
  double acc[3][kPerThread];
#pragma unroll
  for (int r = 0; r < kPerThread; ++r) acc[0][r] = acc[1][r] = acc[2][r] = 0.0;

  for (int64_t q = blockIdx.x; q < a.nsamples; q += gridDim.x) {
    const int64_t f = q / a.npix;
    const int p = __ldg(&a.pix[q - f * a.npix]);
    const float* zf = a.zern + (size_t)f * a.Z * a.HW + p;
    for (int j = t; j < a.Z; j += kThreads) coef[j] = j == 0 ? 0.f : __ldg(&zf[(size_t)j * a.HW]);
    __syncthreads();
    float s0 = 0.f, s1 = 0.f, s2 = 0.f;
    for (int s = t; s < kPD * kPD; s += kThreads) {
      float v = 0.f;
      for (int j = 1; j < a.Z; ++j) v = fmaf(coef[j], __ldg(&a.ztab[(size_t)j * kPD * kPD + s]), v);
      const int g = (s / kPD) * kGW + kGW / 3 + (s % kPD);
      v *= msk[g];
      phi[g] = v;
      const float X = (s % kPD + 0.5f - kPD / 2.f) / (kPD / 2.f), Y = (s / kPD + 0.5f - kPD / 2.f) / (kPD / 2.f);
      s0 += v;
      s1 += v * X;
      s2 += v * Y;
    }
    const float c0 = block_sum(s0, red) / sM, ax = block_sum(s1, red) / sX2, ay = block_sum(s2, red) / sY2;
    for (int s = t; s < kPD * kPD; s += kThreads) {
      const int g = (s / kPD) * kGW + kGW / 3 + (s % kPD);
      const float X = (s % kPD + 0.5f - kPD / 2.f) / (kPD / 2.f), Y = (s / kPD + 0.5f - kPD / 2.f) / (kPD / 2.f);
      vph[g] = msk[g] * (phi[g] - (c0 + ax * X + ay * Y));
    }
    __syncthreads();
    float sf[kPerThread], le[kPerThread], se[kPerThread];
#pragma unroll
    for (int r = 0; r < kPerThread; ++r) sf[r] = le[r] = se[r] = 0.f;
    for (int i = 0; i < npos; ++i) {
      const int g = pos[i];
      const float v1 = phi[g], w1 = vph[g];
#pragma unroll
      for (int r = 0; r < kPerThread; ++r) {
        const int h = g + off[r];
        const float m2 = msk[h];
        const float d = v1 - phi[h], e = w1 - vph[h];
        sf[r] = fmaf(m2 * d, d, sf[r]);
        le[r] = fmaf(m2, cos_red(d), le[r]);
        se[r] = fmaf(m2, cos_red(e), se[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kPerThread; ++r) {
      acc[0][r] += sf[r];
      acc[1][r] += le[r];
      acc[2][r] += se[r];
    }
    __syncthreads();  // coef / phi reuse
  }
  double* out = a.partial + (size_t)blockIdx.x * 4 * kSlots;
#pragma unroll
  for (int r = 0; r < kPerThread; ++r) {
    const int slot = t + r * kThreads;
    out[slot] = acc[0][r];
    out[kSlots + slot] = acc[1][r];
    out[2 * kSlots + slot] = acc[2][r];
    float c = 0.f;
    if (blockIdx.x == 0 && live[r])
      for (int i = 0; i < npos; ++i) c += msk[pos[i] + off[r]];
    if (blockIdx.x == 0) out[3 * kSlots + slot] = c;
  }
}

// out[3][32][63]: SF = sum / (n cnt), LE, SE = sum / (n cnt(0)); fixed-order reduction.
__global__ void k_aperture_reduce(const double* partial, int grid, int64_t nsamples, double* out) {
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= kSlots || (slot & 63) == 63) return;
  const double cnt = partial[3 * kSlots + slot], cnt0 = partial[3 * kSlots + (kPD - 1)];
  double s[3] = {0.0, 0.0, 0.0};
  for (int b = 0; b < grid; ++b)
#pragma unroll
    for (int k = 0; k < 3; ++k) s[k] += partial[(size_t)b * 4 * kSlots + k * kSlots + slot];
  const int dy = slot >> 6, dxi = slot & 63;
  const size_t o = (size_t)dy * (2 * kPD - 1) + dxi, plane = (size_t)kPD * (2 * kPD - 1);
  const double n = (double)nsamples;
  out[o] = cnt > 0 ? s[0] / (n * cnt) : 0.0;
  out[plane + o] = s[1] / (n * cnt0);
  out[2 * plane + o] = s[2] / (n * cnt0);
}

size_t aperture_smem() {
  return (size_t)3 * kGH * kGW * sizeof(float) + kPD * kPD * sizeof(int) + (72 + 16) * sizeof(float) + 17 * sizeof(int);
}

}  // namespace

int aperture_grid(int64_t nsamples) {
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::min<int64_t>(nsamples, (int64_t)2 * sms);
}

size_t aperture_partial_bytes(int64_t nsamples) {
  return (size_t)aperture_grid(nsamples) * 4 * kSlots * sizeof(double);
}

int launch_aperture(const p2s_plan_s* p, const float* zern, int nframes, const int* pix, int npix, double* partial,
                    double* out, cudaStream_t s) {
  ApArgs a{zern, p->d_ztab, pix, partial, (int64_t)nframes * npix, npix, p->Z, (int64_t)p->H * p->W};
  const int grid = aperture_grid(a.nsamples);
  const size_t sm = aperture_smem();
  P2S_SMEM_OPTIN(k_aperture, sm);
  k_aperture<<<grid, kThreads, sm, s>>>(a);
  k_aperture_reduce<<<kSlots / 256, 256, 0, s>>>(partial, grid, a.nsamples, out);
  return (int)cudaGetLastError();
}

}  // namespace p2s
