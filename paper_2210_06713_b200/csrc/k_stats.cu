// k_stats.cu -- validation battery: spatial statistics of sampled
// Zernike coefficient fields at GPU scale.
//
// The paper's sampler reproduces, per mode, the spatial auto-correlation A_jj(s) of the
// Zernike coefficients between pixels (block-diagonal model Eq.10, P:318-330:
// E[a_j(x) a_j(x+s)] = sum_k L_jk^2 c_k(s)), and the tilt statistics follow from j = 2, 3
// (differential tilt variance D(s) = 2 (A_22(0) - A_22(s))).  k_acorr measures
// the empirical auto-correlation of every mode along x and y,
//     R_j(dir, l) = 1/(F H W) sum_{f, y, x} a_j(f, y, x) a_j(f, (y, x) + l e_dir)   (periodic),
// from thousands of frames, for comparison with the analytic kernels.
//
// One CTA per (frame, mode, 32-column block) streams the rows of its column block, 8 at a
// time with the next 8 already in flight, through a shared-memory ring of L + 8 rows (row
// segments of 32 + L columns for the x lags, wrap mod W); each thread accumulates 8 lags
// of one column in fp32; per-CTA sums go to a partial buffer, a second kernel reduces them
// in fp64 in a fixed order (deterministic).
#include "p2s_dev.cuh"
#include "p2s_internal.h"

namespace p2s {

constexpr int kCorrCols = 32;
constexpr int kCorrMaxLag = 64;

constexpr int kCorrRows = 8;  // rows streamed per iteration (loads of the next batch in flight)

__global__ void __launch_bounds__(256) k_acorr(const float* __restrict__ zern, int Z, int H, int W, int L,
                                               double* __restrict__ partial) {
  extern __shared__ float ring[];  // [L + kCorrRows][kCorrCols + L]
  const int seg = kCorrCols + L;
  const int nslot = L + kCorrRows;
  const int ncb = (W + kCorrCols - 1) / kCorrCols;
  const int cb = blockIdx.x % ncb, plane = blockIdx.x / ncb;  // plane = f * Z + j
  const float* a = zern + (size_t)plane * H * W;
  const int x0 = cb * kCorrCols;
  const int tid = threadIdx.x;
  const int col = tid & (kCorrCols - 1), lg = tid >> 5;  // lags lg*8 .. lg*8+7
  const bool col_ok = x0 + col < W;
  const int nrows = H + L;  // periodic y lags: the first L rows again at the end
  const int per = kCorrRows * seg;  // values per batch (<= 8 * 96 = 768 = 3 per thread)
  float sx[8], sy[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) sx[i] = sy[i] = 0.f;
  // loop-invariant pieces of the batch loads and ring offsets (no divisions in the loop)
  float pre[3];
  int ld_r[3], ld_x[3], st_c[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int i = tid + k * 256;
    ld_r[k] = i < per ? i / seg : -1;  // row within the batch (-1: idle)
    st_c[k] = i < per ? i - ld_r[k] * seg : 0;
    ld_x[k] = (x0 + st_c[k]) % W;
  }
  auto fetch = [&](int y0b) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int yp = y0b + ld_r[k];
      const int yr = yp < H ? yp : yp - H;  // yp < H + L <= 2H
      pre[k] = (ld_r[k] >= 0 && yp < nrows) ? __ldg(&a[(size_t)yr * W + ld_x[k]]) : 0.f;
    }
  };
  fetch(0);
  int slot0 = 0;  // ring slot of row y0b
  for (int y0b = 0; y0b < nrows; y0b += kCorrRows) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (ld_r[k] >= 0) {
        int sl = slot0 + ld_r[k];
        if (sl >= nslot) sl -= nslot;
        ring[(size_t)sl * seg + st_c[k]] = pre[k];
      }
    }
    __syncthreads();
    fetch(y0b + kCorrRows);  // next batch in flight while this one is used
    if (col_ok) {
      int sl = slot0;
      for (int r = 0; r < kCorrRows; ++r, sl = (sl + 1 == nslot) ? 0 : sl + 1) {
        const int yp = y0b + r;
        if (yp >= nrows) break;
        const float* slot = ring + (size_t)sl * seg;
        const float v = slot[col];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int l = lg * 8 + i;
          if (l < L) {
            if (yp < H) sx[i] = fmaf(v, slot[col + l], sx[i]);  // a(y, x) a(y, x + l)
            if (yp >= l && yp - l < H) {
              const int sm_ = sl >= l ? sl - l : sl - l + nslot;
              sy[i] = fmaf(ring[(size_t)sm_ * seg + col], v, sy[i]);
            }
          }
        }
      }
    }
    slot0 += kCorrRows;
    if (slot0 >= nslot) slot0 -= nslot;
    __syncthreads();
  }
  // reduce the 32 columns of each lag: shuffle within the warp (one warp = one lag group)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double dx = col_ok ? (double)sx[i] : 0.0, dy = col_ok ? (double)sy[i] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      dx += __shfl_xor_sync(0xffffffffu, dx, o);
      dy += __shfl_xor_sync(0xffffffffu, dy, o);
    }
    const int l = lg * 8 + i;
    if (col == 0 && l < L) {
      partial[((size_t)blockIdx.x * 2 + 0) * L + l] = dx;
      partial[((size_t)blockIdx.x * 2 + 1) * L + l] = dy;
    }
  }
}

// out[j][dir][l] = sum over frames and column blocks of partial / (F H W).  One CTA per
// output element; each thread sums a fixed strided subset, then a fixed-shape tree: the
// result does not depend on scheduling (deterministic).
__global__ void __launch_bounds__(128) k_acorr_reduce(const double* __restrict__ partial, int F, int Z, int ncb,
                                                      int L, double inv, double* __restrict__ out) {
  __shared__ double red[128];
  const int i = blockIdx.x;  // (j, dir, l)
  const int j = i / (2 * L), r = i - j * 2 * L;
  const int n = F * ncb;
  double s = 0.0;
  for (int k = threadIdx.x; k < n; k += 128) {
    const int f = k / ncb, cb = k - f * ncb;
    s += partial[((size_t)((f * Z + j) * ncb + cb) * 2) * L + r];
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 64; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[i] = red[0] * inv;
}

size_t acorr_partial_bytes(int F, int Z, int W, int L) {
  const int ncb = (W + kCorrCols - 1) / kCorrCols;
  return (size_t)F * Z * ncb * 2 * L * sizeof(double);
}

int launch_acorr(const float* zern, int F, int Z, int H, int W, int L, double* partial, double* out, cudaStream_t s) {
  if (L < 1 || L > kCorrMaxLag) return (int)cudaErrorInvalidValue;
  const int ncb = (W + kCorrCols - 1) / kCorrCols;
  const size_t sm = (size_t)(L + kCorrRows) * (kCorrCols + L) * sizeof(float);
  k_acorr<<<F * Z * ncb, 256, sm, s>>>(zern, Z, H, W, L, partial);
  k_acorr_reduce<<<Z * 2 * L, 128, 0, s>>>(partial, F, Z, ncb, L, 1.0 / ((double)F * H * W), out);
  return (int)cudaGetLastError();
}

}  // namespace p2s
