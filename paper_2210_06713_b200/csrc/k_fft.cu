// k_fft.cu -- step 1 of DF-P2S on the GPU: Fourier sampling of the Zernike fields.
//
// Paper: homogeneous auto-covariance slices are circulant, so y = F^{-1}(S^{1/2} F(e))
// (P:234-238); N unit-variance fields are drawn this way and mixed point-wise
// with L, L L^T = A_0 (Eq.10).  Two real fields per complex inverse DFT with
// Hermitian spectral noise per mode (reading Q8):
//     Y_p[k] = sqrt(S_a[k]) eta_a[k] + i sqrt(S_b[k]) eta_b[k],  f_a = Re y, f_b = Im y.
//
// K1  k_rows : Philox noise + PSD filter (+ AR(1)) fused into the row inverse
//              DFT (shared-memory Stockham, radix 8/4/2/3/5); the spectrum is never
//              written.  One CTA per (spectral row, mode pair); the CTA loops over the
//              frame batch so its sqrt(S) row is read from HBM once per batch.
// K2  k_cols : column inverse DFT of TC interleaved columns, Re/Im split, crop to H x W;
//              writes fp32 Zernike planes (API) or bf16 MLP inputs + fp32 tilt planes
//              (fused simulate path).
// K3  k_mix  : a = L f per pixel (API p2s_sample_zernike only; simulate folds L into
//              the MLP's first layer and the warp coefficients).
#include "p2s_dev.cuh"
#include "p2s_internal.h"

#include <algorithm>

#include <cstdlib>

namespace p2s {

// ------------------------------------------------------------------ small inverse DFTs
template <int R>
__device__ __forceinline__ void dft_inv(float2* v);

template <>
__device__ __forceinline__ void dft_inv<2>(float2* v) {
  float2 a = v[0], b = v[1];
  v[0] = make_float2(a.x + b.x, a.y + b.y);
  v[1] = make_float2(a.x - b.x, a.y - b.y);
}
template <>
__device__ __forceinline__ void dft_inv<4>(float2* v) {
  float2 a = v[0], b = v[1], c = v[2], d = v[3];
  float2 s0 = make_float2(a.x + c.x, a.y + c.y), s1 = make_float2(a.x - c.x, a.y - c.y);
  float2 s2 = make_float2(b.x + d.x, b.y + d.y), s3 = make_float2(b.x - d.x, b.y - d.y);
  v[0] = make_float2(s0.x + s2.x, s0.y + s2.y);
  v[2] = make_float2(s0.x - s2.x, s0.y - s2.y);
  // a + i b - c - i d = s1 + i s3
  v[1] = make_float2(s1.x - s3.y, s1.y + s3.x);
  v[3] = make_float2(s1.x + s3.y, s1.y - s3.x);
}
template <>
__device__ __forceinline__ void dft_inv<8>(float2* v) {
  float2 e[4] = {v[0], v[2], v[4], v[6]};
  float2 o[4] = {v[1], v[3], v[5], v[7]};
  dft_inv<4>(e);
  dft_inv<4>(o);
  const float r = 0.70710678118654752f;
  float2 w1 = make_float2(r * (o[1].x - o[1].y), r * (o[1].x + o[1].y));  // (1+i)/sqrt2 * o1
  float2 w2 = make_float2(-o[2].y, o[2].x);                              // i * o2
  float2 w3 = make_float2(-r * (o[3].x + o[3].y), r * (o[3].x - o[3].y)); // (-1+i)/sqrt2 * o3
  v[0] = make_float2(e[0].x + o[0].x, e[0].y + o[0].y);
  v[4] = make_float2(e[0].x - o[0].x, e[0].y - o[0].y);
  v[1] = make_float2(e[1].x + w1.x, e[1].y + w1.y);
  v[5] = make_float2(e[1].x - w1.x, e[1].y - w1.y);
  v[2] = make_float2(e[2].x + w2.x, e[2].y + w2.y);
  v[6] = make_float2(e[2].x - w2.x, e[2].y - w2.y);
  v[3] = make_float2(e[3].x + w3.x, e[3].y + w3.y);
  v[7] = make_float2(e[3].x - w3.x, e[3].y - w3.y);
}
template <>
__device__ __forceinline__ void dft_inv<3>(float2* v) {
  const float h = 0.86602540378443865f;
  float2 t = make_float2(v[1].x + v[2].x, v[1].y + v[2].y);
  float2 a = make_float2(v[0].x - 0.5f * t.x, v[0].y - 0.5f * t.y);
  float2 b = make_float2(h * (v[1].x - v[2].x), h * (v[1].y - v[2].y));
  v[0] = make_float2(v[0].x + t.x, v[0].y + t.y);
  v[1] = make_float2(a.x - b.y, a.y + b.x);
  v[2] = make_float2(a.x + b.y, a.y - b.x);
}
template <>
__device__ __forceinline__ void dft_inv<5>(float2* v) {
  const float c1 = 0.30901699437494742f, c2 = -0.80901699437494742f;
  const float s1 = 0.95105651629515357f, s2 = 0.58778525229247313f;
  float2 t1 = make_float2(v[1].x + v[4].x, v[1].y + v[4].y);
  float2 t2 = make_float2(v[2].x + v[3].x, v[2].y + v[3].y);
  float2 t3 = make_float2(v[1].x - v[4].x, v[1].y - v[4].y);
  float2 t4 = make_float2(v[2].x - v[3].x, v[2].y - v[3].y);
  float2 a1 = make_float2(v[0].x + c1 * t1.x + c2 * t2.x, v[0].y + c1 * t1.y + c2 * t2.y);
  float2 a2 = make_float2(v[0].x + c2 * t1.x + c1 * t2.x, v[0].y + c2 * t1.y + c1 * t2.y);
  float2 b1 = make_float2(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y);
  float2 b2 = make_float2(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y);
  v[0] = make_float2(v[0].x + t1.x + t2.x, v[0].y + t1.y + t2.y);
  v[1] = make_float2(a1.x - b1.y, a1.y + b1.x);
  v[4] = make_float2(a1.x + b1.y, a1.y - b1.x);
  v[2] = make_float2(a2.x - b2.y, a2.y + b2.x);
  v[3] = make_float2(a2.x + b2.y, a2.y - b2.x);
}

// Twiddles e^{+2 pi i j / R} of the composite radices: local constant tables, indexed
// with compile-time j after unrolling (folded into immediates).
template <int R>
__device__ __forceinline__ float2 twr(int j);
template <>
__device__ __forceinline__ float2 twr<6>(int j) {
  const float2 t[6] = {{1.0f, 0.0f}, {0.50000000000000011f, 0.8660254037844386f}, {-0.49999999999999978f, 0.86602540378443871f}, {-1.0f, 1.2246467991473532e-16f}, {-0.50000000000000044f, -0.86602540378443837f}, {0.50000000000000011f, -0.8660254037844386f}};
  return t[j];
}
template <>
__device__ __forceinline__ float2 twr<9>(int j) {
  const float2 t[9] = {{1.0f, 0.0f}, {0.76604444311897801f, 0.64278760968653925f}, {0.17364817766693041f, 0.98480775301220802f}, {-0.49999999999999978f, 0.86602540378443871f}, {-0.93969262078590832f, 0.34202014332566888f}, {-0.93969262078590843f, -0.34202014332566866f}, {-0.50000000000000044f, -0.86602540378443837f}, {0.17364817766692997f, -0.98480775301220813f}, {0.76604444311897779f, -0.64278760968653958f}};
  return t[j];
}
template <>
__device__ __forceinline__ float2 twr<10>(int j) {
  const float2 t[10] = {{1.0f, 0.0f}, {0.80901699437494745f, 0.58778525229247314f}, {0.30901699437494745f, 0.95105651629515353f}, {-0.30901699437494734f, 0.95105651629515364f}, {-0.80901699437494734f, 0.58778525229247325f}, {-1.0f, 1.2246467991473532e-16f}, {-0.80901699437494756f, -0.58778525229247303f}, {-0.30901699437494756f, -0.95105651629515353f}, {0.30901699437494723f, -0.95105651629515364f}, {0.80901699437494734f, -0.58778525229247336f}};
  return t[j];
}
template <>
__device__ __forceinline__ float2 twr<12>(int j) {
  const float2 t[12] = {{1.0f, 0.0f}, {0.86602540378443871f, 0.49999999999999994f}, {0.50000000000000011f, 0.8660254037844386f}, {6.123233995736766e-17f, 1.0f}, {-0.49999999999999978f, 0.86602540378443871f}, {-0.86602540378443871f, 0.49999999999999994f}, {-1.0f, 1.2246467991473532e-16f}, {-0.86602540378443882f, -0.49999999999999972f}, {-0.50000000000000044f, -0.86602540378443837f}, {-1.8369701987210297e-16f, -1.0f}, {0.50000000000000011f, -0.8660254037844386f}, {0.86602540378443837f, -0.50000000000000044f}};
  return t[j];
}
template <>
__device__ __forceinline__ float2 twr<15>(int j) {
  const float2 t[15] = {{1.0f, 0.0f}, {0.91354545764260087f, 0.40673664307580015f}, {0.66913060635885824f, 0.74314482547739413f}, {0.30901699437494745f, 0.95105651629515353f}, {-0.10452846326765333f, 0.9945218953682734f}, {-0.49999999999999978f, 0.86602540378443871f}, {-0.80901699437494734f, 0.58778525229247325f}, {-0.97814760073380569f, 0.20791169081775931f}, {-0.97814760073380569f, -0.20791169081775907f}, {-0.80901699437494756f, -0.58778525229247303f}, {-0.50000000000000044f, -0.86602540378443837f}, {-0.10452846326765423f, -0.99452189536827329f}, {0.30901699437494723f, -0.95105651629515364f}, {0.66913060635885846f, -0.74314482547739402f}, {0.91354545764260098f, -0.40673664307580015f}};
  return t[j];
}
template <>
__device__ __forceinline__ float2 twr<16>(int j) {
  const float2 t[16] = {{1.0f, 0.0f}, {0.92387953251128674f, 0.38268343236508978f}, {0.70710678118654757f, 0.70710678118654746f}, {0.38268343236508984f, 0.92387953251128674f}, {6.123233995736766e-17f, 1.0f}, {-0.38268343236508973f, 0.92387953251128674f}, {-0.70710678118654746f, 0.70710678118654757f}, {-0.92387953251128674f, 0.38268343236508989f}, {-1.0f, 1.2246467991473532e-16f}, {-0.92387953251128685f, -0.38268343236508967f}, {-0.70710678118654768f, -0.70710678118654746f}, {-0.38268343236509034f, -0.92387953251128652f}, {-1.8369701987210297e-16f, -1.0f}, {0.38268343236509f, -0.92387953251128663f}, {0.70710678118654735f, -0.70710678118654768f}, {0.92387953251128652f, -0.38268343236509039f}};
  return t[j];
}
// Composite radix R = A * B in registers (Cooley-Tukey): n = a + A b, k = kb + B ka;
// DFT_B over b for each a, twiddle e^{+2 pi i a kb / R}, DFT_A over a for each kb.
template <int A, int B>
__device__ __forceinline__ void dft_inv_ct(float2* v) {
  constexpr int R = A * B;
  float2 y[A][B];
#pragma unroll
  for (int a = 0; a < A; ++a) {
#pragma unroll
    for (int b = 0; b < B; ++b) y[a][b] = v[a + A * b];
    dft_inv<B>(y[a]);
#pragma unroll
    for (int kb = 1; kb < B; ++kb) {
      const int j = (a * kb) % R;
      if (j) y[a][kb] = cmul(y[a][kb], twr<R>(j));
    }
  }
#pragma unroll
  for (int kb = 0; kb < B; ++kb) {
    float2 t[A];
#pragma unroll
    for (int a = 0; a < A; ++a) t[a] = y[a][kb];
    dft_inv<A>(t);
#pragma unroll
    for (int ka = 0; ka < A; ++ka) v[kb + B * ka] = t[ka];
  }
}
template <>
__device__ __forceinline__ void dft_inv<6>(float2* v) { dft_inv_ct<2, 3>(v); }
template <>
__device__ __forceinline__ void dft_inv<9>(float2* v) { dft_inv_ct<3, 3>(v); }
template <>
__device__ __forceinline__ void dft_inv<10>(float2* v) { dft_inv_ct<2, 5>(v); }
template <>
__device__ __forceinline__ void dft_inv<12>(float2* v) { dft_inv_ct<4, 3>(v); }
template <>
__device__ __forceinline__ void dft_inv<15>(float2* v) { dft_inv_ct<3, 5>(v); }
template <>
__device__ __forceinline__ void dft_inv<16>(float2* v) { dft_inv_ct<4, 4>(v); }


// ------------------------------------------------------------------ shared-memory Stockham IDFT
// TC interleaved sequences of length N live in shared memory, element i of sequence c at
// x[i*TC + c] (TC = 2^tc_log2).  Out-of-place (ping-pong) passes of radix 8/4/2/3/5; the
// divisions by Ns (product of earlier radices) use a multiply-high magic number.
constexpr int kColElems = 4608;  // P * TC per column CTA (2 x 36 KB ping-pong)

struct FFTArgs {
  int N;
  int nrad;
  int rad[kMaxRadix];
  uint32_t magic[kMaxRadix];  // floor(2^32 / Ns) + 1 of each pass (0 when Ns == 1)
  const float2* tw;           // e^{+2 pi i k / N}
};

// The radix plan is staged in shared memory so the kernel-parameter struct is never
// addressed dynamically (which would copy it to local memory).
struct FFTPlanSmem {
  int nrad, N;
  int rad[kMaxRadix];
  uint32_t magic[kMaxRadix];
  const float2* tw;
};

// Stage the radix plan and the twiddle table (N float2) in shared memory.
__device__ __forceinline__ void stage_fft_plan(FFTPlanSmem* sp, const FFTArgs& f, float2* tw_smem) {
  for (int k = threadIdx.x; k < f.N; k += blockDim.x) tw_smem[k] = __ldg(&f.tw[k]);
  if (threadIdx.x == 0) {
    sp->nrad = f.nrad;
    sp->N = f.N;
    sp->tw = tw_smem;
  }
  if (threadIdx.x < kMaxRadix) {
    sp->rad[threadIdx.x] = f.rad[threadIdx.x];
    sp->magic[threadIdx.x] = f.magic[threadIdx.x];
  }
}

// Shared-memory index with one float2 of padding per 16: spreads the strided Stockham
// writes over the banks.
__device__ __forceinline__ int pidx(int i) { return i + (i >> 4); }
__host__ __device__ constexpr size_t padded_len(size_t n) { return (n + (n >> 4) + 2) & ~(size_t)1; }

template <int R, int NT>
__device__ __forceinline__ void ifft_pass(const float2* __restrict__ x, float2* __restrict__ y, int N, int Ns,
                                          uint32_t mag, int tc_log2, const float2* __restrict__ tw) {
  const int NR = N / R;
  const int TC1 = (1 << tc_log2) - 1;
  const int total = NR << tc_log2;
  const int ts = N / (Ns * R);
  for (int w = threadIdx.x; w < total; w += NT) {
    const int c = w & TC1, j = w >> tc_log2;
    const int q = Ns == 1 ? j : (int)__umulhi((uint32_t)j, mag);
    const int k = j - q * Ns;
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = x[pidx(((j + r * NR) << tc_log2) + c)];
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[r * k * ts]);
    }
    dft_inv<R>(v);
    const int base = q * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) y[pidx(((base + r * Ns) << tc_log2) + c)] = v[r];
  }
}

// Inverse DFT (e^{+2 pi i}, unnormalised) of TC interleaved sequences, ping-pong between a
// and b; returns the buffer holding the result.
template <int NT>
__device__ __forceinline__ float2* smem_ifft(float2* a, float2* b, const FFTPlanSmem* f, int tc_log2) {
  int Ns = 1;
  const int nrad = f->nrad;
  for (int ip = 0; ip < nrad; ++ip) {
    const int R = f->rad[ip];
    const uint32_t mg = f->magic[ip];
    switch (R) {
      case 16: ifft_pass<16, NT>(a, b, f->N, Ns, mg, tc_log2, f->tw); break;
      case 15: ifft_pass<15, NT>(a, b, f->N, Ns, mg, tc_log2, f->tw); break;
      case 12: ifft_pass<12, NT>(a, b, f->N, Ns, mg, tc_log2, f->tw); break;
      case 10: ifft_pass<10, NT>(a, b, f->N, Ns, mg, tc_log2, f->tw); break;
      case 9: ifft_pass<9, NT>(a, b, f->N, Ns, mg, tc_log2, f->tw); break;
      case 6: ifft_pass<6, NT>(a, b, f->N, Ns, mg, tc_log2, f->tw); break;
      case 8: ifft_pass<8, NT>(a, b, f->N, Ns, mg, tc_log2, f->tw); break;
      case 4: ifft_pass<4, NT>(a, b, f->N, Ns, mg, tc_log2, f->tw); break;
      case 2: ifft_pass<2, NT>(a, b, f->N, Ns, mg, tc_log2, f->tw); break;
      case 3: ifft_pass<3, NT>(a, b, f->N, Ns, mg, tc_log2, f->tw); break;
      default: ifft_pass<5, NT>(a, b, f->N, Ns, mg, tc_log2, f->tw); break;
    }
    __syncthreads();
    float2* t = a;
    a = b;
    b = t;
    Ns *= R;
  }
  return a;
}

// In-place variant for plans where every pass has at most one butterfly per thread
// ((N / R) * TC <= NT): each thread loads its butterfly into registers, the CTA
// synchronises, and the results overwrite the same buffer, so one buffer serves (the
// persistent column kernel spends the second one on prefetching the next block).
template <int R, int NT>
__device__ __forceinline__ void ifft_pass_inplace(float2* __restrict__ x, int N, int Ns, uint32_t mag, int tc_log2,
                                                  const float2* __restrict__ tw) {
  const int NR = N / R;
  const int total = NR << tc_log2;
  const int ts = N / (Ns * R);
  const int w = threadIdx.x;
  const bool act = w < total;
  const int c = w & ((1 << tc_log2) - 1), j = act ? w >> tc_log2 : 0;
  float2 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = x[pidx(((j + r * NR) << tc_log2) + c)];
  __syncthreads();
  const int q = Ns == 1 ? j : (int)__umulhi((uint32_t)j, mag);
  const int k = j - q * Ns;
  if (Ns > 1) {
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[r * k * ts]);
  }
  dft_inv<R>(v);
  const int base = q * Ns * R + k;
  if (act) {
#pragma unroll
    for (int r = 0; r < R; ++r) x[pidx(((base + r * Ns) << tc_log2) + c)] = v[r];
  }
  __syncthreads();
}

template <int NT>
__device__ __forceinline__ void smem_ifft_inplace(float2* x, const FFTPlanSmem* f, int tc_log2) {
  int Ns = 1;
  const int nrad = f->nrad;
  for (int ip = 0; ip < nrad; ++ip) {
    const int R = f->rad[ip];
    const uint32_t mg = f->magic[ip];
    switch (R) {
      case 16: ifft_pass_inplace<16, NT>(x, f->N, Ns, mg, tc_log2, f->tw); break;
      case 15: ifft_pass_inplace<15, NT>(x, f->N, Ns, mg, tc_log2, f->tw); break;
      case 12: ifft_pass_inplace<12, NT>(x, f->N, Ns, mg, tc_log2, f->tw); break;
      case 10: ifft_pass_inplace<10, NT>(x, f->N, Ns, mg, tc_log2, f->tw); break;
      case 9: ifft_pass_inplace<9, NT>(x, f->N, Ns, mg, tc_log2, f->tw); break;
      case 6: ifft_pass_inplace<6, NT>(x, f->N, Ns, mg, tc_log2, f->tw); break;
      case 8: ifft_pass_inplace<8, NT>(x, f->N, Ns, mg, tc_log2, f->tw); break;
      case 4: ifft_pass_inplace<4, NT>(x, f->N, Ns, mg, tc_log2, f->tw); break;
      case 2: ifft_pass_inplace<2, NT>(x, f->N, Ns, mg, tc_log2, f->tw); break;
      case 3: ifft_pass_inplace<3, NT>(x, f->N, Ns, mg, tc_log2, f->tw); break;
      default: ifft_pass_inplace<5, NT>(x, f->N, Ns, mg, tc_log2, f->tw); break;
    }
    Ns *= R;
  }
}

// Compile-time three-pass plans (N = R1 R2 R3) for the long axes of the BASELINE grids
// (1080 = 12 x 10 x 9, 2160 = 16 x 15 x 9): the same Stockham passes as smem_ifft_inplace,
// with constant radices and spans (index division by the span is a multiply-shift) and
// per-pass twiddle tables laid out [r-1][k], so the butterflies of consecutive threads read
// consecutive entries (the shared e^{2 pi i m / N} table is read at stride r k N/(Ns R) by
// consecutive k, which conflicts on the banks).
template <int N, int R1, int R2, int R3>
struct Plan3 {
  static_assert(R1 * R2 * R3 == N, "three-pass plan");
  static constexpr int tw2 = (R2 - 1) * R1;       // pass 2: span Ns = R1
  static constexpr int tw3 = (R3 - 1) * R1 * R2;  // pass 3: span Ns = R1 R2
  static constexpr int ntw = tw2 + tw3;
};
template <int N, int R1, int R2, int R3>
__device__ __forceinline__ void build_twp3(float2* __restrict__ twp, const float2* __restrict__ tw) {
  using PL = Plan3<N, R1, R2, R3>;
  for (int i = threadIdx.x; i < PL::ntw; i += blockDim.x) {
    int m;
    if (i < PL::tw2) {
      const int r = 1 + i / R1, k = i % R1;
      m = r * k * (N / (R1 * R2));
    } else {
      const int o = i - PL::tw2, r = 1 + o / (R1 * R2), k = o % (R1 * R2);
      m = r * k;
    }
    twp[i] = __ldg(&tw[m]);
  }
}
template <int R, int NS, int N, int NT, int TCL>
__device__ __forceinline__ void ifft_pass_ip_ct(float2* __restrict__ x, const float2* __restrict__ twp) {
  constexpr int NR = N / R, TC = 1 << TCL, total = NR * TC;
  constexpr int NB = (total + NT - 1) / NT;  // butterflies per thread (all loaded before any store)
  float2 v[NB][R];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int w = threadIdx.x + b * NT;
    const int c = w & (TC - 1), j = w < total ? w >> TCL : 0;
#pragma unroll
    for (int r = 0; r < R; ++r) v[b][r] = x[pidx(((j + r * NR) << TCL) + c)];
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int w = threadIdx.x + b * NT;
    const int c = w & (TC - 1), j = w < total ? w >> TCL : 0;
    const int k = j % NS, q = j / NS;
    if (NS > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[b][r] = cmul(v[b][r], twp[(r - 1) * NS + k]);
    }
    dft_inv<R>(v[b]);
    if (w < total) {
#pragma unroll
      for (int r = 0; r < R; ++r) x[pidx(((q * NS * R + k + r * NS) << TCL) + c)] = v[b][r];
    }
  }
  __syncthreads();
}
template <int N, int R1, int R2, int R3, int NT, int TCL>
__device__ __forceinline__ void smem_ifft3_inplace(float2* x, const float2* twp) {
  using PL = Plan3<N, R1, R2, R3>;
  ifft_pass_ip_ct<R1, 1, N, NT, TCL>(x, twp);
  ifft_pass_ip_ct<R2, R1, N, NT, TCL>(x, twp);
  ifft_pass_ip_ct<R3, R1 * R2, N, NT, TCL>(x, twp + PL::tw2);
}

static void fill_fft_args(FFTArgs& a, const AxisFFT& ax) {
  a.N = ax.N;
  a.nrad = ax.nrad;
  int Ns = 1;
  for (int i = 0; i < kMaxRadix; ++i) {
    a.rad[i] = ax.rad[i];
    a.magic[i] = 0;
    if (i < ax.nrad) {
      a.magic[i] = Ns == 1 ? 0u : (uint32_t)((1ull << 32) / (uint64_t)Ns + 1ull);
      Ns *= ax.rad[i];
    }
  }
  a.tw = ax.tw;
}

// ------------------------------------------------------------------ register-resident N = 512
// Fast path for 512-point axes (the bench grid): the same Stockham radix-8 passes as
// smem_ifft (8 x 8 x 8, identical twiddles and butterflies), but each butterfly's eight
// points stay in the registers of one thread (butterfly j holds x[j + 64 r]); the two
// shared-memory exchanges between passes are the only data movement, all index arithmetic
// is compile-time, and the last pass leaves the result in natural order (thread j holds
// y[j + 64 r]), so it is stored straight from registers.
constexpr int kRegN = 512, kRegB = 64;  // points, butterflies per pass

template <int NS>
__device__ __forceinline__ void reg_pass(float2 (&v)[8], int j, const float2* __restrict__ tw) {
  if (NS > 1) {
    const int step = (j & (NS - 1)) * (kRegN / (8 * NS));
#pragma unroll
    for (int r = 1; r < 8; ++r) v[r] = cmul(v[r], tw[r * step]);
  }
  dft_inv<8>(v);
}
// Per-pass twiddle table (same values as tw[r * k * N / (8 NS)]) laid out [r-1][k] so that
// consecutive butterflies read consecutive entries (no bank conflicts): NS = 8 at offset 0
// (7 x 8 entries), NS = 64 at offset 56 (7 x 64 entries); 504 entries in all.
template <int NS>
__device__ __forceinline__ constexpr int twp_base() { return NS == 8 ? 0 : 56; }
__device__ __forceinline__ void build_twp(float2* __restrict__ twp, const float2* __restrict__ tw, int tid, int nt) {
  for (int i = tid; i < 504; i += nt) {
    const bool second = i >= 56;
    const int ns = second ? 64 : 8, o = second ? i - 56 : i;
    const int r = 1 + o / ns, k = o % ns;
    twp[i] = __ldg(&tw[r * k * (kRegN / (8 * ns))]);
  }
}
template <int NS>
__device__ __forceinline__ void reg_pass_t(float2 (&v)[8], int j, const float2* __restrict__ twp) {
  if (NS > 1) {
    const int k = j & (NS - 1);
#pragma unroll
    for (int r = 1; r < 8; ++r) v[r] = cmul(v[r], twp[twp_base<NS>() + (r - 1) * NS + k]);
  }
  dft_inv<8>(v);
}
// Stockham output position of point r of butterfly j after the pass with span NS.
template <int NS>
__device__ __forceinline__ int reg_out(int j, int r) {
  const int k = j & (NS - 1);
  return (j - k) * 8 + k + r * NS;
}

// ------------------------------------------------------------------ K1: noise + PSD + row IDFT
struct RowArgs {
  FFTArgs fq;
  const float2* sqrtS;  // [npairs][P][Q] scaled amplitudes (sa, sb)
  float4* ar;           // [npairs][P][Q] AR state (zeta_a, zeta_b), or null
  float2* Zout;         // [F][npairs][P][Q]
  int P, Q, npairs;
  uint32_t k0, k1;
  int64_t frame0;
  int F;
  float alpha, calpha;
  int64_t t_start;      // first frame evolved (AR replay starts at 0)
  const float2* eta;    // caller-supplied spectral noise [F][nslots][P][Q] (from_noise entry), or null
  int nslots;
  int load_state;       // AR: state holds eta_{frame0-1}
  int flow;             // frozen flow: frame-0 noise translated by (vx, vy) * frame pixels
  double vx, vy;
  int ky0;              // first Hermitian row pair of the launch (slab mode; 0 otherwise)
};

// Frozen flow (reading Q23): shift factor of bin k of an n-point axis for a
// translation by s pixels: exp(-2 pi i f_k s) with the signed frequency f_k, and the real
// cos(pi s) at the Nyquist bin (its own mirror), so the spectrum stays Hermitian.  The
// phase is reduced in fp64 before the fp32 sincos.
__device__ __forceinline__ float2 flow_phase(int k, int n, double s) {
  if (k == 0) return make_float2(1.f, 0.f);
  if (2 * k == n) return make_float2((float)cospi(s), 0.f);
  const int ks = 2 * k < n ? k : k - n;
  double a = (double)ks * s / (double)n;
  a -= rint(a);
  float sn, cs;
  sincospif((float)(-2.0 * a), &sn, &cs);
  return make_float2(cs, sn);
}

// Unit-variance Hermitian noise zeta (eta / sqrt(PQ/2)) for both modes of pair p at bin (ky, kx).
__device__ __forceinline__ float4 spectral_noise(int ky, int kx, int P, int Q, int p, int64_t frame, uint32_t k0,
                                                 uint32_t k1) {
  const uint32_t lin = (uint32_t)ky * Q + kx;
  const int kym = ky ? P - ky : 0, kxm = kx ? Q - kx : 0;
  const uint32_t linm = (uint32_t)kym * Q + kxm;
  const uint32_t canon = lin < linm ? lin : linm;
  uint4 x = philox4x32_10(make_uint4(canon, (uint32_t)p, (uint32_t)frame, (uint32_t)((uint64_t)frame >> 32)), k0, k1);
  float2 ga = box_muller_fast(x.x, x.y), gb = box_muller_fast(x.z, x.w);
  if (lin == linm) {  // self-conjugate: sqrt(PQ) g1 = sqrt(2) sqrt(PQ/2) g1
    const float r2 = 1.41421356237309515f;
    return make_float4(r2 * ga.x, 0.f, r2 * gb.x, 0.f);
  }
  const float sg = (lin == canon) ? 1.f : -1.f;
  return make_float4(ga.x, sg * ga.y, gb.x, sg * gb.y);
}

// Y = sa zeta_a + i sb zeta_b
__device__ __forceinline__ float2 spectrum(float2 s, float4 z) {
  return make_float2(s.x * z.x - s.y * z.w, s.x * z.y + s.y * z.z);
}

// White-noise path: one CTA per Hermitian row pair {ky, P-ky}: each Philox draw serves the
// bin and its mirror (the mirror's noise is the conjugate), the two rows are transformed
// as two interleaved sequences, and the CTA loops over the frame batch.
// ETA: caller-supplied noise (p2s_sample_zernike_from_noise) instead of the Philox draw; a
// separate instantiation so the generated-noise kernel keeps its register budget.
template <int NT, bool ETA = false>
__global__ void __launch_bounds__(NT) k_rows_pair(RowArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int Q = a.Q;
  float2* twq = reinterpret_cast<float2*>(smem);  // [Q] twiddles
  float2* sS = twq + Q;                            // [2][Q]
  float2* X = sS + 2 * Q;                          // [Q][2] interleaved rows (padded)
  float2* Xb = X + padded_len(2 * Q);              // ping-pong partner
  __shared__ FFTPlanSmem fpl;
  stage_fft_plan(&fpl, a.fq, twq);
  const int ky = a.ky0 + (int)blockIdx.x, p = blockIdx.y;
  const int k1 = ky ? a.P - ky : 0;
  const size_t plane = (size_t)p * a.P * Q;
  for (int kx = threadIdx.x; kx < Q; kx += NT) {
    sS[kx] = a.sqrtS[plane + (size_t)ky * Q + kx];
    sS[Q + kx] = a.sqrtS[plane + (size_t)k1 * Q + kx];
  }
  __syncthreads();
  for (int t = 0; t < a.F; ++t) {
    const int64_t fr = a.frame0 + t;
    const int64_t fr_noise = a.flow ? 0 : fr;  // frozen flow: one realisation, translated
    const float2 phy = a.flow ? flow_phase(ky, a.P, a.vy * (double)fr) : make_float2(1.f, 0.f);
    for (int kx = threadIdx.x; kx < Q; kx += NT) {
      const int km = kx ? Q - kx : 0;
      float4 z, zm;
      if (ETA) {  // given eta (reading Q8 scaling): zeta = eta / sqrt(PQ/2), each bin read as stored
        const float inv = rsqrtf(0.5f * (float)a.P * (float)Q);
        const size_t PQ = (size_t)a.P * Q;
        const float2* ea = a.eta + ((size_t)t * a.nslots + 2 * p) * PQ;
        const bool hb = 2 * p + 1 < a.nslots;
        const float2 a0 = ea[(size_t)ky * Q + kx], b0 = hb ? ea[PQ + (size_t)ky * Q + kx] : make_float2(0.f, 0.f);
        const float2 a1 = ea[(size_t)k1 * Q + km], b1 = hb ? ea[PQ + (size_t)k1 * Q + km] : make_float2(0.f, 0.f);
        z = make_float4(a0.x * inv, a0.y * inv, b0.x * inv, b0.y * inv);
        zm = make_float4(a1.x * inv, a1.y * inv, b1.x * inv, b1.y * inv);
      } else {
        z = spectral_noise(ky, kx, a.P, Q, p, fr_noise, a.k0, a.k1);
        zm = make_float4(z.x, -z.y, z.z, -z.w);  // mirror: conjugate noise
      }
      float2 y0 = spectrum(sS[kx], z);
      float2 y1 = spectrum(sS[Q + km], zm);
      if (a.flow) {  // the mirror bin's factor is the conjugate (Hermitian shift factors)
        const float2 ph = cmul(phy, flow_phase(kx, Q, a.vx * (double)fr));
        y0 = cmul(y0, ph);
        y1 = cmul(y1, make_float2(ph.x, -ph.y));
      }
      X[pidx(2 * kx)] = y0;
      X[pidx(2 * km + 1)] = y1;
    }
    __syncthreads();
    const float2* R = smem_ifft<NT>(X, Xb, &fpl, 1);
    float2* dst = a.Zout + (size_t)t * a.npairs * a.P * Q + plane;
    for (int x = threadIdx.x; x < Q; x += NT) {
      dst[(size_t)ky * Q + x] = R[pidx(2 * x)];
      if (k1 != ky) dst[(size_t)k1 * Q + x] = R[pidx(2 * x + 1)];
    }
    __syncthreads();
  }
}

// In-place variant for long rows whose plan has at most one butterfly per thread per pass
// ((Q/R)*2 <= NT): one exchange buffer and the sqrt(S) rows read straight from global memory
// (once per frame and bin) halve the shared memory (4K: 222 -> 95 KB), so two CTAs share
// an SM and one's Philox/butterfly work overlaps the other's barriers and stores.
// QN > 0: the compile-time plan QN = R1 R2 R3 (smem_ifft3_inplace, per-pass twiddles).
template <int NT, bool ETA = false, int QN = 0, int R1 = 1, int R2 = 1, int R3 = 1>
__global__ void __launch_bounds__(NT, 2) k_rows_pair_ip(RowArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int Q = a.Q;
  float2* twq = reinterpret_cast<float2*>(smem);  // [Q] twiddles
  float2* X = twq + Q;                             // [Q][2] interleaved rows (padded)
  __shared__ FFTPlanSmem fpl;
  if constexpr (QN > 0)
    build_twp3<QN, R1, R2, R3>(twq, a.fq.tw);
  else
    stage_fft_plan(&fpl, a.fq, twq);
  const int ky = a.ky0 + (int)blockIdx.x, p = blockIdx.y;
  const int k1 = ky ? a.P - ky : 0;
  const size_t plane = (size_t)p * a.P * Q;
  const float2* sS0 = a.sqrtS + plane + (size_t)ky * Q;
  const float2* sS1 = a.sqrtS + plane + (size_t)k1 * Q;
  __syncthreads();
  for (int t = 0; t < a.F; ++t) {
    const int64_t fr = a.frame0 + t;
    const int64_t fr_noise = a.flow ? 0 : fr;  // frozen flow: one realisation, translated
    const float2 phy = a.flow ? flow_phase(ky, a.P, a.vy * (double)fr) : make_float2(1.f, 0.f);
    for (int kx = threadIdx.x; kx < Q; kx += NT) {
      const int km = kx ? Q - kx : 0;
      float4 z, zm;
      if (ETA) {  // given eta (reading Q8 scaling): zeta = eta / sqrt(PQ/2), each bin read as stored
        const float inv = rsqrtf(0.5f * (float)a.P * (float)Q);
        const size_t PQ = (size_t)a.P * Q;
        const float2* ea = a.eta + ((size_t)t * a.nslots + 2 * p) * PQ;
        const bool hb = 2 * p + 1 < a.nslots;
        const float2 a0 = ea[(size_t)ky * Q + kx], b0 = hb ? ea[PQ + (size_t)ky * Q + kx] : make_float2(0.f, 0.f);
        const float2 a1 = ea[(size_t)k1 * Q + km], b1 = hb ? ea[PQ + (size_t)k1 * Q + km] : make_float2(0.f, 0.f);
        z = make_float4(a0.x * inv, a0.y * inv, b0.x * inv, b0.y * inv);
        zm = make_float4(a1.x * inv, a1.y * inv, b1.x * inv, b1.y * inv);
      } else {
        z = spectral_noise(ky, kx, a.P, Q, p, fr_noise, a.k0, a.k1);
        zm = make_float4(z.x, -z.y, z.z, -z.w);  // mirror: conjugate noise
      }
      float2 y0 = spectrum(__ldg(&sS0[kx]), z);
      float2 y1 = spectrum(__ldg(&sS1[km]), zm);
      if (a.flow) {  // the mirror bin's factor is the conjugate (Hermitian shift factors)
        const float2 ph = cmul(phy, flow_phase(kx, Q, a.vx * (double)fr));
        y0 = cmul(y0, ph);
        y1 = cmul(y1, make_float2(ph.x, -ph.y));
      }
      X[pidx(2 * kx)] = y0;
      X[pidx(2 * km + 1)] = y1;
    }
    __syncthreads();
    if constexpr (QN > 0)
      smem_ifft3_inplace<QN, R1, R2, R3, NT, 1>(X, twq);
    else
      smem_ifft_inplace<NT>(X, &fpl, 1);
    const float2* R = X;
    float2* dst = a.Zout + (size_t)t * a.npairs * a.P * Q + plane;
    for (int x = threadIdx.x; x < Q; x += NT) {
      dst[(size_t)ky * Q + x] = R[pidx(2 * x)];
      if (k1 != ky) dst[(size_t)k1 * Q + x] = R[pidx(2 * x + 1)];
    }
    __syncthreads();
  }
}

// White-noise rows at Q = 512: one CTA per (Hermitian row pair, mode pair); NG groups of
// 64 threads, each group transforms one frame at a time (frames g, g + NG, ...).  Thread t
// owns butterfly t of row ky and butterfly (64 - t) % 64 of row P - ky, which holds exactly
// the mirror bins of its own: one Philox draw feeds both (the mirror takes the conjugate).
template <int NG>
__global__ void __launch_bounds__(64 * NG, 3) k_rows_pair512(RowArgs a) {
  constexpr int N = kRegN, B = kRegB, XL = N + N / 8;
  extern __shared__ __align__(16) unsigned char smem[];
  float2* tw = reinterpret_cast<float2*>(smem);  // [N] per-pass twiddle table (build_twp)
  float2* sS = tw + N;                           // [2][N] sqrt(S) of both rows
  float2* xb = sS + 2 * N;                       // [NG][2][XL] exchange buffers
  const int ky = a.ky0 + (int)blockIdx.x, p = blockIdx.y;
  const int k1 = ky ? a.P - ky : 0;
  const size_t plane = (size_t)p * a.P * N;
  build_twp(tw, a.fq.tw, threadIdx.x, 64 * NG);
  for (int i = threadIdx.x; i < N; i += 64 * NG) {
    sS[i] = __ldg(&a.sqrtS[plane + (size_t)ky * N + i]);
    sS[N + i] = __ldg(&a.sqrtS[plane + (size_t)k1 * N + i]);
  }
  __syncthreads();
  const int g = threadIdx.x >> 6, t = threadIdx.x & (B - 1);
  const int tm = (B - t) & (B - 1);
  float2* x0 = xb + (size_t)g * 2 * XL;
  float2* x1 = x0 + XL;
  auto gsync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(1 + g) : "memory"); };
  auto xi = [](int i) { return i + (i >> 3); };  // exchange padding: conflict-free pass writes
  for (int fi = g; fi < a.F; fi += NG) {
    const int64_t fr = a.frame0 + fi;
    const int64_t fr_noise = a.flow ? 0 : fr;  // frozen flow: one realisation, translated
    float2 phy = make_float2(1.f, 0.f);
    if (a.flow) phy = flow_phase(ky, a.P, a.vy * (double)fr);
    float2 u[8], w[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int kx = t + B * r;
      const float4 z = spectral_noise(ky, kx, a.P, N, p, fr_noise, a.k0, a.k1);
      u[r] = spectrum(sS[kx], z);
      const float4 zc = make_float4(z.x, -z.y, z.z, -z.w);
      // mirror bin (N - kx) % N = tm + 64 (7 - r) for t > 0, 64 ((8 - r) % 8) for t == 0
      const int rm = t ? 7 - r : (8 - r) & 7;
      float2 wv = spectrum(sS[N + tm + B * rm], zc);
      if (a.flow) {  // the mirror bin's factor is the conjugate (Hermitian shift factors)
        const float2 ph = cmul(phy, flow_phase(kx, N, a.vx * (double)fr));
        u[r] = cmul(u[r], ph);
        wv = cmul(wv, make_float2(ph.x, -ph.y));
      }
      if (t)
        w[7 - r] = wv;
      else
        w[(8 - r) & 7] = wv;
    }
    reg_pass_t<1>(u, t, tw);
    reg_pass_t<1>(w, tm, tw);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      x0[xi(reg_out<1>(t, r))] = u[r];
      x1[xi(reg_out<1>(tm, r))] = w[r];
    }
    gsync();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      u[r] = x0[xi(t + B * r)];
      w[r] = x1[xi(tm + B * r)];
    }
    gsync();
    reg_pass_t<8>(u, t, tw);
    reg_pass_t<8>(w, tm, tw);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      x0[xi(reg_out<8>(t, r))] = u[r];
      x1[xi(reg_out<8>(tm, r))] = w[r];
    }
    gsync();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      u[r] = x0[xi(t + B * r)];
      w[r] = x1[xi(tm + B * r)];
    }
    gsync();
    reg_pass_t<64>(u, t, tw);
    reg_pass_t<64>(w, tm, tw);
    float2* dst = a.Zout + (size_t)fi * a.npairs * a.P * N + plane;
#pragma unroll
    for (int r = 0; r < 8; ++r) dst[(size_t)ky * N + t + B * r] = u[r];
    if (k1 != ky) {
#pragma unroll
      for (int r = 0; r < 8; ++r) dst[(size_t)k1 * N + tm + B * r] = w[r];
    }
  }
}

// AR(1) path: one CTA per spectral row with the per-bin state in shared memory;
// frames are evolved sequentially (including the replay of frames before frame0).
template <int NT>
__global__ void __launch_bounds__(NT) k_rows_ar(RowArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int Q = a.Q;
  float4* st = reinterpret_cast<float4*>(smem);  // AR state first: 16-byte aligned
  float2* twq = reinterpret_cast<float2*>(st + Q);
  float2* sS = twq + Q;
  float2* X = sS + Q;
  float2* Xb = X + padded_len(Q);
  __shared__ FFTPlanSmem fpl;
  stage_fft_plan(&fpl, a.fq, twq);
  const int ky = a.ky0 + (int)blockIdx.x, p = blockIdx.y;
  const size_t row = ((size_t)p * a.P + ky) * Q;
  for (int kx = threadIdx.x; kx < Q; kx += NT) {
    sS[kx] = a.sqrtS[row + kx];
    if (a.load_state) st[kx] = a.ar[row + kx];
  }
  __syncthreads();
  const int64_t t_end = a.frame0 + a.F;
  for (int64_t t = a.t_start; t < t_end; ++t) {
    const bool out = t >= a.frame0;
    for (int kx = threadIdx.x; kx < Q; kx += NT) {
      float4 z = spectral_noise(ky, kx, a.P, Q, p, t, a.k0, a.k1);
      if (t > 0) {
        const float4 o = st[kx];
        z = make_float4(a.alpha * o.x + a.calpha * z.x, a.alpha * o.y + a.calpha * z.y,
                        a.alpha * o.z + a.calpha * z.z, a.alpha * o.w + a.calpha * z.w);
      }
      st[kx] = z;
      if (out) X[pidx(kx)] = spectrum(sS[kx], z);
    }
    if (!out) continue;  // replay: state only
    __syncthreads();
    const float2* R = smem_ifft<NT>(X, Xb, &fpl, 0);
    float2* dst = a.Zout + (size_t)(t - a.frame0) * a.npairs * a.P * Q + row;
    for (int x = threadIdx.x; x < Q; x += NT) dst[x] = R[pidx(x)];
    __syncthreads();
  }
  __syncthreads();
  for (int kx = threadIdx.x; kx < Q; kx += NT) a.ar[row + kx] = st[kx];
}

// AR(1) path, Hermitian row pairs: one CTA per row pair {ky, P-ky} as in k_rows_pair.  The
// state of a mirror bin is the conjugate of its canonical bin's (the draws are conjugate and
// the recursion has real coefficients, so this holds exactly, negation being exact), so the
// CTA keeps only row ky's state, in registers (bins kx = tid + NT i, MB per thread), draws
// Philox once per bin pair and feeds the mirror row with the conjugate.  Half the draws and
// half the state traffic of k_rows_ar; the same values up to the FFT's rounding order.
// It pays where the rows are long (Q > 1024: 4K AR rows 5.48 -> 3.84 ms, 1080p 3.89 -> 3.56
// per launch).  Rows of up to 512 points run it with 128-thread CTAs (MB = 4 bins per
// thread): at Q = 256 (cfg2, 100 sequential frames per CTA) that beats both k_rows_ar
// (1.38 vs 1.57 ms) and 256-thread pair CTAs (1.84 ms, half the CTAs); 512 < Q <= 1024
// keeps k_rows_ar (rows_variant).  128 registers, no spills (an 80-register cap spills and
// is slower at 1080p).
// QN > 0: compile-time in-place plan QN = R1 R2 R3 (one exchange buffer, per-pass twiddles).
template <int NT, int MB, int QN = 0, int R1 = 1, int R2 = 1, int R3 = 1>
__global__ void __launch_bounds__(NT) k_rows_ar_pair(RowArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int Q = a.Q;
  float2* twq = reinterpret_cast<float2*>(smem);  // [Q] twiddles
  float2* sS = twq + Q;                            // [2][Q]
  float2* X = sS + 2 * Q;                          // [Q][2] interleaved rows (padded)
  float2* Xb = X + padded_len(2 * Q);
  __shared__ FFTPlanSmem fpl;
  if constexpr (QN > 0)
    build_twp3<QN, R1, R2, R3>(twq, a.fq.tw);
  else
    stage_fft_plan(&fpl, a.fq, twq);
  const int ky = a.ky0 + (int)blockIdx.x, p = blockIdx.y;
  const int k1 = ky ? a.P - ky : 0;
  const size_t plane = (size_t)p * a.P * Q;
  const size_t row = plane + (size_t)ky * Q, rowm = plane + (size_t)k1 * Q;
  for (int kx = threadIdx.x; kx < Q; kx += NT) {
    sS[kx] = a.sqrtS[row + kx];
    sS[Q + kx] = a.sqrtS[rowm + kx];
  }
  float4 st[MB];
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int kx = threadIdx.x + NT * i;
    st[i] = (a.load_state && kx < Q) ? a.ar[row + kx] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  const int64_t t_end = a.frame0 + a.F;
  for (int64_t t = a.t_start; t < t_end; ++t) {
    const bool out = t >= a.frame0;
#pragma unroll
    for (int i = 0; i < MB; ++i) {
      const int kx = threadIdx.x + NT * i;
      if (kx < Q) {
        float4 z = spectral_noise(ky, kx, a.P, Q, p, t, a.k0, a.k1);
        if (t > 0) {
          const float4 o = st[i];
          z = make_float4(a.alpha * o.x + a.calpha * z.x, a.alpha * o.y + a.calpha * z.y,
                          a.alpha * o.z + a.calpha * z.z, a.alpha * o.w + a.calpha * z.w);
        }
        st[i] = z;
        if (out) {
          const int km = kx ? Q - kx : 0;
          X[pidx(2 * kx)] = spectrum(sS[kx], z);
          X[pidx(2 * km + 1)] = spectrum(sS[Q + km], make_float4(z.x, -z.y, z.z, -z.w));
        }
      }
    }
    if (!out) continue;  // replay: state only
    __syncthreads();
    const float2* R;
    if constexpr (QN > 0) {
      smem_ifft3_inplace<QN, R1, R2, R3, NT, 1>(X, twq);
      R = X;
    } else {
      R = smem_ifft<NT>(X, Xb, &fpl, 1);
    }
    float2* dst = a.Zout + (size_t)(t - a.frame0) * a.npairs * a.P * Q + plane;
    for (int x = threadIdx.x; x < Q; x += NT) {
      dst[(size_t)ky * Q + x] = R[pidx(2 * x)];
      if (k1 != ky) dst[(size_t)k1 * Q + x] = R[pidx(2 * x + 1)];
    }
    __syncthreads();
  }
  // Write back both rows (the mirror row as the conjugate) so the stored state is complete.
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int kx = threadIdx.x + NT * i;
    if (kx < Q) {
      const float4 z = st[i];
      a.ar[row + kx] = z;
      a.ar[rowm + (kx ? Q - kx : 0)] = make_float4(z.x, -z.y, z.z, -z.w);
    }
  }
}

// The 512-point register fast path needs a 512-point axis planned as radix 8 x 8 x 8.
static bool reg512(const AxisFFT& ax) {
  return ax.N == kRegN && ax.nrad == 3 && ax.rad[0] == 8 && ax.rad[1] == 8 && ax.rad[2] == 8;
}

// MLP input layout shared by its producers (k_cols*, k_zern_to_x) and k_mlp, decided once
// at plan creation (p2s_plan_s::xtile).  Octet-pair tiles (x_index, xtile 2) from 1M pixels
// per frame (1080p, 4K): contiguous 9 KB tile blocks (r1 measured 2.05 -> 1.36 ms at 4K for
// the tile-major layout against planes), the long-column kernel's stores unchanged, and
// k_mlp's TMA box over them (r2) 1.20 ms at 1080p against 1.45 for planes with per-thread
// copies and 2.28 for planes by TMA (35 plane rows 4 MB apart per box); planes at 512^2
// and below, where k_cols512 writes one column per thread and the tiled addressing cost it
// 0.13 ms (octets + TMA at 512^2: k_mlp 1.24 vs 1.28, k_cols 1.24 vs 1.10).
// P2S_FORCE_X_PLANES / _X_TILES / _X_OCTETS force a layout.
int x_tile_layout(const p2s_plan_s* pl) {
  if (pl->force & P2S_FORCE_X_PLANES) return 0;
  if (pl->force & P2S_FORCE_X_TILES) return 1;
  if (pl->force & P2S_FORCE_X_OCTETS) return 2;
  return (size_t)pl->H * pl->W >= ((size_t)1 << 20) ? 2 : 0;
}

// Row-pass kernel variants (one per dispatch outcome of rows_variant).
enum RowVariant {
  RV_GIVEN_NOISE,   // k_rows_pair<256, true>: caller-supplied spectral noise
  RV_AR_PAIR_128,   // k_rows_ar_pair<128, 4>: AR(1), Q <= 512
  RV_AR_PAIR_256_1, RV_AR_PAIR_256_2, RV_AR_PAIR_256_4, RV_AR_PAIR_512_4, RV_AR_PAIR_512_8,
  RV_AR_PAIR_3840, RV_AR_PAIR_1920,  // k_rows_ar_pair with the compile-time in-place plans
  RV_AR_ROW_128, RV_AR_ROW_512,  // k_rows_ar<NT>: one CTA per spectral row
  RV_REG512,        // k_rows_pair512<4>
  RV_PAIR_IP_512,   // k_rows_pair_ip<512>: in place, long rows
  RV_PAIR_IP_3840,  // k_rows_pair_ip<512, false, 3840, 16, 16, 15>: compile-time plan
  RV_PAIR_IP_1920,  // k_rows_pair_ip<512, false, 1920, 16, 15, 8>
  RV_PAIR_256, RV_PAIR_512  // k_rows_pair<NT>: ping-pong
};

static size_t smem_pair(int Q) { return ((size_t)3 * Q + 2 * padded_len(2 * (size_t)Q)) * sizeof(float2); }
static size_t smem_ar_row(int Q) {
  return ((size_t)2 * Q + 2 * padded_len(Q)) * sizeof(float2) + (size_t)Q * sizeof(float4) + 16;
}
static size_t smem_pair_ip(int Q) { return ((size_t)Q + padded_len(2 * (size_t)Q)) * sizeof(float2); }
constexpr size_t kSmemMax = 227 * 1024;

// The row kernel the plan runs for white noise / AR(1) / given noise, and its dynamic shared
// memory.  Where the preferred kernel would exceed the per-CTA limit the next one that fits
// is taken; plan creation rejects a plan whose row pass fits none (rows_smem_bytes).
static RowVariant rows_variant(const p2s_plan_s* pl, bool ar, bool given, size_t* sm) {
  const int Q = pl->Q, NTp = Q > 1024 ? 512 : 256, mb = (Q + NTp - 1) / NTp;
  if (given) {
    *sm = smem_pair(Q);
    return RV_GIVEN_NOISE;
  }
  // in place: every pass at most one butterfly per thread (two interleaved rows)
  bool one = true;
  for (int i = 0; i < pl->fq.nrad; ++i) one = one && (Q / pl->fq.rad[i]) * 2 <= 512;
  if (ar) {
    // 1: always k_rows_ar, 2: the 256/512-thread pair kernel (P2S_FORCE_AR_*)
    int ar_rows = (pl->force & P2S_FORCE_AR_ROW_KERNEL) ? 1 : (pl->force & P2S_FORCE_AR_PAIR_KERNEL) ? 2 : 0;
    // slab mode: the row-pair kernels transform only this rank's pairs; the one-CTA-per-row
    // kernel (still correct: every row, of which the pack takes this rank's) only if no
    // pair kernel fits
    if (pl->slab_G > 1 && ar_rows == 0 && Q > 512) ar_rows = 2;
    if (ar_rows == 0 && Q <= 512) {
      // short rows: 128-thread row-pair CTAs keep the grid's CTA count up where each CTA
      // runs a long frame sequence (cfg2, Q = 256, 100 frames: 1.57 -> 1.38 ms vs k_rows_ar;
      // 256-thread pair CTAs 1.84 ms)
      *sm = smem_pair(Q);
      return RV_AR_PAIR_128;
    }
    const auto& rq = pl->fq;
    if (ar_rows != 1 && !(pl->force & P2S_FORCE_FFT_GENERIC) && rq.nrad == 3) {
      const size_t sm_ip = ((size_t)3 * Q + padded_len(2 * (size_t)Q)) * sizeof(float2);
      if (Q == 3840 && rq.rad[0] == 16 && rq.rad[1] == 16 && rq.rad[2] == 15) {
        *sm = sm_ip;
        return RV_AR_PAIR_3840;
      }
      if (Q == 1920 && rq.rad[0] == 16 && rq.rad[1] == 15 && rq.rad[2] == 8) {
        *sm = sm_ip;
        return RV_AR_PAIR_1920;
      }
    }
    if (mb <= 8 && ar_rows != 1 && (Q > 1024 || ar_rows == 2) && smem_pair(Q) <= kSmemMax) {
      *sm = smem_pair(Q);
      if (NTp == 512) return mb <= 4 ? RV_AR_PAIR_512_4 : RV_AR_PAIR_512_8;
      return mb <= 1 ? RV_AR_PAIR_256_1 : mb <= 2 ? RV_AR_PAIR_256_2 : RV_AR_PAIR_256_4;
    }
    *sm = smem_ar_row(Q);
    return Q > 1024 ? RV_AR_ROW_512 : RV_AR_ROW_128;
  }
  if (reg512(pl->fq) && !(pl->force & P2S_FORCE_FFT_GENERIC)) {
    *sm = ((size_t)3 * kRegN + (size_t)4 * 2 * (kRegN + kRegN / 8)) * sizeof(float2);
    return RV_REG512;
  }
  // in place only where the ping-pong kernel fits one CTA per SM (4K: 222 KB; at 1920
  // points it already fits two, and the in-place variant measured slower there: 2.94 vs
  // 2.50 ms), or does not fit at all (4096 = 16 x 16 x 16)
  // compile-time in-place plans for the BASELINE row lengths (per-pass twiddles, constant
  // index arithmetic): two CTAs per SM at both
  const auto& rq = pl->fq;
  if (!(pl->force & (P2S_FORCE_ROWS_PINGPONG | P2S_FORCE_FFT_GENERIC)) && rq.nrad == 3) {
    if (Q == 3840 && rq.rad[0] == 16 && rq.rad[1] == 16 && rq.rad[2] == 15) {
      *sm = smem_pair_ip(Q);
      return RV_PAIR_IP_3840;
    }
    if (Q == 1920 && rq.rad[0] == 16 && rq.rad[1] == 15 && rq.rad[2] == 8) {
      *sm = smem_pair_ip(Q);
      return RV_PAIR_IP_1920;
    }
  }
  if (Q > 1024 && 2 * smem_pair(Q) > kSmemMax && one && !(pl->force & P2S_FORCE_ROWS_PINGPONG)) {
    *sm = smem_pair_ip(Q);
    return RV_PAIR_IP_512;
  }
  *sm = smem_pair(Q);
  return Q > 1024 ? RV_PAIR_512 : RV_PAIR_256;
}

size_t rows_smem_bytes(const p2s_plan_s* pl, bool ar, bool given_noise) {
  size_t sm = 0;
  rows_variant(pl, ar, given_noise, &sm);
  return sm;
}

template <int NT, int MB, int QN = 0, int R1 = 1, int R2 = 1, int R3 = 1>
static int launch_rows_ar_pair(const RowArgs& a, int npr, int npairs, size_t sm, cudaStream_t s) {
  dim3 grid(npr, npairs);  // Hermitian row pairs [a.ky0, a.ky0 + npr)
  P2S_SMEM_OPTIN((k_rows_ar_pair<NT, MB, QN, R1, R2, R3>), sm);
  k_rows_ar_pair<NT, MB, QN, R1, R2, R3><<<grid, NT, sm, s>>>(a);
  return (int)cudaGetLastError();
}

int launch_rows(const p2s_plan_s* pl, uint64_t seed, int64_t frame0, int F, bool ar, int ar_mode,
                int64_t replay_from, cudaStream_t s, const float2* eta) {
  RowArgs a;
  fill_fft_args(a.fq, pl->fq);
  a.sqrtS = pl->d_sqrtS;
  a.ar = pl->d_ar;
  a.Zout = pl->d_Z;
  a.P = pl->P;
  a.Q = pl->Q;
  a.npairs = pl->npairs;
  a.k0 = (uint32_t)seed;
  a.k1 = (uint32_t)(seed >> 32);
  a.frame0 = frame0;
  a.F = F;
  a.alpha = pl->ar_alpha;
  a.calpha = sqrtf(1.0f - pl->ar_alpha * pl->ar_alpha);
  a.t_start = ar ? replay_from : frame0;
  a.load_state = (ar && ar_mode == 0) ? 1 : 0;
  a.flow = (pl->flow_vx != 0.0 || pl->flow_vy != 0.0) ? 1 : 0;
  a.vx = pl->flow_vx;
  a.vy = pl->flow_vy;
  a.eta = eta;
  a.nslots = pl->nslots;
  if (eta) a.flow = 0;  // caller-supplied noise: generic row kernel, no AR state, no flow
  size_t sm = 0;
  const RowVariant v = rows_variant(pl, ar, eta != nullptr, &sm);
  if (sm > kSmemMax) return (int)cudaErrorInvalidConfiguration;
  // slab mode: this rank's Hermitian row pairs [kp0, kp1) only (white noise)
  a.ky0 = pl->slab_G > 1 ? pl->slab_kp0 : 0;
  const int npr = pl->slab_G > 1 ? pl->slab_kp1 - pl->slab_kp0 : pl->P / 2 + 1;
  if (npr <= 0) return 0;
  const dim3 gpair(npr, pl->npairs), grow(pl->P, pl->npairs);
  switch (v) {
    case RV_GIVEN_NOISE:
      P2S_SMEM_OPTIN((k_rows_pair<256, true>), sm);
      k_rows_pair<256, true><<<gpair, 256, sm, s>>>(a);
      break;
    case RV_AR_PAIR_128: return launch_rows_ar_pair<128, 4>(a, npr, pl->npairs, sm, s);
    case RV_AR_PAIR_256_1: return launch_rows_ar_pair<256, 1>(a, npr, pl->npairs, sm, s);
    case RV_AR_PAIR_256_2: return launch_rows_ar_pair<256, 2>(a, npr, pl->npairs, sm, s);
    case RV_AR_PAIR_256_4: return launch_rows_ar_pair<256, 4>(a, npr, pl->npairs, sm, s);
    case RV_AR_PAIR_512_4: return launch_rows_ar_pair<512, 4>(a, npr, pl->npairs, sm, s);
    case RV_AR_PAIR_512_8: return launch_rows_ar_pair<512, 8>(a, npr, pl->npairs, sm, s);
    case RV_AR_PAIR_3840: return launch_rows_ar_pair<512, 8, 3840, 16, 16, 15>(a, npr, pl->npairs, sm, s);
    case RV_AR_PAIR_1920: return launch_rows_ar_pair<512, 4, 1920, 16, 15, 8>(a, npr, pl->npairs, sm, s);
    case RV_AR_ROW_512:
      a.ky0 = 0;  // one CTA per row over all P rows (slab mode: the pack takes this rank's)
      P2S_SMEM_OPTIN(k_rows_ar<512>, sm);
      k_rows_ar<512><<<grow, 512, sm, s>>>(a);
      break;
    case RV_AR_ROW_128:
      a.ky0 = 0;
      P2S_SMEM_OPTIN(k_rows_ar<128>, sm);
      k_rows_ar<128><<<grow, 128, sm, s>>>(a);
      break;
    case RV_REG512:
      P2S_SMEM_OPTIN(k_rows_pair512<4>, sm);
      k_rows_pair512<4><<<gpair, 64 * 4, sm, s>>>(a);
      break;
    case RV_PAIR_IP_512:
      P2S_SMEM_OPTIN(k_rows_pair_ip<512>, sm);
      k_rows_pair_ip<512><<<gpair, 512, sm, s>>>(a);
      break;
    case RV_PAIR_IP_3840:
      P2S_SMEM_OPTIN((k_rows_pair_ip<512, false, 3840, 16, 16, 15>), sm);
      k_rows_pair_ip<512, false, 3840, 16, 16, 15><<<gpair, 512, sm, s>>>(a);
      break;
    case RV_PAIR_IP_1920:
      P2S_SMEM_OPTIN((k_rows_pair_ip<512, false, 1920, 16, 15, 8>), sm);
      k_rows_pair_ip<512, false, 1920, 16, 15, 8><<<gpair, 512, sm, s>>>(a);
      break;
    case RV_PAIR_512:
      P2S_SMEM_OPTIN((k_rows_pair<512>), sm);
      k_rows_pair<512><<<gpair, 512, sm, s>>>(a);
      break;
    case RV_PAIR_256:
      P2S_SMEM_OPTIN((k_rows_pair<256>), sm);
      k_rows_pair<256><<<gpair, 256, sm, s>>>(a);
      break;
  }
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ K2: column IDFT
struct ColArgs {
  FFTArgs fp;
  const float2* Zin;  // [F][npairs][P][Q]
  int P, Q, H, W, npairs, nslots, Z;
  int F;  // frames (the persistent column kernel's tile count)
  int ntx, xtile;  // MLP input layout (x_index)
  int tc_log2;
  float* zern;        // mode 0: [F][Z][H][W]
  uint16_t* X;        // mode 1: bf16 [F][nslots][H*W]
  float* tilt;        // mode 1: [F][2][H*W]
  // mode 1, fused step 2 (512-point columns): the mode-pair-0 CTAs hold f_2, f_3 and warp
  // the image directly (no tilt planes): Iw(x) = bilinear(I, x + (cx f2, cy0 f2 + cy1 f3))
  int fuse_warp;
  const float* img;   // [F or 1][C][H][W]
  int64_t img_stride; // floats between frames (0 = broadcast)
  int C;
  float cx, cy0, cy1;
  uint16_t* Iw;       // bf16 [F][C][H][W]
};

// Step 2 at one pixel (the arithmetic of k_warp: clamp-to-edge bilinear gather).
__device__ __forceinline__ void warp_pixel(const ColArgs& a, int f, int y, int x, float u, float v) {
  const int HW = a.H * a.W;
  const float X = (float)x + a.cx * u;
  const float Y = (float)y + a.cy0 * u + a.cy1 * v;
  const float fx = floorf(X), fy = floorf(Y);
  const float tx = X - fx, ty = Y - fy;
  int xa = (int)fmaxf(fminf(fx, (float)(a.W - 1)), -1.f);
  int ya = (int)fmaxf(fminf(fy, (float)(a.H - 1)), -1.f);
  const int xb = min(xa + 1, a.W - 1), yb = min(ya + 1, a.H - 1);
  xa = max(xa, 0);
  ya = max(ya, 0);
  const float* I = a.img + (size_t)f * a.img_stride;
  const int pix = y * a.W + x;
#pragma unroll 1
  for (int c = 0; c < a.C; ++c) {
    const float* Ic = I + (size_t)c * HW;
    const float i00 = __ldg(&Ic[ya * a.W + xa]), i01 = __ldg(&Ic[ya * a.W + xb]);
    const float i10 = __ldg(&Ic[yb * a.W + xa]), i11 = __ldg(&Ic[yb * a.W + xb]);
    const float val = (1.f - ty) * ((1.f - tx) * i00 + tx * i01) + ty * ((1.f - tx) * i10 + tx * i11);
    a.Iw[((size_t)f * a.C + c) * HW + pix] = f_to_bf16(val);
  }
}

template <int MODE, int NT>
__global__ void __launch_bounds__(NT) k_cols(ColArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int TC = 1 << a.tc_log2;
  float2* twp = reinterpret_cast<float2*>(smem);
  float2* X = twp + a.P;
  float2* Xb = X + padded_len((size_t)a.P << a.tc_log2);
  __shared__ FFTPlanSmem fpl;
  stage_fft_plan(&fpl, a.fp, twp);
  const int x0 = blockIdx.x * TC, p = blockIdx.y, f = blockIdx.z;
  const float2* src = a.Zin + ((size_t)f * a.npairs + p) * a.P * a.Q;
  const int n = a.P << a.tc_log2;
  constexpr int U = 8;  // batch the global loads so they are in flight together
  for (int w0 = threadIdx.x; w0 < n; w0 += NT * U) {
    float2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int w = w0 + u * NT;
      const int c = w & (TC - 1), ky = w >> a.tc_log2;
      const int x = x0 + c;
      v[u] = (w < n && x < a.Q) ? __ldg(&src[(size_t)ky * a.Q + x]) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int w = w0 + u * NT;
      if (w < n) X[pidx(w)] = v[u];
    }
  }
  __syncthreads();
  const float2* R = smem_ifft<NT>(X, Xb, &fpl, a.tc_log2);
  const int sa = 2 * p, sb = 2 * p + 1;
  const size_t HW = (size_t)a.H * a.W;
  const int m = a.H << a.tc_log2;
  for (int w = threadIdx.x; w < m; w += NT) {
    const int c = w & (TC - 1), yy = w >> a.tc_log2;
    const int x = x0 + c;
    if (x >= a.W) continue;
    const float2 v = R[pidx(w)];
    const size_t pix = (size_t)yy * a.W + x;
    if (MODE == 0) {
      float* z = a.zern + (size_t)f * a.Z * HW;
      z[(size_t)(sa + 1) * HW + pix] = v.x;
      if (sb < a.nslots) z[(size_t)(sb + 1) * HW + pix] = v.y;
    } else {
      if (a.xtile) {  // tile-major (x_index); the plane path below keeps its cheaper addressing
        uint16_t* Xt = a.X + x_index(a.xtile, f, sa, a.nslots, a.H, a.W, a.ntx, yy, x);
        Xt[0] = f_to_bf16(v.x);
        if (sb < a.nslots) Xt[a.xtile == 2 ? 8 : 128] = f_to_bf16(v.y);
      } else {
        uint16_t* Xo = a.X + (size_t)f * a.nslots * HW;
        Xo[(size_t)sa * HW + pix] = f_to_bf16(v.x);
        if (sb < a.nslots) Xo[(size_t)sb * HW + pix] = f_to_bf16(v.y);
      }
      if (p == 0) {
        float* t = a.tilt + (size_t)f * 2 * HW;
        t[pix] = v.x;
        t[HW + pix] = v.y;
      }
    }
  }
}

__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Long columns (1080p / 4K), in place, two CTAs per SM: one CTA per (block of TC = 2^TCL
// columns, mode pair, frame), one shared buffer transformed in place (every pass has at
// most one butterfly per thread, (P / R) TC <= NT), twiddles staged in shared memory.  The
// second resident CTA's loads and stores overlap this one's barrier-separated passes (the
// persistent single-CTA kernel below serialises them: its transform phase is
// barrier-bound).  Each thread then writes the TC adjacent columns of a row with one
// vector store per output plane (TC bf16 = 4 or 8 bytes, TC fp32 tilt / zern values).
// PN > 0: the compile-time plan PN = R1 R2 R3 (smem_ifft3_inplace), else the runtime plan.
template <int MODE, int NT, int TCL, int PN = 0, int R1 = 1, int R2 = 1, int R3 = 1>
__global__ void __launch_bounds__(NT, NT <= 512 ? 2 : 1) k_cols_ip(ColArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int TC = 1 << TCL;
  float2* twp = reinterpret_cast<float2*>(smem);
  float2* X = twp + a.P;
  __shared__ FFTPlanSmem fpl;
  if constexpr (PN > 0)
    build_twp3<PN, R1, R2, R3>(twp, a.fp.tw);
  else
    stage_fft_plan(&fpl, a.fp, twp);
  const int x0 = blockIdx.x * TC, p = blockIdx.y, f = blockIdx.z;
  const float2* src = a.Zin + ((size_t)f * a.npairs + p) * a.P * a.Q + x0;
  const bool full = x0 + TC <= a.Q && (a.Q & 1) == 0;  // 16-byte loads need an even row length
  // loads: row ky of the block is TC consecutive float2 (16 or 32 bytes)
  constexpr int U = 4;
  for (int r0 = threadIdx.x; r0 < a.P * (TC / 2); r0 += NT * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u * NT;
      const int ky = r / (TC / 2), h = r % (TC / 2);
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < a.P * (TC / 2)) {
        if (full) {
          v[u] = __ldg(reinterpret_cast<const float4*>(src + (size_t)ky * a.Q) + h);
        } else {
          if (x0 + 2 * h < a.Q) {
            const float2 e = __ldg(src + (size_t)ky * a.Q + 2 * h);
            v[u].x = e.x;
            v[u].y = e.y;
          }
          if (x0 + 2 * h + 1 < a.Q) {
            const float2 e = __ldg(src + (size_t)ky * a.Q + 2 * h + 1);
            v[u].z = e.x;
            v[u].w = e.y;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u * NT;
      if (r < a.P * (TC / 2)) {
        const int w = 2 * r;  // element index (ky << TCL) + 2 h
        X[pidx(w)] = make_float2(v[u].x, v[u].y);
        X[pidx(w + 1)] = make_float2(v[u].z, v[u].w);
      }
    }
  }
  __syncthreads();
  if constexpr (PN > 0)
    smem_ifft3_inplace<PN, R1, R2, R3, NT, TCL>(X, twp);
  else
    smem_ifft_inplace<NT>(X, &fpl, TCL);
  const int sa = 2 * p, sb = 2 * p + 1;
  const size_t HW = (size_t)a.H * a.W;
  const bool vec = (a.W % TC == 0) && x0 + TC <= a.W;
  for (int yy = threadIdx.x; yy < a.H; yy += NT) {
    float2 v[TC];
#pragma unroll
    for (int c = 0; c < TC; ++c) v[c] = X[pidx((yy << TCL) + c)];
    const size_t pix = (size_t)yy * a.W + x0;
    if (MODE == 0) {
      float* za = a.zern + ((size_t)f * a.Z + sa + 1) * HW + pix;
      float* zb = a.zern + ((size_t)f * a.Z + sb + 1) * HW + pix;
      const bool hb = sb < a.nslots;
      if (vec) {
        if (TC == 2) {
          *reinterpret_cast<float2*>(za) = make_float2(v[0].x, v[1].x);
          if (hb) *reinterpret_cast<float2*>(zb) = make_float2(v[0].y, v[1].y);
        } else {
#pragma unroll
          for (int c = 0; c < TC; c += 4) {
            *reinterpret_cast<float4*>(za + c) = make_float4(v[c].x, v[c + 1].x, v[c + 2].x, v[c + 3].x);
            if (hb) *reinterpret_cast<float4*>(zb + c) = make_float4(v[c].y, v[c + 1].y, v[c + 2].y, v[c + 3].y);
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < TC; ++c)
          if (x0 + c < a.W) {
            za[c] = v[c].x;
            if (hb) zb[c] = v[c].y;
          }
      }
    } else {
      uint16_t* Xa = a.X + x_index(a.xtile, f, sa, a.nslots, a.H, a.W, a.ntx, yy, x0);
      // the second mode of the pair: the next plane (planes) or the next 128-pixel row of the tile
      const size_t db = a.xtile == 2 ? 8 : a.xtile ? 128 : HW;
      const bool hb = sb < a.nslots;
      if (vec) {
        uint32_t ua[TC / 2], ub[TC / 2];
#pragma unroll
        for (int c = 0; c < TC; c += 2) {
          ua[c / 2] = pack_bf16x2(v[c].x, v[c + 1].x);
          ub[c / 2] = pack_bf16x2(v[c].y, v[c + 1].y);
        }
        if (TC == 2) {
          *reinterpret_cast<uint32_t*>(Xa) = ua[0];
          if (hb) *reinterpret_cast<uint32_t*>(Xa + db) = ub[0];
        } else {
#pragma unroll
          for (int c = 0; c < TC; c += 4) {
            *reinterpret_cast<uint2*>(Xa + c) = make_uint2(ua[c / 2], ua[c / 2 + 1]);
            if (hb) *reinterpret_cast<uint2*>(Xa + db + c) = make_uint2(ub[c / 2], ub[c / 2 + 1]);
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < TC; ++c)
          if (x0 + c < a.W) {
            Xa[c] = f_to_bf16(v[c].x);
            if (hb) Xa[db + c] = f_to_bf16(v[c].y);
          }
      }
      if (p == 0) {
        float* t = a.tilt + (size_t)f * 2 * HW + pix;
        if (vec && TC == 2) {
          *reinterpret_cast<float2*>(t) = make_float2(v[0].x, v[1].x);
          *reinterpret_cast<float2*>(t + HW) = make_float2(v[0].y, v[1].y);
        } else if (vec) {
#pragma unroll
          for (int c = 0; c < TC; c += 4) {
            *reinterpret_cast<float4*>(t + c) = make_float4(v[c].x, v[c + 1].x, v[c + 2].x, v[c + 3].x);
            *reinterpret_cast<float4*>(t + HW + c) = make_float4(v[c].y, v[c + 1].y, v[c + 2].y, v[c + 3].y);
          }
        } else {
#pragma unroll
          for (int c = 0; c < TC; ++c)
            if (x0 + c < a.W) {
              t[c] = v[c].x;
              t[HW + c] = v[c].y;
            }
        }
      }
    }
  }
}

// Long columns (1080p / 4K), persistent: one CTA per SM walks the column blocks; the next
// block's loads (cp.async, zero-filled past Q) land in the second buffer while the current
// block is transformed in place (smem_ifft_inplace) and written out.  k_cols runs one
// 164 KB CTA per SM whose load, transform and store phases serialise (ncu at 4K: DRAM 11%
// of peak, stalls on the load scoreboard and on barriers).
template <int MODE, int NT>
__global__ void __launch_bounds__(NT) k_cols_p(ColArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int TC = 1 << a.tc_log2;
  float2* twp = reinterpret_cast<float2*>(smem);
  float2* Xw = twp + a.P;
  float2* Xn = Xw + padded_len((size_t)a.P << a.tc_log2);
  __shared__ FFTPlanSmem fpl;
  stage_fft_plan(&fpl, a.fp, twp);
  const int nxb = (a.W + TC - 1) / TC;
  const int ntiles = nxb * a.npairs * a.F;
  const int n = a.P << a.tc_log2;
  auto prefetch = [&](int tile, float2* dst) {
    const int xk = tile % nxb, r = tile / nxb;
    const int p = r % a.npairs, f = r / a.npairs;
    const float2* src = a.Zin + ((size_t)f * a.npairs + p) * a.P * a.Q;
    for (int w = threadIdx.x; w < n; w += NT) {
      const int c = w & (TC - 1), ky = w >> a.tc_log2;
      const int x = xk * TC + c;
      cp_async8(dst + pidx(w), x < a.Q ? &src[(size_t)ky * a.Q + x] : src, x < a.Q ? 8u : 0u);
    }
    cp_async_commit();
  };
  if ((int)blockIdx.x < ntiles) prefetch(blockIdx.x, Xw);
  const size_t HW = (size_t)a.H * a.W;
  const int m = a.H << a.tc_log2;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    cp_async_wait<0>();
    __syncthreads();  // this block landed; every thread is done with the previous one (Xn)
    if (tile + (int)gridDim.x < ntiles) prefetch(tile + gridDim.x, Xn);
    smem_ifft_inplace<NT>(Xw, &fpl, a.tc_log2);
    const int xk = tile % nxb, r = tile / nxb;
    const int p = r % a.npairs, f = r / a.npairs;
    const int x0 = xk * TC, sa = 2 * p, sb = 2 * p + 1;
    for (int w = threadIdx.x; w < m; w += NT) {
      const int c = w & (TC - 1), yy = w >> a.tc_log2;
      const int x = x0 + c;
      if (x >= a.W) continue;
      const float2 v = Xw[pidx(w)];
      const size_t pix = (size_t)yy * a.W + x;
      if (MODE == 0) {
        float* z = a.zern + (size_t)f * a.Z * HW;
        z[(size_t)(sa + 1) * HW + pix] = v.x;
        if (sb < a.nslots) z[(size_t)(sb + 1) * HW + pix] = v.y;
      } else {
        if (a.xtile) {  // tile-major (x_index)
          uint16_t* Xt = a.X + x_index(a.xtile, f, sa, a.nslots, a.H, a.W, a.ntx, yy, x);
          Xt[0] = f_to_bf16(v.x);
          if (sb < a.nslots) Xt[a.xtile == 2 ? 8 : 128] = f_to_bf16(v.y);
        } else {
          uint16_t* Xo = a.X + (size_t)f * a.nslots * HW;
          Xo[(size_t)sa * HW + pix] = f_to_bf16(v.x);
          if (sb < a.nslots) Xo[(size_t)sb * HW + pix] = f_to_bf16(v.y);
        }
        if (p == 0) {
          float* t = a.tilt + (size_t)f * 2 * HW;
          t[pix] = v.x;
          t[HW + pix] = v.y;
        }
      }
    }
    float2* t = Xw;
    Xw = Xn;
    Xn = t;
  }
}

// Column IDFT at P = 512: 16 interleaved columns per CTA, 512 threads; thread (c, jj) owns
// butterflies jj and jj + 32 of column c (16 independent 8-byte loads in flight per thread,
// 128-byte row segments per half-warp).  Exchange buffer column-interleaved (x[i*16 + c]):
// every half-warp access is 128 contiguous bytes.
template <int MODE>
__global__ void __launch_bounds__(512) k_cols512(ColArgs a) {
  constexpr int N = kRegN, B = kRegB, TC = 16;
  extern __shared__ __align__(16) unsigned char smem[];
  float2* tw = reinterpret_cast<float2*>(smem);  // [N]
  float2* xb = tw + N;                           // [N][TC]
  for (int i = threadIdx.x; i < N; i += 512) tw[i] = __ldg(&a.fp.tw[i]);
  const int c = threadIdx.x & (TC - 1), jj = threadIdx.x >> 4;
  const int x0 = blockIdx.x * TC, p = blockIdx.y, f = blockIdx.z;
  const int x = x0 + c;
  const float2* src = a.Zin + ((size_t)f * a.npairs + p) * (size_t)N * a.Q + x;
  float2 u[8], w[8];
  const bool xin = x < a.Q;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    u[r] = xin ? __ldg(src + (size_t)(jj + B * r) * a.Q) : make_float2(0.f, 0.f);
    w[r] = xin ? __ldg(src + (size_t)(jj + 32 + B * r) * a.Q) : make_float2(0.f, 0.f);
  }
  __syncthreads();  // twiddles staged
  const int j0 = jj, j1 = jj + 32;
  reg_pass<1>(u, j0, tw);
  reg_pass<1>(w, j1, tw);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    xb[reg_out<1>(j0, r) * TC + c] = u[r];
    xb[reg_out<1>(j1, r) * TC + c] = w[r];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    u[r] = xb[(j0 + B * r) * TC + c];
    w[r] = xb[(j1 + B * r) * TC + c];
  }
  __syncthreads();
  reg_pass<8>(u, j0, tw);
  reg_pass<8>(w, j1, tw);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    xb[reg_out<8>(j0, r) * TC + c] = u[r];
    xb[reg_out<8>(j1, r) * TC + c] = w[r];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    u[r] = xb[(j0 + B * r) * TC + c];
    w[r] = xb[(j1 + B * r) * TC + c];
  }
  reg_pass<64>(u, j0, tw);
  reg_pass<64>(w, j1, tw);
  const bool fused_warp_cta = MODE == 1 && a.fuse_warp && p == 0;  // uniform per CTA
  if (x >= a.W && !fused_warp_cta) return;
  const int sa = 2 * p, sb = 2 * p + 1;
  const size_t HW = (size_t)a.H * a.W;
  auto put = [&](int yy, float2 v) {
    if (yy >= a.H || x >= a.W) return;
    const size_t pix = (size_t)yy * a.W + x;
    if (MODE == 0) {
      float* z = a.zern + (size_t)f * a.Z * HW;
      z[(size_t)(sa + 1) * HW + pix] = v.x;
      if (sb < a.nslots) z[(size_t)(sb + 1) * HW + pix] = v.y;
    } else {
      if (a.xtile) {  // tile-major (x_index); the plane path below keeps its cheaper addressing
        uint16_t* Xt = a.X + x_index(a.xtile, f, sa, a.nslots, a.H, a.W, a.ntx, yy, x);
        Xt[0] = f_to_bf16(v.x);
        if (sb < a.nslots) Xt[a.xtile == 2 ? 8 : 128] = f_to_bf16(v.y);
      } else {
        uint16_t* Xo = a.X + (size_t)f * a.nslots * HW;
        Xo[(size_t)sa * HW + pix] = f_to_bf16(v.x);
        if (sb < a.nslots) Xo[(size_t)sb * HW + pix] = f_to_bf16(v.y);
      }
      if (p == 0 && !a.fuse_warp) {
        float* tl = a.tilt + (size_t)f * 2 * HW;
        tl[pix] = v.x;
        tl[HW + pix] = v.y;
      }
    }
  };
  if (fused_warp_cta) {
    // fused step 2: stash f_2, f_3 of the 16 columns in the (now free) exchange buffer,
    // then warp with the field registers dead (keeps the kernel's register budget)
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      xb[(j0 + B * r) * TC + c] = u[r];
      xb[(j1 + B * r) * TC + c] = w[r];
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      put(j0 + B * r, u[r]);
      put(j1 + B * r, w[r]);
    }
    __syncwarp();
    if (x < a.W) {
#pragma unroll 1
      for (int r = 0; r < 16; ++r) {
        const int yy = (r & 1 ? j1 : j0) + B * (r >> 1);
        if (yy < a.H) {
          const float2 v = xb[yy * TC + c];
          warp_pixel(a, f, yy, x, v.x, v.y);
        }
      }
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    put(j0 + B * r, u[r]);
    put(j1 + B * r, w[r]);
  }
}

int launch_cols(const p2s_plan_s* pl, int F, int mode, float* zern, cudaStream_t s, const float* img,
                int64_t img_stride, bool* warp_fused) {
  ColArgs a;
  fill_fft_args(a.fp, pl->fp);
  a.Zin = pl->d_Z;
  a.P = pl->P;
  a.Q = pl->slab_G > 1 ? pl->W : pl->Q;  // slab mode: the unpacked halo strip [npairs][P][W]
  a.H = pl->H;
  a.W = pl->W;
  a.npairs = pl->npairs;
  a.nslots = pl->nslots;
  a.Z = pl->Z;
  a.F = F;
  a.ntx = pl->ntx;
  a.xtile = pl->xtile;
  int tcl = 4;
  while (tcl > 0 && pl->P * (1 << tcl) > kColElems) --tcl;
  a.tc_log2 = tcl;
  a.zern = zern;
  a.X = pl->d_X;
  a.tilt = pl->d_tilt;
  a.fuse_warp = 0;
  if (warp_fused) *warp_fused = false;
  if (reg512(pl->fp) && !(pl->force & P2S_FORCE_FFT_GENERIC)) {
    if (mode == 1 && img && warp_fused && cols_fuse_warp(pl)) {
      const int Z = pl->Z;
      a.fuse_warp = 1;
      a.img = img;
      a.img_stride = img_stride;
      a.C = pl->C;
      a.cx = (float)(pl->kappa * pl->Lc[1 * Z + 1]);
      a.cy0 = (float)(pl->kappa * pl->Lc[2 * Z + 1]);
      a.cy1 = (float)(pl->kappa * pl->Lc[2 * Z + 2]);
      a.Iw = pl->d_Iw;
      *warp_fused = true;
    }
    dim3 grid((pl->W + 15) / 16, pl->npairs, F);  // only the W cropped columns are needed
    size_t sm = (size_t)kRegN * 17 * sizeof(float2);
    if (mode == 0) {
      P2S_SMEM_OPTIN((k_cols512<0>), sm);
      k_cols512<0><<<grid, 512, sm, s>>>(a);
    } else {
      P2S_SMEM_OPTIN((k_cols512<1>), sm);
      k_cols512<1><<<grid, 512, sm, s>>>(a);
    }
    return (int)cudaGetLastError();
  }
  // Long columns whose plan has at most 512 / TC butterflies per pass: the in-place
  // two-CTAs-per-SM kernel with the widest block that fits (TC = 4 at 1080 = 12 x 10 x 9,
  // TC = 2 at 2160 = 16 x 15 x 9).
  if (pl->P > 512 && !(pl->force & (P2S_FORCE_COLS_PER_BLOCK | P2S_FORCE_COLS_PERSISTENT))) {
    // (step 2 stays a kernel of its own here: fused into the mode-pair-0 CTAs it made them
    // stragglers -- 4K k_cols 2.59 -> 3.47 ms against k_warp's 0.29 ms; 1080p 2.30 -> 3.17)
    const auto& rp = pl->fp;
    const bool ct = !(pl->force & P2S_FORCE_FFT_GENERIC) && rp.nrad == 3;
#define P2S_COLS_CT(NT_, TL_, ...)                                                       \
  do {                                                                                   \
    a.tc_log2 = TL_;                                                                     \
    const size_t sm = ((size_t)pl->P + padded_len((size_t)pl->P << TL_)) * sizeof(float2); \
    dim3 grid((pl->W + (1 << TL_) - 1) >> TL_, pl->npairs, F);                           \
    if (mode == 0) {                                                                     \
      P2S_SMEM_OPTIN((k_cols_ip<0, NT_, TL_, __VA_ARGS__>), sm);                         \
      k_cols_ip<0, NT_, TL_, __VA_ARGS__><<<grid, NT_, sm, s>>>(a);                      \
    } else {                                                                             \
      P2S_SMEM_OPTIN((k_cols_ip<1, NT_, TL_, __VA_ARGS__>), sm);                         \
      k_cols_ip<1, NT_, TL_, __VA_ARGS__><<<grid, NT_, sm, s>>>(a);                      \
    }                                                                                    \
    return (int)cudaGetLastError();                                                      \
  } while (0)
    // measured (cfg5 / cfg4, per launch): 2160 with 4 columns and 384 threads, two CTAs per
    // SM (up to 3 butterflies per thread): 2.58 ms per 2 frames (8 columns, 768 threads, one
    // CTA: 2.66; 2 columns, 512 threads: 3.86; the persistent k_cols_p: 3.81); 1080 with 8
    // columns and 512 threads: 2.28 ms per 8 frames (4 columns: 2.57; k_cols_p: 2.73).  The
    // stores set the pace: TC columns of a row are TC * 2 bytes per output plane.
    if (ct && pl->P == 2160 && rp.rad[0] == 16 && rp.rad[1] == 15 && rp.rad[2] == 9)
      P2S_COLS_CT(384, 2, 2160, 16, 15, 9);
    if (ct && pl->P == 1080 && rp.rad[0] == 12 && rp.rad[1] == 10 && rp.rad[2] == 9)
      P2S_COLS_CT(512, 3, 1080, 12, 10, 9);
#undef P2S_COLS_CT
    for (int tl = 2; tl >= 1; --tl) {
      bool one = true;
      for (int i = 0; i < pl->fp.nrad; ++i) one = one && ((pl->P / pl->fp.rad[i]) << tl) <= 512;
      const size_t sm = ((size_t)pl->P + padded_len((size_t)pl->P << tl)) * sizeof(float2);
      if (!one || 2 * (sm + 1024) > kSmemMax) continue;
      a.tc_log2 = tl;
      dim3 grid((pl->W + (1 << tl) - 1) >> tl, pl->npairs, F);
#define P2S_COLS_IP(...)                                \
  do {                                                  \
    P2S_SMEM_OPTIN((k_cols_ip<__VA_ARGS__>), sm);       \
    k_cols_ip<__VA_ARGS__><<<grid, 512, sm, s>>>(a);    \
  } while (0)
      if (mode == 0) {
        if (tl == 2) P2S_COLS_IP(0, 512, 2); else P2S_COLS_IP(0, 512, 1);
      } else {
        if (tl == 2) P2S_COLS_IP(1, 512, 2); else P2S_COLS_IP(1, 512, 1);
      }
#undef P2S_COLS_IP
      return (int)cudaGetLastError();
    }
  }

  // Long columns: 1024 threads and up to 8640 elements per CTA double the columns per CTA
  // where that is still below 16 (1080 points: 8 columns, 64-byte row segments, 3.26 ->
  // 3.10 ms per 8 frames; 2160: 4 columns, 5.53 -> 4.67 ms per 2 frames).
  int tw = 4;
  while (tw > 0 && pl->P * (1 << tw) > 8640) --tw;
  const int wide = tw > tcl;
  if (wide) {
    tcl = tw;
    a.tc_log2 = tcl;
  }
  const int TC = 1 << tcl;
  if (wide && !(pl->force & P2S_FORCE_COLS_PER_BLOCK)) {
    bool one = true;  // every pass at most one butterfly per thread: in-place persistent kernel
    for (int i = 0; i < pl->fp.nrad; ++i) one = one && (pl->P / pl->fp.rad[i]) * TC <= 1024;
    if (one) {
      const int ntiles = (pl->W + TC - 1) / TC * pl->npairs * F;
      const int grid = std::min(ntiles, pl->num_sms);
      size_t sm = ((size_t)pl->P + 2 * padded_len((size_t)pl->P * TC)) * sizeof(float2);
      if (mode == 0) {
        P2S_SMEM_OPTIN((k_cols_p<0, 1024>), sm);
        k_cols_p<0, 1024><<<grid, 1024, sm, s>>>(a);
      } else {
        P2S_SMEM_OPTIN((k_cols_p<1, 1024>), sm);
        k_cols_p<1, 1024><<<grid, 1024, sm, s>>>(a);
      }
      return (int)cudaGetLastError();
    }
  }
  dim3 grid((pl->W + TC - 1) / TC, pl->npairs, F);
  size_t sm = ((size_t)pl->P + 2 * padded_len((size_t)pl->P * TC)) * sizeof(float2);
  if (wide) {
    if (mode == 0) {
      P2S_SMEM_OPTIN((k_cols<0, 1024>), sm);
      k_cols<0, 1024><<<grid, 1024, sm, s>>>(a);
    } else {
      P2S_SMEM_OPTIN((k_cols<1, 1024>), sm);
      k_cols<1, 1024><<<grid, 1024, sm, s>>>(a);
    }
  } else if (mode == 0) {
    P2S_SMEM_OPTIN((k_cols<0, 256>), sm);
    k_cols<0, 256><<<grid, 256, sm, s>>>(a);
  } else {
    P2S_SMEM_OPTIN((k_cols<1, 256>), sm);
    k_cols<1, 256><<<grid, 256, sm, s>>>(a);
  }
  return (int)cudaGetLastError();
}

// Step 2 inside k_cols512 (the mode-pair-0 CTAs gather the warp) is a forced variant: the
// separate TMA-window warp (k_warp_tma) after an unfused k_cols512 measured 0.04 ms per 64
// frames faster at 512^2 RGB (1.05 + 0.095 vs 1.19 ms), the fused CTAs being stragglers.
bool cols_fuse_warp(const p2s_plan_s* pl) {
  return reg512(pl->fp) && !(pl->force & P2S_FORCE_FFT_GENERIC) && (pl->force & P2S_FORCE_WARP_FUSION) &&
         pl->slab_G < 2;
}

// ------------------------------------------------------------------ K3: Noll mixing a = L f
__global__ void __launch_bounds__(256) k_mix(float* __restrict__ zern, const float* __restrict__ Lm, int Z,
                                             size_t HW) {
  const size_t pix = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= HW) return;
  float* z = zern + (size_t)blockIdx.y * Z * HW + pix;
  const int n = Z - 1;
  float f[65];
#pragma unroll 1
  for (int i = 0; i < n; ++i) f[i] = z[(size_t)(i + 1) * HW];
  z[0] = 0.f;
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    float acc = 0.f;
    for (int k = 0; k <= i; ++k) acc = fmaf(__ldg(&Lm[i * n + k]), f[k], acc);
    z[(size_t)(i + 1) * HW] = acc;
  }
}

int launch_mix(const p2s_plan_s* pl, int F, float* zern, cudaStream_t s) {
  size_t HW = (size_t)pl->H * pl->W;
  dim3 grid((unsigned)((HW + 255) / 256), F);
  k_mix<<<grid, 256, 0, s>>>(zern, pl->d_L, pl->Z, HW);
  return (int)cudaGetLastError();
}

// a_4..a_Z (fp32 Zernike planes) -> bf16 MLP input planes (p2s_blur API path).
__global__ void k_zern_to_x(const float* __restrict__ zern, uint16_t* __restrict__ X, int Z, int H, int W, int ntx,
                            int xtile) {
  const size_t HW = (size_t)H * W;
  const size_t pix = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= HW) return;
  const int f = blockIdx.y, y = (int)(pix / W), x = (int)(pix - (size_t)y * W);
  const float* z = zern + (size_t)f * Z * HW + pix;
  for (int k = 0; k < Z - 3; ++k) X[x_index(xtile, f, k, Z - 3, H, W, ntx, y, x)] = f_to_bf16(z[(size_t)(k + 3) * HW]);
}

int launch_zern_to_x(const p2s_plan_s* pl, int F, const float* zern, cudaStream_t s) {
  size_t HW = (size_t)pl->H * pl->W;
  dim3 grid((unsigned)((HW + 255) / 256), F);
  k_zern_to_x<<<grid, 256, 0, s>>>(zern, pl->d_X, pl->Z, pl->H, pl->W, pl->ntx, pl->xtile);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ test support
__global__ void k_philox_fill(uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1, int64_t n,
                              uint4* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = philox4x32_10(make_uint4((uint32_t)i, c1, c2, c3), k0, k1);
}

int launch_philox_fill(uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1, int64_t n, uint32_t* out,
                       cudaStream_t s) {
  if (n <= 0) return 0;
  k_philox_fill<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c1, c2, c3, k0, k1, n, reinterpret_cast<uint4*>(out));
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ slab mode (NEXT-4)
// Rank r's geometry: output columns [x0, x1) balanced over G, halo T/2 each side clipped to
// the frame, Hermitian row pairs [kp0, kp1) of the P/2 + 1 balanced over G, and the number
// of spectral rows they hold (pair 0 and, for even P, pair P/2 are their own mirror).
SlabGeom slab_geometry(int W, int T, int P, int G, int r) {
  SlabGeom g;
  const int c = T / 2;
  g.x0 = (int)((int64_t)W * r / G);
  g.x1 = (int)((int64_t)W * (r + 1) / G);
  g.hx0 = std::max(0, g.x0 - c);
  g.hx1 = std::min(W, g.x1 + c);
  const int npr = P / 2 + 1;
  g.kp0 = (int)((int64_t)npr * r / G);
  g.kp1 = (int)((int64_t)npr * (r + 1) / G);
  g.rows = 0;
  for (int kp = g.kp0; kp < g.kp1; ++kp) g.rows += (kp == 0 || 2 * kp == P) ? 1 : 2;
  return g;
}

// Pack this rank's row-transformed rows (d_Z [npairs][P][Q]) into the send blocks:
// block d = [rows_r][npairs][Ws(d)], columns [hx0(d), hx0(d) + Ws(d)) of each row.
__global__ void k_slab_pack(const float2* __restrict__ Z, float2* __restrict__ send, const int* __restrict__ ky_of,
                            const int* __restrict__ dest, int G, int P, int Q, int npairs, int rows) {
  const int l = blockIdx.x, p = blockIdx.y;
  const int ky = ky_of[l];
  const float2* src = Z + ((size_t)p * P + ky) * Q;
  for (int d = 0; d < G; ++d) {
    const int hx0 = dest[3 * d], ws = dest[3 * d + 1];
    float2* dst = send + (size_t)dest[3 * d + 2] + ((size_t)l * npairs + p) * ws;
    for (int x = threadIdx.x; x < ws; x += blockDim.x) dst[x] = src[hx0 + x];
  }
}

// Unpack the received rows (recv [G src][rows_src][npairs][Ws], i.e. rows in source order)
// into the strip spectrum d_Z [npairs][P][Ws] for the column pass.
__global__ void k_slab_unpack(const float2* __restrict__ recv, float2* __restrict__ Z, const int* __restrict__ ky_of,
                              int P, int npairs, int ws) {
  const int i = blockIdx.x, p = blockIdx.y;
  const float2* src = recv + ((size_t)i * npairs + p) * ws;
  float2* dst = Z + ((size_t)p * P + ky_of[i]) * ws;
  for (int x = threadIdx.x; x < ws; x += blockDim.x) dst[x] = src[x];
}

int launch_slab_pack(const p2s_plan_s* pl, float2* send, cudaStream_t s) {
  if (pl->slab_rows == 0) return 0;
  dim3 grid(pl->slab_rows, pl->npairs);
  k_slab_pack<<<grid, 256, 0, s>>>(pl->d_Z, send, pl->d_slab_ky, pl->d_slab_dest, pl->slab_G, pl->P, pl->Q,
                                   pl->npairs, pl->slab_rows);
  return (int)cudaGetLastError();
}

int launch_slab_unpack(const p2s_plan_s* pl, const float2* recv, cudaStream_t s) {
  dim3 grid(pl->P, pl->npairs);
  k_slab_unpack<<<grid, 256, 0, s>>>(recv, pl->d_Z, pl->d_slab_ky + pl->slab_rows, pl->P, pl->npairs, pl->W);
  return (int)cudaGetLastError();
}

}  // namespace p2s
