// k_warp.cu -- step 2: tilt warp Iw_c(x) = I_c(x + d(x)), d = kappa (a_2, a_3)
// (BASELINE north_star step 2; reading Q12: gather warp, bilinear, clamp-to-edge,
// +a_2 -> +x columns, +a_3 -> +y rows).
//
// One thread per output pixel handles all C channels (the displacement is shared,
// Q17).  The clean image is small and broadcast over frames, so its gathers hit L2;
// the kernel streams the two tilt planes in and the warped planes out (HBM-bound).
#include "p2s_dev.cuh"
#include "p2s_internal.h"

#include <cudaTypedefs.h>

namespace p2s {

struct WarpArgs {
  const float* img;
  int64_t img_stride;  // floats between frames (0 = broadcast)
  const float* t0;     // tilt source plane 0 of frame 0
  const float* t1;     // tilt source plane 1 of frame 0
  int64_t t_stride;    // floats between frames of the tilt source
  float cx, cy0, cy1;  // dx = cx t0 ; dy = cy0 t0 + cy1 t1
  void* out;           // [F][C][H][W] fp32 or bf16
  int C, H, W;
  int x_off, W_img;    // output column x samples image column x_off + x of an H x W_img image
                       // (slab mode: the rank's halo strip of the frame; else 0, W)
};

template <bool BF16_OUT>
__global__ void __launch_bounds__(256) k_warp(WarpArgs a) {
  const int HW = a.H * a.W;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= HW) return;
  const int f = blockIdx.y;
  const int y = pix / a.W, x = pix - y * a.W;
  const float u = __ldg(&a.t0[(size_t)f * a.t_stride + pix]);
  const float v = __ldg(&a.t1[(size_t)f * a.t_stride + pix]);
  const float X = (float)(a.x_off + x) + a.cx * u;
  const float Y = (float)y + a.cy0 * u + a.cy1 * v;
  const float fx = floorf(X), fy = floorf(Y);
  const float tx = X - fx, ty = Y - fy;
  const int Wi = a.W_img;
  int xa = (int)fmaxf(fminf(fx, (float)(Wi - 1)), -1.f);
  int ya = (int)fmaxf(fminf(fy, (float)(a.H - 1)), -1.f);
  int xb = min(xa + 1, Wi - 1), yb = min(ya + 1, a.H - 1);
  xa = max(xa, 0);
  ya = max(ya, 0);
  const float* I = a.img + (size_t)f * a.img_stride;
  const size_t HWi = (size_t)a.H * Wi;
  for (int c = 0; c < a.C; ++c) {
    const float* Ic = I + (size_t)c * HWi;
    const float i00 = __ldg(&Ic[ya * Wi + xa]), i01 = __ldg(&Ic[ya * Wi + xb]);
    const float i10 = __ldg(&Ic[yb * Wi + xa]), i11 = __ldg(&Ic[yb * Wi + xb]);
    const float val = (1.f - ty) * ((1.f - tx) * i00 + tx * i01) + ty * ((1.f - tx) * i10 + tx * i11);
    const size_t o = ((size_t)f * a.C + c) * HW + pix;
    if (BF16_OUT)
      reinterpret_cast<uint16_t*>(a.out)[o] = f_to_bf16(val);
    else
      reinterpret_cast<float*>(a.out)[o] = val;
  }
}

// TMA-staged variant (north_star step 2: "a fused warp+gather kernel using TMA-staged tiles"):
// one CTA per 64 x 32 output tile and frame; one 3-D TMA box brings the image window of the
// tile plus a margin of kWarpM pixels on every side (5-8 on the right: the window start is
// rounded down to 16 bytes) (all channels, zero-filled outside the
// image) into shared memory, and the bilinear taps are read from there; a tap outside the
// window (|d| > kWarpM px, a few percent of pixels at D/r0 = 5) is read from global memory.
// Same arithmetic as k_warp (bit-identical results).
constexpr int kWarpTX = 64, kWarpTY = 32, kWarpM = 8;
constexpr int kWarpBX = kWarpTX + 2 * kWarpM, kWarpBY = kWarpTY + 2 * kWarpM;

template <int C>
__global__ void __launch_bounds__(256) k_warp_tma(WarpArgs a, const __grid_constant__ CUtensorMap tmap_img, int img_frames) {
  extern __shared__ __align__(128) float win[];  // [C][kWarpBY][kWarpBX]
  __shared__ __align__(8) uint64_t bar;
  // window origin in image columns, rounded down to 16 bytes (a TMA box starts on a 16-byte
  // boundary in its innermost dimension; slab strips start at any column)
  const int wx0 = (a.x_off + (int)blockIdx.x * kWarpTX - kWarpM) & ~3;
  const int by0 = blockIdx.y * kWarpTY - kWarpM, f = blockIdx.z;
  const int fi = img_frames > 1 ? f : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, (uint32_t)(C * kWarpBX * kWarpBY * 4));
    tma_load_4d(win, &tmap_img, wx0, by0, 0, fi, &bar);
  }
  // tilt values of this thread's pixels while the window lands
  constexpr int PPT = kWarpTX * kWarpTY / 256;
  const int HW = a.H * a.W;
  const int Wi = a.W_img;
  const size_t HWi = (size_t)a.H * Wi;
  float u[PPT], v[PPT];
#pragma unroll
  for (int i = 0; i < PPT; ++i) {
    const int e = threadIdx.x + 256 * i, x = blockIdx.x * kWarpTX + (e % kWarpTX), y = blockIdx.y * kWarpTY + e / kWarpTX;
    u[i] = v[i] = 0.f;
    if (x < a.W && y < a.H) {
      u[i] = __ldg(&a.t0[(size_t)f * a.t_stride + (size_t)y * a.W + x]);
      v[i] = __ldg(&a.t1[(size_t)f * a.t_stride + (size_t)y * a.W + x]);
    }
  }
  mbar_wait(&bar, 0);
  const float* I = a.img + (size_t)f * a.img_stride;
#pragma unroll
  for (int i = 0; i < PPT; ++i) {
    const int e = threadIdx.x + 256 * i, x = blockIdx.x * kWarpTX + (e % kWarpTX), y = blockIdx.y * kWarpTY + e / kWarpTX;
    if (x >= a.W || y >= a.H) continue;
    const float X = (float)(a.x_off + x) + a.cx * u[i];
    const float Y = (float)y + a.cy0 * u[i] + a.cy1 * v[i];
    const float fx = floorf(X), fy = floorf(Y);
    const float tx = X - fx, ty = Y - fy;
    int xa = (int)fmaxf(fminf(fx, (float)(Wi - 1)), -1.f);
    int ya = (int)fmaxf(fminf(fy, (float)(a.H - 1)), -1.f);
    const int xb = min(xa + 1, Wi - 1), yb = min(ya + 1, a.H - 1);
    xa = max(xa, 0);
    ya = max(ya, 0);
    // window coordinates (the window starts at image column wx0, row by0)
    const int wxa = xa - wx0, wxb = xb - wx0, wya = ya - by0, wyb = yb - by0;
    const bool in = wxa >= 0 && wxb < kWarpBX && wya >= 0 && wyb < kWarpBY;
    const int pix = y * a.W + x;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      float i00, i01, i10, i11;
      if (in) {
        const float* wc = win + c * kWarpBX * kWarpBY;
        i00 = wc[wya * kWarpBX + wxa];
        i01 = wc[wya * kWarpBX + wxb];
        i10 = wc[wyb * kWarpBX + wxa];
        i11 = wc[wyb * kWarpBX + wxb];
      } else {
        const float* Ic = I + (size_t)c * HWi;
        i00 = __ldg(&Ic[ya * Wi + xa]);
        i01 = __ldg(&Ic[ya * Wi + xb]);
        i10 = __ldg(&Ic[yb * Wi + xa]);
        i11 = __ldg(&Ic[yb * Wi + xb]);
      }
      const float val = (1.f - ty) * ((1.f - tx) * i00 + tx * i01) + ty * ((1.f - tx) * i10 + tx * i11);
      reinterpret_cast<uint16_t*>(a.out)[((size_t)f * C + c) * HW + pix] = f_to_bf16(val);
    }
  }
}

// 4-D tensor map over the image [F_img][C][H][W_img] fp32 (box = the warp window, all channels).
static bool encode_img_map(CUtensorMap* m, const float* img, int C, int H, int Wi, int Fimg, int64_t stride) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode)
      return false;
  }
  const uint64_t fstride = (uint64_t)(Fimg > 1 ? stride : (int64_t)C * H * Wi) * 4;
  if (((uintptr_t)img & 15) || ((uint64_t)Wi * 4) % 16 || fstride % 16) return false;
  cuuint64_t dims[4] = {(cuuint64_t)Wi, (cuuint64_t)H, (cuuint64_t)C, (cuuint64_t)Fimg};
  cuuint64_t strides[3] = {(cuuint64_t)Wi * 4, (cuuint64_t)H * Wi * 4, fstride};
  cuuint32_t box[4] = {(cuuint32_t)kWarpBX, (cuuint32_t)kWarpBY, (cuuint32_t)C, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(img), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int launch_warp_f32(const p2s_plan_s* p, int F, const float* img, int64_t stride, const float* zern, float* out,
                    cudaStream_t s) {
  const size_t HW = (size_t)p->H * p->W;
  WarpArgs a;
  a.img = img;
  a.img_stride = stride;
  a.t0 = zern + 1 * HW;  // a_2
  a.t1 = zern + 2 * HW;  // a_3
  a.t_stride = (int64_t)p->Z * HW;
  a.cx = (float)p->kappa;
  a.cy0 = 0.f;
  a.cy1 = (float)p->kappa;
  a.out = out;
  a.C = p->C;
  a.H = p->H;
  a.W = p->W;
  a.x_off = 0;
  a.W_img = p->W;
  dim3 grid((unsigned)((HW + 255) / 256), F);
  k_warp<false><<<grid, 256, 0, s>>>(a);
  return (int)cudaGetLastError();
}

// Fused path: the tilt planes hold the unmixed f_2, f_3; a_2 = L22 f_2, a_3 = L32 f_2 + L33 f_3.
int launch_warp_sim(const p2s_plan_s* p, int F, const float* img, int64_t stride, cudaStream_t s) {
  const size_t HW = (size_t)p->H * p->W;
  const int Z = p->Z;
  WarpArgs a;
  a.img = img;
  a.img_stride = stride;
  a.t0 = p->d_tilt;
  a.t1 = p->d_tilt + HW;
  a.t_stride = (int64_t)2 * HW;
  a.cx = (float)(p->kappa * p->Lc[1 * Z + 1]);
  a.cy0 = (float)(p->kappa * p->Lc[2 * Z + 1]);
  a.cy1 = (float)(p->kappa * p->Lc[2 * Z + 2]);
  a.out = p->d_Iw;
  a.C = p->C;
  a.H = p->H;
  a.W = p->W;
  a.x_off = p->slab_G > 1 ? p->slab_hx0 : 0;
  a.W_img = p->slab_G > 1 ? p->W_glob : p->W;
  CUtensorMap tm;
  const int Fimg = stride == 0 ? 1 : F;
  if (!(p->force & P2S_FORCE_WARP_GATHER) && F <= 65535 &&
      encode_img_map(&tm, img, p->C, p->H, a.W_img, Fimg, stride)) {
    dim3 g((p->W + kWarpTX - 1) / kWarpTX, (p->H + kWarpTY - 1) / kWarpTY, F);
    const size_t sm = (size_t)p->C * kWarpBX * kWarpBY * 4;
#define P2S_WARP_TMA(CC)                                      \
  do {                                                        \
    P2S_SMEM_OPTIN(k_warp_tma<CC>, sm);                       \
    k_warp_tma<CC><<<g, 256, sm, s>>>(a, tm, Fimg);           \
  } while (0)
    switch (p->C) {
      case 1: P2S_WARP_TMA(1); break;
      case 2: P2S_WARP_TMA(2); break;
      case 3: P2S_WARP_TMA(3); break;
      default: P2S_WARP_TMA(4); break;
    }
#undef P2S_WARP_TMA
    return (int)cudaGetLastError();
  }
  dim3 grid((unsigned)((HW + 255) / 256), F);
  k_warp<true><<<grid, 256, 0, s>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace p2s
