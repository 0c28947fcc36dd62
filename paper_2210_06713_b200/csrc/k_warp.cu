// k_warp.cu -- step 2: tilt warp Iw_c(x) = I_c(x + d(x)), d = kappa (a_2, a_3)
// (BASELINE north_star step 2; reading Q12: gather warp, bilinear, clamp-to-edge,
// +a_2 -> +x columns, +a_3 -> +y rows).
//
// One thread per output pixel handles all C channels (the displacement is shared,
// Q17).  The clean image is small and broadcast over frames, so its gathers hit L2;
// the kernel streams the two tilt planes in and the warped planes out (HBM-bound).
#include "p2s_dev.cuh"
#include "p2s_internal.h"

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
  dim3 grid((unsigned)((HW + 255) / 256), F);
  k_warp<true><<<grid, 256, 0, s>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace p2s
