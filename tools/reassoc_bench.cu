// Microbenchmark (development tool, not part of libp2s): the per-pixel patch-dot phase of
// the RE-ASSOCIATED Eq.9 blur (h_x = sum_k w_k(x) h_k per pixel on the tensor cores, then
// out_c(x) = sum_u h_x[u] Iw_c(x - u)), which DESIGN.md section 6c argues is shared-memory
// bound.  Steady state on one CTA per SM: the 128 pixels of an output row are TMEM lanes;
// 16 warps (4 per TMEM lane quarter) each take a quarter of the 1089 taps, read the
// per-pixel PSF values from TMEM with tcgen05.ld.32x32b.x16 (16 taps per load; TMEM content
// is not initialised -- timing only) and the source pixels (3 channels packed in one float4)
// from the shared-memory tile, 3 FMAs per tap, partial sums reduced through shared memory.
// Reports cycles per output row of 128 pixels per SM, to compare with the direct implicit
// GEMM's 69 K-steps x 3 MMAs x 56 cycles = 11.6k cycles per 256-pixel CTA-pair row (one
// 128-pixel row per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2210_06713_b200/csrc \
//        tools/reassoc_bench.cu -o tools/reassoc_bench
#include <cstdio>
#include <cstdlib>

#include "p2s_dev.cuh"

using namespace p2s;

constexpr int T = 33, C0 = T / 2, NTAP = T * T, RB = 8, SEGW = 128 + T - 1, ROWS = RB + T - 1;

__global__ void __launch_bounds__(512, 1) k_patchdot(float* out, int reps, unsigned long long* cycles) {
  extern __shared__ __align__(16) unsigned char smem[];
  float4* tile = reinterpret_cast<float4*>(smem);                      // [ROWS][SEGW] RGB(+pad)
  float* part = reinterpret_cast<float*>(smem + ROWS * SEGW * 16);     // [4 parts][3][128]
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < ROWS * SEGW; i += 512) tile[i] = make_float4(1e-3f * (i % 97), 2e-3f, 3e-3f, 0.f);
  if (warp == 0) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int qd = warp & 3, h = warp >> 2;  // lane quarter, tap quarter
  const int m = qd * 32 + lane;            // pixel of the row
  const int t0 = (NTAP * h) / 4, t1 = (NTAP * (h + 1)) / 4;
  const uint32_t tl = tmem + ((uint32_t)(qd * 32) << 16);
  const unsigned long long c0 = clock64();
  float keep = 0.f;
  for (int rep = 0; rep < reps; ++rep) {
    for (int r = 0; r < RB; ++r) {
      float a0 = 0.f, a1 = 0.f, a2 = 0.f;
      for (int tb = t0 & ~15; tb < t1; tb += 16) {
        uint32_t v[16];
        tmem_ld16_issue(tl + (uint32_t)(tb % 512), v);  // PSF values of taps tb..tb+15 (lane = pixel)
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int t = tb + i;
          if (t < t0 || t >= t1) continue;
          const int ty = t / T, tx = t - ty * T;
          const float4 s = tile[(r + 2 * C0 - ty) * SEGW + (m + 2 * C0 - tx)];
          const float hv = __uint_as_float(v[i]);
          a0 = fmaf(hv, s.x, a0);
          a1 = fmaf(hv, s.y, a1);
          a2 = fmaf(hv, s.z, a2);
        }
      }
      if (h) {
        part[((h - 1) * 3 + 0) * 128 + m] = a0;
        part[((h - 1) * 3 + 1) * 128 + m] = a1;
        part[((h - 1) * 3 + 2) * 128 + m] = a2;
      }
      __syncthreads();
      if (!h) {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          a0 += part[(p * 3 + 0) * 128 + m];
          a1 += part[(p * 3 + 1) * 128 + m];
          a2 += part[(p * 3 + 2) * 128 + m];
        }
        keep += a0 + a1 + a2;
      }
      __syncthreads();
    }
  }
  const unsigned long long c1 = clock64();
  if (!h) out[blockIdx.x * 128 + m] = keep;
  if (tid == 0) atomicAdd(cycles, c1 - c0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t sm = (size_t)ROWS * SEGW * 16 + 4 * 3 * 128 * 4;
  cudaFuncSetAttribute(k_patchdot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, sizeof(float) * nsm * 128);
  cudaMalloc(&cyc, sizeof(unsigned long long));
  const int reps = 20;
  k_patchdot<<<nsm, 512, sm>>>(out, 2, cyc);  // warm-up
  cudaMemset(cyc, 0, sizeof(unsigned long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_patchdot<<<nsm, 512, sm>>>(out, reps, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
    return 1;
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double rows = (double)reps * RB;
  const double cyc_row = (double)c / nsm / rows;
  // time per frame of 512^2 RGB: 512 rows x 4 tiles of 128 px over nsm SMs
  const double us_frame = ms * 1e3 / (rows * nsm) * (512.0 * 4.0);
  printf("{\"patch_dot_cycles_per_128px_row_per_SM\": %.0f, \"direct_implicit_gemm_cycles\": 11592, "
         "\"patch_dot_us_per_512x512_rgb_frame\": %.1f, \"direct_blur_us_per_frame_measured\": 119}\n",
         cyc_row, us_frame);
  return 0;
}
