// k_blur.cu -- steps 4+5: the spatially varying blur of Eq.9 on tcgen05 tensor cores.
//
// Paper P:166-171 (Eq.9): I(x) = sum_m beta_{x,m} (phi_m (*) I_g)(x), "a set of spatially
// invariant convolutions".  Here conv_k(x) = (h_k (*) Iw_c)(x) for all K bases at once is
// an implicit GEMM  D[pixel][k] = sum_taps A[pixel][tap] B[tap][k]  with
//   M = 128 pixels of one output row (lane m <-> pixel x0 + 16 (m % 8) + m / 8),
//   N = np (K padded to 16), fp32 accumulators in TMEM (4 output rows in flight),
//   K = taps, ordered as groups of 8 consecutive tap rows ty at one tap column tx.
// The A operand is never materialised as im2col: the source tile is stored ONCE in
// shared memory as 16-byte chunks, chunk cc of source row r holding the 8 pixels at
// window offsets cc + 16 j (j = 0..7).  With the lane permutation above, the
// [128 x 8-tap-row] slab of any (output row, tx, tap-row group) is a canonical
// MN-major SWIZZLE_NONE layout (8 k-rows at 16 B, m-groups at SBO = one chunk
// column), so every K-step is pure descriptor arithmetic: start = tile + chunk
// (2c - tx) + rows, and the second 8-row group of the K-step is reached through the
// descriptor's leading-byte offset.  The B operand (taps x bases, precomputed per
// K-step on the host) streams through a TMA bulk-copy ring shared by the 4 rows.
// The epilogue (4 warps) reads the accumulator rows with tcgen05.ld, forms
// sum_k w_k(x) conv_k(x) with the P2S weights, and applies step 5 (normalise,
// Philox noise, clamp) before the only HBM write of the frame.
#include "p2s_dev.cuh"
#include "p2s_internal.h"

namespace p2s {

constexpr int kBlurStages = 6;
constexpr int kBlurThreads = 192;  // warp 0 TMA producer, warp 1 MMA issuer, warps 2-5 epilogue
constexpr int kRowsInFlight = 4;
constexpr int kAccStride = 128;    // TMEM columns per accumulator row

struct BlurArgs {
  const void* src;          // Iw [F][C][H][W] (bf16 or fp32)
  const uint16_t* w;        // bf16 [F][HW][np]
  float* out;               // [F][C][H][W]
  const uint8_t* bimg;      // [nks][np*32]
  const uint32_t* koff;     // [nks]
  const uint32_t* klbo;     // [nks]
  const float* hsum;        // [np]
  int C, H, W, T, c, NC, RB, RS, nks, np;
  uint32_t k0, k1;
  int64_t frame0;
  float sigma;
  int normalize, clamp01;
};

__device__ __forceinline__ int reflect_idx(int i, int n) {
  if (i < 0) i = -i;
  if (i >= n) i = 2 * n - 2 - i;
  return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

template <bool SRC_F32>
__device__ __forceinline__ float load_src(const void* src, size_t idx) {
  if (SRC_F32) return __ldg(reinterpret_cast<const float*>(src) + idx);
  return bf16_to_f(__ldg(reinterpret_cast<const uint16_t*>(src) + idx));
}

template <bool SRC_F32>
__global__ void __launch_bounds__(kBlurThreads, 1) k_blur(BlurArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbo_src = (uint32_t)a.RS * 16;
  uint8_t* tile = smem;
  const uint32_t tile_bytes = ((uint32_t)a.NC * sbo_src + 127) & ~127u;
  const uint32_t bbytes = (uint32_t)a.np * 32;
  uint8_t* ring = tile + tile_bytes;
  uint32_t* s_koff = reinterpret_cast<uint32_t*>(ring + kBlurStages * bbytes);
  uint32_t* s_klbo = s_koff + a.nks;
  float* s_hsum = reinterpret_cast<float*>(s_klbo + a.nks);
  uint64_t* bars = reinterpret_cast<uint64_t*>(((uintptr_t)(s_hsum + a.np) + 7) & ~(uintptr_t)7);
  uint64_t* full = bars;
  uint64_t* empty = bars + kBlurStages;
  uint64_t* tfull = bars + 2 * kBlurStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int x0 = blockIdx.x * 128, y0 = blockIdx.y * a.RB, f = blockIdx.z;
  const int HW = a.H * a.W;

  for (int i = tid; i < a.nks; i += kBlurThreads) {
    s_koff[i] = a.koff[i];
    s_klbo[i] = a.klbo[i];
  }
  for (int i = tid; i < a.np; i += kBlurThreads) s_hsum[i] = a.hsum[i];
  if (tid == 0) {
    for (int s = 0; s < kBlurStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  const uint32_t idesc = umma_idesc_bf16(128, a.np, true, false);
  const uint32_t s_tile = smem_u32(tile);
  uint32_t p_stage = 0, p_phase = 0;  // producer ring position
  uint32_t m_stage = 0, m_phase = 0;  // MMA ring position
  uint32_t rg_count = 0;
  const int n_rg = a.RB / kRowsInFlight;

  for (int ch = 0; ch < a.C; ++ch) {
    // ---- source tile: chunk cc, row rl <- pixels (x0 - c + cc + 16 j, y0 - c + rl), mirror boundary
    const size_t plane = ((size_t)f * a.C + ch) * HW;
    const int rows_real = a.RB + a.T - 1;
    for (int idx = tid; idx < a.NC * a.RS; idx += kBlurThreads) {
      const int cc = idx / a.RS, rl = idx - cc * a.RS;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (rl < rows_real) {
        const int sy = reflect_idx(y0 - a.c + rl, a.H);
        const size_t rowb = plane + (size_t)sy * a.W;
        float e[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) e[j] = load_src<SRC_F32>(a.src, rowb + reflect_idx(x0 - a.c + cc + 16 * j, a.W));
        v = make_uint4(pack_bf16x2(e[0], e[1]), pack_bf16x2(e[2], e[3]), pack_bf16x2(e[4], e[5]),
                       pack_bf16x2(e[6], e[7]));
      }
      *reinterpret_cast<uint4*>(tile + (size_t)cc * sbo_src + rl * 16) = v;
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp == 0) {
      if (lane == 0) {  // ---- TMA producer: B tiles of every K-step, once per row group
        for (int rg = 0; rg < n_rg; ++rg)
          for (int t = 0; t < a.nks; ++t) {
            mbar_wait(&empty[p_stage], p_phase ^ 1);
            mbar_arrive_expect_tx(&full[p_stage], bbytes);
            bulk_g2s(ring + p_stage * bbytes, a.bimg + (size_t)t * bbytes, bbytes, &full[p_stage]);
            if (++p_stage == kBlurStages) {
              p_stage = 0;
              p_phase ^= 1;
            }
          }
      }
    } else if (warp == 1) {
      if (lane == 0) {  // ---- MMA issuer
        for (int rg = 0; rg < n_rg; ++rg) {
          mbar_wait(tempty, (rg_count & 1) ^ 1);
          tc_fence_after();
          const uint32_t arow = s_tile + (uint32_t)(rg * kRowsInFlight) * 16;
          for (int t = 0; t < a.nks; ++t) {
            mbar_wait(&full[m_stage], m_phase);
            tc_fence_after();
            const uint64_t bdesc = umma_desc(smem_u32(ring + m_stage * bbytes), 128, 256);
            const uint32_t ko = s_koff[t], lbo = s_klbo[t];
#pragma unroll
            for (int r = 0; r < kRowsInFlight; ++r)
              umma_bf16(tmem + r * kAccStride, umma_desc(arow + r * 16 + ko, lbo, sbo_src), bdesc, idesc, t > 0);
            umma_commit(&empty[m_stage]);
            if (++m_stage == kBlurStages) {
              m_stage = 0;
              m_phase ^= 1;
            }
          }
          umma_commit(tfull);
          ++rg_count;
        }
      }
    } else {  // ---- epilogue warps 2..5: TMEM lane quarter = warp % 4
      const int qd = warp & 3;
      const int m = qd * 32 + lane;
      const int x = x0 + 16 * (m & 7) + (m >> 3);
      const uint32_t tl = tmem + ((uint32_t)(qd * 32) << 16);
      for (int rg = 0; rg < n_rg; ++rg) {
        mbar_wait(tfull, rg_count & 1);
        tc_fence_after();
        for (int r = 0; r < kRowsInFlight; ++r) {
          const int y = y0 + rg * kRowsInFlight + r;
          const bool valid = (y < a.H) && (x < a.W);
          const uint16_t* wrow = a.w + ((size_t)f * HW + (size_t)(valid ? y : 0) * a.W + (valid ? x : 0)) * a.np;
          float acc = 0.f, g = 0.f;
          for (int cb = 0; cb < a.np / 16; ++cb) {
            float v[16];
            tmem_ld16(tl + r * kAccStride + cb * 16, v);
            if (valid) {
              const uint4 w0 = __ldg(reinterpret_cast<const uint4*>(wrow + cb * 16));
              const uint4 w1 = __ldg(reinterpret_cast<const uint4*>(wrow + cb * 16 + 8));
              const uint32_t wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float wa = bf16_lo(wv[i]), wb = bf16_hi(wv[i]);
                acc = fmaf(wa, v[2 * i], acc);
                acc = fmaf(wb, v[2 * i + 1], acc);
                g = fmaf(wa, s_hsum[cb * 16 + 2 * i], g);
                g = fmaf(wb, s_hsum[cb * 16 + 2 * i + 1], g);
              }
            }
          }
          if (valid) {
            float o = acc;
            if (a.normalize) o = o / g;
            if (a.sigma != 0.f) {
              const int64_t fr = a.frame0 + f;
              uint4 rx = philox4x32_10(
                  make_uint4((uint32_t)(y * a.W + x), (uint32_t)ch | (1u << 16), (uint32_t)fr,
                             (uint32_t)((uint64_t)fr >> 32)),
                  a.k0, a.k1);
              o += a.sigma * box_muller(rx.x, rx.y).x;
            }
            if (a.clamp01) o = fminf(fmaxf(o, 0.f), 1.f);
            a.out[((size_t)f * a.C + ch) * HW + (size_t)y * a.W + x] = o;
          }
        }
        tc_fence_before();
        mbar_arrive(tempty);
        ++rg_count;
      }
    }
    __syncthreads();  // channel done: all MMAs retired (epilogue saw the last tfull)
  }
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int launch_blur(const p2s_plan_s* p, int F, const void* src, bool src_f32, uint64_t seed, int64_t frame0, float* out,
                cudaStream_t s) {
  const BlurGeom& g = p->bg;
  BlurArgs a;
  a.src = src;
  a.w = p->d_w;
  a.out = out;
  a.bimg = g.bimg;
  a.koff = g.koff;
  a.klbo = g.klbo;
  a.hsum = g.hsum;
  a.C = p->C;
  a.H = p->H;
  a.W = p->W;
  a.T = g.T;
  a.c = g.c;
  a.NC = g.NC;
  a.RB = g.RB;
  a.RS = g.RS;
  a.nks = g.nks;
  a.np = g.np;
  a.k0 = (uint32_t)seed;
  a.k1 = (uint32_t)(seed >> 32);
  a.frame0 = frame0;
  a.sigma = p->noise_sigma;
  a.normalize = p->normalize;
  a.clamp01 = p->clamp01;
  size_t tile_bytes = ((size_t)g.NC * g.RS * 16 + 127) & ~(size_t)127;
  size_t sm = tile_bytes + kBlurStages * (size_t)g.np * 32 + (size_t)g.nks * 8 + g.np * 4 + 8 +
              (2 * kBlurStages + 2) * 8 + 16;
  // TMEM: this kernel owns all 512 columns of its SM; keep shared memory above half the SM
  // so that two CTAs never co-reside and contend for tcgen05.alloc.
  if (sm < 116 * 1024) sm = 116 * 1024;
  dim3 grid((p->W + 127) / 128, (p->H + g.RB - 1) / g.RB, F);
  if (src_f32) {
    cudaFuncSetAttribute(k_blur<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_blur<true><<<grid, kBlurThreads, sm, s>>>(a);
  } else {
    cudaFuncSetAttribute(k_blur<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_blur<false><<<grid, kBlurThreads, sm, s>>>(a);
  }
  return (int)cudaGetLastError();
}

}  // namespace p2s
