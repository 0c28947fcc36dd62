// k_mlp.cu -- step 3: the Phase-to-Space network on 5th-generation tensor cores.
//
// Paper P:172: "train a small neural network to convert the coefficients from the
// Zernike coefficients a_x ... to the PSF coefficients beta_x".  Shape (reading Q13):
// n_in -> h1 -> h2 -> K with ReLU hidden layers, linear output.  In the fused
// simulate path the Noll mixing a = L f is folded into layer 1 (W1' = W1 L),
// so the inputs are the unmixed unit-variance fields f_2..f_Z.
//
// Per 128-pixel tile (M = 128) the three layers are tcgen05.mma kind::f16 GEMMs
// (bf16 operands in shared memory, fp32 accumulators in TMEM):
//   layer 1: A1 [128 x k1] MN-major (pixels contiguous per input plane, as stored in
//            HBM), B = W1 image [n1 x k1] K-major
//   layer 2: A2 [128 x n1] K-major (written by the layer-1 epilogue), B = W2 image
//   layer 3: A2 [128 x n2] K-major, B = W3 image
// Epilogues read TMEM with tcgen05.ld (32 lanes x 16 columns per warp), add bias,
// ReLU, repack bf16 into the next layer's A operand; the last one writes the basis
// weights w as [F][H][ntx][n3/8][128 px][8] bf16: each 128-pixel row tile is one
// contiguous block (one bulk store), and the blur epilogue thread of a pixel reads 8
// consecutive bases with one 16-byte load.
// Persistent grid, one CTA per SM holding the weight images once in shared memory and
// running four independent 128-pixel tile pipelines (one per warpgroup, 128 TMEM columns
// each), so the tensor core always has another warpgroup's GEMM to run while one
// warpgroup is in an epilogue; the output tile leaves through one bulk copy.  Tiles are
// 128-pixel segments of one image row (the blur's x-tiles).
#include "p2s_dev.cuh"
#include "p2s_internal.h"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

namespace p2s {

struct MlpArgs {
  const uint16_t* X;    // bf16 [F][nin][HW]
  uint16_t* wout;       // bf16 [F][H][ntx][n3/8][128][8]
  const uint8_t* blob;  // W1img | W2img | W3img | b1 | b2 | b3
  int nin, k1, n1, n2, n3;
  uint32_t off_w2, off_w3, off_b1, off_b2, off_b3, blob_bytes;
  int HW, H, W, ntx, F, tiles_per_frame;
  int bias_folded;  // A1 column nin is the constant 1; biases live in the weight images
  int xtile;        // X layout (x_index): 1 = tile-major [F][H][ntx][nin][128]
  int a1_tma;       // A1 tiles by TMA (tmap_x valid)
  unsigned long long* probe;  // P2S_MLP_PROBE builds: [8] phase cycle sums, else null
};

// Epilogue of a hidden layer: TMEM columns [0, ncols) of this thread's row -> +bias -> ReLU
// -> bf16 -> the next layer's K-major A operand (row m of a [128 x ncols] SWIZZLE_NONE
// image, core matrices of 8 rows x 16 B, k-chunks at 128 B, 8-row groups at sbo).
// One 16-column TMEM load per wait (measured: 32 or 64 columns per wait are slower).
template <bool BIAS>
__device__ __forceinline__ void mlp_hidden_epilogue(uint32_t taddr, int ncols, const float* bias, uint8_t* a_smem,
                                                    uint32_t sbo, int m) {
  uint8_t* rowbase = a_smem + (m & 7) * 16 + (m >> 3) * sbo;
  for (int c0 = 0; c0 < ncols; c0 += 16) {  // 16 columns per TMEM wait
    uint32_t r[16];
    tmem_ld16_issue(taddr + c0, r);
    tmem_wait_ld();
    uint32_t pk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float x0 = __uint_as_float(r[2 * i]), x1 = __uint_as_float(r[2 * i + 1]);
      if (BIAS) {
        x0 += bias[c0 + 2 * i];
        x1 += bias[c0 + 2 * i + 1];
      }
      x0 = fmaxf(x0, 0.f);
      x1 = fmaxf(x1, 0.f);
      pk[i] = pack_bf16x2(x0, x1);
    }
    uint8_t* base = rowbase + (c0 / 8) * 128;
    *reinterpret_cast<uint4*>(base) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    *reinterpret_cast<uint4*>(base + 128) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
  }
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void wg_sync(int wg) {  // named barrier of one 128-thread warpgroup
  asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
}

// A1 tile (nin planes x 128 pixels, MN-major, k linear at 16 B): pixels [pix0, pix0 + n) of
// frame f (one row segment, n <= 128; the rest of the tile is zero).
// NIN > 0: the input count at compile time (35 on the simulate path, 33 on the blur API
// path), so the chunk index splits by constant division.
template <int NIN>
__device__ __forceinline__ void load_a1(const MlpArgs& a, uint8_t* A1, int tile, int f, int pix0, int n, int ltid,
                                        bool async) {
  const int nin = NIN > 0 ? NIN : a.nin;
  const uint16_t* Xf = a.X + (size_t)f * nin * a.HW;
  const int nin2 = a.xtile == 2 ? (nin + 1) & ~1 : nin;
  const uint16_t* Xt = a.X + (size_t)tile * 128 * nin2;  // tile-major: this tile's block
  for (int idx = ltid; idx < nin * 16; idx += 128) {
    const int k = idx % nin, g = idx / nin;
    const int o = 8 * g;
    // tile-major: plane k of this tile at k * 128 elements of its contiguous block; octet-pair
    // layout (xtile 2): the chunk of mode k, octet g at ((k/2) 16 + g) 16 + (k%2) 8
    const uint16_t* src = a.xtile == 2 ? Xt + (size_t)(((k >> 1) * 16 + g) * 16 + (k & 1) * 8)
                        : a.xtile     ? Xt + (size_t)k * 128 + o
                                      : Xf + (size_t)k * a.HW + pix0 + o;
    uint8_t* dst = A1 + g * (a.k1 * 16) + k * 16;
    if (async) {  // W % 8 == 0: whole 16-byte chunks, zero-filled past the row segment
      cp_async16(dst, o < n ? src : a.X, o < n ? 16u : 0u);
    } else {
      uint16_t t[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) t[e] = (o + e < n) ? src[e] : (uint16_t)0;
      *reinterpret_cast<uint4*>(dst) =
          make_uint4(t[0] | (t[1] << 16), t[2] | (t[3] << 16), t[4] | (t[5] << 16), t[6] | (t[7] << 16));
    }
  }
}

// Tile index -> (frame, first pixel, pixel count); tiles are 128-pixel segments of rows.
__device__ __forceinline__ void tile_pixels(const MlpArgs& a, int tile, int& f, int& pix0, int& n) {
  f = tile / a.tiles_per_frame;
  const int r = tile - f * a.tiles_per_frame;
  const int y = r / a.ntx, xt = r - y * a.ntx;
  pix0 = y * a.W + xt * 128;
  n = min(128, a.W - xt * 128);
}

// One layer GEMM: nsteps K-steps of 16; descriptors advance by 256 bytes (16 in the
// 16-byte-unit address field) per step, so the issuing thread does one add per operand.
__device__ __forceinline__ void mlp_issue_layer(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, int nsteps) {
#pragma unroll 8
  for (int s = 0; s < nsteps; ++s) umma_bf16(tmem, da + (uint64_t)(16 * s), db + (uint64_t)(16 * s), idesc, s > 0);
}

constexpr int kMlpWG = 4;  // independent 128-pixel tile pipelines per CTA

// kMlpWG warpgroups per CTA, each an independent tile pipeline (own A1, A2, 128 TMEM
// columns, mbarrier), sharing one resident copy of the weight images; while one warpgroup
// runs an epilogue the tensor core serves the others.
template <int NIN>
__global__ void __launch_bounds__(128 * kMlpWG, 1)
    k_mlp(const __grid_constant__ MlpArgs a, const __grid_constant__ CUtensorMap tmap_x) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sw = smem;  // weight blob
  const uint32_t blob_al = (a.blob_bytes + 127) & ~127u;
  const uint32_t a1_bytes = 128u * a.k1 * 2;
  const int nmax = a.n1 > a.n2 ? a.n1 : a.n2;
  const int na2 = nmax > a.n3 ? nmax : a.n3;  // A2 also stages the output tile
  const uint32_t a2_bytes = 128u * na2 * 2;
  const uint32_t wg_bytes = a1_bytes + a2_bytes;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wg = tid >> 7, ltid = tid & 127;
  const int nwg = blockDim.x >> 7;
  uint8_t* A1 = sw + blob_al + wg * wg_bytes;
  uint8_t* A2 = A1 + a1_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sw + blob_al + nwg * wg_bytes);
  uint64_t* bar = bars + wg;                 // layer MMAs done
  uint64_t* a1bar = bars + kMlpWG + wg;      // A1 bulk copy landed (xtile 3)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * kMlpWG);

  for (uint32_t i = tid * 16; i < a.blob_bytes; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(sw + i) = __ldg(reinterpret_cast<const uint4*>(a.blob + i));
  // zero the padded input planes (k in [nin, k1)) of every A1 buffer once
  if (a.k1 > a.nin) {
    const int per = (a.k1 - a.nin) * 16;
    for (int idx = tid; idx < nwg * per; idx += blockDim.x) {
      const int b = idx / per, r = idx % per;
      const int k = a.nin + r % (a.k1 - a.nin), g = r / (a.k1 - a.nin);
      // padding planes are zero; with folded biases plane nin is the constant 1 (bf16 0x3F80)
      const uint32_t one = (a.bias_folded && k == a.nin) ? 0x3F803F80u : 0u;
      *reinterpret_cast<uint4*>(sw + blob_al + b * wg_bytes + g * (a.k1 * 16) + k * 16) = make_uint4(one, one, one, one);
    }
  }
  if (tid == 0) {
    for (int i = 0; i < 2 * kMlpWG; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  const int wmax = na2;  // widest accumulator (n1, n2 or n3)
  const uint32_t cols_wg = wmax <= 32 ? 32 : wmax <= 64 ? 64 : wmax <= 128 ? 128 : 256;
  uint32_t ncols = 32;  // tcgen05.alloc takes a power of two >= 32: round nwg * cols_wg up
  while (ncols < nwg * cols_wg) ncols <<= 1;  // <= 512 (the launcher picks nwg)
  if (warp == 0) tmem_alloc(tslot, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot + wg * cols_wg;
  const int qd = warp & 3;
  const uint32_t taddr = tmem + ((uint32_t)(qd * 32) << 16);
  const int m = qd * 32 + lane;  // TMEM lane = tile row = pixel offset

  const float* b1 = reinterpret_cast<const float*>(sw + a.off_b1);
  const float* b2 = reinterpret_cast<const float*>(sw + a.off_b2);
  const float* b3 = reinterpret_cast<const float*>(sw + a.off_b3);
  const uint32_t sA1 = smem_u32(A1), sA2 = smem_u32(A2);
  const uint32_t sW1 = smem_u32(sw), sW2 = smem_u32(sw + a.off_w2), sW3 = smem_u32(sw + a.off_w3);
  const uint64_t dA1 = umma_desc(sA1, 128, a.k1 * 16), dW1 = umma_desc(sW1, 128, (a.k1 / 8) * 128);
  const uint64_t dA2a = umma_desc(sA2, 128, (a.n1 / 8) * 128), dW2 = umma_desc(sW2, 128, (a.n1 / 8) * 128);
  const uint64_t dA2b = umma_desc(sA2, 128, (a.n2 / 8) * 128), dW3 = umma_desc(sW3, 128, (a.n2 / 8) * 128);
  const uint32_t id1 = umma_idesc_bf16(128, a.n1, true, false);
  const uint32_t id2 = umma_idesc_bf16(128, a.n2, false, false);
  const uint32_t id3 = umma_idesc_bf16(128, a.n3, false, false);
  uint32_t phase = 0, a1phase = 0;
  const int ntiles = a.F * a.tiles_per_frame;
  const bool async = (a.W % 8) == 0;
  const bool bulk = a.a1_tma != 0;  // A1 by one TMA box per tile (tensor map over X)
  const int stride = nwg * gridDim.x;
  auto fetch_a1 = [&](int t) {
    if (bulk) {
      if (ltid == 32) {  // warp 1: warp 0 already issues the layer MMAs and waits on the w store
        mbar_arrive_expect_tx(a1bar, a1_bytes);
        if (a.xtile == 2) {
          tma_load_5d(A1, &tmap_x, 0, 0, 0, 0, t, a1bar);
        } else {
          int f, pix0, n;
          tile_pixels(a, t, f, pix0, n);
          tma_load_4d(A1, &tmap_x, 0, 0, pix0 >> 3, f, a1bar);
        }
      }
    } else {
      int f, pix0, n;
      tile_pixels(a, t, f, pix0, n);
      load_a1<NIN>(a, A1, t, f, pix0, n, ltid, async);
    }
  };

#ifdef P2S_MLP_PROBE  // phase cycle counters of a tuning build (tools/blur_probe.py prints them)
  unsigned long long pr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto pclk = []() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    return t;
  };
#define MLP_T(i) const unsigned long long tt##i = pclk()
#define MLP_ACC(i, a, b) pr[i] += tt##b - tt##a
#else
#define MLP_T(i)
#define MLP_ACC(i, a, b)
#endif
  int tile = nwg * blockIdx.x + wg;
  if (tile < ntiles) fetch_a1(tile);
  cp_async_commit();
  for (; tile < ntiles; tile += stride) {
    MLP_T(0);
    if (bulk) {  // this tile's A1 (issued during the previous tile's layers 2-3); then the
                 // padding planes [nin, k1): 0, the bias plane 1 (the box fills them with
                 // zeros or, on octet-pair tiles, the odd plane of the last pair unwritten)
      mbar_wait(a1bar, a1phase);
      a1phase ^= 1;
      const int npad = a.k1 - a.nin;
      for (int idx = ltid; idx < npad * 16; idx += 128) {
        const int k = a.nin + idx % npad, g = idx / npad;
        const uint32_t one = (a.bias_folded && k == a.nin) ? 0x3F803F80u : 0u;
        *reinterpret_cast<uint4*>(A1 + g * (a.k1 * 16) + k * 16) = make_uint4(one, one, one, one);
      }
    } else {
      cp_async_wait<0>();  // this tile's A1 (issued during the previous tile's layers 2-3)
    }
    fence_async_smem();
    tc_fence_before();
    wg_sync(wg);
    MLP_T(1);
    // ---- layer 1
    if (ltid == 0) {
      tma_store_wait_read();  // the previous tile's w store has finished reading A2
      tc_fence_after();
      mlp_issue_layer(tmem, dA1, dW1, id1, a.k1 / 16);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    MLP_T(2);
    {  // A1 is free once layer 1 has completed: prefetch the next tile's inputs
      const int nxt = tile + stride;
      if (nxt < ntiles) fetch_a1(nxt);
      cp_async_commit();
    }
    if (a.bias_folded)
      mlp_hidden_epilogue<false>(taddr, a.n1, b1, A2, (a.n1 / 8) * 128, m);
    else
      mlp_hidden_epilogue<true>(taddr, a.n1, b1, A2, (a.n1 / 8) * 128, m);
    MLP_T(3);
    fence_async_smem();
    tc_fence_before();
    wg_sync(wg);
    MLP_T(4);
    // ---- layer 2
    if (ltid == 0) {
      tc_fence_after();
      mlp_issue_layer(tmem, dA2a, dW2, id2, a.n1 / 16);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    MLP_T(5);
    if (a.bias_folded)
      mlp_hidden_epilogue<false>(taddr, a.n2, b2, A2, (a.n2 / 8) * 128, m);
    else
      mlp_hidden_epilogue<true>(taddr, a.n2, b2, A2, (a.n2 / 8) * 128, m);
    MLP_T(6);
    fence_async_smem();
    tc_fence_before();
    wg_sync(wg);
    // ---- layer 3
    if (ltid == 0) {
      tc_fence_after();
      mlp_issue_layer(tmem, dA2b, dW3, id3, a.n2 / 16);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    MLP_T(7);
    // w tile -> A2 as [n3/8][128 px][8] bf16 (16-byte stores, consecutive lanes adjacent),
    // then one bulk copy of the whole tile.
    {
      uint4* st = reinterpret_cast<uint4*>(A2) + m;
      for (int c0 = 0; c0 < a.n3; c0 += 16) {
        uint32_t r[16];
        tmem_ld16_issue(taddr + c0, r);
        tmem_wait_ld();
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float v0 = __uint_as_float(r[2 * i]), v1 = __uint_as_float(r[2 * i + 1]);
          if (!a.bias_folded) {
            v0 += b3[c0 + 2 * i];
            v1 += b3[c0 + 2 * i + 1];
          }
          pk[i] = pack_bf16x2(v0, v1);
        }
        st[(c0 / 8) * 128] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        st[(c0 / 8 + 1) * 128] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
    fence_async_smem();
    tc_fence_before();
    wg_sync(wg);
    // tile index == (f * H + y) * ntx + xt: the output block of this row tile
    if (ltid == 0) bulk_s2g(a.wout + (size_t)tile * a.n3 * 128, A2, (uint32_t)a.n3 * 256);
    MLP_T(8);
    MLP_ACC(0, 0, 1);  // A1 wait (+ padding planes) + group sync
    MLP_ACC(1, 1, 2);  // layer 1 (after the previous w store has read A2)
    MLP_ACC(2, 2, 3);  // next tile's A1 prefetch issue + epilogue 1
    MLP_ACC(3, 3, 4);  // sync
    MLP_ACC(4, 4, 5);  // layer 2
    MLP_ACC(5, 5, 6);  // epilogue 2
    MLP_ACC(6, 6, 7);  // sync + layer 3
    MLP_ACC(7, 7, 8);  // output epilogue + sync + store issue
  }
#ifdef P2S_MLP_PROBE
  if (ltid == 0 && a.probe)
    for (int i = 0; i < 8; ++i) atomicAdd(&a.probe[i], pr[i]);
#endif
  if (ltid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(*tslot, ncols);
}

// User-supplied basis weights (p2s_blur_weights): fp32 planes [F][K][H][W] -> the blur's
// bf16 row-tile layout [F][H][ntx][np/8][128][8] (bases >= K and pixels >= W are zero).
__global__ void k_pack_weights(const float* __restrict__ wts, int K, int np, int H, int W, int ntx,
                               uint16_t* __restrict__ out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // one 8-basis chunk of one pixel
  const int nk8 = np / 8;
  const size_t per_row = (size_t)ntx * nk8 * 128;
  const int f = blockIdx.y;
  if (i >= (size_t)H * per_row) return;
  const int y = (int)(i / per_row);
  size_t r = i - (size_t)y * per_row;
  const int xt = (int)(r / ((size_t)nk8 * 128));
  r -= (size_t)xt * nk8 * 128;
  const int k8 = (int)(r / 128), px = (int)(r % 128);
  const int x = xt * 128 + px;
  uint32_t pk[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float v[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = k8 * 8 + 2 * e + h;
      v[h] = (k < K && x < W) ? __ldg(&wts[(((size_t)f * K + k) * H + y) * W + x]) : 0.f;
    }
    pk[e] = pack_bf16x2(v[0], v[1]);
  }
  reinterpret_cast<uint4*>(out + (size_t)f * H * per_row * 8)[i] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
}

int launch_pack_weights(const p2s_plan_s* p, int F, const float* wts, cudaStream_t s) {
  const int np = p->mg_fold.n3;
  const size_t n = (size_t)p->H * p->ntx * (np / 8) * 128;
  dim3 grid((unsigned)((n + 255) / 256), F);
  k_pack_weights<<<grid, 256, 0, s>>>(wts, p->K, np, p->H, p->W, p->ntx, p->d_w);
  return (int)cudaGetLastError();
}

// Tensor map that delivers a 128-pixel tile's inputs as the A1 operand image
// [16 octets][k1 planes][8 px] in one TMA box; the dimension order is the smem order, the
// strides are X's layout (planes past nin are outside the map: zero-filled).
//   planes (xtile 0) [F][nin][HW]: dims {8 px, nin, HW/8 octets, F}, box {8, k1, 16, 1}
//   octet-pair tiles (xtile 2) [tiles][nin2/2][16][2][8]: dims {8 px, 2, nin2/2, 16 octets,
//   tiles}, box {8, 2, k1/2, 16, 1}
// Returns false when the layout / alignment does not allow it (k_mlp then loads A1 with
// per-thread copies).
static bool encode_x_map(CUtensorMap* m, const p2s_plan_s* p, const MlpArgs& a) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode)
      return false;
  }
  if (((uintptr_t)a.X & 15) || a.k1 > 256) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  if (a.xtile == 0) {
    // a box gathers 35 plane rows HW*2 bytes apart: measured faster than per-thread copies up
    // to 512^2 (k_mlp 1.43 -> 1.28 ms), much slower at 1080p (4 MB apart: 1.45 -> 2.28 ms);
    // the plan picks octet-pair tiles from 1M pixels, so larger plane strides only occur
    // when forced
    if (a.W % 8 || a.HW % 8 || a.HW > 512 * 512) return false;
    cuuint64_t dims[4] = {8, (cuuint64_t)a.nin, (cuuint64_t)a.HW / 8, (cuuint64_t)a.F};
    cuuint64_t strides[3] = {(cuuint64_t)a.HW * 2, 16, (cuuint64_t)a.nin * a.HW * 2};
    cuuint32_t box[4] = {8, (cuuint32_t)a.k1, 16, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(a.X), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  if (a.xtile == 2) {
    const int nin2 = (a.nin + 1) & ~1;
    cuuint64_t dims[5] = {8, 2, (cuuint64_t)nin2 / 2, 16, (cuuint64_t)a.F * a.tiles_per_frame};
    cuuint64_t strides[4] = {16, 512, 32, (cuuint64_t)nin2 * 256};
    cuuint32_t box[5] = {8, 2, (cuuint32_t)a.k1 / 2, 16, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<uint16_t*>(a.X), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  return false;
}

int launch_mlp(const p2s_plan_s* p, int F, bool folded, cudaStream_t s) {
  const MlpGeom& g = folded ? p->mg_fold : p->mg_plain;
  MlpArgs a;
  a.X = p->d_X;
  a.wout = p->d_w;
  a.blob = folded ? p->d_mlp_fold : p->d_mlp_plain;
  a.nin = g.nin;
  a.k1 = g.k1;
  a.n1 = g.n1;
  a.n2 = g.n2;
  a.n3 = g.n3;
  a.off_w2 = (uint32_t)g.off_w2;
  a.off_w3 = (uint32_t)g.off_w3;
  a.off_b1 = (uint32_t)g.off_b1;
  a.off_b2 = (uint32_t)g.off_b2;
  a.off_b3 = (uint32_t)g.off_b3;
  a.blob_bytes = (uint32_t)g.blob_bytes;
  a.HW = p->H * p->W;
  a.H = p->H;
  a.W = p->W;
  a.ntx = p->ntx;
  a.bias_folded = g.bias_folded ? 1 : 0;
  a.xtile = p->xtile;
  a.F = F;
  a.tiles_per_frame = p->H * p->ntx;
  const int nmax = std::max(std::max(g.n1, g.n2), g.n3);
  const int cols_wg = nmax <= 32 ? 32 : nmax <= 64 ? 64 : nmax <= 128 ? 128 : 256;
  const size_t blob_al = (g.blob_bytes + 127) & ~(size_t)127;
  const size_t per_wg = 128 * g.k1 * 2 + 128 * nmax * 2;
  int nwg = std::min(kMlpWG, 512 / cols_wg);
  while (nwg > 1 && blob_al + nwg * per_wg + 128 > 227 * 1024) --nwg;
  size_t sm = blob_al + nwg * per_wg + 128;
  auto kern = a.nin == 35 ? k_mlp<35> : a.nin == 33 ? k_mlp<33> : k_mlp<0>;
  P2S_SMEM_OPTIN(kern, sm);
  const int ntiles = F * a.tiles_per_frame;
  int grid = p->num_sms;  // persistent: one CTA (nwg tile pipelines) per SM
  if (nwg * grid > ntiles) grid = (ntiles + nwg - 1) / nwg;
  CUtensorMap tmap_x;
  std::memset(&tmap_x, 0, sizeof(tmap_x));
  a.a1_tma = (p->force & P2S_FORCE_MLP_A1_THREADS) ? 0 : encode_x_map(&tmap_x, p, a) ? 1 : 0;
  a.probe = nullptr;
#ifdef P2S_MLP_PROBE
  static unsigned long long* probe = nullptr;
  if (!probe) cudaMalloc(&probe, 8 * sizeof(unsigned long long));
  cudaMemsetAsync(probe, 0, 8 * sizeof(unsigned long long), s);
  a.probe = probe;
#endif
  kern<<<grid, 128 * nwg, sm, s>>>(a, tmap_x);
#ifdef P2S_MLP_PROBE
  {
    unsigned long long h[8];
    cudaMemcpyAsync(h, probe, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double nt = (double)ntiles;
    fprintf(stderr,
            "[mlp probe] tiles %.0f A1 %s | per tile cycles: A1 wait %.0f | L1 %.0f | prefetch+epi1 %.0f | sync %.0f | "
            "L2 %.0f | epi2 %.0f | sync+L3 %.0f | epi3+store %.0f\n",
            nt, a.a1_tma ? "TMA" : "threads", h[0] / nt, h[1] / nt, h[2] / nt, h[3] / nt, h[4] / nt, h[5] / nt,
            h[6] / nt, h[7] / nt);
  }
#endif
  return (int)cudaGetLastError();
}

}  // namespace p2s
