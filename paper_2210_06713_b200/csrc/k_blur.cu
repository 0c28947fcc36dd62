// k_blur.cu -- steps 4+5: the spatially varying blur of Eq.9 on tcgen05 tensor cores.
//
// Paper P:166-171 (Eq.9): I(x) = sum_m beta_{x,m} (phi_m (*) I_g)(x), "a set of spatially
// invariant convolutions".  Here conv_k(x) = (h_k (*) Iw_c)(x) for all K bases at once is
// an implicit GEMM  D[pixel][k] = sum_taps A[pixel][tap] B[tap][k]  with
//   M = 128 pixels of one output row (lane m <-> pixel x0 + 16 (m % 8) + m / 8),
//   N = np (K padded to 16), fp32 accumulators in TMEM, one per (channel, row) in flight,
//   K = taps: groups of 8 consecutive tap rows ty at one tap column tx, and for the T % 8
//   leftover tap rows, groups of 8 tap columns on transposed copies of single source rows
//   (chunks of the row contiguous: m-groups 16 B apart), written per row group into a
//   2-slot ring by the producer warp.
// The A operand is never materialised as im2col: the source tile of each channel is stored
// ONCE in shared memory as 16-byte chunks, chunk cc of source row r holding the 8 pixels
// at window offsets cc + 16 j (j = 0..7).  With the lane permutation above, the
// [128 x 8-tap-row] slab of any (output row, tx, tap-row group) is a canonical MN-major
// SWIZZLE_NONE layout (8 k-rows at 16 B, m-groups at SBO = one chunk column), so every
// K-step is pure descriptor arithmetic: start = tile + chunk (2c - tx) + rows, and the
// second 8-row group of the K-step is reached through the descriptor's leading-byte
// offset.  Descriptors of all K-steps are precomputed once per CTA in shared memory; the
// MMA warp issues C x RACC tcgen05.mma per K-step under elect.sync.
// The B operand (taps x bases, precomputed per K-step on the host) streams through a TMA
// bulk-copy ring shared by all accumulators (4 K-steps per stage).  The 16 epilogue warps
// read the accumulators with tcgen05.ld, release TMEM as soon as their reads have landed,
// form sum_k w_k(x) conv_k(x) with the P2S weights w (per-pixel 16-byte loads from HBM,
// prefetched one row group ahead), apply step 5 (normalise, Philox noise, clamp) and
// write the output: the only HBM write of the frame.
// PAIR mode (CTA pairs on adjacent x-tiles, cluster of 2): the even CTA issues
// tcgen05.mma.cta_group::2 with M = 256; each CTA supplies its own 128 pixels of A and half
// of the bases of B, halving the shared-memory and L2 traffic of the B operand per SM.
#include "p2s_dev.cuh"
#include "p2s_internal.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace p2s {

constexpr int kStepsPerStage = kBlurStepsPerStage;  // K-steps (B tiles) moved per ring stage
constexpr int kEpiWarps = 16;      // four warps per TMEM lane quarter, each owning two 16-basis chunks
constexpr int kBlurThreads = 64 + 32 * kEpiWarps;  // warp 0 TMA producer, warp 1 MMA issuer, epilogue
constexpr int kAccStride = 128;    // TMEM columns per accumulator
constexpr int kBlurLagStages = 1;  // B stages run for accumulator 0 alone at a row-group start (LAG)
constexpr int kLoadRows = 4;       // source rows staged per warp by the tile loader
constexpr int kSeg = 192;          // staged pixels per source row (>= 128 + T - 1 for T <= 63)

struct BlurArgs {
  const void* src;          // Iw [F][C][H][W] (bf16 or fp32)
  float* out;               // [F][C][H][W]
  const uint16_t* w;        // P2S weights [F][H][ntx][np/8][128 px][8] bf16 (k_mlp output)
  const uint8_t* bimg;      // [nks][np*32]
  const uint64_t* adesc;    // [nks] A descriptor of each K-step relative to tile base 0 (start, LBO, SBO)
  uint32_t idesc;           // instruction descriptor (M, N = np, A MN-major)
  const float* hsum;        // [np]
  int H, W, T, c, NC, RB, RS, nks, np, stages, ntx;
  int nks_main, g8, lr, nct;  // K-steps over 8-row groups; leftover tap rows on transposed rows
  uint32_t k0, k1;
  int64_t frame0;
  float sigma;
  int normalize, clamp01;
  int noise_x0, noise_W;    // step-5 noise counter y * noise_W + noise_x0 + x (slab strips: frame coordinates)
  int band0;                // first row band of the launch (a frame's blur split in two launches)
  unsigned long long* probe;  // optional [8] cycle counters (P2S_BLUR_PROBE), else null
  int brep, brows;            // B image copies; rows between copies (pair mode tensor map)
  size_t bstride;             // bytes between copies (bulk path)
};

__device__ __forceinline__ uint64_t clk() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int reflect_idx(int i, int n) {
  if (i < 0) i = -i;
  if (i >= n) i = 2 * n - 2 - i;
  return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

template <bool SRC_F32>
__device__ __forceinline__ uint16_t load_src_bf16(const void* src, size_t idx) {
  if (SRC_F32) return f_to_bf16(__ldg(reinterpret_cast<const float*>(src) + idx));
  return __ldg(reinterpret_cast<const uint16_t*>(src) + idx);
}

struct BlurSmem {
  uint32_t tile_bytes, b_bytes, ring_bytes;
  uint32_t off_ring, off_desc, off_hsum, off_part, off_bar, total;
};

__host__ __device__ inline BlurSmem blur_smem_layout(int C, int NC, int RS, int racc, int np, int nks, bool pair,
                                                     int stages, int lr, int nct) {
  BlurSmem L;
  // per channel: the column-ordered tile, then kBlurTSlots slots of racc x lr transposed rows
  L.tile_bytes = (blur_main_bytes(NC, RS) + (uint32_t)kBlurTSlots * racc * lr * nct * 16 + 127) & ~127u;
  L.b_bytes = (uint32_t)np * 32 / (pair ? 2 : 1);  // per K-step: this CTA's rows of B
  L.ring_bytes = stages * kStepsPerStage * L.b_bytes;
  const uint32_t stg_bytes = (kBlurThreads / 32) * kLoadRows * kSeg * 2;  // the loader's staging (bf16)
  L.off_ring = C * L.tile_bytes;
  L.off_desc = L.off_ring + (L.ring_bytes > stg_bytes ? L.ring_bytes : stg_bytes);
  L.off_hsum = L.off_desc + 8 * nks;
  L.off_part = (L.off_hsum + 4 * np + 15) & ~15u;  // [2 parity][3 parts][racc][C+1][128] partial sums
  L.off_bar = L.off_part + 2u * 3 * racc * (C + 1) * 128 * 4;
  L.total = L.off_bar + (2 * stages + 2 + 2 * kBlurTSlots) * 8 + 16;
  return L;
}

template <bool SRC_F32, int C, int RACC, bool PAIR>
__global__ void __launch_bounds__(kBlurThreads, 1)
    k_blur(const __grid_constant__ BlurArgs a, const __grid_constant__ CUtensorMap tmap_b) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const BlurSmem L = blur_smem_layout(C, a.NC, a.RS, RACC, a.np, a.nks, PAIR, a.stages, a.lr, a.nct);
  const int kBlurStages = a.stages;
  const uint32_t main_bytes = blur_main_bytes(a.NC, a.RS);
  const uint32_t sbo_src = (uint32_t)blur_rs_pad(a.RS) * 16;
  uint8_t* ring = smem + L.off_ring;
  float* s_hsum = reinterpret_cast<float*>(smem + L.off_hsum);
  uint64_t* s_adesc = reinterpret_cast<uint64_t*>(smem + L.off_desc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* full = bars;
  uint64_t* empty = bars + kBlurStages;
  uint64_t* tfull = bars + 2 * kBlurStages;
  uint64_t* tempty = tfull + 1;  // TMEM free (on the MMA-issuing CTA; one arrival per epilogue warp)
  uint64_t* trow_full = tempty + 1;               // [kBlurTSlots] transposed rows written (leader)
  uint64_t* trow_empty = trow_full + kBlurTSlots;  // [kBlurTSlots] their MMAs done (both CTAs)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(trow_empty + kBlurTSlots);
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  // TMEM columns of accumulator a (= ch * RACC + r) of row group rg (see the MMA issuer)
  constexpr bool LAG = C * RACC == 3;
  auto acc_col = [](int rg, int ac) -> uint32_t {
    return (uint32_t)((LAG ? ((3 * rg + ac) & 3) : ac) * kAccStride);
  };

  const int x0 = blockIdx.x * 128, y0 = (a.band0 + (int)blockIdx.y) * a.RB, f = blockIdx.z;
  const int HW = a.H * a.W;
  const uint32_t s_tile = smem_u32(smem);
  const uint64_t t_start = clk();

  for (int i = tid; i < a.nks; i += kBlurThreads) s_adesc[i] = a.adesc[i] + (uint64_t)(s_tile >> 4);
  for (int i = tid; i < a.np; i += kBlurThreads) s_hsum[i] = a.hsum[i];
  if (tid == 0) {
    for (int s = 0; s < kBlurStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, PAIR ? 2 * kEpiWarps : kEpiWarps);
    for (int s = 0; s < kBlurTSlots; ++s) {
      mbar_init(&trow_full[s], PAIR ? 2 : 1);
      mbar_init(&trow_empty[s], 1);
    }
    mbar_fence_init();
  }
  if (warp == 0) {
    if (PAIR)
      tmem_alloc_pair(tslot, 512);
    else
      tmem_alloc(tslot, 512);
  }

  {
    // ---- source tiles of every channel: chunk cc of row rl holds the 8 pixels at window
  // offsets cc + 16 j of source row y0 - c + rl (mirror boundary).  Each warp stages
  // kLoadRows row segments (bf16, all loads in flight together) in the not-yet-used B ring,
  // then packs the chunks.
  {
    constexpr int kE = (kSeg + 31) / 32;
    uint16_t* stg = reinterpret_cast<uint16_t*>(ring) + warp * kLoadRows * kSeg;
    const int rows_real = a.RB + a.T - 1;
    const int seg = 128 + a.T - 1;
    const int nwarps = kBlurThreads / 32;
    for (int ch = 0; ch < C; ++ch) {
      uint8_t* tile = smem + ch * L.tile_bytes;
      const size_t plane = ((size_t)f * C + ch) * HW;
      for (int rl0 = warp * kLoadRows; rl0 < a.RS; rl0 += nwarps * kLoadRows) {
        uint16_t v[kLoadRows][kE];
#pragma unroll
        for (int u = 0; u < kLoadRows; ++u) {
          const int rl = rl0 + u;
          const size_t rowb = plane + (size_t)reflect_idx(y0 - a.c + rl, a.H) * a.W;
#pragma unroll
          for (int e = 0; e < kE; ++e) {
            const int i = lane + 32 * e;
            v[u][e] = (rl < rows_real && i < seg) ? load_src_bf16<SRC_F32>(a.src, rowb + reflect_idx(x0 - a.c + i, a.W))
                                                  : (uint16_t)0;
          }
        }
#pragma unroll
        for (int u = 0; u < kLoadRows; ++u)
#pragma unroll
          for (int e = 0; e < kE; ++e)
            if (lane + 32 * e < kSeg) stg[u * kSeg + lane + 32 * e] = v[u][e];
        __syncwarp();
        for (int u = 0; u < kLoadRows; ++u) {
          const int rl = rl0 + u;
          if (rl >= a.RS) break;
          const uint16_t* sr = stg + u * kSeg;
          for (int cc = lane; cc < a.NC; cc += 32) {
            uint4 q = make_uint4(0, 0, 0, 0);
            if (rl < rows_real)
              q = make_uint4(sr[cc] | ((uint32_t)sr[cc + 16] << 16), sr[cc + 32] | ((uint32_t)sr[cc + 48] << 16),
                             sr[cc + 64] | ((uint32_t)sr[cc + 80] << 16), sr[cc + 96] | ((uint32_t)sr[cc + 112] << 16));
            *reinterpret_cast<uint4*>(tile + (size_t)cc * sbo_src + rl * 16) = q;
          }
        }
        __syncwarp();
      }
    }
  }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();  // both source tiles and all barrier inits visible to the pair
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (a.probe && tid == 0) atomicAdd(&a.probe[0], (unsigned long long)(clk() - t_start));

  const int n_rg = (a.RB + RACC - 1) / RACC;
  const int nst = (a.nks + kStepsPerStage - 1) / kStepsPerStage;
  const uint32_t bbytes = L.b_bytes;

  if (warp == 0) {
    // ---- TMA producer: the B tiles of every row group stream through the ring.
    uint32_t stage = 0, phase = 0;
    const int bcopy = (int)((blockIdx.x / 2 + blockIdx.y * 7 + blockIdx.z * 13) % a.brep);
    const uint8_t* bsrc = a.bimg + (size_t)bcopy * a.bstride;
    const int brow0 = bcopy * a.brows;
    const uint32_t trow_full_leader = PAIR ? mapa_shared(trow_full, 0) : smem_u32(trow_full);
    uint64_t p_fill = 0, p_wait = 0;
    // transposed copies of the leftover tap rows' source rows of row group rg:
    // slot[r][l][cc] = chunk cc of tile row rg*RACC + r + 8 g8 + l (zero beyond NC).  Issued
    // half-way through the previous row group's B loads, so it never drains the ring.
    auto fill_trows = [&](int rg) {
      const uint64_t tf0 = clk();
      const int slot = rg % kBlurTSlots;
      mbar_wait(&trow_empty[slot], ((rg / kBlurTSlots) & 1) ^ 1);
#pragma unroll
      for (int ch = 0; ch < C; ++ch) {
        uint8_t* tb = smem + ch * L.tile_bytes;
#pragma unroll
        for (int r = 0; r < RACC; ++r)
          for (int l = 0; l < a.lr; ++l) {
            const uint8_t* srow = tb + (rg * RACC + r + 8 * a.g8 + l) * 16;
            uint8_t* drow = tb + main_bytes + (((size_t)slot * RACC + r) * a.lr + l) * a.nct * 16;
            for (int cc = lane; cc < a.nct; cc += 32) {
              uint4 q = make_uint4(0, 0, 0, 0);
              if (cc < a.NC) q = *reinterpret_cast<const uint4*>(srow + (size_t)cc * sbo_src);
              *reinterpret_cast<uint4*>(drow + cc * 16) = q;
            }
          }
      }
      fence_async_smem();
      __syncwarp();
      // CTA-scope release: the rows are read by this CTA's own tensor-core half of the pair
      // MMA; fence.proxy.async above orders them for the async proxy.
      if (lane == 0) mbar_arrive_cluster(trow_full_leader + 8u * slot);
      p_fill += clk() - tf0;
    };
    if (a.lr > 0) fill_trows(0);
    for (int rg = 0; rg < n_rg; ++rg) {
      for (int st = 0; st < nst; ++st) {
        const uint64_t tw0 = clk();
        mbar_wait(&empty[stage], phase ^ 1);
        p_wait += clk() - tw0;
        const int t0 = st * kStepsPerStage;
        const int nt = min(kStepsPerStage, a.nks - t0);
        if (elect_one()) {
          if (PAIR) {  // both CTAs load their half; the bytes count on the leader's barrier
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kStepsPerStage * bbytes);
            tma_load_2d_pair(ring + stage * kStepsPerStage * bbytes, &tmap_b, 0,
                             brow0 + ((int)rank * a.nks + t0) * (int)(bbytes / 256), &full[stage]);
          } else {
            mbar_arrive_expect_tx(&full[stage], nt * bbytes);
            bulk_g2s(ring + stage * kStepsPerStage * bbytes, bsrc + (size_t)t0 * bbytes, nt * bbytes, &full[stage]);
          }
        }
        __syncwarp();
        if (++stage == kBlurStages) {
          stage = 0;
          phase ^= 1;
        }
        if (a.lr > 0 && st == nst / 2 && rg + 1 < n_rg) fill_trows(rg + 1);
      }
    }
    if (a.probe && lane == 0) {
      atomicAdd(&a.probe[10], (unsigned long long)p_fill);
      atomicAdd(&a.probe[11], (unsigned long long)p_wait);
    }
  } else if (warp == 1 && leader) {
    // ---- MMA issuer (one elected lane): C x RACC accumulators per K-step, kStepsPerStage
    // K-steps per ring stage so the issuing thread stays ahead of the tensor pipe.
    // LAG (3 accumulators, the 4th TMEM slot free): accumulator a of row group rg lives in
    // slot (3 rg + a) mod 4, so accumulator 0 of the next row group starts in the free slot
    // on the first kBlurLagStages B stages while the epilogue drains the previous group;
    // accumulators 1-2 catch up on the same stages once it has released its slots.  The K
    // order within each accumulator is unchanged (results are bit-identical to no lag).
    // The epilogue's tcgen05.ld waits behind MMAs already in flight, so a longer lag delays
    // the drain by as much as it hides (measured, DESIGN 6c): one stage.
    uint32_t stage = 0, phase = 0;
    const uint64_t ch_step = (uint64_t)(L.tile_bytes >> 4);
    const uint64_t b_desc_base = umma_desc(smem_u32(ring), 128, 256);
    if (tmem != 0) __trap();  // accumulators are addressed from column 0
    uint64_t w_full = 0, w_tempty = 0, w_trow = 0, p_a = 0, p_b = 0, p_c = 0;
    const uint64_t t_mma0 = clk();
    const int st_tr = a.nks_main / kStepsPerStage;  // first stage with a transposed K-step
    for (int rg = 0; rg < n_rg; ++rg) {
      const uint64_t a_row_desc = (uint64_t)(rg * RACC);  // start address += rows of this group
      const int slot = rg % kBlurTSlots;
      const uint64_t t_row_desc = (uint64_t)(slot * RACC * a.lr * a.nct);  // transposed rows of this group
      const uint64_t t_rstep = (uint64_t)(a.lr * a.nct);
      const int nA = (LAG && rg > 0) ? min(kBlurLagStages, nst) : 0;  // lagged stages
      // one ring stage: MMAs of accumulators [a0, a1) on its K-steps; optionally release it
      auto issue_stage = [&](int st, int acc0, int acc1, bool release) {
        const uint64_t bdesc0 = b_desc_base + (uint64_t)((stage * kStepsPerStage * bbytes) >> 4);
        const int t0 = st * kStepsPerStage;
        if (elect_one()) {
#pragma unroll
          for (int u = 0; u < kStepsPerStage; ++u) {
            const int t = t0 + u;
            if (t < a.nks) {
              const uint64_t bd = bdesc0 + (uint64_t)((u * bbytes) >> 4);
              const bool tr = t >= a.nks_main;
              const uint64_t ad = s_adesc[t] + (tr ? t_row_desc : a_row_desc);
              const uint64_t rstep = tr ? t_rstep : 1ull;
              const uint32_t acc = t > 0 ? 1u : 0u;
#pragma unroll
              for (int ac = 0; ac < C * RACC; ++ac) {
                if (ac < acc0 || ac >= acc1) continue;
                const int ch = ac / RACC, r = ac - ch * RACC;
                const uint32_t d = acc_col(rg, ac);
                if (PAIR)
                  umma_bf16_pair(d, ad + ch * ch_step + r * rstep, bd, a.idesc, acc);
                else
                  umma_bf16(d, ad + ch * ch_step + r * rstep, bd, a.idesc, acc);
              }
            }
          }
          if (release) {
            if (PAIR)
              umma_commit_pair(&empty[stage]);
            else
              umma_commit(&empty[stage]);
          }
        }
        __syncwarp();
      };
      auto wait_stage = [&](int st) {
        const uint64_t t1c = clk();
        mbar_wait(&full[stage], phase);
        w_full += clk() - t1c;
        if (st == st_tr && a.nks > a.nks_main) {
          const uint64_t t2c = clk();
          if (PAIR)
            mbar_wait_cluster(&trow_full[slot], (rg / kBlurTSlots) & 1);
          else
            mbar_wait(&trow_full[slot], (rg / kBlurTSlots) & 1);
          w_trow += clk() - t2c;
        }
        tc_fence_after();
      };
      auto next_stage = [&]() {
        if (++stage == kBlurStages) {
          stage = 0;
          phase ^= 1;
        }
      };
      const uint32_t stage_a = stage, phase_a = phase;
      const uint64_t ph0 = clk();
      for (int st = 0; st < nA; ++st) {  // phase A: accumulator 0 alone, stages kept
        wait_stage(st);
        issue_stage(st, 0, 1, false);
        next_stage();
      }
      {
        uint64_t t0c = clk();
        mbar_wait(tempty, (rg & 1) ^ 1);  // the previous row group's slots are drained
        w_tempty += clk() - t0c;
        tc_fence_after();
      }
      const uint64_t ph1 = clk();
      if (nA > 0) {  // phase B: the other accumulators on the same stages, then release them
        stage = stage_a;
        phase = phase_a;
        for (int st = 0; st < nA; ++st) {
          issue_stage(st, 1, C * RACC, true);
          next_stage();
        }
      }
      const uint64_t ph2 = clk();
      for (int st = nA; st < nst; ++st) {
        wait_stage(st);
        issue_stage(st, 0, C * RACC, true);
        next_stage();
      }
      const uint64_t ph3 = clk();
      p_a += ph1 - ph0;
      p_b += ph2 - ph1;
      p_c += ph3 - ph2;
      if (elect_one()) {
        if (PAIR) {
          umma_commit_pair(tfull);
          if (a.lr > 0) umma_commit_pair(&trow_empty[slot]);
        } else {
          umma_commit(tfull);
          if (a.lr > 0) umma_commit(&trow_empty[slot]);
        }
      }
      __syncwarp();
    }
    if (a.probe && lane == 0) {
      atomicAdd(&a.probe[1], (unsigned long long)w_full);
      atomicAdd(&a.probe[2], (unsigned long long)w_tempty);
      atomicAdd(&a.probe[3], (unsigned long long)(clk() - t_mma0));
      atomicAdd(&a.probe[9], (unsigned long long)w_trow);
      atomicAdd(&a.probe[12], (unsigned long long)p_a);
      atomicAdd(&a.probe[13], (unsigned long long)p_b);
      atomicAdd(&a.probe[14], (unsigned long long)p_c);
    }
  } else if (warp >= 2) {
    // ---- epilogue warps 2..17: TMEM lane quarter qd = warp % 4; part h = 0..3 owns the
    // 16-basis chunks 2h and 2h+1.  Each warp reads its accumulator columns, releases TMEM
    // right after its last tcgen05.ld has landed (the next row group's MMAs start while the
    // sums are formed), weights them with w (prefetched from HBM one group ahead, 16-byte
    // loads of 8 bases), and parts 1-3 hand partial sums to part 0, which applies step 5.
    const int qd = warp & 3;
    const int h = (warp - 2) >> 2;
    const int m = qd * 32 + lane;
    const int q = 16 * (m & 7) + (m >> 3);
    const int x = x0 + q;
    const uint32_t tl = tmem + ((uint32_t)(qd * 32) << 16);
    const uint32_t t_tempty_leader = PAIR ? mapa_shared(tempty, 0) : 0u;
    float* part = reinterpret_cast<float*>(smem + L.off_part);
    const int nch = a.np / 16;
    const int xt = blockIdx.x;
    const size_t wrow = (size_t)a.ntx * a.np * 128;  // elements per image row of w
    const uint16_t* wpix = a.w + ((size_t)f * a.H * a.ntx + xt) * a.np * 128 + (size_t)q * 8;
    const bool xin = x0 < a.W;
    uint4 wn[RACC][2][2];
    auto load_w = [&](int rg) {
#pragma unroll
      for (int r = 0; r < RACC; ++r) {
        const int y = y0 + rg * RACC + r;
        const bool ok = xin && y < a.H;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int cb = 2 * h + c;
#pragma unroll
          for (int k8 = 0; k8 < 2; ++k8) {
            wn[r][c][k8] = make_uint4(0, 0, 0, 0);
            if (ok && cb < nch)
              wn[r][c][k8] = __ldg(reinterpret_cast<const uint4*>(wpix + (size_t)y * wrow + (size_t)(2 * cb + k8) * 1024));
          }
        }
      }
    };
    load_w(0);
    // last (r, c) with a chunk: the release point
    const int c_last = (2 * h + 1 < nch) ? 1 : 0;
    const bool has_any = 2 * h < nch;
    uint64_t e_wait = 0, e_work = 0, e_rel = 0;
    for (int rg = 0; rg < n_rg; ++rg) {
      uint4 wc[RACC][2][2];
#pragma unroll
      for (int r = 0; r < RACC; ++r)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          wc[r][c][0] = wn[r][c][0];
          wc[r][c][1] = wn[r][c][1];
        }
      const uint64_t t0c = clk();
      mbar_wait(tfull, rg & 1);
      tc_fence_after();
      const uint64_t t1c = clk();
      e_wait += t1c - t0c;
      auto release = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR)
            mbar_arrive_cluster(t_tempty_leader);
          else
            mbar_arrive(tempty);
        }
        e_rel += clk() - t1c;
      };
      if (!has_any) release();
      float accs[RACC][C + 1];
#pragma unroll
      for (int r = 0; r < RACC; ++r) {
#pragma unroll
        for (int ch = 0; ch <= C; ++ch) accs[r][ch] = 0.f;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int cb = 2 * h + c;
          if (cb < nch) {
            uint32_t v[C][16];
#pragma unroll
            for (int ch = 0; ch < C; ++ch) tmem_ld16_issue(tl + acc_col(rg, ch * RACC + r) + cb * 16, v[ch]);
            float wf[16];
            {
              const uint32_t* wp = reinterpret_cast<const uint32_t*>(&wc[r][c][0]);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                wf[2 * i] = __uint_as_float(wp[i] << 16);
                wf[2 * i + 1] = __uint_as_float(wp[i] & 0xFFFF0000u);
              }
            }
            if (a.normalize) {
#pragma unroll
              for (int i = 0; i < 16; ++i) accs[r][C] = fmaf(wf[i], s_hsum[cb * 16 + i], accs[r][C]);
            }
            tmem_wait_ld();
            if (r == RACC - 1 && c == c_last) release();
#pragma unroll
            for (int ch = 0; ch < C; ++ch)
#pragma unroll
              for (int i = 0; i < 16; ++i) accs[r][ch] = fmaf(wf[i], __uint_as_float(v[ch][i]), accs[r][ch]);
          }
        }
      }
      if (rg + 1 < n_rg) load_w(rg + 1);
      // parts 1-3 -> shared memory (double-buffered by group parity, one named barrier per
      // parity so a fast part cannot complete the other group's barrier)
      float* pb = part + (size_t)(rg & 1) * 3 * RACC * (C + 1) * 128;
      const int bar_id = 1 + (rg & 1);
      if (h != 0) {
#pragma unroll
        for (int r = 0; r < RACC; ++r)
#pragma unroll
          for (int ch = 0; ch <= C; ++ch) pb[(((size_t)(h - 1) * RACC + r) * (C + 1) + ch) * 128 + m] = accs[r][ch];
        asm volatile("bar.arrive %0, %1;" ::"r"(bar_id), "n"(kEpiWarps * 32) : "memory");
      } else {
        asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(kEpiWarps * 32) : "memory");
#pragma unroll
        for (int r = 0; r < RACC; ++r) {
          const int y = y0 + rg * RACC + r;
#pragma unroll
          for (int p3 = 0; p3 < 3; ++p3)
#pragma unroll
            for (int ch = 0; ch <= C; ++ch) accs[r][ch] += pb[(((size_t)p3 * RACC + r) * (C + 1) + ch) * 128 + m];
          if (y < a.H && x < a.W) {
            const float g = accs[r][C];
#pragma unroll
            for (int ch = 0; ch < C; ++ch) {
              float o = accs[r][ch];
              if (a.normalize) o = o / g;
              if (a.sigma != 0.f) {
                const int64_t fr = a.frame0 + f;
                uint4 rx = philox4x32_10(make_uint4((uint32_t)(y * a.noise_W + a.noise_x0 + x), (uint32_t)ch | (1u << 16), (uint32_t)fr,
                                                    (uint32_t)((uint64_t)fr >> 32)),
                                         a.k0, a.k1);
                o += a.sigma * box_muller(rx.x, rx.y).x;
              }
              if (a.clamp01) o = fminf(fmaxf(o, 0.f), 1.f);
              a.out[((size_t)f * C + ch) * HW + (size_t)y * a.W + x] = o;
            }
          }
        }
      }
      e_work += clk() - t1c;
    }
    if (a.probe && warp == 2 && lane == 0) {
      atomicAdd(&a.probe[4], (unsigned long long)e_wait);
      atomicAdd(&a.probe[5], (unsigned long long)e_work);
      atomicAdd(&a.probe[8], (unsigned long long)e_rel);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (a.probe && tid == 0) {
    atomicAdd(&a.probe[6], (unsigned long long)(clk() - t_start));
    atomicAdd(&a.probe[7], 1ull);
  }
  if (PAIR) cluster_sync_all();  // the pair's MMAs and remote arrivals are all done
  tc_fence_after();
  if (warp == 0) {
    if (PAIR)
      tmem_dealloc_pair(tmem, 512);
    else
      tmem_dealloc(tmem, 512);
  }
}

template <bool SRC_F32, int C, int RACC, bool PAIR>
static int launch_blur_t(const BlurArgs& a, const CUtensorMap& tb, dim3 grid, size_t sm, cudaStream_t s) {
  auto kern = k_blur<SRC_F32, C, RACC, PAIR>;
  P2S_SMEM_OPTIN(kern, sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kBlurThreads);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a, tb);
  return (int)cudaGetLastError();
}

template <bool SRC_F32, bool PAIR>
static int launch_blur_c(int C, const BlurArgs& a, const CUtensorMap& tb, dim3 grid, size_t sm, cudaStream_t s) {
  switch (C) {
    case 1: return launch_blur_t<SRC_F32, 1, 4, PAIR>(a, tb, grid, sm, s);
    case 2: return launch_blur_t<SRC_F32, 2, 2, PAIR>(a, tb, grid, sm, s);
    case 3: return launch_blur_t<SRC_F32, 3, 1, PAIR>(a, tb, grid, sm, s);
    default: return launch_blur_t<SRC_F32, 4, 1, PAIR>(a, tb, grid, sm, s);
  }
}

int launch_blur(const p2s_plan_s* p, int F, const void* src, bool src_f32, uint64_t seed, int64_t frame0, float* out,
                cudaStream_t s, int band0, int nbands) {
  const BlurGeom& g = p->bg;
  BlurArgs a;
  a.src = src;
  a.out = out;
  a.w = p->d_w;
  a.bimg = g.bimg;
  a.adesc = g.adesc;
  a.idesc = umma_idesc_bf16(g.pair ? 256 : 128, g.np, true, false);
  a.hsum = g.hsum;
  a.brep = g.brep;
  a.brows = g.brows;
  a.bstride = g.bstride;
  a.H = p->H;
  a.W = p->W;
  a.ntx = p->ntx;
  a.T = g.T;
  a.c = g.c;
  a.NC = g.NC;
  a.RB = g.RB;
  a.RS = g.RS;
  a.nks = g.nks;
  a.nks_main = g.nks_main;
  a.g8 = g.g8;
  a.lr = g.lr;
  a.nct = g.nct;
  a.np = g.np;
  a.k0 = (uint32_t)seed;
  a.k1 = (uint32_t)(seed >> 32);
  a.frame0 = frame0;
  a.sigma = p->noise_sigma;
  a.noise_x0 = p->slab_G > 1 ? p->slab_hx0 : 0;
  a.noise_W = p->slab_G > 1 ? p->W_glob : p->W;
  a.normalize = p->normalize;
  a.clamp01 = p->clamp01;
  a.probe = nullptr;
  // phase cycle counters: a tuning build only (make EXTRA=-DP2S_BLUR_PROBE)
#ifdef P2S_BLUR_PROBE
  static unsigned long long* probe = nullptr;
  const bool want_probe = true;
#else
  unsigned long long* probe = nullptr;
  const bool want_probe = false;
#endif
  if (want_probe) {
    if (!probe) cudaMalloc(&probe, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(probe, 0, 16 * sizeof(unsigned long long), s);
    a.probe = probe;
  }
  const bool pair = g.pair;
  a.stages = g.stages;
  const BlurSmem L = blur_smem_layout(p->C, a.NC, a.RS, g.racc, a.np, a.nks, pair, g.stages, a.lr, a.nct);
  // TMEM: this kernel owns all 512 columns of its SM; keep shared memory above half the SM
  // so that two CTAs never co-reside and contend for tcgen05.alloc.
  size_t sm = L.total < 116 * 1024 ? 116 * 1024 : L.total;
  int gx = p->ntx;
  if (pair) gx = (gx + 1) / 2 * 2;  // whole CTA pairs; a trailing dummy CTA stores nothing
  const int bands = (p->H + g.RB - 1) / g.RB;
  a.band0 = std::max(0, std::min(band0, bands));
  const int nb = nbands < 0 ? bands - a.band0 : std::min(nbands, bands - a.band0);
  if (nb <= 0) return 0;
  dim3 grid(gx, nb, F);
  int rc;
  if (pair)
    rc = src_f32 ? launch_blur_c<true, true>(p->C, a, p->tmap_b, grid, sm, s)
                 : launch_blur_c<false, true>(p->C, a, p->tmap_b, grid, sm, s);
  else
    rc = src_f32 ? launch_blur_c<true, false>(p->C, a, p->tmap_b, grid, sm, s)
                 : launch_blur_c<false, false>(p->C, a, p->tmap_b, grid, sm, s);
  if (want_probe) {  // debug: per-CTA averages of the phase cycle counters
    unsigned long long h[16];
    cudaMemcpyAsync(h, probe, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double n = h[7] ? (double)h[7] : 1.0, nm = pair ? n / 2 : n;
    fprintf(stderr,
            "[blur probe] CTAs %llu  per CTA cycles: total %.0f prologue %.0f | MMA warp: loop %.0f wait_full %.0f "
            "wait_tmem %.0f wait_trow %.0f | epilogue warp 2: wait %.0f work %.0f (tfull to release %.0f) | "
            "producer: trow fill %.0f ring wait %.0f | issuer phases A+wait %.0f B %.0f C %.0f\n",
            h[7], h[6] / n, h[0] / n, h[3] / nm, h[1] / nm, h[2] / nm, h[9] / nm, h[4] / n, h[5] / n, h[8] / n,
            h[10] / n, h[11] / n, h[12] / nm, h[13] / nm, h[14] / nm);
  }
  return rc;
}

// Host helper: rows per CTA that fit the shared-memory budget, balanced over the bands.
// Output rows per CTA: the largest that fits shared memory is the cheapest per row (the
// tile's halo and prologue are amortised), but the band count also sets how many CTA
// (pairs) a launch of F frames has, and a last wave that is mostly empty costs a full wave.
// Cost model in output-row units: waves(bands) x (RB + 2.5), the 2.5 rows being the
// per-CTA fixed cost (measured at 512^2 RGB: prologue ~28k cycles = 1.8 rows of 15.4k,
// plus the last row's epilogue that no MMA overlaps); the cheapest band count wins.
int blur_rows_per_cta(int C, int T, int np, int racc, int H, int W, bool pair, int stages, int F, int nsm) {
  const int NC = T + 15, nct = NC > 23 ? NC : 23;
  int g8, lr;
  blur_tap_split(T, &g8, &lr);
  const int nks = (T * g8 + 1) / 2 + (lr * ((T + 7) / 8) + 1) / 2;
  int best = racc;
  for (int RB = racc; RB <= 64; RB += racc) {
    const int RS = blur_tile_rows(RB, T, g8, lr);
    if (blur_smem_layout(C, NC, RS, racc, np, nks, pair, stages, lr, nct).total <= 227 * 1024) best = RB;
  }
  const int ntx = (W + 127) / 128;
  const int ux = pair ? (ntx + 1) / 2 : ntx;
  const int slots = std::max(1, pair ? nsm / 2 : nsm);
  const int b0 = (H + best - 1) / best;
  int pick = -1;
  double pick_cost = 0.0;
  for (int bands = b0; bands <= std::min(H, 3 * b0); ++bands) {
    int rb = (H + bands - 1) / bands;
    rb = (rb + racc - 1) / racc * racc;
    if (rb > best) continue;
    const int be = (H + rb - 1) / rb;
    const long long units = (long long)ux * be * std::max(1, F);
    const long long waves = (units + slots - 1) / slots;
    const double cost = (double)waves * (rb + 2.5);
    if (pick < 0 || cost < pick_cost - 1e-9) {
      pick = rb;
      pick_cost = cost;
    }
  }
  return pick > 0 ? pick : best;
}

// Blur waves of a launch of F frames (CTA pairs or CTAs over the SM slots).
int blur_waves(const p2s_plan_s* p, int F) {
  const BlurGeom& g = p->bg;
  const int bands = (p->H + g.RB - 1) / g.RB;
  const int ux = g.pair ? (p->ntx + 1) / 2 : p->ntx;
  const int slots = std::max(1, g.pair ? p->nsm / 2 : p->nsm);
  return (int)(((long long)ux * bands * F + slots - 1) / slots);
}

}  // namespace p2s
