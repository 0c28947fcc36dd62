// Microbenchmark (development tool, not part of libp2s): steady-state issue-to-completion
// cycles per tcgen05.mma kind::f16 for the operand layouts the blur uses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2210_06713_b200/csrc \
//        tools/mma_bench.cu -o tools/mma_bench -lcuda
// One CTA per SM, zero-filled shared memory, NMMA back-to-back MMAs into one accumulator.
#include <cstdio>
#include <cstdlib>

#include "p2s_dev.cuh"

using namespace p2s;

struct Cfg {
  int a_mn, b_mn, N, nmma;
  uint32_t a_lbo, a_sbo, b_lbo, b_sbo;
  int a_stride;   // bytes added to the A start address per MMA (cycled over 64 values)
  int pair;       // cta_group::2
  int nacc;       // accumulators rotated over (column stride N)
  int a_swz, b_swz;  // layout type field (bits 61-63): 0 none, 2 = 128B swizzle
  int a_tiles;       // >1: rotate A over this many tiles 48 KB apart (channels)
  int b_ring;        // >1: rotate B over this many 2 KB slots
  int commit_every;  // >0: tcgen05.commit to a scratch barrier every this many MMAs
  int rnd;           // random operand data instead of zeros
  int tile_dist;     // bytes between the A tiles (default 40960)
};

__device__ __forceinline__ void umma_bf16_2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc));
}

template <bool PAIR>
__global__ void __launch_bounds__(128, 1) k_mma_bench(Cfg c, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid * 16; i < 200 * 1024; i += 128 * 16) {
    uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x;
    uint32_t w[4];
    for (int k = 0; k < 4; ++k) {
      h ^= h >> 13;
      h *= 0x5bd1e995u;
      h ^= h >> 15;
      // two bf16 values in [-1, 1): sign, exponent 126/127, random mantissa
      w[k] = c.rnd ? ((h & 0x807F807Fu) | 0x3F003F00u) : 0u;
    }
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    mbar_fence_init();
  }
  if (tid < 32) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc(&slot, 512);
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 128 * 1024);
  const uint32_t idesc = umma_idesc_bf16(PAIR ? 256 : 128, c.N, c.a_mn, c.b_mn);
  if (tid < 32 && rank == 0) {
    const uint64_t bd = umma_desc(sb, c.b_lbo, c.b_sbo) | ((uint64_t)c.b_swz << 61);
    const uint64_t t0 = clock64();
    if (elect_one()) {
      if (c.a_tiles > 1 || c.b_ring > 1 || c.commit_every > 0) {
        // blur-like issue: per K-step one MMA per channel tile (3), B slot per K-step, commit every 2 K-steps
        const uint64_t ad0 = umma_desc(sa, c.a_lbo, c.a_sbo);
        const int nt = c.a_tiles;
        if (nt == 2) {
          const uint64_t d1 = (uint64_t)((c.tile_dist ? c.tile_dist : 40960) >> 4);
          for (int i = 0, ks = 0; i < c.nmma; i += 4, ks += 2) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const uint64_t bdi = bd + (uint64_t)((((ks + u) & (c.b_ring - 1)) * 2048) >> 4);
              const uint64_t adk = ad0 + (uint64_t)(((ks + u) & 63) * c.a_stride >> 4);
              const uint32_t acc = (ks + u) > 0 ? 1u : 0u;
              if (PAIR) {
                umma_bf16_2(tmem, adk, bdi, idesc, acc);
                umma_bf16_2(tmem + c.N, adk + d1, bdi, idesc, acc);
              } else {
                umma_bf16(tmem, adk, bdi, idesc, acc);
                umma_bf16(tmem + c.N, adk + d1, bdi, idesc, acc);
              }
            }
            if (c.commit_every > 0) {
              if (PAIR)
                asm volatile(
                    "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                        smem_u32(&bar2)),
                    "h"((uint16_t)3)
                    : "memory");
              else
                umma_commit(&bar2);
            }
          }
        } else
        for (int i = 0, ks = 0; i < c.nmma; i += 2 * nt, ks += 2) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const uint64_t bdi = bd + (uint64_t)((((ks + u) & (c.b_ring - 1)) * 2048) >> 4);
            const uint64_t adk = ad0 + (uint64_t)(((ks + u) & 63) * c.a_stride >> 4);
#pragma unroll 4
            for (int ch = 0; ch < nt; ++ch) {
              const uint32_t acc = (ks + u) > 0 ? 1u : 0u;
              if (PAIR)
                umma_bf16_2(tmem + ch * c.N, adk + (uint64_t)(ch * ((c.tile_dist ? c.tile_dist : 40960) >> 4)), bdi, idesc, acc);
              else
                umma_bf16(tmem + ch * c.N, adk + (uint64_t)(ch * ((c.tile_dist ? c.tile_dist : 40960) >> 4)), bdi, idesc, acc);
            }
          }
          if (c.commit_every > 0) {
            if (PAIR)
              asm volatile(
                  "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                      smem_u32(&bar2)),
                  "h"((uint16_t)3)
                  : "memory");
            else
              umma_commit(&bar2);
          }
        }
      } else {
        for (int i = 0; i < c.nmma; ++i) {
          const uint64_t ad = umma_desc(sa + (uint32_t)((i & 63) * c.a_stride), c.a_lbo, c.a_sbo) | ((uint64_t)c.a_swz << 61);
          if (PAIR)
            umma_bf16_2(tmem + (i % c.nacc) * c.N, ad, bd, idesc, i >= c.nacc);
          else
            umma_bf16(tmem + (i % c.nacc) * c.N, ad, bd, idesc, i >= c.nacc);
        }
      }
      if (PAIR)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"((uint16_t)3)
            : "memory");
      else
        umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    const uint64_t t1 = clock64();
    if (tid == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
  } else if (PAIR && tid < 32) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  if (tid < 32) {
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    else
      tmem_dealloc(tmem, 512);
  }
}

template <bool PAIR>
static cudaError_t launch(Cfg c, unsigned long long* d) {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_mma_bench<PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_mma_bench<PAIR>, c, d);
}

static void run(const char* name, Cfg c) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  cudaError_t e = c.pair ? launch<true>(c, d) : launch<false>(c, d);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const int issuers = c.pair ? 74 : 148;
  const double cyc = (double)h / issuers / c.nmma;
  printf("%-44s N=%3d acc=%d %7.1f cyc/MMA  (floor %.0f)  %s\n", name, c.N, c.nacc, cyc, 128.0 * c.N / 256.0,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  const int n = 8196;  // multiple of 6
  // blur-like pair issue, 3 channel tiles, N = 112: A m-groups one chunk column apart
  // (SBO = padded rows x 16, the column-ordered tile) vs one 16-byte chunk apart (SBO = 16,
  // the transposed leftover rows)
  for (uint32_t sbo : {1232u, 1264u, 16u, 32u}) {
    for (int rnd : {0, 1}) {
      Cfg c = {1, 0, 112, n, 128, sbo, 128, 256, 16, 1, 1, 0, 0, 3, 16, 1, rnd, 40960};
      char name[128];
      snprintf(name, sizeof(name), "PAIR 3 tiles A sbo=%u rnd=%d", sbo, rnd);
      run(name, c);
    }
  }
  // accumulator chains: consecutive MMAs into 1..4 rotating accumulators (a run of MMAs into
  // one accumulator waits on its own result)
  for (int nacc : {1, 2, 3, 4}) {
    Cfg c = {1, 0, 112, n, 128, 1232u, 128, 256, 16, 1, nacc, 0, 0, 3, 16, 1, 1, 40960};
    char name[128];
    snprintf(name, sizeof(name), "PAIR 3 tiles, %d accumulator(s)", nacc);
    run(name, c);
  }
  return 0;
}
