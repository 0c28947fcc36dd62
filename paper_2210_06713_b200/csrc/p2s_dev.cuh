// p2s_dev.cuh -- device helpers: Philox4x32-10, Box-Muller, bf16 packing, and the
// sm_100a tcgen05 / TMEM / mbarrier / bulk-copy PTX wrappers used by the MLP and
// blur kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace p2s {

// ------------------------------------------------------------------ Philox4x32-10
// Salmon et al. SC'11; constants as in Random123.  Counter layout:
// (index, slot | stream << 16, frame_lo, frame_hi), key (seed_lo, seed_hi).
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// (g1, g2) = sqrt(-2 ln u1) (cos 2 pi u2, sin 2 pi u2), u1 = (a+1) 2^-32, u2 = b 2^-32.
// -ln u1 is evaluated as -log1p(-(2^32-1-a) 2^-32) for u1 > 1/2 to keep relative accuracy.
__device__ __forceinline__ float2 box_muller(uint32_t a, uint32_t b) {
  const float k = 2.3283064365386963e-10f;  // 2^-32
  float nl;
  if (a >= 0x80000000u) {
    nl = -log1pf(-(float)(0xFFFFFFFFu - a) * k);
  } else {
    nl = -logf(((float)a + 1.0f) * k);
  }
  float r = sqrtf(2.0f * nl);
  float s, c;
  sincospif((float)b * (2.0f * k), &s, &c);
  return make_float2(r * c, r * s);
}

// Same transform with the SFU approximations (MUFU lg2/sin/cos): -ln u1 from lg2.approx,
// the angle folded to [-pi, pi) (cos/sin(2 pi u2) = -cos/sin(2 pi (u2 - 1/2))).  Absolute
// error ~1e-6; used on the per-bin spectral noise hot path.
__device__ __forceinline__ float2 box_muller_fast(uint32_t a, uint32_t b) {
  const float k = 2.3283064365386963e-10f;  // 2^-32
  const float u1 = fmaf((float)a, k, k);    // (a + 1) 2^-32 in (0, 1]
  const float r = sqrtf(-2.0f * 0.69314718055994531f * __log2f(u1));
  float s, c;
  __sincosf(6.28318530717958648f * fmaf((float)b, k, -0.5f), &s, &c);
  return make_float2(-r * c, -r * s);
}

// MLP input X (bf16): xtile = 1 -> per 128-pixel row tile, [F][H][ntx][nin][128 px] (one
// tile's inputs are one contiguous 256*nin-byte block, so k_mlp's 16-byte chunk loads stay
// within a few pages; consecutive pixels stay adjacent, so the column kernels' stores keep
// their full-sector runs); xtile = 0 -> planes [F][nin][H][W].
// xtile = 2 -> per 128-pixel row tile, [F][H][ntx][nin/2 mode pairs][16 octets][2 modes][8 px]
// (nin rounded up to even): the two modes of a pair for 8 adjacent pixels are one 32-byte
// sector, so a long-column CTA writes a row of its block as one full-sector store, and each
// (mode, octet) is still the 16-byte chunk of 8 pixels the MLP's A operand loads.
__device__ __forceinline__ size_t x_index(int xtile, int f, int k, int nin, int H, int W, int ntx, int y, int x) {
  if (!xtile) return ((size_t)f * nin + k) * (size_t)H * W + (size_t)y * W + x;
  const int xt = x >> 7, px = x & 127;
  if (xtile == 2) {
    const int nin2 = (nin + 1) & ~1;
    return (((size_t)f * H + y) * ntx + xt) * (size_t)(nin2 * 128) + (size_t)(((k >> 1) * 16 + (px >> 3)) * 16 +
                                                                             (k & 1) * 8 + (px & 7));
  }
  return ((((size_t)f * H + y) * ntx + xt) * nin + k) * 128 + px;
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
__device__ __forceinline__ float bf16_to_f(uint16_t v) { return __uint_as_float(((uint32_t)v) << 16); }
__device__ __forceinline__ uint16_t f_to_bf16(float f) {
  __nv_bfloat16 b = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&b);
}

// ------------------------------------------------------------------ sm_100a async / tensor-core PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory matrix descriptor, SWIZZLE_NONE (canonical "interleave" layout):
//   K-major : element (row r, k) at (r%8)*16 + (r/8)*SBO + (k/8)*LBO + (k%8)*2
//   MN-major: element (mn, k)    at (mn%8)*2 + (mn/8)*SBO + (k%8)*16 + (k/8)*LBO
// bits [0,14) start>>4, [16,30) LBO>>4, [32,46) SBO>>4, [46,48) version = 1 (sm_100),
// [49,52) base offset 0, bit 52 LBO mode 0, [61,64) layout 0 = SWIZZLE_NONE.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// Instruction descriptor, kind::f16: D f32, A/B bf16, dense.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N, bool a_mn_major, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Arrive on an mbarrier when all prior tcgen05.mma of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// Make generic-proxy shared-memory writes visible to the async proxy (tensor core / TMA).
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}


// Issue-only variant (batch several, then one tmem_wait_ld()); registers are valid after the wait.
__device__ __forceinline__ void tmem_ld16_issue(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Wait for the phase with the given parity.  Watchdog: a pipeline bug must not hang
// the GPU, so after ~4 s of waiting the kernel traps (launch error on the host).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, parity)) return;
  const uint64_t t0 = global_ns();
  uint32_t n = 0;
  while (!mbar_try_wait(a, parity)) {
    if ((++n & 1023u) == 0 && global_ns() - t0 > 4000000000ull) __trap();
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared (TMA engine, non-tensor), completes tx bytes on bar.
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// One lane of the (converged) warp returns true.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

// 2-D TMA tiled load (tensor map in kernel parameter space) into shared memory.
__device__ __forceinline__ void tma_load_2d(void* sdst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(sdst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// 4-D / 5-D TMA tiled loads (tensor map in kernel parameter space).
__device__ __forceinline__ void tma_load_4d(void* sdst, const void* tmap, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          smem_u32(sdst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* sdst, const void* tmap, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
      "[%7];" ::"r"(smem_u32(sdst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}

// 1-D bulk copy shared -> global (TMA engine), committed as its own bulk group.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ---- CTA-pair (cluster of 2) helpers for cta_group::2 tensor-core work
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// Wait on a barrier that receives cluster-scope (remote) arrivals: acquire at cluster scope,
// polled with the non-suspending test_wait.
__device__ __forceinline__ bool mbar_test_wait_cluster(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
  if (mbar_test_wait_cluster(a, parity)) return;
  const uint64_t t0 = global_ns();
  uint32_t n = 0;
  while (!mbar_test_wait_cluster(a, parity)) {
    if ((++n & 4095u) == 0 && global_ns() - t0 > 4000000000ull) __trap();
  }
}
// Arrive on a (possibly remote) barrier of the cluster.  Default .release.cta semantics: the
// data this arrival publishes is TMEM/shared-memory state already ordered by the caller's
// tcgen05.wait + fence; a .release.cluster arrive would wait ~1-2k cycles for every
// outstanding global store of the warp.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// D[256 x N] (+)= A[256 x 16] B[16 x N]: each CTA of the pair supplies 128 rows of A and N/2
// rows of B from its own shared memory at the same offsets; issued by the even CTA.
__device__ __forceinline__ void umma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// Arrive (when all prior pair MMAs complete) on the barrier at the same offset in both CTAs.
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// 2-D TMA load into this CTA's smem whose completion bytes count on the even CTA's barrier.
__device__ __forceinline__ void tma_load_2d_pair(void* sdst, const void* tmap, int c0, int c1, uint64_t* bar) {
  const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;  // peer bit cleared: the leader CTA's copy
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(sdst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(b)
      : "memory");
}

}  // namespace p2s
