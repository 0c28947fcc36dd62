// api.cpp -- the C ABI of include/p2s.h: plan construction (host tables, bf16
// tensor-core images, workspace) and the per-frame entry points that enqueue the
// sm_100a kernels of k_fft.cu, k_warp.cu, k_mlp.cu and k_blur.cu.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "p2s_internal.h"

namespace p2s {

static thread_local std::string g_err;

p2s_status set_error(p2s_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

static p2s_status cuda_fail(const char* what, cudaError_t e) {
  return set_error(e == cudaErrorMemoryAllocation ? P2S_ERR_OUT_OF_MEMORY : P2S_ERR_CUDA,
                   std::string(what) + ": " + cudaGetErrorString(e));
}

#define P2S_CUDA(call, what)                    \
  do {                                          \
    cudaError_t e_ = (call);                    \
    if (e_ != cudaSuccess) return cuda_fail(what, e_); \
  } while (0)

#define P2S_LAUNCH(call, what)                                   \
  do {                                                           \
    int e_ = (call);                                             \
    if (e_ != 0) return cuda_fail(what, (cudaError_t)e_);         \
  } while (0)

static inline int round16(int x) { return (x + 15) / 16 * 16; }

static uint16_t host_bf16(float f) {
  __nv_bfloat16 b = __float2bfloat16_rn(f);
  uint16_t u;
  std::memcpy(&u, &b, 2);
  return u;
}

static void radix_plan(int N, AxisFFT& a, bool columns, bool small_only) {
  a.N = N;
  a.nrad = 0;
  int m = N;
  // composite radices up to 16 done in registers: 1080, 1920, 2160, 3840 take three
  // shared-memory passes instead of five or six, 256 two instead of three; 512 keeps the
  // radix-8 plan the 512-point register kernels match on
  // (powers of two: columns only -- the row kernels run one or two sequences per CTA and
  // a radix-16 pass of a 256-point row leaves most of their threads idle)
  const bool pow2 = (N & (N - 1)) == 0;
  if (N != 512 && (!pow2 || columns || N == 4096) && !small_only) {
    // columns: prefer three radices >= 9 (1080 = 12 x 10 x 9 rather than 15 x 12 x 6), so
    // every pass has at most one butterfly per thread and the persistent in-place column
    // kernel (k_cols_p) applies
    static const int wide[] = {16, 15, 12, 10, 9};
    if (columns && !pow2)
      for (int r1 : wide)
        for (int r2 : wide)
          for (int r3 : wide)
            if (r1 >= r2 && r2 >= r3 && r1 * r2 * r3 == N) {
              a.rad[0] = r1;
              a.rad[1] = r2;
              a.rad[2] = r3;
              a.nrad = 3;
              return;
            }
    static const int big[] = {16, 15, 12, 10, 9, 8, 6, 5, 4, 3, 2};
    while (m > 1) {
      for (int r : big)
        if (m % r == 0) {
          a.rad[a.nrad++] = r;
          m /= r;
          break;
        }
    }
    return;
  }
  while (m % 8 == 0) { a.rad[a.nrad++] = 8; m /= 8; }
  while (m % 4 == 0) { a.rad[a.nrad++] = 4; m /= 4; }
  while (m % 2 == 0) { a.rad[a.nrad++] = 2; m /= 2; }
  while (m % 3 == 0) { a.rad[a.nrad++] = 3; m /= 3; }
  while (m % 5 == 0) { a.rad[a.nrad++] = 5; m /= 5; }
}

static p2s_status upload_twiddles(AxisFFT& a) {
  std::vector<float2> tw(a.N);
  const double pi = 3.14159265358979323846;
  for (int k = 0; k < a.N; ++k) {
    double ang = 2.0 * pi * (double)k / a.N;  // inverse transform: e^{+2 pi i k/N}
    tw[k] = make_float2((float)std::cos(ang), (float)std::sin(ang));
  }
  P2S_CUDA(cudaMalloc(&a.tw, sizeof(float2) * a.N), "cudaMalloc twiddles");
  P2S_CUDA(cudaMemcpy(a.tw, tw.data(), sizeof(float2) * a.N, cudaMemcpyHostToDevice), "copy twiddles");
  return P2S_OK;
}

// K-major SWIZZLE_NONE image of a [rows x cols] matrix (rows padded to R, cols to Kp).
static void kmajor_image(const std::vector<double>& Mtx, int rows, int cols, int R, int Kp, uint8_t* dst) {
  std::memset(dst, 0, (size_t)R * Kp * 2);
  const size_t sbo = (size_t)(Kp / 8) * 128;
  for (int n = 0; n < rows; ++n)
    for (int k = 0; k < cols; ++k) {
      size_t off = (n % 8) * 16 + (n / 8) * sbo + (k / 8) * 128 + (k % 8) * 2;
      uint16_t v = host_bf16((float)Mtx[(size_t)n * cols + k]);
      std::memcpy(dst + off, &v, 2);
    }
}

// Pack W1 (n_in x h1 as [h1][nin]), W2, W3 and biases into the smem image of k_mlp.
static p2s_status build_mlp_blob(const std::vector<double>& W1, int nin, int h1, const std::vector<double>& b1,
                                 const std::vector<double>& W2, int h2, const std::vector<double>& b2,
                                 const std::vector<double>& W3, int K, const std::vector<double>& b3, MlpGeom& g,
                                 uint8_t** dblob) {
  g.nin = nin;
  g.k1 = round16(nin);
  g.n1 = round16(h1);
  g.n2 = round16(h2);
  g.n3 = round16(K);
  g.kout = K;
  size_t w1 = (size_t)g.n1 * g.k1 * 2, w2 = (size_t)g.n2 * g.n1 * 2, w3 = (size_t)g.n3 * g.n2 * 2;
  g.off_w2 = w1;
  g.off_w3 = w1 + w2;
  g.off_b1 = w1 + w2 + w3;
  g.off_b2 = g.off_b1 + (size_t)g.n1 * 4;
  g.off_b3 = g.off_b2 + (size_t)g.n2 * 4;
  g.blob_bytes = (g.off_b3 + (size_t)g.n3 * 4 + 15) / 16 * 16;
  std::vector<uint8_t> blob(g.blob_bytes, 0);
  // Bias folding: when every layer has a padding column, a constant-1 input (A1 column nin,
  // set once in smem) is carried through the network in the first padding unit of each
  // hidden layer, and the biases become GEMM weights of that unit (bf16).
  g.bias_folded = (g.k1 > nin) && (g.n1 > h1) && (g.n2 > h2);
  if (g.bias_folded) {
    std::vector<double> A1((size_t)g.n1 * g.k1, 0.0), A2((size_t)g.n2 * g.n1, 0.0), A3((size_t)g.n3 * g.n2, 0.0);
    for (int n = 0; n < h1; ++n) {
      for (int k = 0; k < nin; ++k) A1[(size_t)n * g.k1 + k] = W1[(size_t)n * nin + k];
      A1[(size_t)n * g.k1 + nin] = b1[n];
    }
    A1[(size_t)h1 * g.k1 + nin] = 1.0;
    for (int n = 0; n < h2; ++n) {
      for (int k = 0; k < h1; ++k) A2[(size_t)n * g.n1 + k] = W2[(size_t)n * h1 + k];
      A2[(size_t)n * g.n1 + h1] = b2[n];
    }
    A2[(size_t)h2 * g.n1 + h1] = 1.0;
    for (int n = 0; n < K; ++n) {
      for (int k = 0; k < h2; ++k) A3[(size_t)n * g.n2 + k] = W3[(size_t)n * h2 + k];
      A3[(size_t)n * g.n2 + h2] = b3[n];
    }
    kmajor_image(A1, g.n1, g.k1, g.n1, g.k1, blob.data());
    kmajor_image(A2, g.n2, g.n1, g.n2, g.n1, blob.data() + g.off_w2);
    kmajor_image(A3, g.n3, g.n2, g.n3, g.n2, blob.data() + g.off_w3);
  } else {
    kmajor_image(W1, h1, nin, g.n1, g.k1, blob.data());
    kmajor_image(W2, h2, h1, g.n2, g.n1, blob.data() + g.off_w2);
    kmajor_image(W3, K, h2, g.n3, g.n2, blob.data() + g.off_w3);
    float* fb1 = reinterpret_cast<float*>(blob.data() + g.off_b1);
    float* fb2 = reinterpret_cast<float*>(blob.data() + g.off_b2);
    float* fb3 = reinterpret_cast<float*>(blob.data() + g.off_b3);
    for (int i = 0; i < h1; ++i) fb1[i] = (float)b1[i];
    for (int i = 0; i < h2; ++i) fb2[i] = (float)b2[i];
    for (int i = 0; i < K; ++i) fb3[i] = (float)b3[i];
  }
  P2S_CUDA(cudaMalloc(dblob, g.blob_bytes), "cudaMalloc mlp blob");
  P2S_CUDA(cudaMemcpy(*dblob, blob.data(), g.blob_bytes, cudaMemcpyHostToDevice), "copy mlp blob");
  return P2S_OK;
}

// Blur K-step schedule (see k_blur.cu).  The T x T taps are covered by 1 x 8 groups:
// g8 = T / 8 groups of 8 consecutive tap rows at each tap column (MN-major slabs of the
// column-ordered source tile), and the lr = T % 8 leftover tap rows run along the tap
// columns on transposed copies of single source rows (groups of 8 tap columns, the top
// one partial), so only the partial groups carry zero B rows: 69 K-steps per output row at
// T = 33 instead of 83 with 8-row groups alone.  Groups are paired two per K-step within
// each kind, ordered by shared-memory offset.
static p2s_status build_blur(p2s_plan_s* p, const float* basis) {
  BlurGeom& g = p->bg;
  const int T = p->T, K = p->K;
  g.T = T;
  g.c = T / 2;
  g.NC = T + 15;
  blur_tap_split(T, &g.g8, &g.lr);
  g.nct = std::max(g.NC, 23);  // the partial column group reaches chunk 22 when T < 8
  g.np = round16(K);
  g.racc = std::max(1, 4 / p->C);
  g.pair = !(p->force & P2S_FORCE_BLUR_SINGLE);
  // B ring: a stage is kBlurStepsPerStage (7) K-steps x C*racc MMAs.  Large stages keep
  // the single MMA-issuing thread ahead of the tensor pipe (one barrier wait + commit per
  // 21 MMAs; measured 4 -> 7: 8.3 -> 7.6 ms per 64 frames); 4 stages cover the L2 latency
  // of the B reloads.  Pair mode halves the bytes.
  g.stages = g.pair ? 4 : 3;
  {
    int nsm = 148;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device) != cudaSuccess) nsm = 148;
    p->nsm = nsm;
  }
  p->ntx = (p->W + 127) / 128;
  g.RB = blur_rows_per_cta(p->C, T, g.np, g.racc, p->H, p->W, g.pair, g.stages, p->max_batch, p->nsm);
  g.RS = blur_tile_rows(g.RB, T, g.g8, g.lr);
  const uint32_t sbo = (uint32_t)blur_rs_pad(g.RS) * 16;
  const uint32_t main_bytes = blur_main_bytes(g.NC, g.RS);
  struct Grp {
    bool tr;      // transposed (leftover tap row l = gi) or 8-row group gi
    int tx, gi;   // main: tap column, row group; tr: top tap column of the group, leftover row
    int width;    // tr: valid tap columns tx, tx-1, .., tx-width+1
    uint32_t off;
  };
  std::vector<Grp> mains, trs;
  for (int tx = T - 1; tx >= 0; --tx)
    for (int gi = 0; gi < g.g8; ++gi) mains.push_back({false, tx, gi, 8, (uint32_t)(2 * g.c - tx) * sbo + 128u * gi});
  for (int l = 0; l < g.lr; ++l) {
    if (T % 8) trs.push_back({true, T - 1, l, T % 8, main_bytes + (uint32_t)(l * g.nct + 2 * g.c - (T - 1)) * 16});
    for (int i = T / 8 - 1; i >= 0; --i)
      trs.push_back({true, 8 * i + 7, l, 8, main_bytes + (uint32_t)(l * g.nct + 2 * g.c - (8 * i + 7)) * 16});
  }
  // K-steps of one kind: a lone lowest-address group first (its second half reads the next
  // group against zero B rows), then consecutive pairs.
  struct Step { const Grp* a; const Grp* b; uint32_t lbo; };
  std::vector<Step> steps;
  auto pair_up = [&](const std::vector<Grp>& v) {
    size_t i = 0;
    if (v.size() % 2 == 1) {
      steps.push_back({&v[0], nullptr, v.size() > 1 ? v[1].off - v[0].off : 0u});
      i = 1;
    }
    for (; i < v.size(); i += 2) steps.push_back({&v[i], &v[i + 1], v[i + 1].off - v[i].off});
  };
  pair_up(mains);
  g.nks_main = (int)steps.size();
  pair_up(trs);
  g.nks = (int)steps.size();
  const size_t bbytes = (size_t)g.np * 32;
  std::vector<uint8_t> img((size_t)g.nks * bbytes, 0);
  std::vector<uint32_t> koff(g.nks), klbo(g.nks);
  for (int t = 0; t < g.nks; ++t) {
    const Step& st = steps[t];
    koff[t] = st.a->off;
    klbo[t] = st.lbo;
    uint8_t* dst = img.data() + (size_t)t * bbytes;
    for (int k = 0; k < 16; ++k) {
      const Grp* gr = k < 8 ? st.a : st.b;
      if (!gr) continue;  // dummy half: zero B rows
      const int j = k & 7;
      int ty, tx;
      if (gr->tr) {
        if (j >= gr->width) continue;
        ty = 2 * g.c - (8 * g.g8 + gr->gi);
        tx = gr->tx - j;
      } else {
        ty = 2 * g.c - 8 * gr->gi - j;
        tx = gr->tx;
      }
      if (ty < 0 || ty >= T || tx < 0 || tx >= T) continue;
      for (int n = 0; n < K; ++n) {
        float v = basis[((size_t)n * T + ty) * T + tx];
        uint16_t b = host_bf16(v);
        size_t off = (n % 8) * 16 + (n / 8) * 256 + (k / 8) * 128 + (k % 8) * 2;
        std::memcpy(dst + off, &b, 2);
      }
    }
  }
  std::vector<float> hs(g.np, 0.f);
  for (int n = 0; n < K; ++n) {
    double s = 0;
    for (int i = 0; i < T * T; ++i) s += basis[(size_t)n * T * T + i];
    hs[n] = (float)s;
  }
  // Every CTA streams the same B tiles at about the same time; brep copies (CTA picks one by
  // its index) spread those reads over more L2 slices.
  g.brep = 8;
  g.bstride = (img.size() + 4095) & ~(size_t)4095;
  P2S_CUDA(cudaMalloc(&g.bimg, g.bstride * g.brep), "cudaMalloc blur B");
  for (int r = 0; r < g.brep; ++r)
    P2S_CUDA(cudaMemcpy(g.bimg + r * g.bstride, img.data(), img.size(), cudaMemcpyHostToDevice), "copy blur B");
  {  // pair-mode copy: [half][t][np/2 rows x 32 B], + 16 zero rows, brep times
    const size_t hb = bbytes / 2;
    std::vector<uint8_t> img2(img.size() + kBlurStepsPerStage * bbytes + 4096, 0);  // a whole stage of slack
    for (int h = 0; h < 2; ++h)
      for (int t = 0; t < g.nks; ++t)
        std::memcpy(img2.data() + ((size_t)h * g.nks + t) * hb, img.data() + (size_t)t * bbytes + h * hb, hb);
    g.brows = (int)(img2.size() / 256);
    P2S_CUDA(cudaMalloc(&g.bimg2, img2.size() * g.brep), "cudaMalloc blur B2");
    for (int r = 0; r < g.brep; ++r)
      P2S_CUDA(cudaMemcpy(g.bimg2 + r * img2.size(), img2.data(), img2.size(), cudaMemcpyHostToDevice),
               "copy blur B2");
  }
  {
    std::vector<uint64_t> ad(g.nks);
    for (int t = 0; t < g.nks; ++t) {
      uint64_t d = (uint64_t)((koff[t] >> 4) & 0x3FFFu);
      d |= (uint64_t)((klbo[t] >> 4) & 0x3FFFu) << 16;
      d |= (uint64_t)(((t < g.nks_main ? sbo : 16u) >> 4) & 0x3FFFu) << 32;  // transposed rows: m-groups 1 chunk apart
      d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
      ad[t] = d;
    }
    P2S_CUDA(cudaMalloc(&g.adesc, sizeof(uint64_t) * g.nks), "cudaMalloc adesc");
    P2S_CUDA(cudaMemcpy(g.adesc, ad.data(), sizeof(uint64_t) * g.nks, cudaMemcpyHostToDevice), "copy adesc");
  }
  P2S_CUDA(cudaMalloc(&g.koff, sizeof(uint32_t) * g.nks), "cudaMalloc koff");
  P2S_CUDA(cudaMemcpy(g.koff, koff.data(), sizeof(uint32_t) * g.nks, cudaMemcpyHostToDevice), "copy koff");
  P2S_CUDA(cudaMalloc(&g.klbo, sizeof(uint32_t) * g.nks), "cudaMalloc klbo");
  P2S_CUDA(cudaMemcpy(g.klbo, klbo.data(), sizeof(uint32_t) * g.nks, cudaMemcpyHostToDevice), "copy klbo");
  P2S_CUDA(cudaMalloc(&g.hsum, sizeof(float) * g.np), "cudaMalloc hsum");
  P2S_CUDA(cudaMemcpy(g.hsum, hs.data(), sizeof(float) * g.np, cudaMemcpyHostToDevice), "copy hsum");
  return P2S_OK;
}

// Device sqrt(S) pairs scaled by sqrt(PQ/2)/PQ (noise amplitude and the 1/PQ of the IDFT).
static p2s_status upload_sqrtS(p2s_plan_s* p) {
  const size_t PQ = (size_t)p->P * p->Q;
  std::vector<float2> dev(PQ * p->npairs);
  const double sc = 1.0 / std::sqrt(2.0 * (double)PQ);
  for (int pr = 0; pr < p->npairs; ++pr)
    for (size_t k = 0; k < PQ; ++k) {
      int sa = 2 * pr, sb = 2 * pr + 1;
      float a = (float)(p->sqrtS_host[(size_t)sa * PQ + k] * sc);
      float b = sb < p->nslots ? (float)(p->sqrtS_host[(size_t)sb * PQ + k] * sc) : 0.f;
      dev[(size_t)pr * PQ + k] = make_float2(a, b);
    }
  if (!p->d_sqrtS) P2S_CUDA(cudaMalloc(&p->d_sqrtS, sizeof(float2) * dev.size()), "cudaMalloc sqrtS");
  P2S_CUDA(cudaMemcpy(p->d_sqrtS, dev.data(), sizeof(float2) * dev.size(), cudaMemcpyHostToDevice), "copy sqrtS");
  return P2S_OK;
}

static size_t frame_bytes(const p2s_plan_s* p) {
  const size_t HW = (size_t)p->H * p->W, PQ = (size_t)p->P * p->Q;
  size_t b = 0;
  b += PQ * p->npairs * sizeof(float2);
  b += (size_t)p->H * ((p->W + 127) / 128) * 128 * (size_t)((std::max(p->nslots, p->Z - 3) + 1) & ~1) * 2;
  b += 2 * HW * 4;
  b += (size_t)p->C * HW * 2;
  b += (size_t)p->H * ((p->W + 127) / 128) * 128 * (size_t)p->mg_fold.n3 * 2;
  b += 2 * (size_t)p->C * HW * 4;
  return b + 5 * 256;
}

static p2s_status alloc_workspace(p2s_plan_s* p) {
  const size_t HW = (size_t)p->H * p->W, PQ = (size_t)p->P * p->Q, mb = p->max_batch;
  p->ws_bytes = frame_bytes(p) * mb;
  P2S_CUDA(cudaMalloc(&p->d_ws, p->ws_bytes), "cudaMalloc workspace");
  uint8_t* c = reinterpret_cast<uint8_t*>(p->d_ws);
  auto take = [&](size_t bytes) {
    uint8_t* r = c;
    c += (bytes + 255) / 256 * 256;
    return r;
  };
  p->d_Z = reinterpret_cast<float2*>(take(mb * PQ * p->npairs * sizeof(float2)));
  p->d_X = reinterpret_cast<uint16_t*>(
      take(mb * (size_t)p->H * ((p->W + 127) / 128) * 128 * (size_t)((std::max(p->nslots, p->Z - 3) + 1) & ~1) * 2));
  p->d_tilt = reinterpret_cast<float*>(take(mb * 2 * HW * 4));
  p->d_Iw = reinterpret_cast<uint16_t*>(take(mb * (size_t)p->C * HW * 2));
  p->ntx = (p->W + 127) / 128;
  p->d_w = reinterpret_cast<uint16_t*>(take(mb * (size_t)p->H * p->ntx * 128 * p->mg_fold.n3 * 2));
  p->d_img = reinterpret_cast<float*>(take(mb * (size_t)p->C * HW * 4));
  p->d_out = reinterpret_cast<float*>(take(mb * (size_t)p->C * HW * 4));
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !encode)
    return set_error(P2S_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int np = p->mg_fold.n3;
  cuuint32_t estr[2] = {1, 1};
  CUresult r;
  {  // B halves for the CTA-pair blur: rows of 256 B; one box = one ring stage of K-steps of one half
    const int rows_per_step = np / 16;  // (np/2 rows x 32 B) / 256 B
    cuuint64_t bd[2] = {128, (cuuint64_t)p->bg.brows * p->bg.brep};
    cuuint64_t bs[1] = {256};
    cuuint32_t bb[2] = {128, (cuuint32_t)(kBlurStepsPerStage * rows_per_step)};
    r = encode(&p->tmap_b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p->bg.bimg2, bd, bs, bb, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(P2S_ERR_CUDA, "cuTensorMapEncodeTiled (B) failed");
  }
  return P2S_OK;
}

static void clear_timing(p2s_plan_s* p);

static void free_plan(p2s_plan_s* p) {
  if (!p) return;
  clear_timing(p);
  cudaFree(p->d_slab_ky);
  cudaFree(p->d_slab_dest);
  cudaFree(p->d_sqrtS);
  cudaFree(p->d_ar);
  cudaFree(p->d_L);
  cudaFree(p->d_mlp_fold);
  cudaFree(p->d_mlp_plain);
  cudaFree(p->bg.bimg);
  cudaFree(p->bg.bimg2);
  if (p->copy_stream) {
    cudaStreamDestroy(p->copy_stream);
    cudaEventDestroy(p->ev_sub);
    cudaEventDestroy(p->ev_copied);
    cudaEventDestroy(p->ev_img);
    cudaEventDestroy(p->ev_half);
  }
  cudaFree(p->d_ztab);
  cudaFree(p->bg.koff);
  cudaFree(p->bg.adesc);
  cudaFree(p->bg.klbo);
  cudaFree(p->bg.hsum);
  cudaFree(p->fq.tw);
  cudaFree(p->fp.tw);
  cudaFree(p->d_ws);
  delete p;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// AR(1) bookkeeping: 0 = continue from the stored state, 1 = fresh start at frame 0,
// 2 = replay frames 0..frame0-1 into the state first.
static int ar_mode_for(p2s_plan_s* p, uint64_t seed, int64_t frame0) {
  if (p->ar_valid && p->ar_seed == seed && p->ar_next == frame0) return 0;
  return frame0 == 0 ? 1 : 2;
}

// Event pair around one launch when stage timing is on.
struct StageScope {
  p2s_plan_s* p;
  cudaStream_t s;
  cudaEvent_t b = nullptr, e = nullptr;
  StageScope(p2s_plan_s* p_, int stage, cudaStream_t s_) : p(p_), s(s_) {
    if (!p->timing) return;
    cudaEventCreate(&b);
    cudaEventCreate(&e);
    cudaEventRecord(b, s);
    p->t_stage.push_back(stage);
  }
  ~StageScope() {
    if (!p->timing) return;
    cudaEventRecord(e, s);
    p->t_ev.push_back(b);
    p->t_ev.push_back(e);
  }
};

static void clear_timing(p2s_plan_s* p) {
  for (cudaEvent_t ev : p->t_ev) cudaEventDestroy(ev);
  p->t_ev.clear();
  p->t_stage.clear();
}

static p2s_status run_step1(p2s_plan_s* p, uint64_t seed, int64_t f0, int F, cudaStream_t s) {
  const bool ar = p->ar_alpha != 0.f;
  int mode = ar ? ar_mode_for(p, seed, f0) : 1;
  {
    StageScope sc(p, 0, s);
    P2S_LAUNCH(launch_rows(p, seed, f0, F, ar, mode, mode == 2 ? 0 : f0, s), "k_rows");
  }
  if (ar) {
    p->ar_valid = true;
    p->ar_seed = seed;
    p->ar_next = f0 + F;
  }
  return P2S_OK;
}

// Slab-mode tables (NEXT-4): this rank's spectral rows in pack order, the destinations'
// strip columns and block offsets, the rows of the receive buffer in source order, and the
// per-peer float counts of the all-to-all.
static p2s_status build_slab_tables(p2s_plan_s* p) {
  const int G = p->slab_G, P = p->P, W = p->W_glob, T = p->T, np = p->npairs;
  auto rows_of = [&](const SlabGeom& g, std::vector<int>& v) {
    for (int kp = g.kp0; kp < g.kp1; ++kp) {
      v.push_back(kp);
      if (kp != 0 && 2 * kp != P) v.push_back(P - kp);
    }
  };
  const SlabGeom me = slab_geometry(W, T, P, G, p->slab_r);
  std::vector<int> ky;  // [rows_r] pack order, then [P] receive order
  rows_of(me, ky);
  std::vector<int> dest(3 * (size_t)G);
  p->slab_send.assign(G, 0);
  p->slab_recv.assign(G, 0);
  int64_t off = 0;
  const int ws_me = p->W;
  for (int d = 0; d < G; ++d) {
    const SlabGeom gd = slab_geometry(W, T, P, G, d);
    const int ws = gd.hx1 - gd.hx0;
    dest[3 * d] = gd.hx0;
    dest[3 * d + 1] = ws;
    if (off > INT32_MAX) return set_error(P2S_ERR_UNSUPPORTED, "slab send buffer above 2^31 complex values");
    dest[3 * d + 2] = (int)off;
    const int64_t n = (int64_t)me.rows * np * ws;
    off += n;
    p->slab_send[d] = 2 * n;
    rows_of(gd, ky);  // rows sent by rank d, in its pack order = their order in our recv buffer
    p->slab_recv[d] = 2 * (int64_t)gd.rows * np * ws_me;
  }
  if ((int)ky.size() != me.rows + P) return set_error(P2S_ERR_NUMERIC, "slab row partition does not cover the grid");
  P2S_CUDA(cudaMalloc(&p->d_slab_ky, sizeof(int) * ky.size()), "cudaMalloc slab rows");
  P2S_CUDA(cudaMemcpy(p->d_slab_ky, ky.data(), sizeof(int) * ky.size(), cudaMemcpyHostToDevice), "copy slab rows");
  P2S_CUDA(cudaMalloc(&p->d_slab_dest, sizeof(int) * dest.size()), "cudaMalloc slab dests");
  P2S_CUDA(cudaMemcpy(p->d_slab_dest, dest.data(), sizeof(int) * dest.size(), cudaMemcpyHostToDevice),
           "copy slab dests");
  return P2S_OK;
}

}  // namespace p2s

using namespace p2s;

extern "C" const char* p2s_last_error(void) { return g_err.c_str(); }

extern "C" p2s_status p2s_plan_create(p2s_plan* out, int H, int W, int C, double d_over_r0, double L_m, int Z, int K,
                                      const float* basis, const float* mlp_weights, const p2s_options* opt) {
  g_err.clear();
  if (!out) return set_error(P2S_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  p2s_options o;
  std::memset(&o, 0, sizeof(o));
  if (opt) o = *opt;
  const int T = o.taps;
  if (T < 3 || T > 63 || T % 2 == 0) return set_error(P2S_ERR_INVALID_ARGUMENT, "taps must be odd in [3, 63]");
  if (H < T || W < T || H > 8192 || W > 8192) return set_error(P2S_ERR_INVALID_ARGUMENT, "H, W must be in [T, 8192]");
  if (T / 2 > std::min(H, W) - 1) return set_error(P2S_ERR_INVALID_ARGUMENT, "T/2 must be <= min(H,W)-1");
  if (C < 1 || C > 4) return set_error(P2S_ERR_INVALID_ARGUMENT, "C must be in [1, 4]");
  if (!(d_over_r0 >= 0) || !std::isfinite(d_over_r0)) return set_error(P2S_ERR_INVALID_ARGUMENT, "D/r0 must be >= 0");
  if (!(L_m > 0) || !std::isfinite(L_m)) return set_error(P2S_ERR_INVALID_ARGUMENT, "L must be > 0");
  if (Z < 4 || Z > 66) return set_error(P2S_ERR_INVALID_ARGUMENT, "Z must be in [4, 66]");
  if (K < 1 || K > 128) return set_error(P2S_ERR_INVALID_ARGUMENT, "K must be in [1, 128]");
  if (!basis || !mlp_weights) return set_error(P2S_ERR_INVALID_ARGUMENT, "basis / mlp_weights is NULL");
  const int h1 = o.mlp_hidden[0] > 0 ? o.mlp_hidden[0] : 100;
  const int h2 = o.mlp_hidden[1] > 0 ? o.mlp_hidden[1] : 100;
  if (h1 > 256 || h2 > 256) return set_error(P2S_ERR_INVALID_ARGUMENT, "mlp_hidden must be <= 256");
  if (!(o.ar_alpha >= 0.f && o.ar_alpha < 1.f)) return set_error(P2S_ERR_INVALID_ARGUMENT, "ar_alpha in [0,1)");
  if (!std::isfinite(o.flow_px_per_frame[0]) || !std::isfinite(o.flow_px_per_frame[1]))
    return set_error(P2S_ERR_INVALID_ARGUMENT, "flow_px_per_frame must be finite");
  if ((o.flow_px_per_frame[0] != 0.f || o.flow_px_per_frame[1] != 0.f) && o.ar_alpha != 0.f)
    return set_error(P2S_ERR_INVALID_ARGUMENT, "frozen flow and ar_alpha are exclusive");
  const double D = o.aperture_m > 0 ? o.aperture_m : 0.1;
  const double lam = o.wavelength_m > 0 ? o.wavelength_m : 525e-9;
  const int pad = o.pad > 0 ? o.pad : 1;
  if (o.device < 0) return set_error(P2S_ERR_INVALID_ARGUMENT, "device must be >= 0");
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  if (o.device > 0) dev = o.device;  // 0 selects the calling thread's current device

  p2s_plan_s* p = new (std::nothrow) p2s_plan_s();
  if (!p) return set_error(P2S_ERR_OUT_OF_MEMORY, "host allocation failed");
  p->H = H; p->W = W; p->C = C; p->Z = Z; p->K = K; p->T = T;
  p->h1 = h1; p->h2 = h2;
  p->d_over_r0 = d_over_r0; p->L_m = L_m;
  p->s_px = o.s_per_px > 0 ? o.s_per_px : L_m * (lam / (2.0 * D)) / D;
  p->kappa = o.tilt_px_per_rad > 0 ? o.tilt_px_per_rad : 4.0 / 3.14159265358979323846;
  p->ar_alpha = o.ar_alpha;
  p->flow_vx = o.flow_px_per_frame[0];
  p->flow_vy = o.flow_px_per_frame[1];
  p->noise_sigma = o.noise_sigma;
  p->normalize = o.normalize_psf_sum;
  p->clamp01 = o.clamp01;
  p->device = dev;
  p->force = o.force;
  if (__builtin_popcount(o.force & (P2S_FORCE_X_PLANES | P2S_FORCE_X_TILES | P2S_FORCE_X_OCTETS)) > 1)
    return delete p, set_error(P2S_ERR_INVALID_ARGUMENT, "P2S_FORCE_X_PLANES, _X_TILES and _X_OCTETS are exclusive");
  if ((o.force & P2S_FORCE_AR_ROW_KERNEL) && (o.force & P2S_FORCE_AR_PAIR_KERNEL))
    return delete p, set_error(P2S_ERR_INVALID_ARGUMENT, "P2S_FORCE_AR_ROW_KERNEL and _AR_PAIR_KERNEL are exclusive");
  p->P = grid_size(pad * H);
  p->Q = grid_size(pad * W);
  if (p->P > 4096 || p->Q > 4096) {
    delete p;
    return set_error(P2S_ERR_UNSUPPORTED, "FFT grid larger than 4096 per axis");
  }
  p->W_glob = W;
  if (o.slab_count > 1) {  // NEXT-4: this rank's share of one frame; steps 1b-5 on its halo strip
    const int G = o.slab_count, r = o.slab_rank;
    if (r < 0 || r >= G || G > 64)
      return delete p, set_error(P2S_ERR_INVALID_ARGUMENT, "slab_rank must be in [0, slab_count), slab_count <= 64");
    const SlabGeom g = slab_geometry(W, T, p->P, G, r);
    for (int d = 0; d < G; ++d) {
      const SlabGeom gd = slab_geometry(W, T, p->P, G, d);
      if (gd.hx1 - gd.hx0 < T || gd.x1 <= gd.x0)
        return delete p, set_error(P2S_ERR_INVALID_ARGUMENT, "slab strips narrower than the taps: fewer ranks");
    }
    p->slab_G = G;
    p->slab_r = r;
    p->slab_x0 = g.x0;
    p->slab_x1 = g.x1;
    p->slab_hx0 = g.hx0;
    p->slab_kp0 = g.kp0;
    p->slab_kp1 = g.kp1;
    p->slab_rows = g.rows;
    p->W = g.hx1 - g.hx0;
    o.max_batch = 1;
  }
  p->xtile = x_tile_layout(p);
  p->nslots = Z - 1;
  p->npairs = (p->nslots + 1) / 2;

  DeviceGuard guard(dev);
  p2s_status st;
#define P2S_TRY(expr)              \
  do {                             \
    st = (expr);                   \
    if (st != P2S_OK) {            \
      free_plan(p);                \
      return st;                   \
    }                              \
  } while (0)
  {
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, dev);
    if (e != cudaSuccess) {
      delete p;
      return cuda_fail("cudaGetDeviceProperties", e);
    }
    p->num_sms = prop.multiProcessorCount;
    if (prop.major < 10) {
      delete p;
      return set_error(P2S_ERR_UNSUPPORTED, "requires an sm_100a (Blackwell B200) device");
    }
  }
  // ---- step-1 tables (host fp64)
  noll_matrix(Z, d_over_r0, p->A0);
  if (!noll_cholesky(Z, p->A0, p->Lc)) {
    delete p;
    return set_error(P2S_ERR_NUMERIC, "Cholesky of the Noll matrix failed after regularisation");
  }
  {
    std::vector<double> sq, cl;
    psd_tables(p->P, p->Q, p->s_px, Z, sq, cl);
    p->sqrtS_host.assign(sq.begin(), sq.end());
    p->clamped_max = *std::max_element(cl.begin(), cl.end());
  }
  P2S_TRY(upload_sqrtS(p));
  radix_plan(p->Q, p->fq, false, p->force & P2S_FORCE_FFT_SMALL_RADIX);
  radix_plan(p->P, p->fp, true, p->force & P2S_FORCE_FFT_SMALL_RADIX);
  if (rows_smem_bytes(p, p->ar_alpha != 0.f, false) > 227 * 1024) {
    free_plan(p);
    return set_error(P2S_ERR_UNSUPPORTED, "no row-pass kernel fits shared memory for this FFT row length");
  }
  P2S_TRY(upload_twiddles(p->fq));
  P2S_TRY(upload_twiddles(p->fp));
  {
    const int n = Z - 1;
    std::vector<float> Lf((size_t)n * n);
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < n; ++k) Lf[(size_t)i * n + k] = (float)p->Lc[(size_t)(i + 1) * Z + (k + 1)];
    cudaError_t e = cudaMalloc(&p->d_L, sizeof(float) * Lf.size());
    if (e == cudaSuccess) e = cudaMemcpy(p->d_L, Lf.data(), sizeof(float) * Lf.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      free_plan(p);
      return cuda_fail("upload L", e);
    }
  }
  // ---- P2S MLP (steps 3): plain (inputs a_4..a_Z) and folded (inputs f_2..f_Z, W1' = W1 L)
  {
    const int nin = Z - 3;
    const size_t need = (size_t)h1 * nin + h1 + (size_t)h2 * h1 + h2 + (size_t)K * h2 + K;
    p->mlp_host.assign(mlp_weights, mlp_weights + need);
    const float* q = mlp_weights;
    std::vector<double> W1(q, q + (size_t)h1 * nin); q += (size_t)h1 * nin;
    std::vector<double> b1(q, q + h1); q += h1;
    std::vector<double> W2(q, q + (size_t)h2 * h1); q += (size_t)h2 * h1;
    std::vector<double> b2(q, q + h2); q += h2;
    std::vector<double> W3(q, q + (size_t)K * h2); q += (size_t)K * h2;
    std::vector<double> b3(q, q + K);
    P2S_TRY(build_mlp_blob(W1, nin, h1, b1, W2, h2, b2, W3, K, b3, p->mg_plain, &p->d_mlp_plain));
    const int nf = Z - 1;
    std::vector<double> W1f((size_t)h1 * nf, 0.0);
    for (int h = 0; h < h1; ++h)
      for (int s = 0; s < nf; ++s) {
        double acc = 0;
        for (int r = 0; r < nin; ++r) acc += W1[(size_t)h * nin + r] * p->Lc[(size_t)(r + 3) * Z + (s + 1)];
        W1f[(size_t)h * nf + s] = acc;
      }
    P2S_TRY(build_mlp_blob(W1f, nf, h1, b1, W2, h2, b2, W3, K, b3, p->mg_fold, &p->d_mlp_fold));
    // k_mlp keeps all three weight images resident in shared memory next to at least one
    // tile pipeline (A1 + A2 images): wide hidden layers with many modes may not fit.
    for (const MlpGeom* g : {&p->mg_plain, &p->mg_fold}) {
      const size_t need = ((g->blob_bytes + 127) & ~(size_t)127) + 128 * (size_t)g->k1 * 2 +
                          128 * (size_t)std::max(std::max(g->n1, g->n2), g->n3) * 2 + 96;
      if (need > 227 * 1024) {
        free_plan(p);
        return set_error(P2S_ERR_UNSUPPORTED, "MLP weights + one tile pipeline exceed 227 KB of shared memory "
                                              "(reduce mlp_hidden or Z)");
      }
    }
  }
  // ---- workspace size (frames per launch; the blur's band choice depends on it)
  {
    size_t fb = frame_bytes(p);
    int mb = o.max_batch > 0 ? o.max_batch : (int)std::min<size_t>(64, std::max<size_t>(1, ((size_t)12 << 30) / fb));
    p->max_batch = mb;
  }
  // ---- basis (step 4)
  p->basis_host.assign(basis, basis + (size_t)K * T * T);
  P2S_TRY(build_blur(p, basis));
  P2S_TRY(alloc_workspace(p));
  if (p->slab_G > 1) P2S_TRY(build_slab_tables(p));
  if (p->ar_alpha != 0.f) {
    cudaError_t e = cudaMalloc(&p->d_ar, sizeof(float4) * (size_t)p->npairs * p->P * p->Q);
    if (e != cudaSuccess) {
      free_plan(p);
      return cuda_fail("cudaMalloc AR state", e);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    free_plan(p);
    return cuda_fail("plan create", e);
  }
  *out = p;
  return P2S_OK;
}

extern "C" p2s_status p2s_plan_destroy(p2s_plan p) {
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");
  DeviceGuard guard(p->device);
  cudaDeviceSynchronize();
  free_plan(p);
  return P2S_OK;
}

#define CHECK_PLAN()                                                         \
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");       \
  if (p->slab_G > 1)                                                         \
    return set_error(P2S_ERR_INVALID_ARGUMENT, "slab plans run through p2s_slab_rows / p2s_slab_finish"); \
  if (nframes < 0) return set_error(P2S_ERR_INVALID_ARGUMENT, "nframes < 0"); \
  if (frame0 < 0) return set_error(P2S_ERR_INVALID_ARGUMENT, "frame0 < 0");

extern "C" p2s_status p2s_sample_zernike(p2s_plan p, uint64_t seed, int64_t frame0, int nframes, float* zern,
                                         void* stream) {
  CHECK_PLAN();
  if (nframes == 0) return P2S_OK;
  if (!zern) return set_error(P2S_ERR_INVALID_ARGUMENT, "zern is NULL");
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t per = (size_t)p->Z * p->H * p->W;
  for (int i0 = 0; i0 < nframes; i0 += p->max_batch) {
    const int F = std::min(p->max_batch, nframes - i0);
    p2s_status st = run_step1(p, seed, frame0 + i0, F, s);
    if (st != P2S_OK) return st;
    P2S_LAUNCH(launch_cols(p, F, 0, zern + per * i0, s), "k_cols");
    P2S_LAUNCH(launch_mix(p, F, zern + per * i0, s), "k_mix");
  }
  return P2S_OK;
}

extern "C" p2s_status p2s_sample_zernike_from_noise(p2s_plan p, const float* eta, int nframes, float* zern,
                                                    void* stream) {
  const int64_t frame0 = 0;
  CHECK_PLAN();
  if (nframes == 0) return P2S_OK;
  if (!eta || !zern) return set_error(P2S_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (rows_smem_bytes(p, false, true) > 227 * 1024)
    return set_error(P2S_ERR_UNSUPPORTED, "the given-noise row kernel does not fit shared memory at this row length");
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t per = (size_t)p->Z * p->H * p->W;
  const size_t eper = (size_t)p->nslots * p->P * p->Q;  // complex values per frame
  for (int i0 = 0; i0 < nframes; i0 += p->max_batch) {
    const int F = std::min(p->max_batch, nframes - i0);
    P2S_LAUNCH(launch_rows(p, 0, 0, F, false, 0, 0, s, reinterpret_cast<const float2*>(eta) + eper * i0),
               "k_rows (given noise)");
    P2S_LAUNCH(launch_cols(p, F, 0, zern + per * i0, s), "k_cols");
    P2S_LAUNCH(launch_mix(p, F, zern + per * i0, s), "k_mix");
  }
  return P2S_OK;
}

extern "C" p2s_status p2s_warp(p2s_plan p, const float* img, int64_t img_frame_stride, const float* zern,
                               float* warped, int nframes, void* stream) {
  const int64_t frame0 = 0;
  CHECK_PLAN();
  if (nframes == 0) return P2S_OK;
  if (!img || !zern || !warped) return set_error(P2S_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (img_frame_stride < 0) return set_error(P2S_ERR_INVALID_ARGUMENT, "img_frame_stride < 0");
  if (nframes > 65535) return set_error(P2S_ERR_INVALID_ARGUMENT, "nframes > 65535 per call");
  DeviceGuard guard(p->device);
  P2S_LAUNCH(launch_warp_f32(p, nframes, img, img_frame_stride, zern, warped, (cudaStream_t)stream), "k_warp");
  return P2S_OK;
}

extern "C" p2s_status p2s_blur(p2s_plan p, const float* warped, const float* zern, uint64_t seed, int64_t frame0,
                               float* out, int nframes, void* stream) {
  CHECK_PLAN();
  if (nframes == 0) return P2S_OK;
  if (!warped || !zern || !out) return set_error(P2S_ERR_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t HW = (size_t)p->H * p->W;
  for (int i0 = 0; i0 < nframes; i0 += p->max_batch) {
    const int F = std::min(p->max_batch, nframes - i0);
    P2S_LAUNCH(launch_zern_to_x(p, F, zern + (size_t)i0 * p->Z * HW, s), "k_zern_to_x");
    P2S_LAUNCH(launch_mlp(p, F, false, s), "k_mlp");
    P2S_LAUNCH(launch_blur(p, F, warped + (size_t)i0 * p->C * HW, true, seed, frame0 + i0,
                           out + (size_t)i0 * p->C * HW, s),
               "k_blur");
  }
  return P2S_OK;
}

extern "C" p2s_status p2s_blur_weights(p2s_plan p, const float* warped, const float* weights, uint64_t seed,
                                       int64_t frame0, float* out, int nframes, void* stream) {
  CHECK_PLAN();
  if (nframes == 0) return P2S_OK;
  if (!warped || !weights || !out) return set_error(P2S_ERR_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t HW = (size_t)p->H * p->W;
  for (int i0 = 0; i0 < nframes; i0 += p->max_batch) {
    const int F = std::min(p->max_batch, nframes - i0);
    P2S_LAUNCH(launch_pack_weights(p, F, weights + (size_t)i0 * p->K * HW, s), "k_pack_weights");
    P2S_LAUNCH(launch_blur(p, F, warped + (size_t)i0 * p->C * HW, true, seed, frame0 + i0,
                           out + (size_t)i0 * p->C * HW, s),
               "k_blur");
  }
  return P2S_OK;
}

// Steps 1-5; img_ready (nullable): an event the image upload records -- step 1 does not
// read the image, so the upload overlaps the row pass and (when step 2 is its own kernel)
// the column pass too; only the stage that reads the image waits.  half_done (nullable,
// one-frame calls): the blur runs as two launches over the top and bottom halves of the
// row bands and half_done is recorded between them, so the caller can copy rows
// [0, *split_row) out while the bottom half is computed.
static p2s_status simulate_impl(p2s_plan_s* p, const float* img, int64_t img_frame_stride, uint64_t seed,
                                int64_t frame0, int nframes, float* out, cudaStream_t s, cudaEvent_t img_ready,
                                cudaEvent_t half_done = nullptr, int* split_row = nullptr) {
  const size_t HW = (size_t)p->H * p->W;
  const bool fused = cols_fuse_warp(p);
  for (int i0 = 0; i0 < nframes; i0 += p->max_batch) {
    const int F = std::min(p->max_batch, nframes - i0);
    p2s_status st = run_step1(p, seed, frame0 + i0, F, s);
    if (st != P2S_OK) return st;
    if (img_ready && fused) P2S_CUDA(cudaStreamWaitEvent(s, img_ready, 0), "wait image upload");
    bool warp_fused = false;  // 512-point columns: step 2 runs inside the column kernel
    {
      StageScope sc(p, 1, s);
      P2S_LAUNCH(launch_cols(p, F, 1, nullptr, s, img + (size_t)i0 * img_frame_stride, img_frame_stride, &warp_fused),
                 "k_cols");
    }
    if (!warp_fused) {
      if (img_ready && !fused) P2S_CUDA(cudaStreamWaitEvent(s, img_ready, 0), "wait image upload");
      StageScope sc(p, 2, s);
      P2S_LAUNCH(launch_warp_sim(p, F, img + (size_t)i0 * img_frame_stride, img_frame_stride, s), "k_warp");
    }
    {
      StageScope sc(p, 3, s);
      P2S_LAUNCH(launch_mlp(p, F, true, s), "k_mlp");
    }
    float* o = out + (size_t)i0 * p->C * HW;
    const int bands = (p->H + p->bg.RB - 1) / p->bg.RB;
    if (half_done && F == 1 && nframes == 1 && bands >= 2) {
      const int b1 = bands / 2;
      {
        StageScope sc(p, 4, s);
        P2S_LAUNCH(launch_blur(p, F, p->d_Iw, false, seed, frame0 + i0, o, s, 0, b1), "k_blur (top)");
      }
      P2S_CUDA(cudaEventRecord(half_done, s), "event record");
      {
        StageScope sc(p, 4, s);
        P2S_LAUNCH(launch_blur(p, F, p->d_Iw, false, seed, frame0 + i0, o, s, b1, bands - b1), "k_blur (bottom)");
      }
      if (split_row) *split_row = b1 * p->bg.RB;
    } else {
      StageScope sc(p, 4, s);
      P2S_LAUNCH(launch_blur(p, F, p->d_Iw, false, seed, frame0 + i0, o, s), "k_blur");
    }
  }
  return P2S_OK;
}

extern "C" p2s_status p2s_simulate_frames(p2s_plan p, const float* img, int64_t img_frame_stride, uint64_t seed,
                                          int64_t frame0, int nframes, float* out, void* stream) {
  CHECK_PLAN();
  if (nframes == 0) return P2S_OK;
  if (!img || !out) return set_error(P2S_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (img_frame_stride < 0) return set_error(P2S_ERR_INVALID_ARGUMENT, "img_frame_stride < 0");
  DeviceGuard guard(p->device);
  return simulate_impl(p, img, img_frame_stride, seed, frame0, nframes, out, (cudaStream_t)stream, nullptr);
}

// Sub-batch sizes for the host entry point.  Modelled compute time of a sub-batch of s frames:
//   blur_waves(s) x wave time (a partly empty last wave costs a full one)
//   + ceil(s / 4) x the 512-point row kernel's 4-frame step + s x the linear rest + launches;
// each sub-batch's device->host copy runs under the next sub-batch's compute (constraint:
// compute(next) >= copy(previous)), the last copy is the exposed tail.  Minimum over
// non-increasing size sequences by dynamic programming over (remaining, previous size).
static std::vector<int> host_schedule_uncached(const p2s_plan_s* p, int F) {
  const BlurGeom& g = p->bg;
  const double px = (double)p->H * p->W / 262144.0;
  const double row_ms = 8.1e-3 * (double)p->C * g.racc * g.nks / (3.0 * 69.0);
  const double wave_ms = (g.RB + 2.5) * row_ms;
  const bool r512 = p->Q == 512 && p->ar_alpha == 0.f;
  const double r4_ms = r512 ? 0.09 * ((double)p->P * p->Q / 262144.0) * (p->npairs / 18.0) : 0.0;
  const double lin_ms = 0.04 * px;  // columns + MLP per frame (512^2: ~2.6 ms / 64)
  const double c_ms = (double)p->C * p->H * p->W * 4.0 / 50e9 * 1e3;
  std::vector<double> compv(F + 1, 0.0);
  for (int s = 1; s <= F; ++s) compv[s] = blur_waves(p, s) * wave_ms + ((s + 3) / 4) * r4_ms + s * lin_ms + 0.03;
  auto comp = [&](int s) { return compv[s]; };
  // best[r][q]: minimal time of r remaining frames after a sub-batch of q frames (q = 0: none)
  const size_t W1 = (size_t)F + 1;
  std::vector<double> best(W1 * W1, -1.0);
  std::vector<int> choice(W1 * W1, 0);
  for (int r = 1; r <= F; ++r)
    for (int q = 0; q <= F; ++q) {
      double bv = 1e300;
      int bs = 0;
      const int smax = q ? std::min(r, q) : r;
      for (int s = 1; s <= smax; ++s) {
        const double cs = comp(s);
        if (q && cs < c_ms * q) continue;  // the previous copy would not hide
        const double rest = s == r ? c_ms * s : best[(size_t)(r - s) * W1 + s];
        if (rest < 0) continue;
        if (cs + rest < bv - 1e-12) {
          bv = cs + rest;
          bs = s;
        }
      }
      if (bs) {
        best[(size_t)r * W1 + q] = bv;
        choice[(size_t)r * W1 + q] = bs;
      }
    }
  std::vector<int> out;
  int r = F, q = 0;
  while (r > 0) {
    int s = choice[(size_t)r * W1 + q];
    if (s <= 0) s = r;  // no feasible taper (copies slower than compute): one launch
    out.push_back(s);
    r -= s;
    q = s;
  }
  return out;
}

static const std::vector<int>& host_schedule(p2s_plan_s* p, int F) {
  auto it = p->host_sched.find(F);
  if (it == p->host_sched.end()) it = p->host_sched.emplace(F, host_schedule_uncached(p, F)).first;
  return it->second;
}

extern "C" p2s_status p2s_simulate_frames_host(p2s_plan p, const float* img_host, int64_t img_frame_stride,
                                               uint64_t seed, int64_t frame0, int nframes, float* out_host,
                                               void* stream) {
  CHECK_PLAN();
  if (nframes == 0) return P2S_OK;
  if (!img_host || !out_host) return set_error(P2S_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (img_frame_stride < 0) return set_error(P2S_ERR_INVALID_ARGUMENT, "img_frame_stride < 0");
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t img_floats = (size_t)p->C * p->H * p->W;
  if (!p->copy_stream) {
    P2S_CUDA(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    P2S_CUDA(cudaEventCreateWithFlags(&p->ev_sub, cudaEventDisableTiming), "cudaEventCreate");
    P2S_CUDA(cudaEventCreateWithFlags(&p->ev_copied, cudaEventDisableTiming), "cudaEventCreate");
    P2S_CUDA(cudaEventCreateWithFlags(&p->ev_img, cudaEventDisableTiming), "cudaEventCreate");
    P2S_CUDA(cudaEventCreateWithFlags(&p->ev_half, cudaEventDisableTiming), "cudaEventCreate");
  }
  // The device->host copy of each sub-batch runs on a second stream while the next
  // sub-batch computes, so the PCIe transfer of the outputs hides behind the kernels; the
  // sub-batch sizes come from host_schedule (wave-aligned blur launches, short copy tail).
  bool pending = false;
  for (int i0 = 0; i0 < nframes; i0 += p->max_batch) {
    const int F = std::min(p->max_batch, nframes - i0);
    const std::vector<int>& subs = host_schedule(p, F);
    if (pending) P2S_CUDA(cudaStreamWaitEvent(s, p->ev_copied, 0), "wait copies");  // d_out reuse
    // image upload on the copy stream (after the previous chunk's compute has read d_img);
    // the compute stream waits for it only before the column/warp stage
    if (pending) P2S_CUDA(cudaStreamWaitEvent(p->copy_stream, p->ev_sub, 0), "wait compute");
    if (img_frame_stride == 0) {
      P2S_CUDA(cudaMemcpyAsync(p->d_img, img_host, img_floats * 4, cudaMemcpyHostToDevice, p->copy_stream),
               "H2D img");
    } else {
      for (int i = 0; i < F; ++i)
        P2S_CUDA(cudaMemcpyAsync(p->d_img + i * img_floats, img_host + (size_t)(i0 + i) * img_frame_stride,
                                 img_floats * 4, cudaMemcpyHostToDevice, p->copy_stream),
                 "H2D img");
    }
    P2S_CUDA(cudaEventRecord(p->ev_img, p->copy_stream), "event record");
    int j0 = 0;
    for (size_t si = 0; si < subs.size(); ++si) {
      const int Fs = subs[si];
      // the exposed copy tail: a one-frame last sub-batch runs its blur as two halves and
      // its top rows leave while the bottom half is computed (4K: half of a 100 MB copy)
      const bool split = si + 1 == subs.size() && i0 + F == nframes && Fs == 1 && p->H >= 256;
      int ysplit = 0;
      p2s_status st = simulate_impl(p, p->d_img + (img_frame_stride ? (size_t)j0 * img_floats : 0),
                                    img_frame_stride ? (int64_t)img_floats : 0, seed, frame0 + i0 + j0, Fs,
                                    p->d_out + (size_t)j0 * img_floats, s, p->ev_img, split ? p->ev_half : nullptr,
                                    split ? &ysplit : nullptr);
      if (st != P2S_OK) return st;
      const size_t plane = (size_t)p->H * p->W;
      if (split && ysplit > 0) {
        P2S_CUDA(cudaStreamWaitEvent(p->copy_stream, p->ev_half, 0), "wait top half");
        for (int c = 0; c < p->C; ++c)
          P2S_CUDA(cudaMemcpyAsync(out_host + (size_t)(i0 + j0) * img_floats + c * plane,
                                   p->d_out + (size_t)j0 * img_floats + c * plane, (size_t)ysplit * p->W * 4,
                                   cudaMemcpyDeviceToHost, p->copy_stream),
                   "D2H out (top)");
      }
      P2S_CUDA(cudaEventRecord(p->ev_sub, s), "event record");
      P2S_CUDA(cudaStreamWaitEvent(p->copy_stream, p->ev_sub, 0), "wait sub-batch");
      if (split && ysplit > 0) {
        for (int c = 0; c < p->C; ++c)
          P2S_CUDA(cudaMemcpyAsync(out_host + (size_t)(i0 + j0) * img_floats + c * plane + (size_t)ysplit * p->W,
                                   p->d_out + (size_t)j0 * img_floats + c * plane + (size_t)ysplit * p->W,
                                   (plane - (size_t)ysplit * p->W) * 4, cudaMemcpyDeviceToHost, p->copy_stream),
                   "D2H out (bottom)");
      } else {
        P2S_CUDA(cudaMemcpyAsync(out_host + (size_t)(i0 + j0) * img_floats, p->d_out + (size_t)j0 * img_floats,
                                 (size_t)Fs * img_floats * 4, cudaMemcpyDeviceToHost, p->copy_stream),
                 "D2H out");
      }
      j0 += Fs;
    }
    P2S_CUDA(cudaEventRecord(p->ev_copied, p->copy_stream), "event record");
    pending = true;
  }
  P2S_CUDA(cudaStreamSynchronize(p->copy_stream), "copy stream sync");
  P2S_CUDA(cudaStreamSynchronize(s), "stream sync");
  return P2S_OK;
}

extern "C" p2s_status p2s_field_autocorr(p2s_plan p, const float* zern, int nframes, int max_lag, double* out,
                                         void* stream) {
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (!zern || !out) return set_error(P2S_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (nframes < 1 || max_lag < 1 || max_lag > 64 || max_lag > p->H || max_lag > p->W)
    return set_error(P2S_ERR_INVALID_ARGUMENT, "nframes >= 1 and 1 <= max_lag <= min(64, H, W) required");
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  double* partial = nullptr;
  P2S_CUDA(cudaMallocAsync(&partial, acorr_partial_bytes(nframes, p->Z, p->W, max_lag), s), "cudaMallocAsync");
  const int rc = launch_acorr(zern, nframes, p->Z, p->H, p->W, max_lag, partial, out, s);
  cudaFreeAsync(partial, s);
  if (rc != 0) return set_error(P2S_ERR_CUDA, std::string("k_acorr: ") + cudaGetErrorString((cudaError_t)rc));
  return P2S_OK;
}

extern "C" p2s_status p2s_exact_psf(p2s_plan p, const float* zern, const int32_t* pixels, int n, int include_tilt,
                                    float* out, void* stream) {
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (!zern || !pixels || !out || n < 1) return set_error(P2S_ERR_INVALID_ARGUMENT, "NULL buffer or n < 1");
  DeviceGuard guard(p->device);
  P2S_LAUNCH(ensure_pupil_table(p), "pupil table");
  P2S_LAUNCH(launch_exact_psf(p, zern, pixels, n, include_tilt, out, (cudaStream_t)stream), "k_exact_psf");
  return P2S_OK;
}

extern "C" p2s_status p2s_render_exact(p2s_plan p, const float* img, const float* zern, int include_tilt, float* out,
                                       void* stream) {
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (!img || !zern || !out) return set_error(P2S_ERR_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  P2S_LAUNCH(ensure_pupil_table(p), "pupil table");
  P2S_LAUNCH(launch_render_exact(p, img, zern, include_tilt, out, (cudaStream_t)stream), "k_render_exact");
  return P2S_OK;
}

extern "C" p2s_status p2s_aperture_stats(p2s_plan p, const float* zern, int nframes, const int32_t* pixels,
                                         int npix, double* out, void* stream) {
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (!zern || !pixels || !out) return set_error(P2S_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (nframes < 1 || npix < 1) return set_error(P2S_ERR_INVALID_ARGUMENT, "nframes >= 1 and npix >= 1 required");
  if (p->Z > 72) return set_error(P2S_ERR_UNSUPPORTED, "Z <= 72 required");
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  P2S_LAUNCH(ensure_pupil_table(p), "pupil table");
  double* partial = nullptr;
  P2S_CUDA(cudaMallocAsync(&partial, aperture_partial_bytes((int64_t)nframes * npix), s), "cudaMallocAsync");
  const int rc = launch_aperture(p, zern, nframes, pixels, npix, partial, out, s);
  cudaFreeAsync(partial, s);
  if (rc != 0) return set_error(P2S_ERR_CUDA, std::string("k_aperture: ") + cudaGetErrorString((cudaError_t)rc));
  return P2S_OK;
}

extern "C" p2s_status p2s_plan_info(p2s_plan p, int* P, int* Q, size_t* ws, double* clamped, int* max_batch) {
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (P) *P = p->P;
  if (Q) *Q = p->Q;
  if (ws) *ws = p->ws_bytes;
  if (clamped) *clamped = p->clamped_max;
  if (max_batch) *max_batch = p->max_batch;
  return P2S_OK;
}

extern "C" p2s_status p2s_plan_stage_timing(p2s_plan p, int enable) {
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");
  DeviceGuard guard(p->device);
  clear_timing(p);
  p->timing = enable != 0;
  return P2S_OK;
}

extern "C" p2s_status p2s_plan_stage_times(p2s_plan p, double* ms, int64_t* launches) {
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");
  DeviceGuard guard(p->device);
  double acc[5] = {0, 0, 0, 0, 0};
  int64_t cnt[5] = {0, 0, 0, 0, 0};
  for (size_t i = 0; i < p->t_stage.size(); ++i) {
    cudaEvent_t b = p->t_ev[2 * i], e = p->t_ev[2 * i + 1];
    P2S_CUDA(cudaEventSynchronize(e), "cudaEventSynchronize");
    float t = 0.f;
    P2S_CUDA(cudaEventElapsedTime(&t, b, e), "cudaEventElapsedTime");
    acc[p->t_stage[i]] += t;
    cnt[p->t_stage[i]] += 1;
  }
  for (int k = 0; k < 5; ++k) {
    if (ms) ms[k] = acc[k];
    if (launches) launches[k] = cnt[k];
  }
  return P2S_OK;
}

extern "C" p2s_status p2s_plan_export_tables(p2s_plan p, double* A0, double* chol, float* sqrtS) {
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (A0) std::memcpy(A0, p->A0.data(), sizeof(double) * p->A0.size());
  if (chol) std::memcpy(chol, p->Lc.data(), sizeof(double) * p->Lc.size());
  if (sqrtS) std::memcpy(sqrtS, p->sqrtS_host.data(), sizeof(float) * p->sqrtS_host.size());
  return P2S_OK;
}

extern "C" p2s_status p2s_plan_import_sqrtS(p2s_plan p, const float* sqrtS) {
  if (!p || !sqrtS) return set_error(P2S_ERR_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard guard(p->device);
  std::memcpy(p->sqrtS_host.data(), sqrtS, sizeof(float) * p->sqrtS_host.size());
  return upload_sqrtS(p);
}

extern "C" p2s_status p2s_philox_fill(uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1, int64_t n,
                                      uint32_t* out, void* stream) {
  if (n < 0 || (n > 0 && !out)) return set_error(P2S_ERR_INVALID_ARGUMENT, "bad argument");
  P2S_LAUNCH(launch_philox_fill(c1, c2, c3, k0, k1, n, out, (cudaStream_t)stream), "k_philox_fill");
  return P2S_OK;
}

// ------------------------------------------------------------------ slab mode (NEXT-4)
extern "C" p2s_status p2s_slab_geometry(int H, int W, int T, int pad, int G, int rank, int64_t* info) {
  g_err.clear();
  if (!info) return set_error(P2S_ERR_INVALID_ARGUMENT, "info is NULL");
  if (H < 1 || W < 1 || T < 1 || G < 1 || rank < 0 || rank >= G)
    return set_error(P2S_ERR_INVALID_ARGUMENT, "bad slab geometry arguments");
  const int P = grid_size((pad > 0 ? pad : 1) * H), Q = grid_size((pad > 0 ? pad : 1) * W);
  const SlabGeom g = slab_geometry(W, T, P, G, rank);
  const int64_t v[9] = {g.x0, g.x1, g.hx0, g.hx1, g.kp0, g.kp1, g.rows, P, Q};
  std::memcpy(info, v, sizeof(v));
  return P2S_OK;
}

extern "C" p2s_status p2s_slab_counts(p2s_plan p, int64_t* send_counts, int64_t* recv_counts) {
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (p->slab_G < 2) return set_error(P2S_ERR_INVALID_ARGUMENT, "not a slab plan");
  for (int d = 0; d < p->slab_G; ++d) {
    if (send_counts) send_counts[d] = p->slab_send[d];
    if (recv_counts) recv_counts[d] = p->slab_recv[d];
  }
  return P2S_OK;
}

extern "C" p2s_status p2s_slab_rows(p2s_plan p, uint64_t seed, int64_t frame, float* send, void* stream) {
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (p->slab_G < 2) return set_error(P2S_ERR_INVALID_ARGUMENT, "not a slab plan");
  if (frame < 0) return set_error(P2S_ERR_INVALID_ARGUMENT, "frame < 0");
  if (!send) return set_error(P2S_ERR_INVALID_ARGUMENT, "send is NULL");
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  // row pass of this rank's pairs: white noise, frozen flow or AR(1) (the rank keeps the
  // state of its own rows; a frame that does not continue the previous call replays)
  p2s_status st = run_step1(p, seed, frame, 1, s);
  if (st != P2S_OK) return st;
  {
    StageScope sc(p, 0, s);
    P2S_LAUNCH(launch_slab_pack(p, reinterpret_cast<float2*>(send), s), "k_slab_pack");
  }
  return P2S_OK;
}

extern "C" p2s_status p2s_slab_finish(p2s_plan p, const float* recv, const float* img, uint64_t seed, int64_t frame,
                                      float* out_strip, void* stream) {
  if (!p) return set_error(P2S_ERR_INVALID_ARGUMENT, "plan is NULL");
  if (p->slab_G < 2) return set_error(P2S_ERR_INVALID_ARGUMENT, "not a slab plan");
  if (frame < 0) return set_error(P2S_ERR_INVALID_ARGUMENT, "frame < 0");
  if (!recv || !img || !out_strip) return set_error(P2S_ERR_INVALID_ARGUMENT, "NULL buffer");
  DeviceGuard guard(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  {
    StageScope sc(p, 1, s);
    P2S_LAUNCH(launch_slab_unpack(p, reinterpret_cast<const float2*>(recv), s), "k_slab_unpack");
    P2S_LAUNCH(launch_cols(p, 1, 1, nullptr, s, nullptr, 0, nullptr), "k_cols (slab strip)");
  }
  {
    StageScope sc(p, 2, s);
    P2S_LAUNCH(launch_warp_sim(p, 1, img, 0, s), "k_warp (slab strip)");
  }
  {
    StageScope sc(p, 3, s);
    P2S_LAUNCH(launch_mlp(p, 1, true, s), "k_mlp");
  }
  const size_t HWs = (size_t)p->H * p->W;
  {
    StageScope sc(p, 4, s);
    P2S_LAUNCH(launch_blur(p, 1, p->d_Iw, false, seed, frame, p->d_out, s), "k_blur");
  }
  const int wo = p->slab_x1 - p->slab_x0;
  P2S_CUDA(cudaMemcpy2DAsync(out_strip, (size_t)wo * 4, p->d_out + (p->slab_x0 - p->slab_hx0), (size_t)p->W * 4,
                             (size_t)wo * 4, (size_t)p->C * p->H, cudaMemcpyDeviceToDevice, s),
           "copy slab strip");
  (void)HWs;
  return P2S_OK;
}
