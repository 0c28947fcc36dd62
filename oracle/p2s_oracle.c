/*
 * p2s_oracle.c -- the DF-P2S per-frame steps 1-5 in plain fp64 C (OpenMP over rows and
 * pixels), written from the paper (arXiv 2210.06713, PAPER.md "P:line") and the readings
 * of SURVEY.md 8(c) ("Q<n>").
 *
 * TEST INFRASTRUCTURE ONLY, like the rest of oracle/: only tests/ and bench.py's
 * reference / cpu_baseline legs load it (through ctypes, libp2s_oracle.so built by
 * __graft_entry__.build()).  The product path never links it; it shares no code, header
 * or table with paper_2210_06713_b200/.
 *
 * It is the CPU-baseline program BASELINE.md describes and the "naive DFT, direct
 * convolution, scalar MLP" form of the definitions (north_star):
 *   - Philox4x32-10 (Salmon et al. SC'11) with the counter layout of Q10;
 *   - Hermitian spectral white noise per mode pair (Q8), AR(1) update (Q18);
 *   - the inverse DFT of Y = sqrt(S_a) eta_a + i sqrt(S_b) eta_b as a direct separable
 *     sum y[x] = (1/PQ) sum_k Y[k] e^{+2 pi i k.x} (Q9), cropped to H x W;
 *   - per-pixel Noll mixing a = L f (Eq.10);
 *   - bilinear clamp-to-edge tilt warp (Q12);
 *   - scalar-loop MLP n_in -> h1 -> h2 -> K, ReLU hidden (Q13);
 *   - Eq.9 direct convolution, true convolution, centre tap, whole-sample mirror (Q14);
 *   - step 5: normalisation, Philox noise (stream 1), clamp (Q16).
 * Pins: tests/test_oracle_c_cpu.py checks every function against the pinned numpy oracle
 * (oracle/pipeline.py) to 1e-12 and the Philox words against the Random123 vectors, and
 * pins the IDFT sign with a single-tone spectrum.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define PI 3.14159265358979323846

/* ------------------------------------------------------------------ Philox4x32-10 */
void p2so_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* Box-Muller on two words (Q10): u1 = (x+1) 2^-32 in (0,1], u2 = x' 2^-32. */
static void box_muller(uint32_t xa, uint32_t xb, double* g1, double* g2) {
  const double u1 = ((double)xa + 1.0) * 0x1p-32, u2 = (double)xb * 0x1p-32;
  const double r = sqrt(-2.0 * log(u1));
  *g1 = r * cos(2.0 * PI * u2);
  *g2 = r * sin(2.0 * PI * u2);
}

/* The four Gaussians of counter (index, slot | stream << 16, frame) under key seed. */
static void gaussians(uint32_t index, int slot, int stream, int64_t frame, uint64_t seed, double g[4]) {
  const uint32_t ctr[4] = {index, (uint32_t)slot | ((uint32_t)stream << 16), (uint32_t)frame,
                           (uint32_t)((uint64_t)frame >> 32)};
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t x[4];
  p2so_philox(ctr, key, x);
  box_muller(x[0], x[1], &g[0], &g[1]);
  box_muller(x[2], x[3], &g[2], &g[3]);
}

/* ------------------------------------------------------------------ step 1: noise */
/* xi for frame `frame`: eta [N-1][P][Q] complex (re, im interleaved).  Bin k and its mirror
 * -k share the draw at the smaller linear index (canonical): eta = sqrt(PQ/2)(g1 + i g2) there,
 * the conjugate on the mirror, sqrt(PQ) g1 on self-conjugate bins.  Pair p = modes 2p+2, 2p+3:
 * words (x0, x1) for mode a, (x2, x3) for mode b (Q8, Q10). */
void p2so_white_noise(uint64_t seed, int64_t frame, int P, int Q, int N, double* eta) {
  const int M = N - 1, npairs = (M + 1) / 2;
  const double s2 = sqrt((double)P * Q / 2.0), s1 = sqrt((double)P * Q);
#pragma omp parallel for schedule(static)
  for (int ky = 0; ky < P; ++ky)
    for (int kx = 0; kx < Q; ++kx) {
      const uint32_t lin = (uint32_t)ky * Q + kx;
      const uint32_t linm = (uint32_t)((P - ky) % P) * Q + (uint32_t)((Q - kx) % Q);
      const uint32_t canon = lin < linm ? lin : linm;
      for (int p = 0; p < npairs; ++p) {
        double g[4];
        gaussians(canon, p, 0, frame, seed, g);
        for (int h = 0; h < 2; ++h) {
          const int m = 2 * p + h;
          if (m >= M) break;
          double* e = eta + 2 * (((size_t)m * P + ky) * Q + kx);
          if (lin == linm) {
            e[0] = s1 * g[2 * h];
            e[1] = 0.0;
          } else {
            e[0] = s2 * g[2 * h];
            e[1] = (lin == canon ? 1.0 : -1.0) * s2 * g[2 * h + 1];
          }
        }
      }
    }
}

/* AR(1) update eta <- alpha eta + sqrt(1 - alpha^2) xi (Q18). */
void p2so_ar_update(double* eta, const double* xi, size_t n, double alpha) {
  const double c = sqrt(1.0 - alpha * alpha);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) eta[i] = alpha * eta[i] + c * xi[i];
}

/* ------------------------------------------------------------------ step 1: fields */
/* f [N-1][H][W]: f_a = Re y, f_b = Im y, y = IDFT(sqrt(S_a) eta_a + i sqrt(S_b) eta_b),
 * y[yy][xx] = (1/PQ) sum_{ky,kx} Y[ky][kx] e^{+2 pi i (ky yy / P + kx xx / Q)}, evaluated
 * as the direct separable sum (rows over kx, then columns over ky), only at the cropped
 * pixels.  sqrtS [N-1][P][Q]. */
void p2so_fields(const double* eta, const double* sqrtS, int P, int Q, int H, int W, int N, double* f) {
  const int M = N - 1, npairs = (M + 1) / 2;
  double* cq = malloc(sizeof(double) * 2 * Q);
  double* cp = malloc(sizeof(double) * 2 * P);
  for (int m = 0; m < Q; ++m) {
    cq[2 * m] = cos(2.0 * PI * m / Q);
    cq[2 * m + 1] = sin(2.0 * PI * m / Q);
  }
  for (int m = 0; m < P; ++m) {
    cp[2 * m] = cos(2.0 * PI * m / P);
    cp[2 * m + 1] = sin(2.0 * PI * m / P);
  }
  double* T = malloc(sizeof(double) * 2 * (size_t)P * W);  /* row pass: T[ky][xx] */
  for (int p = 0; p < npairs; ++p) {
    const int a = 2 * p, b = 2 * p + 1;
    const double* ea = eta + 2 * (size_t)a * P * Q;
    const double* eb = b < M ? eta + 2 * (size_t)b * P * Q : NULL;
    const double* sa = sqrtS + (size_t)a * P * Q;
    const double* sb = b < M ? sqrtS + (size_t)b * P * Q : NULL;
#pragma omp parallel for schedule(static)
    for (int ky = 0; ky < P; ++ky)
      for (int xx = 0; xx < W; ++xx) {
        double re = 0.0, im = 0.0;
        for (int kx = 0; kx < Q; ++kx) {
          const size_t k = (size_t)ky * Q + kx;
          /* Y = sa eta_a + i sb eta_b */
          double yr = sa[k] * ea[2 * k], yi = sa[k] * ea[2 * k + 1];
          if (eb) {
            yr -= sb[k] * eb[2 * k + 1];
            yi += sb[k] * eb[2 * k];
          }
          const int m = (int)(((int64_t)kx * xx) % Q);
          re += yr * cq[2 * m] - yi * cq[2 * m + 1];
          im += yr * cq[2 * m + 1] + yi * cq[2 * m];
        }
        T[2 * ((size_t)ky * W + xx)] = re;
        T[2 * ((size_t)ky * W + xx) + 1] = im;
      }
    const double inv = 1.0 / ((double)P * Q);
#pragma omp parallel for schedule(static)
    for (int yy = 0; yy < H; ++yy)
      for (int xx = 0; xx < W; ++xx) {
        double re = 0.0, im = 0.0;
        for (int ky = 0; ky < P; ++ky) {
          const int m = (int)(((int64_t)ky * yy) % P);
          const double tr = T[2 * ((size_t)ky * W + xx)], ti = T[2 * ((size_t)ky * W + xx) + 1];
          re += tr * cp[2 * m] - ti * cp[2 * m + 1];
          im += tr * cp[2 * m + 1] + ti * cp[2 * m];
        }
        f[((size_t)a * H + yy) * W + xx] = re * inv;
        if (b < M) f[((size_t)b * H + yy) * W + xx] = im * inv;
      }
  }
  free(T);
  free(cp);
  free(cq);
}

/* a [N][H W] = L f per pixel, a_1 = 0 (Eq.10); L [N][N] (row/col 0 = piston). */
void p2so_mix(const double* f, const double* L, int N, size_t HW, double* a) {
#pragma omp parallel for schedule(static)
  for (size_t x = 0; x < HW; ++x) {
    a[x] = 0.0;
    for (int i = 1; i < N; ++i) {
      double s = 0.0;
      for (int j = 1; j <= i; ++j) s += L[(size_t)i * N + j] * f[(size_t)(j - 1) * HW + x];
      a[(size_t)i * HW + x] = s;
    }
  }
}

/* ------------------------------------------------------------------ step 2: warp */
/* Iw_c(y, x) = bilinear(I_c, x + kappa a2, y + kappa a3), clamp-to-edge (Q12). */
void p2so_warp(const double* img, const double* a2, const double* a3, double kappa, int C, int H, int W, double* Iw) {
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const size_t pix = (size_t)y * W + x;
      const double X = x + kappa * a2[pix], Y = y + kappa * a3[pix];
      const double x0 = floor(X), y0 = floor(Y), tx = X - x0, ty = Y - y0;
      const int xi = (int)x0, yi = (int)y0;
      const int xa = xi < 0 ? 0 : (xi > W - 1 ? W - 1 : xi), xb = xi + 1 < 0 ? 0 : (xi + 1 > W - 1 ? W - 1 : xi + 1);
      const int ya = yi < 0 ? 0 : (yi > H - 1 ? H - 1 : yi), yb = yi + 1 < 0 ? 0 : (yi + 1 > H - 1 ? H - 1 : yi + 1);
      for (int c = 0; c < C; ++c) {
        const double* I = img + (size_t)c * H * W;
        Iw[(size_t)c * H * W + pix] = (1 - ty) * ((1 - tx) * I[(size_t)ya * W + xa] + tx * I[(size_t)ya * W + xb]) +
                                      ty * ((1 - tx) * I[(size_t)yb * W + xa] + tx * I[(size_t)yb * W + xb]);
      }
    }
}

/* ------------------------------------------------------------------ step 3: MLP */
/* w [K][HW] = W3 relu(W2 relu(W1 x + b1) + b2) + b3, x = a_4..a_N [n_in][HW] (Q13);
 * weights packed row-major [out][in]: W1, b1, W2, b2, W3, b3. */
void p2so_mlp(const double* x, size_t HW, int n_in, int h1, int h2, int K, const double* wts, double* w) {
  const double *W1 = wts, *b1 = W1 + (size_t)h1 * n_in, *W2 = b1 + h1, *b2 = W2 + (size_t)h2 * h1;
  const double *W3 = b2 + h2, *b3 = W3 + (size_t)K * h2;
#pragma omp parallel
  {
    double* u = malloc(sizeof(double) * (h1 + h2));
#pragma omp for schedule(static)
    for (size_t p = 0; p < HW; ++p) {
      for (int o = 0; o < h1; ++o) {
        double s = b1[o];
        for (int i = 0; i < n_in; ++i) s += W1[(size_t)o * n_in + i] * x[(size_t)i * HW + p];
        u[o] = s > 0.0 ? s : 0.0;
      }
      for (int o = 0; o < h2; ++o) {
        double s = b2[o];
        for (int i = 0; i < h1; ++i) s += W2[(size_t)o * h1 + i] * u[i];
        u[h1 + o] = s > 0.0 ? s : 0.0;
      }
      for (int o = 0; o < K; ++o) {
        double s = b3[o];
        for (int i = 0; i < h2; ++i) s += W3[(size_t)o * h2 + i] * u[h1 + i];
        w[(size_t)o * HW + p] = s;
      }
    }
    free(u);
  }
}

/* ------------------------------------------------------------------ steps 4 + 5 */
static int reflect(int i, int n) { /* whole-sample mirror (Q14) */
  if (i < 0) i = -i;
  if (i >= n) i = 2 * n - 2 - i;
  return i;
}

/* out_c(x) = sum_k w_k(x) sum_u h_k[u + T/2] Iw_c(refl(x - u)) (Eq.9) for the n
 * pixels (ys[i], xs[i]) (n = -1: every pixel, out [C][H][W]; else out [C][n]). */
void p2so_blur(const double* Iw, const double* w, const double* basis, int C, int H, int W, int K, int T,
               const int* ys, const int* xs, int64_t n, double* out) {
  const int c0 = T / 2;
  const int64_t np = n < 0 ? (int64_t)H * W : n;
#pragma omp parallel
  {
    double* conv = malloc(sizeof(double) * K);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < np; ++i) {
      const int y = n < 0 ? (int)(i / W) : ys[i], x = n < 0 ? (int)(i % W) : xs[i];
      const size_t pix = (size_t)y * W + x;
      for (int c = 0; c < C; ++c) {
        const double* I = Iw + (size_t)c * H * W;
        for (int k = 0; k < K; ++k) conv[k] = 0.0;
        for (int ty = 0; ty < T; ++ty) {
          const int sy = reflect(y - (ty - c0), H);
          for (int tx = 0; tx < T; ++tx) {
            const double v = I[(size_t)sy * W + reflect(x - (tx - c0), W)];
            for (int k = 0; k < K; ++k) conv[k] += basis[((size_t)k * T + ty) * T + tx] * v;
          }
        }
        double s = 0.0;
        for (int k = 0; k < K; ++k) s += w[(size_t)k * H * W + pix] * conv[k];
        out[(size_t)c * np + i] = s;
      }
    }
    free(conv);
  }
}

/* Step 5 (Q16) on out [C][n] at the pixels (ys, xs) (n = -1: every pixel): divide by
 * g = sum_k w_k sum_u h_k if normalize; + sigma xi (Philox stream 1, counter (y W + x, c,
 * frame), first Gaussian); clamp to [0, 1] if clamp01. */
void p2so_step5(double* out, const double* w, const double* basis, int C, int H, int W, int K, int T,
                const int* ys, const int* xs, int64_t n, uint64_t seed, int64_t frame, double sigma, int normalize,
                int clamp01) {
  const int64_t np = n < 0 ? (int64_t)H * W : n;
  double* hs = malloc(sizeof(double) * K);
  for (int k = 0; k < K; ++k) {
    double s = 0.0;
    for (int i = 0; i < T * T; ++i) s += basis[(size_t)k * T * T + i];
    hs[k] = s;
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < np; ++i) {
    const int y = n < 0 ? (int)(i / W) : ys[i], x = n < 0 ? (int)(i % W) : xs[i];
    const size_t pix = (size_t)y * W + x;
    double g = 0.0;
    if (normalize)
      for (int k = 0; k < K; ++k) g += w[(size_t)k * H * W + pix] * hs[k];
    for (int c = 0; c < C; ++c) {
      double o = out[(size_t)c * np + i];
      if (normalize) o /= g;
      if (sigma != 0.0) {
        double gg[4];
        gaussians((uint32_t)pix, c, 1, frame, seed, gg);
        o += sigma * gg[0];
      }
      if (clamp01) o = o < 0.0 ? 0.0 : (o > 1.0 ? 1.0 : o);
      out[(size_t)c * np + i] = o;
    }
  }
  free(hs);
}

/* Steps 1-5 of one white-noise frame on every pixel (the CPU baseline's unit of work):
 * img [C][H][W], sqrtS [N-1][P][Q], L [N][N], packed MLP, basis [K][T][T] -> out [C][H][W]. */
int p2so_simulate_frame(const double* img, uint64_t seed, int64_t frame, const double* sqrtS, int P, int Q,
                        const double* L, int N, int C, int H, int W, double kappa, const double* mlp, int h1, int h2,
                        const double* basis, int K, int T, double sigma, int normalize, int clamp01, double* out) {
  const size_t HW = (size_t)H * W;
  double* eta = malloc(sizeof(double) * 2 * (size_t)(N - 1) * P * Q);
  double* f = malloc(sizeof(double) * (size_t)(N - 1) * HW);
  double* a = malloc(sizeof(double) * (size_t)N * HW);
  double* Iw = malloc(sizeof(double) * (size_t)C * HW);
  double* w = malloc(sizeof(double) * (size_t)K * HW);
  if (!eta || !f || !a || !Iw || !w) {
    free(eta), free(f), free(a), free(Iw), free(w);
    return 1;
  }
  p2so_white_noise(seed, frame, P, Q, N, eta);
  p2so_fields(eta, sqrtS, P, Q, H, W, N, f);
  p2so_mix(f, L, N, HW, a);
  p2so_warp(img, a + HW, a + 2 * HW, kappa, C, H, W, Iw);
  p2so_mlp(a + 3 * HW, HW, N - 3, h1, h2, K, mlp, w);
  p2so_blur(Iw, w, basis, C, H, W, K, T, NULL, NULL, -1, out);
  p2so_step5(out, w, basis, C, H, W, K, T, NULL, NULL, -1, seed, frame, sigma, normalize, clamp01);
  free(eta), free(f), free(a), free(Iw), free(w);
  return 0;
}

int p2so_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
