// train.cpp -- training of the P2S network, host fp64.
//
// a small network maps each pixel's Zernike vector a_x to the PSF-basis
// coefficients beta_x.  Reading Q26 (loss and optimiser are not given): mean squared error
// over the mini-batch and the K outputs, Adam (0.9, 0.999, 1e-8, bias-corrected), one
// update per mini-batch of consecutive entries of the caller's per-epoch sample order.
// Forward/backward per sample, OpenMP over the samples of a batch with per-thread gradient
// buffers summed in thread order.  The packed weight layout is the plan's
// [W1 (h1 x n_in), b1, W2 (h2 x h1), b2, W3 (K x h2), b3], row-major [out][in].
#include <cmath>
#include <cstring>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "p2s_internal.h"

using namespace p2s;

extern "C" p2s_status p2s_train_mlp(const float* mlp_in, int n_in, int h1, int h2, int K, const float* a,
                                    const float* beta, int n, const int32_t* order, int epochs, int batch,
                                    double lr, float* mlp_out, double* loss_curve) {
  if (!mlp_in || !a || !beta || !order || !mlp_out || n_in < 1 || h1 < 1 || h2 < 1 || K < 1 || n < 1 ||
      epochs < 1 || batch < 1 || !(lr > 0))
    return set_error(P2S_ERR_INVALID_ARGUMENT, "p2s_train_mlp: bad argument");
  for (size_t i = 0; i < (size_t)epochs * n; ++i)
    if (order[i] < 0 || order[i] >= n) return set_error(P2S_ERR_INVALID_ARGUMENT, "p2s_train_mlp: order out of range");
  const size_t oW1 = 0, ob1 = oW1 + (size_t)h1 * n_in, oW2 = ob1 + h1, ob2 = oW2 + (size_t)h2 * h1,
               oW3 = ob2 + h2, ob3 = oW3 + (size_t)K * h2, np_ = ob3 + K;
  std::vector<double> th(np_), m(np_, 0.0), v(np_, 0.0);
  for (size_t i = 0; i < np_; ++i) th[i] = mlp_in[i];
  int nth = 1;
#ifdef _OPENMP
  nth = omp_get_max_threads();
#endif
  std::vector<double> gbuf((size_t)nth * np_);
  std::vector<double> lbuf(nth);
  const double b1c = 0.9, b2c = 0.999, eps = 1e-8;
  long long t = 0;
  for (int e = 0; e < epochs; ++e) {
    const int32_t* ord = order + (size_t)e * n;
    double ep_loss = 0.0;
    for (int s0 = 0; s0 < n; s0 += batch) {
      const int B = std::min(batch, n - s0);
      const double scale = 2.0 / ((double)B * K);
      std::fill(gbuf.begin(), gbuf.end(), 0.0);
      std::fill(lbuf.begin(), lbuf.end(), 0.0);
#pragma omp parallel num_threads(nth)
      {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double* g = gbuf.data() + (size_t)tid * np_;
        std::vector<double> z1(h1), hh1(h1), z2(h2), hh2(h2), dy(K), d2(h2), d1(h1);
        double lsum = 0.0;
#pragma omp for schedule(static)
        for (int i = 0; i < B; ++i) {
          const int idx = ord[s0 + i];
          const float* x = a + (size_t)idx * n_in;
          const float* bt = beta + (size_t)idx * K;
          for (int u = 0; u < h1; ++u) {
            double s = th[ob1 + u];
            const double* w = th.data() + oW1 + (size_t)u * n_in;
            for (int k = 0; k < n_in; ++k) s += w[k] * x[k];
            z1[u] = s;
            hh1[u] = s > 0 ? s : 0.0;
          }
          for (int u = 0; u < h2; ++u) {
            double s = th[ob2 + u];
            const double* w = th.data() + oW2 + (size_t)u * h1;
            for (int k = 0; k < h1; ++k) s += w[k] * hh1[k];
            z2[u] = s;
            hh2[u] = s > 0 ? s : 0.0;
          }
          for (int u = 0; u < K; ++u) {
            double s = th[ob3 + u];
            const double* w = th.data() + oW3 + (size_t)u * h2;
            for (int k = 0; k < h2; ++k) s += w[k] * hh2[k];
            const double r = s - bt[u];
            lsum += r * r;
            dy[u] = scale * r;
          }
          // layer 3
          std::fill(d2.begin(), d2.end(), 0.0);
          for (int u = 0; u < K; ++u) {
            double* gw = g + oW3 + (size_t)u * h2;
            const double* w = th.data() + oW3 + (size_t)u * h2;
            for (int k = 0; k < h2; ++k) {
              gw[k] += dy[u] * hh2[k];
              d2[k] += dy[u] * w[k];
            }
            g[ob3 + u] += dy[u];
          }
          for (int k = 0; k < h2; ++k) d2[k] = z2[k] > 0 ? d2[k] : 0.0;
          // layer 2
          std::fill(d1.begin(), d1.end(), 0.0);
          for (int u = 0; u < h2; ++u) {
            if (d2[u] == 0.0) continue;
            double* gw = g + oW2 + (size_t)u * h1;
            const double* w = th.data() + oW2 + (size_t)u * h1;
            for (int k = 0; k < h1; ++k) {
              gw[k] += d2[u] * hh1[k];
              d1[k] += d2[u] * w[k];
            }
            g[ob2 + u] += d2[u];
          }
          for (int k = 0; k < h1; ++k) d1[k] = z1[k] > 0 ? d1[k] : 0.0;
          // layer 1
          for (int u = 0; u < h1; ++u) {
            if (d1[u] == 0.0) continue;
            double* gw = g + oW1 + (size_t)u * n_in;
            for (int k = 0; k < n_in; ++k) gw[k] += d1[u] * x[k];
            g[ob1 + u] += d1[u];
          }
        }
        lbuf[tid] = lsum;
      }
      double bl = 0.0;
      for (int i = 0; i < nth; ++i) bl += lbuf[i];
      ep_loss += bl / K;  // sum over the batch of the per-sample mean over K
      ++t;
      const double c1 = 1.0 - std::pow(b1c, (double)t), c2 = 1.0 - std::pow(b2c, (double)t);
#pragma omp parallel for schedule(static) num_threads(nth)
      for (long long p = 0; p < (long long)np_; ++p) {
        double gp = 0.0;
        for (int i = 0; i < nth; ++i) gp += gbuf[(size_t)i * np_ + p];
        m[p] = b1c * m[p] + (1.0 - b1c) * gp;
        v[p] = b2c * v[p] + (1.0 - b2c) * gp * gp;
        th[p] -= lr * (m[p] / c1) / (std::sqrt(v[p] / c2) + eps);
      }
    }
    if (loss_curve) loss_curve[e] = ep_loss / n;
  }
  for (size_t i = 0; i < np_; ++i) mlp_out[i] = (float)th[i];
  return P2S_OK;
}
