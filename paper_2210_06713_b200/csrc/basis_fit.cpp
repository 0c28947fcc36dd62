// basis_fit.cpp -- PSF basis by principal components (Eq.7; SURVEY NEXT-1 part).
//
// The paper represents every PSF as h_x = sum_m beta_{x,m} phi_m with a basis learned from
// a PSF database by PCA.  p2s_fit_basis takes such a database (e.g. the exact PSFs
// of p2s_exact_psf at the pixels of sampled frames), and returns the mean PSF followed by
// the M leading principal components (unit L2 norm) and the fraction of the centred energy
// the M components leave out.  Host fp64: covariance by an OpenMP-parallel rank update,
// leading eigenvectors by block (subspace) iteration with modified Gram-Schmidt, finished
// by a Rayleigh-Ritz step (cyclic Jacobi on the M x M projected matrix).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "p2s_internal.h"

namespace p2s {

// Cyclic Jacobi eigen-decomposition of a symmetric n x n matrix (row-major, in place):
// on return A holds the eigenvalues on its diagonal and V the eigenvectors as columns.
static void jacobi_eigen(int n, std::vector<double>& A, std::vector<double>& V) {
  V.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += A[(size_t)p * n + q] * A[(size_t)p * n + q];
    if (off < 1e-30) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[(size_t)p * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        const double app = A[(size_t)p * n + p], aqq = A[(size_t)q * n + q];
        const double th = 0.5 * (aqq - app) / apq;
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // A <- J^T A J
          const double akp = A[(size_t)k * n + p], akq = A[(size_t)k * n + q];
          A[(size_t)k * n + p] = c * akp - s * akq;
          A[(size_t)k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[(size_t)p * n + k], aqk = A[(size_t)q * n + k];
          A[(size_t)p * n + k] = c * apk - s * aqk;
          A[(size_t)q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V[(size_t)k * n + p], vkq = V[(size_t)k * n + q];
          V[(size_t)k * n + p] = c * vkp - s * vkq;
          V[(size_t)k * n + q] = s * vkp + c * vkq;
        }
      }
  }
}

// Modified Gram-Schmidt on the M columns (length d, column-major blocks of Q).
static void orthonormalise(int d, int M, std::vector<double>& Q) {
  for (int j = 0; j < M; ++j) {
    double* qj = Q.data() + (size_t)j * d;
    for (int i = 0; i < j; ++i) {
      const double* qi = Q.data() + (size_t)i * d;
      double dot = 0.0;
      for (int k = 0; k < d; ++k) dot += qi[k] * qj[k];
      for (int k = 0; k < d; ++k) qj[k] -= dot * qi[k];
    }
    double nrm = 0.0;
    for (int k = 0; k < d; ++k) nrm += qj[k] * qj[k];
    nrm = std::sqrt(nrm);
    if (nrm < 1e-300) {  // degenerate: restart the column on a coordinate axis
      std::memset(qj, 0, sizeof(double) * d);
      qj[j % d] = 1.0;
    } else {
      for (int k = 0; k < d; ++k) qj[k] /= nrm;
    }
  }
}

}  // namespace p2s

using namespace p2s;

extern "C" p2s_status p2s_fit_basis(const float* psfs, int n, int T, int M, float* basis, double* residual) {
  if (!psfs || !basis || n < 2 || T < 1 || M < 1 || M > T * T || M >= n)
    return set_error(P2S_ERR_INVALID_ARGUMENT, "p2s_fit_basis: need psfs, basis, n >= 2, 1 <= M < n, M <= T*T");
  const int d = T * T;
  std::vector<double> mean(d, 0.0);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) mean[k] += psfs[(size_t)i * d + k];
  for (int k = 0; k < d; ++k) mean[k] /= n;
  // covariance (upper triangle by rows, OpenMP over rows), then mirror
  std::vector<double> Cv((size_t)d * d, 0.0);
#pragma omp parallel for schedule(dynamic, 8)
  for (int a = 0; a < d; ++a)
    for (int i = 0; i < n; ++i) {
      const float* h = psfs + (size_t)i * d;
      const double xa = h[a] - mean[a];
      if (xa == 0.0) continue;
      double* row = Cv.data() + (size_t)a * d;
      for (int b = a; b < d; ++b) row[b] += xa * (h[b] - mean[b]);
    }
  double trace = 0.0;
  for (int a = 0; a < d; ++a) {
    for (int b = a + 1; b < d; ++b) Cv[(size_t)b * d + a] = Cv[(size_t)a * d + b];
    trace += Cv[(size_t)a * d + a];
  }
  // block iteration: Q <- orth(C Q), deterministic start
  std::vector<double> Q((size_t)M * d), Y((size_t)M * d);
  for (int j = 0; j < M; ++j)
    for (int k = 0; k < d; ++k) Q[(size_t)j * d + k] = std::cos(0.37 * (j + 1) * (k + 1)) + (k == j ? 1.0 : 0.0);
  orthonormalise(d, M, Q);
  for (int it = 0; it < 300; ++it) {
#pragma omp parallel for schedule(static)
    for (int j = 0; j < M; ++j) {
      const double* q = Q.data() + (size_t)j * d;
      double* y = Y.data() + (size_t)j * d;
      for (int a = 0; a < d; ++a) {
        const double* row = Cv.data() + (size_t)a * d;
        double s = 0.0;
        for (int b = 0; b < d; ++b) s += row[b] * q[b];
        y[a] = s;
      }
    }
    orthonormalise(d, M, Y);
    double change = 0.0;  // 1 - |<q_j, y_j>| summed
    for (int j = 0; j < M; ++j) {
      double dot = 0.0;
      for (int k = 0; k < d; ++k) dot += Q[(size_t)j * d + k] * Y[(size_t)j * d + k];
      change += 1.0 - std::fabs(dot);
    }
    Q.swap(Y);
    if (change < 1e-13 * M) break;
  }
  // Rayleigh-Ritz: B = Q^T C Q (M x M), eigenvectors rotate Q into the principal axes
  std::vector<double> B((size_t)M * M), CQ((size_t)M * d);
  for (int j = 0; j < M; ++j)
    for (int a = 0; a < d; ++a) {
      const double* row = Cv.data() + (size_t)a * d;
      double s = 0.0;
      for (int b = 0; b < d; ++b) s += row[b] * Q[(size_t)j * d + b];
      CQ[(size_t)j * d + a] = s;
    }
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j) {
      double s = 0.0;
      for (int k = 0; k < d; ++k) s += Q[(size_t)i * d + k] * CQ[(size_t)j * d + k];
      B[(size_t)i * M + j] = s;
    }
  std::vector<double> V;
  jacobi_eigen(M, B, V);
  std::vector<int> order(M);
  for (int j = 0; j < M; ++j) order[j] = j;
  std::sort(order.begin(), order.end(), [&](int x, int y) { return B[(size_t)x * M + x] > B[(size_t)y * M + y]; });
  double kept = 0.0;
  for (int k = 0; k < d; ++k) basis[k] = (float)mean[k];
  for (int r = 0; r < M; ++r) {
    const int j = order[r];
    kept += B[(size_t)j * M + j];
    std::vector<double> v(d, 0.0);
    for (int i = 0; i < M; ++i) {
      const double c = V[(size_t)i * M + j];
      for (int k = 0; k < d; ++k) v[k] += c * Q[(size_t)i * d + k];
    }
    // sign convention: largest-magnitude entry positive (deterministic output)
    int am = 0;
    for (int k = 1; k < d; ++k)
      if (std::fabs(v[k]) > std::fabs(v[am])) am = k;
    const double sg = v[am] < 0 ? -1.0 : 1.0;
    for (int k = 0; k < d; ++k) basis[(size_t)(r + 1) * d + k] = (float)(sg * v[k]);
  }
  if (residual) *residual = trace > 0 ? std::max(0.0, 1.0 - kept / trace) : 0.0;
  return P2S_OK;
}

// Readout fit for the P2S network (NEXT-1): keep the hidden layers of a packed MLP and
// solve the output layer (W3, b3) by ridge regression from the second hidden layer's
// activations to target basis weights beta (e.g. projections of exact PSFs on the PCA
// basis): (X^T X + lambda I) Theta = X^T beta with X = [h2(a), 1], fp64 Cholesky.
extern "C" p2s_status p2s_fit_readout(const float* mlp_in, int n_in, int h1, int h2, int K, const float* a,
                                      const float* beta, int n, double lambda, float* mlp_out,
                                      double* rel_residual) {
  if (!mlp_in || !a || !beta || !mlp_out || n_in < 1 || h1 < 1 || h2 < 1 || K < 1 || n < 1 || lambda < 0)
    return set_error(P2S_ERR_INVALID_ARGUMENT, "p2s_fit_readout: bad argument");
  const size_t oW1 = 0, ob1 = oW1 + (size_t)h1 * n_in, oW2 = ob1 + h1, ob2 = oW2 + (size_t)h2 * h1,
               oW3 = ob2 + h2, ob3 = oW3 + (size_t)K * h2, total = ob3 + K;
  const int d = h2 + 1;
  std::vector<double> G((size_t)d * d, 0.0), R((size_t)d * K, 0.0);
  std::vector<double> Xall((size_t)n * d);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    std::vector<double> z1(h1);
    for (int u = 0; u < h1; ++u) {
      double s = mlp_in[ob1 + u];
      for (int k = 0; k < n_in; ++k) s += (double)mlp_in[oW1 + (size_t)u * n_in + k] * a[(size_t)i * n_in + k];
      z1[u] = s > 0 ? s : 0.0;
    }
    double* x = Xall.data() + (size_t)i * d;
    for (int v = 0; v < h2; ++v) {
      double s = mlp_in[ob2 + v];
      for (int u = 0; u < h1; ++u) s += (double)mlp_in[oW2 + (size_t)v * h1 + u] * z1[u];
      x[v] = s > 0 ? s : 0.0;
    }
    x[h2] = 1.0;
  }
  for (int i = 0; i < n; ++i) {
    const double* x = Xall.data() + (size_t)i * d;
    for (int p = 0; p < d; ++p) {
      if (x[p] == 0.0) continue;
      for (int q = 0; q < d; ++q) G[(size_t)p * d + q] += x[p] * x[q];
      for (int k = 0; k < K; ++k) R[(size_t)p * K + k] += x[p] * beta[(size_t)i * K + k];
    }
  }
  for (int p = 0; p < h2; ++p) G[(size_t)p * d + p] += lambda;  // the bias is not shrunk
  // Cholesky G = C C^T (in place, lower), then two triangular solves per output
  std::vector<double> C = G;
  for (int j = 0; j < d; ++j) {
    double s = C[(size_t)j * d + j];
    for (int k = 0; k < j; ++k) s -= C[(size_t)j * d + k] * C[(size_t)j * d + k];
    if (!(s > 0.0)) return set_error(P2S_ERR_NUMERIC, "p2s_fit_readout: normal matrix not positive definite");
    C[(size_t)j * d + j] = std::sqrt(s);
    for (int i = j + 1; i < d; ++i) {
      double t = C[(size_t)i * d + j];
      for (int k = 0; k < j; ++k) t -= C[(size_t)i * d + k] * C[(size_t)j * d + k];
      C[(size_t)i * d + j] = t / C[(size_t)j * d + j];
    }
  }
  std::vector<double> Th((size_t)d * K);
  for (int k = 0; k < K; ++k) {
    std::vector<double> y(d);
    for (int i = 0; i < d; ++i) {
      double t = R[(size_t)i * K + k];
      for (int j = 0; j < i; ++j) t -= C[(size_t)i * d + j] * y[j];
      y[i] = t / C[(size_t)i * d + i];
    }
    for (int i = d - 1; i >= 0; --i) {
      double t = y[i];
      for (int j = i + 1; j < d; ++j) t -= C[(size_t)j * d + i] * Th[(size_t)j * K + k];
      Th[(size_t)i * K + k] = t / C[(size_t)i * d + i];
    }
  }
  std::memcpy(mlp_out, mlp_in, sizeof(float) * oW3);
  for (int k = 0; k < K; ++k) {
    for (int v = 0; v < h2; ++v) mlp_out[oW3 + (size_t)k * h2 + v] = (float)Th[(size_t)v * K + k];
    mlp_out[ob3 + k] = (float)Th[(size_t)h2 * K + k];
  }
  if (rel_residual) {
    double num = 0.0, den = 0.0;
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < K; ++k) {
        double p = 0.0;
        for (int q = 0; q < d; ++q) p += Xall[(size_t)i * d + q] * Th[(size_t)q * K + k];
        const double b = beta[(size_t)i * K + k];
        num += (p - b) * (p - b);
        den += b * b;
      }
    *rel_residual = den > 0 ? std::sqrt(num / den) : 0.0;
  }
  (void)total;
  return P2S_OK;
}
