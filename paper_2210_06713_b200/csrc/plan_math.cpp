// plan_math.cpp -- host (CPU, fp64) plan-time tables of the DF-P2S simulator.
//
// Everything here runs once per plan, off the per-frame clock:
//   * Noll indexing and the Noll matrix A_0 = [A]_{0,i,j} in Noll's
//     Gamma-function closed form with the exact Kolmogorov constant (reading Q1);
//   * the Cholesky factor L, L L^T = A_0 over j = 2..Z (Eq.10);
//   * the homogeneous auto-correlation slices A_jj(s) (form of
//     reading Q4) as radial Hankel integrals, sampled on the periodic lag grid;
//   * S_j = DFT(c_j) (the circulant eigenvalues), clamped at 0 and
//     renormalised to sum S_j = P*Q (reading Q7), and sqrt(S_j).
// Written independently of oracle/ (own Bessel functions, quadrature, spline,
// FFT and Cholesky).  Exposed for CPU tests through p2s_host_tables().
#include "p2s_internal.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

namespace p2s {

static const double kPi = 3.14159265358979323846;

// ------------------------------------------------------------------ constants
// Eq.4 structure-function constant C_D = 2[(24/5) Gamma(6/5)]^{5/6} (printed 6.88).
double kolmogorov_cd() { return 2.0 * std::pow(4.8 * std::tgamma(1.2), 5.0 / 6.0); }
// Phase PSD coefficient W(f) = C_W r0^{-5/3} f^{-11/3}, from
// C_D = 4 pi C_W (2 pi)^{5/3} * 2^{-5/3} Gamma(1/6) / ((5/3) Gamma(11/6)).
double kolmogorov_cw() {
  double I = std::pow(2.0, -5.0 / 3.0) * std::tgamma(1.0 / 6.0) / ((5.0 / 3.0) * std::tgamma(11.0 / 6.0));
  return kolmogorov_cd() / (4.0 * kPi * std::pow(2.0 * kPi, 5.0 / 3.0) * I);
}
// Noll constant K_N = C_W 2^{-5/3} pi^{8/3} Gamma(14/3) (= 2.246065).
double noll_constant() {
  return kolmogorov_cw() * std::pow(2.0, -5.0 / 3.0) * std::pow(kPi, 8.0 / 3.0) * std::tgamma(14.0 / 3.0);
}

// ------------------------------------------------------------------ Noll index
void noll_nm(int j, int* n_out, int* m_out, int* kind_out) {
  int n = 0;
  while ((n + 1) * (n + 2) / 2 < j) ++n;
  int p = j - n * (n + 1) / 2 - 1;
  int m = (n % 2 == 0) ? 2 * ((p + 1) / 2) : 2 * (p / 2) + 1;
  *n_out = n;
  *m_out = m;
  *kind_out = (m == 0) ? 0 : ((j % 2 == 0) ? 1 : -1);  // 0 rot, +1 cos, -1 sin
}

void noll_matrix(int Z, double d_over_r0, std::vector<double>& A) {
  A.assign((size_t)Z * Z, 0.0);
  const double K = noll_constant();
  const double sc = std::pow(d_over_r0, 5.0 / 3.0);
  for (int i = 2; i <= Z; ++i) {
    int ni, mi, ki;
    noll_nm(i, &ni, &mi, &ki);
    for (int j = 2; j <= Z; ++j) {
      int nj, mj, kj;
      noll_nm(j, &nj, &mj, &kj);
      if (mi != mj) continue;
      if (mi != 0 && ki != kj) continue;
      double sgn = (((ni + nj - 2 * mi) / 2) % 2 == 0) ? 1.0 : -1.0;
      double num = K * sgn * std::sqrt((ni + 1.0) * (nj + 1.0)) * std::tgamma((ni + nj - 5.0 / 3.0) / 2.0);
      double den = std::tgamma((ni - nj + 17.0 / 3.0) / 2.0) * std::tgamma((nj - ni + 17.0 / 3.0) / 2.0) *
                   std::tgamma((ni + nj + 23.0 / 3.0) / 2.0);
      A[(size_t)(i - 1) * Z + (j - 1)] = num / den * sc;
    }
  }
}

// Cholesky of A[1:,1:] into L (Z x Z, row/col 0 zero).  Returns false on failure.
static bool chol_inplace(int n, const double* B, double* Lo) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = B[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) s -= Lo[(size_t)i * n + k] * Lo[(size_t)j * n + k];
      if (i == j) {
        if (!(s > 0.0)) return false;
        Lo[(size_t)i * n + i] = std::sqrt(s);
      } else {
        Lo[(size_t)i * n + j] = s / Lo[(size_t)j * n + j];
      }
    }
  return true;
}

bool noll_cholesky(int Z, const std::vector<double>& A, std::vector<double>& L) {
  L.assign((size_t)Z * Z, 0.0);
  int n = Z - 1;
  std::vector<double> B((size_t)n * n), Lo((size_t)n * n, 0.0);
  bool any = false;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      B[(size_t)i * n + j] = A[(size_t)(i + 1) * Z + (j + 1)];
      any |= B[(size_t)i * n + j] != 0.0;
    }
  if (!any) return true;  // D/r0 = 0: L = 0
  if (!chol_inplace(n, B.data(), Lo.data())) {
    double tr = 0;
    for (int i = 0; i < n; ++i) tr += B[(size_t)i * n + i];
    for (int i = 0; i < n; ++i) B[(size_t)i * n + i] += 1e-12 * tr / n;
    std::fill(Lo.begin(), Lo.end(), 0.0);
    if (!chol_inplace(n, B.data(), Lo.data())) return false;
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) L[(size_t)(i + 1) * Z + (j + 1)] = Lo[(size_t)i * n + j];
  return true;
}

// ------------------------------------------------------------------ Bessel J_0..J_nmax
// Miller backward recurrence (x < 40) normalised by J0 + 2 sum J_2k = 1, or the
// Hankel asymptotic expansion for J0, J1 plus forward recurrence (x >= 40 > nmax).
static void bessel_asym01(double x, double* j0, double* j1) {
  for (int nu = 0; nu <= 1; ++nu) {
    double mu = 4.0 * nu * nu, P = 0, Qs = 0, term = 1.0;
    for (int k = 0; k < 40; ++k) {
      // a_k = prod_{i=1..k} (mu - (2i-1)^2) / (k! 8^k); term = a_k / x^k
      if (k > 0) term *= (mu - (2.0 * k - 1) * (2.0 * k - 1)) / (k * 8.0 * x);
      double t = term;
      if (k % 4 == 0) P += t;
      else if (k % 4 == 1) Qs += t;
      else if (k % 4 == 2) P -= t;
      else Qs -= t;
      if (k > 2 && std::fabs(term) < 1e-17) break;
    }
    double w = x - nu * kPi / 2 - kPi / 4;
    double v = std::sqrt(2.0 / (kPi * x)) * (P * std::cos(w) - Qs * std::sin(w));
    if (nu == 0) *j0 = v; else *j1 = v;
  }
}

void bessel_j_all(double x, int nmax, double* J) {
  if (x == 0.0) {
    J[0] = 1.0;
    for (int k = 1; k <= nmax; ++k) J[k] = 0.0;
    return;
  }
  if (x < 1e-8) {  // leading series term
    double t = 1.0;
    for (int k = 0; k <= nmax; ++k) {
      J[k] = t;
      t *= x / (2.0 * (k + 1));
    }
    return;
  }
  if (x >= 40.0) {
    bessel_asym01(x, &J[0], &J[1]);
    for (int k = 1; k < nmax; ++k) J[k + 1] = (2.0 * k / x) * J[k] - J[k - 1];
    return;
  }
  int M = 2 * ((int)(std::max(x, (double)nmax) + 30.0) / 2 + 1);
  double bkp1 = 0.0, bk = 1e-30, sum = 0.0;
  double tmp[160];
  for (int k = M; k >= 1; --k) {
    double bkm1 = (2.0 * k / x) * bk - bkp1;
    bkp1 = bk;
    bk = bkm1;
    if (k - 1 <= nmax) tmp[k - 1] = bk;
    if ((k - 1) % 2 == 0 && k - 1 > 0) sum += 2.0 * bk;
    if (std::fabs(bk) > 1e250) {  // rescale
      bk *= 1e-250; bkp1 *= 1e-250; sum *= 1e-250;
      for (int q = k - 1; q <= nmax && q <= M; ++q) if (q >= k - 1) tmp[q] *= 1e-250;
    }
  }
  sum += bk;  // b_0
  for (int k = 0; k <= nmax; ++k) J[k] = tmp[k] / sum;
}

// ------------------------------------------------------------------ radial Hankel tables
// R_{n,q}(s) = 2 pi C_W (n+1) Int_0^inf nu^{-8/3} [2 J_{n+1}(pi nu)/(pi nu)]^2 J_q(2 pi nu s) d nu
// (units of (D/r0)^{5/3}; nu in cycles per aperture diameter, s in units of D).
struct RadialSeg {
  double s0 = 0, h = 0.005;
  int ns = 0, nq = 0;
  std::vector<double> tab;  // [(n-1)*nq + q/2][ns]
  double* row(int n, int q) { return &tab[((size_t)(n - 1) * nq + q / 2) * ns]; }
  const double* row(int n, int q) const { return &tab[((size_t)(n - 1) * nq + q / 2) * ns]; }
  // 4-point Lagrange interpolation on the uniform grid s0 + i h
  double eval(int n, int q, double s) const {
    const double* r = row(n, q);
    double u = (s - s0) / h;
    int i = (int)std::floor(u);
    if (i < 1) i = 1;
    if (i > ns - 3) i = ns - 3;
    double t = u - i;  // nodes i-1, i, i+1, i+2 at t = -1, 0, 1, 2
    double l0 = -t * (t - 1) * (t - 2) / 6.0;
    double l1 = (t + 1) * (t - 1) * (t - 2) / 2.0;
    double l2 = -(t + 1) * t * (t - 2) / 2.0;
    double l3 = (t + 1) * t * (t - 1) / 6.0;
    return l0 * r[i - 1] + l1 * r[i] + l2 * r[i + 1] + l3 * r[i + 2];
  }
};

// Fine segment (h = 0.005) for |s| <= 4 where the high modes vary fastest, coarse
// segment (h = 0.05) beyond, where every A_jj varies on scales >> 0.05 (SURVEY C3
// tables) and nu > 20 contributes < 1e-8 relative after the Bessel oscillation.
struct Radial {
  int nmax = 0, qmax = 0;
  double s_split = 4.0;
  RadialSeg fine, coarse;
  bool has_coarse = false;
  double eval(int n, int q, double s) const {
    return (has_coarse && s > s_split) ? coarse.eval(n, q, s) : fine.eval(n, q, s);
  }
  double at0(int n) const { return fine.row(n, 0)[0]; }
};

static void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  x.resize(n);
  w.resize(n);
  for (int i = 0; i < n; ++i) {
    double z = std::cos(kPi * (i + 0.75) / (n + 0.5)), z1, pp;
    do {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; ++j) {
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      z1 = z;
      z = z1 - p1 / pp;
    } while (std::fabs(z - z1) > 1e-15);
    x[i] = -z;
    w[i] = 2.0 / ((1.0 - z * z) * pp * pp);
  }
}

// Quadrature nodes on (0, nu_max]: t = nu^{1/3} on [0, 1] (removes the nu^{-2/3}
// end point of the tilt integrand), then nu in [1, nu_max]; 16-point Gauss
// panels no wider than one period of J_q(2 pi nu s_hi).
static void radial_nodes(double s_hi, double nu_max, std::vector<double>& nu, std::vector<double>& wq) {
  double pw = std::min(0.5, 1.0 / std::max(s_hi, 1e-3));
  std::vector<double> gx, gw;
  gauss_legendre(16, gx, gw);
  nu.clear();
  wq.clear();
  int npa = (int)std::ceil(3.0 / pw);
  for (int p = 0; p < npa; ++p) {
    double a = (double)p / npa, b = (double)(p + 1) / npa;
    for (int i = 0; i < 16; ++i) {
      double t = 0.5 * (b - a) * gx[i] + 0.5 * (a + b);
      nu.push_back(t * t * t);
      wq.push_back(0.5 * (b - a) * gw[i] * 3.0 * t * t);
    }
  }
  int npb = (int)std::ceil((nu_max - 1.0) / pw);
  for (int p = 0; p < npb; ++p) {
    double a = 1.0 + (nu_max - 1.0) * p / npb, b = 1.0 + (nu_max - 1.0) * (p + 1) / npb;
    for (int i = 0; i < 16; ++i) {
      nu.push_back(0.5 * (b - a) * gx[i] + 0.5 * (a + b));
      wq.push_back(0.5 * (b - a) * gw[i]);
    }
  }
}

static void fill_segment(RadialSeg& S, int nmax, int qmax, double nu_max) {
  std::vector<double> nu, wq;
  double s_hi = S.s0 + (S.ns - 1) * S.h;
  radial_nodes(s_hi, nu_max, nu, wq);
  const int nn = (int)nu.size();
  const double cw = kolmogorov_cw();
  std::vector<double> G((size_t)nmax * nn);
  for (int i = 0; i < nn; ++i) {
    double J[64];
    double x = kPi * nu[i];
    bessel_j_all(x, nmax + 1, J);
    for (int n = 1; n <= nmax; ++n) {
      double win = 2.0 * J[n + 1] / x;
      G[(size_t)(n - 1) * nn + i] = 2.0 * kPi * cw * (n + 1.0) * std::pow(nu[i], -8.0 / 3.0) * win * win * wq[i];
    }
  }
  const int nq = S.nq;
#pragma omp parallel for schedule(dynamic, 4)
  for (int is = 0; is < S.ns; ++is) {
    double s = S.s0 + is * S.h;
    std::vector<double> acc((size_t)nmax * nq, 0.0);
    double J[64];
    for (int i = 0; i < nn; ++i) {
      bessel_j_all(2.0 * kPi * nu[i] * s, qmax, J);
      for (int n = 1; n <= nmax; ++n) {
        double g = G[(size_t)(n - 1) * nn + i];
        double* a = &acc[(size_t)(n - 1) * nq];
        for (int qi = 0; qi < nq; ++qi) a[qi] += g * J[2 * qi];
      }
    }
    for (int n = 1; n <= nmax; ++n)
      for (int qi = 0; qi < nq; ++qi) S.row(n, 2 * qi)[is] = acc[(size_t)(n - 1) * nq + qi];
  }
}

static void build_radial(Radial& R, int Z, double s_max) {
  int nmax = 0, qmax = 0;
  for (int j = 2; j <= Z; ++j) {
    int n, m, k;
    noll_nm(j, &n, &m, &k);
    nmax = std::max(nmax, n);
    qmax = std::max(qmax, 2 * m);
  }
  R.nmax = nmax;
  R.qmax = qmax;
  const int nq = qmax / 2 + 1;
  double s_f = std::min(s_max, R.s_split);
  R.fine.s0 = 0.0;
  R.fine.h = 0.005;
  R.fine.nq = nq;
  R.fine.ns = (int)std::ceil(s_f / R.fine.h) + 5;
  R.fine.tab.assign((size_t)nmax * nq * R.fine.ns, 0.0);
  fill_segment(R.fine, nmax, qmax, 60.0);
  R.has_coarse = s_max > R.s_split;
  if (R.has_coarse) {
    R.coarse.h = 0.05;
    R.coarse.s0 = R.s_split - 2 * R.coarse.h;
    R.coarse.nq = nq;
    R.coarse.ns = (int)std::ceil((s_max - R.coarse.s0) / R.coarse.h) + 5;
    R.coarse.tab.assign((size_t)nmax * nq * R.coarse.ns, 0.0);
    fill_segment(R.coarse, nmax, qmax, 20.0);
  }
}

// ------------------------------------------------------------------ fp64 FFT (mixed radix 2,3,4,5)
// Stockham autosort, forward sign -1, unnormalised.
struct FFT1D {
  int N = 0;
  std::vector<int> rad;
  std::vector<std::complex<double>> tw;  // e^{-2 pi i k / N}
  explicit FFT1D(int n) : N(n) {
    int m = n;
    while (m % 4 == 0) { rad.push_back(4); m /= 4; }
    while (m % 2 == 0) { rad.push_back(2); m /= 2; }
    while (m % 3 == 0) { rad.push_back(3); m /= 3; }
    while (m % 5 == 0) { rad.push_back(5); m /= 5; }
    tw.resize(n);
    for (int k = 0; k < n; ++k) tw[k] = std::polar(1.0, -2.0 * kPi * k / n);
  }
  void run(std::complex<double>* x, std::complex<double>* scratch) const {
    std::complex<double>* a = x;
    std::complex<double>* b = scratch;
    int Ns = 1;
    for (int R : rad) {
      int NR = N / R;
      int ts = N / (Ns * R);
      for (int j = 0; j < NR; ++j) {
        int k = j % Ns;
        std::complex<double> v[5], V[5];
        for (int r = 0; r < R; ++r) v[r] = a[j + r * NR];
        for (int r = 1; r < R; ++r) v[r] *= tw[(size_t)r * k * ts % N];
        for (int q = 0; q < R; ++q) {
          std::complex<double> s = 0;
          for (int r = 0; r < R; ++r) s += v[r] * tw[(size_t)(r * q % R) * (N / R)];
          V[q] = s;
        }
        int base = (j / Ns) * Ns * R + k;
        for (int q = 0; q < R; ++q) b[base + q * Ns] = V[q];
      }
      std::swap(a, b);
      Ns *= R;
    }
    if (a != x) std::memcpy(x, a, sizeof(std::complex<double>) * N);
  }
};

static void fft2_inplace(std::vector<std::complex<double>>& d, int P, int Q) {
  FFT1D fq(Q), fp(P);
#pragma omp parallel
  {
    std::vector<std::complex<double>> sc(std::max(P, Q)), col(P);
#pragma omp for schedule(static)
    for (int y = 0; y < P; ++y) fq.run(&d[(size_t)y * Q], sc.data());
#pragma omp for schedule(static)
    for (int x = 0; x < Q; ++x) {
      for (int y = 0; y < P; ++y) col[y] = d[(size_t)y * Q + x];
      fp.run(col.data(), sc.data());
      for (int y = 0; y < P; ++y) d[(size_t)y * Q + x] = col[y];
    }
  }
}

// ------------------------------------------------------------------ tables
int grid_size(int x) {
  for (int n = std::max(x, 1);; ++n) {
    int m = n;
    while (m % 2 == 0) m /= 2;
    while (m % 3 == 0) m /= 3;
    while (m % 5 == 0) m /= 5;
    if (m == 1) return n;
  }
}

// sqrtS: [Z-1][P][Q] (slot j-2), clamped[Z-1].
void psd_tables(int P, int Q, double s_px, int Z, std::vector<double>& sqrtS, std::vector<double>& clamped) {
  int hy = P / 2, hx = Q / 2;
  double s_max = s_px * std::sqrt((double)hy * hy + (double)hx * hx);
  Radial R;
  build_radial(R, Z, s_max);
  const int ns = Z - 1;
  sqrtS.assign((size_t)ns * P * Q, 0.0);
  clamped.assign(ns, 0.0);
  const size_t PQ = (size_t)P * Q;
  std::vector<std::complex<double>> plane(PQ);
  for (int p0 = 0; p0 < ns; p0 += 2) {
    int modes[2] = {p0 + 2, (p0 + 1 < ns) ? p0 + 3 : -1};
    // kernel pair c_a + i c_b on the minimum-image lag grid (even in each axis)
#pragma omp parallel for schedule(static)
    for (int iy = 0; iy < P; ++iy) {
      int dy = (iy <= hy) ? iy : iy - P;
      for (int ix = 0; ix < Q; ++ix) {
        int dx = (ix <= hx) ? ix : ix - Q;
        double s = s_px * std::sqrt((double)dy * dy + (double)dx * dx);
        double phi = std::atan2((double)dy, (double)dx);
        double v[2] = {0, 0};
        for (int t = 0; t < 2; ++t) {
          int j = modes[t];
          if (j < 0) continue;
          int n, m, kind;
          noll_nm(j, &n, &m, &kind);
          double val = R.eval(n, 0, s);
          if (m > 0) val += kind * ((m % 2) ? -1.0 : 1.0) * R.eval(n, 2 * m, s) * std::cos(2.0 * m * phi);
          v[t] = val / R.at0(n);
        }
        plane[(size_t)iy * Q + ix] = std::complex<double>(v[0], v[1]);
      }
    }
    fft2_inplace(plane, P, Q);  // DFT(c_a) + i DFT(c_b); both real
    for (int t = 0; t < 2; ++t) {
      if (modes[t] < 0) continue;
      double neg = 0, tot = 0, sum = 0;
      double* out = &sqrtS[(size_t)(p0 + t) * PQ];
      for (size_t k = 0; k < PQ; ++k) {
        double S = (t == 0) ? plane[k].real() : plane[k].imag();
        tot += std::fabs(S);
        if (S < 0) { neg -= S; S = 0; }
        out[k] = S;
        sum += S;
      }
      double sc = (double)PQ / sum;
      for (size_t k = 0; k < PQ; ++k) out[k] = std::sqrt(out[k] * sc);
      clamped[p0 + t] = neg / tot;
    }
  }
}

}  // namespace p2s

extern "C" int p2s_grid_size(int x) { return p2s::grid_size(x); }

extern "C" p2s_status p2s_host_tables(int P, int Q, double s_per_px, double d_over_r0, int Z, double* A0,
                                      double* chol, double* sqrtS, double* clamped) {
  using namespace p2s;
  if (P < 2 || Q < 2 || Z < 4 || Z > 66 || !(s_per_px > 0) || !(d_over_r0 >= 0))
    return set_error(P2S_ERR_INVALID_ARGUMENT, "p2s_host_tables: bad argument");
  std::vector<double> A, L;
  noll_matrix(Z, d_over_r0, A);
  if (!noll_cholesky(Z, A, L)) return set_error(P2S_ERR_NUMERIC, "Cholesky of A_0 failed");
  if (A0) std::memcpy(A0, A.data(), sizeof(double) * A.size());
  if (chol) std::memcpy(chol, L.data(), sizeof(double) * L.size());
  if (sqrtS || clamped) {
    std::vector<double> sq, cl;
    psd_tables(P, Q, s_per_px, Z, sq, cl);
    if (sqrtS) std::memcpy(sqrtS, sq.data(), sizeof(double) * sq.size());
    if (clamped) std::memcpy(clamped, cl.data(), sizeof(double) * cl.size());
  }
  return P2S_OK;
}

namespace p2s {
// Noll-normalised Zernike polynomial Z_j(rho, theta) on the unit disk (theta from the
// column axis, reading Q4); used for the exact-PSF pupil table (NEXT-1).
double zernike_value(int j, double rho, double theta) {
  int n, m, kind;
  noll_nm(j, &n, &m, &kind);
  double R = 0.0;
  for (int s = 0; s <= (n - m) / 2; ++s) {
    double c = std::tgamma(n - s + 1.0) /
               (std::tgamma(s + 1.0) * std::tgamma((n + m) / 2 - s + 1.0) * std::tgamma((n - m) / 2 - s + 1.0));
    R += ((s & 1) ? -c : c) * std::pow(rho, n - 2 * s);
  }
  if (m == 0) return std::sqrt(n + 1.0) * R;
  return std::sqrt(2.0 * (n + 1.0)) * R * (kind > 0 ? std::cos(m * theta) : std::sin(m * theta));
}
}  // namespace p2s
