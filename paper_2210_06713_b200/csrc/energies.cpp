// energies.cpp -- validation battery: the Zernike cross-correlation
// kernels A_ij(s) and the approximation energies E, E~, E- of P:369-397, host fp64.
//
//   A_ij(s, phi) = 2 pi C_W sqrt((n_i+1)(n_j+1)) Int nu^{-8/3} P_{n_i}(nu) P_{n_j}(nu)
//                  Re{conj(c_i) c_j G_ij(2 pi nu s, phi)} d nu   (units (D/r0)^{5/3})
//   P_n(nu) = 2 J_{n+1}(pi nu)/(pi nu),  c_j = (-1)^{(n_j-m_j)/2} i^{m_j},
//   G_ij = (1/2pi) Int A_i(t) A_j(t) e^{i x cos(t - phi)} dt, A = 1 | sqrt2 cos(m t) | sqrt2 sin(m t),
// expanded into harmonics cos/sin(M t) with (1/2pi) Int trig(M t) e^{i x cos(t-phi)} dt =
// i^M J_M(x) trig(M phi).  The energies integrate tr(A^T A), tr(A~^T A~) and
// |tr(A^T A - A~^T A~)| over the disc |s'| <= s (A~ = L diag(c_k) L^T, Eq.10), either at
// every angle (the printed formulas) or with the angle-averaged functions (reading Q25).
#include <algorithm>
#include <cmath>
#include <vector>

#include "p2s_internal.h"

namespace p2s {
namespace {

constexpr double kPi = 3.14159265358979323846;

struct Term {
  double coef;
  int M;      // signed harmonic
  bool sine;  // trig = sin (else cos)
};

// A_a(t) A_b(t) = sum coef * trig(M t)
void angular_terms(int a, int b, std::vector<Term>& out) {
  int na, ma, ka, nb, mb, kb;
  noll_nm(a, &na, &ma, &ka);
  noll_nm(b, &nb, &mb, &kb);
  out.clear();
  const double r2 = std::sqrt(2.0);
  if (ma == 0 && mb == 0) {
    out.push_back({1.0, 0, false});
  } else if (ma == 0) {
    out.push_back({r2, mb, kb < 0});
  } else if (mb == 0) {
    out.push_back({r2, ma, ka < 0});
  } else if (ka > 0 && kb > 0) {
    out.push_back({1.0, ma - mb, false});
    out.push_back({1.0, ma + mb, false});
  } else if (ka < 0 && kb < 0) {
    out.push_back({1.0, ma - mb, false});
    out.push_back({-1.0, ma + mb, false});
  } else if (ka > 0 && kb < 0) {
    out.push_back({1.0, ma + mb, true});
    out.push_back({-1.0, ma - mb, true});
  } else {
    out.push_back({1.0, ma + mb, true});
    out.push_back({1.0, ma - mb, true});
  }
}

// Re(i^k)
double re_ipow(int k) {
  k = ((k % 4) + 4) % 4;
  return k == 0 ? 1.0 : (k == 2 ? -1.0 : 0.0);
}

}  // namespace
}  // namespace p2s

using namespace p2s;

extern "C" p2s_status p2s_correlation_energies(int Z, double d_over_r0, double s_max, int n_per_unit, int angle_mean,
                                               int mode_lo, double* s_out, double* E, double* Et, double* Em) {
  if (Z < 4 || Z > 66 || !(d_over_r0 >= 0) || !(s_max > 0) || n_per_unit < 1 || mode_lo < 2 || mode_lo > Z ||
      !s_out || !E || !Et || !Em)
    return set_error(P2S_ERR_INVALID_ARGUMENT, "p2s_correlation_energies: bad argument");
  const int ns = std::max(2, (int)std::lround(n_per_unit * s_max));
  const int nphi = angle_mean ? 1 : 32;
  std::vector<double> A0, Lc;
  noll_matrix(Z, d_over_r0, A0);
  noll_cholesky(Z, A0, Lc);
  int nmax = 0, mmax = 0;
  for (int j = 2; j <= Z; ++j) {
    int n, m, k;
    noll_nm(j, &n, &m, &k);
    nmax = std::max(nmax, n);
    mmax = std::max(mmax, m);
  }
  const int Mmax = 2 * mmax;
  // nu quadrature: nu = u^3 on [0, 1], then panels of width <= min(0.25, 1/(2 s_max)) to 60
  std::vector<double> nu, wq;
  {
    const double xg[8] = {-0.9602898564975363, -0.7966664774136267, -0.5255324099163290, -0.1834346424956498,
                          0.1834346424956498,  0.5255324099163290,  0.7966664774136267,  0.9602898564975363};
    const double wg[8] = {0.1012285362903763, 0.2223810344533745, 0.3137066458778873, 0.3626837833783620,
                          0.3626837833783620, 0.3137066458778873, 0.2223810344533745, 0.1012285362903763};
    const double pw = std::min(0.25, 1.0 / (2.0 * s_max));
    const int npa = (int)std::ceil(3.0 / pw);
    for (int p = 0; p < npa; ++p) {
      const double a = (double)p / npa, b = (double)(p + 1) / npa;
      for (int g = 0; g < 8; ++g) {
        const double u = 0.5 * (b - a) * xg[g] + 0.5 * (a + b);
        nu.push_back(u * u * u);
        wq.push_back(0.5 * (b - a) * wg[g] * 3.0 * u * u);
      }
    }
    const double numax = 60.0;
    const int npb = (int)std::ceil((numax - 1.0) / pw);
    for (int p = 0; p < npb; ++p) {
      const double a = 1.0 + (numax - 1.0) * p / npb, b = 1.0 + (numax - 1.0) * (p + 1) / npb;
      for (int g = 0; g < 8; ++g) {
        nu.push_back(0.5 * (b - a) * xg[g] + 0.5 * (a + b));
        wq.push_back(0.5 * (b - a) * wg[g]);
      }
    }
  }
  const int nn = (int)nu.size();
  const int NP = nmax + 1;
  std::vector<double> Pn((size_t)nn * NP), base(nn);  // P_n(nu), quadrature weight x prefactor
  for (int q = 0; q < nn; ++q) {
    std::vector<double> J(NP + 2);
    const double x = kPi * nu[q];
    bessel_j_all(x, NP + 1, J.data());
    for (int n = 0; n <= nmax; ++n) Pn[(size_t)q * NP + n] = 2.0 * J[n + 1] / x;
    base[q] = wq[q] * 2.0 * kPi * kolmogorov_cw() * std::pow(nu[q], -8.0 / 3.0);
  }
  // radial functions R[n_a][n_b][M](s) on the s grid
  std::vector<double> sg(ns + 1);
  for (int i = 0; i <= ns; ++i) sg[i] = s_max * i / ns;
  const size_t rstride = (size_t)NP * NP * (Mmax + 1);
  std::vector<double> R((size_t)(ns + 1) * rstride, 0.0);
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i <= ns; ++i) {
    std::vector<double> JM(Mmax + 1);
    double* Ri = R.data() + (size_t)i * rstride;
    for (int q = 0; q < nn; ++q) {
      bessel_j_all(2.0 * kPi * nu[q] * sg[i], Mmax, JM.data());
      for (int na = 0; na <= nmax; ++na)
        for (int nb = na; nb <= nmax; ++nb) {
          const double f = base[q] * Pn[(size_t)q * NP + na] * Pn[(size_t)q * NP + nb];
          double* r = Ri + ((size_t)na * NP + nb) * (Mmax + 1);
          for (int M = 0; M <= Mmax; ++M) r[M] += f * JM[M];
        }
    }
  }
  const double scale = std::pow(d_over_r0, 5.0 / 3.0);
  // kernel A_ab(s_i, phi_p) for all a, b in [2, Z]
  auto kernel = [&](int a, int b, int i, double phi) {
    int na, ma, ka, nb, mb, kb;
    noll_nm(a, &na, &ma, &ka);
    noll_nm(b, &nb, &mb, &kb);
    const double sgn_c = (((na - ma) / 2 + (nb - mb) / 2) % 2) ? -1.0 : 1.0;
    std::vector<Term> terms;
    angular_terms(a, b, terms);
    const int lo = std::min(na, nb), hi = std::max(na, nb);
    const double* r = R.data() + (size_t)i * rstride + ((size_t)lo * NP + hi) * (Mmax + 1);
    double v = 0.0;
    for (const Term& t : terms) {
      if (angle_mean && (t.M != 0 || t.sine)) continue;
      const int aM = std::abs(t.M);
      const double jsign = (t.M < 0 && (aM & 1)) ? -1.0 : 1.0;  // J_{-M} = (-1)^M J_M
      const double ph = t.sine ? std::sin(t.M * phi) : std::cos(t.M * phi);
      v += sgn_c * t.coef * re_ipow(mb - ma + t.M) * jsign * r[aM] * ph;
    }
    return v * scale * std::sqrt((na + 1.0) * (nb + 1.0));
  };
  std::vector<double> ffull(ns + 1, 0.0), fmodel(ns + 1, 0.0), fdiff(ns + 1, 0.0);
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i <= ns; ++i) {
    double sf = 0.0, sm = 0.0, sd = 0.0;
    for (int p = 0; p < nphi; ++p) {
      const double phi = 2.0 * kPi * p / nphi;
      std::vector<double> c(Z + 1, 0.0);
      for (int k = 2; k <= Z; ++k) {
        const double v = A0[(size_t)(k - 1) * Z + (k - 1)];
        c[k] = v > 0 ? kernel(k, k, i, phi) / v : 0.0;
      }
      double tf = 0.0, tm = 0.0;
      for (int a = mode_lo; a <= Z; ++a)
        for (int b = mode_lo; b <= Z; ++b) {
          const double Aab = kernel(a, b, i, phi);
          double Mab = 0.0;
          for (int k = 2; k <= Z; ++k) Mab += Lc[(size_t)(a - 1) * Z + (k - 1)] * Lc[(size_t)(b - 1) * Z + (k - 1)] * c[k];
          tf += Aab * Aab;
          tm += Mab * Mab;
        }
      sf += tf;
      sm += tm;
      sd += std::fabs(tf - tm);
    }
    ffull[i] = sf / nphi * 2.0 * kPi * sg[i];
    fmodel[i] = sm / nphi * 2.0 * kPi * sg[i];
    fdiff[i] = sd / nphi * 2.0 * kPi * sg[i];
  }
  E[0] = Et[0] = Em[0] = 0.0;
  s_out[0] = 0.0;
  for (int i = 1; i <= ns; ++i) {
    const double h = sg[i] - sg[i - 1];
    s_out[i] = sg[i];
    E[i] = E[i - 1] + 0.5 * h * (ffull[i] + ffull[i - 1]);
    Et[i] = Et[i - 1] + 0.5 * h * (fmodel[i] + fmodel[i - 1]);
    Em[i] = Em[i - 1] + 0.5 * h * (fdiff[i] + fdiff[i - 1]);
  }
  return P2S_OK;
}
