// Dense host linear algebra and the gamma quantile used at setup time:
// the symmetric eigensystem of a reversible generator (substitution.hpp:196-208,
// the Eigen SelfAdjointEigenSolver restated as cyclic Jacobi), Pade-13
// scaling-and-squaring (the Eigen MatrixBase::exp() algorithm, used for
// simulation only) and the regularized incomplete gamma / its quantile
// (Boost gamma_p_inv restated by bisection, substitution.hpp:55-68).
// Shared by libphylograd_b200.so and the workload generator library.
#include <algorithm>
#include <cmath>

#include "pg_common.hpp"

namespace pg {

// ------------------------------------------------------------ linear algebra
RowMat matmul(const RowMat& a, const RowMat& b, int n) {
  RowMat c(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      const double v = a[size_t(i) * n + k];
      if (v == 0.0) continue;
      for (int j = 0; j < n; ++j) c[size_t(i) * n + j] += v * b[size_t(k) * n + j];
    }
  return c;
}

void symmetric_eigen(const RowMat& a_in, int n, std::vector<double>& w, RowMat& v) {
  RowMat a = a_in;
  v.assign(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i) v[size_t(i) * n + i] = 1.0;
  auto A = [&](int i, int j) -> double& { return a[size_t(i) * n + j]; };
  auto V = [&](int i, int j) -> double& { return v[size_t(i) * n + j]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int p = 0; p < n; ++p) {
      diag += A(p, p) * A(p, p);
      for (int q = p + 1; q < n; ++q) off += A(p, q) * A(p, q);
    }
    if (off == 0.0 || off < 1e-36 * diag) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A(p, q);
        if (apq == 0.0) continue;
        const double theta = (A(q, q) - A(p, p)) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - s * akq;
          A(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * aqk;
          A(q, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V(k, p), vkq = V(k, q);
          V(k, p) = c * vkp - s * vkq;
          V(k, q) = s * vkp + c * vkq;
        }
      }
  }
  w.resize(size_t(n));
  for (int i = 0; i < n; ++i) w[size_t(i)] = A(i, i);
}

RowMat expm_host(const RowMat& arg, int n) {
  double l1 = 0.0;
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += std::fabs(arg[size_t(i) * n + j]);
    l1 = std::max(l1, s);
  }
  int sq = 0;
  if (l1 > 5.371920351148152) {
    std::frexp(l1 / 5.371920351148152, &sq);
    if (sq < 0) sq = 0;
  }
  RowMat A = arg;
  for (double& x : A) x = std::ldexp(x, -sq);
  static const double b[] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0, 1187353796428800.0,
                             129060195264000.0,   10559470521600.0,    670442572800.0,    33522128640.0,
                             1323241920.0,        40840800.0,          960960.0,          16380.0,
                             182.0,               1.0};
  RowMat A2 = matmul(A, A, n), A4 = matmul(A2, A2, n), A6 = matmul(A4, A2, n);
  const size_t nn = size_t(n) * n;
  RowMat t(nn), u(nn), vv(nn);
  for (size_t i = 0; i < nn; ++i) t[i] = b[13] * A6[i] + b[11] * A4[i] + b[9] * A2[i];
  RowMat tmp = matmul(A6, t, n);
  for (size_t i = 0; i < nn; ++i) tmp[i] += b[7] * A6[i] + b[5] * A4[i] + b[3] * A2[i];
  for (int i = 0; i < n; ++i) tmp[size_t(i) * n + i] += b[1];
  u = matmul(A, tmp, n);
  for (size_t i = 0; i < nn; ++i) t[i] = b[12] * A6[i] + b[10] * A4[i] + b[8] * A2[i];
  vv = matmul(A6, t, n);
  for (size_t i = 0; i < nn; ++i) vv[i] += b[6] * A6[i] + b[4] * A4[i] + b[2] * A2[i];
  for (int i = 0; i < n; ++i) vv[size_t(i) * n + i] += b[0];
  RowMat num(nn), den(nn);
  for (size_t i = 0; i < nn; ++i) {
    num[i] = vv[i] + u[i];
    den[i] = vv[i] - u[i];
  }
  // solve den X = num (partial pivoting)
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(den[size_t(i) * n + k]) > std::fabs(den[size_t(piv) * n + k])) piv = i;
    if (piv != k)
      for (int j = 0; j < n; ++j) {
        std::swap(den[size_t(k) * n + j], den[size_t(piv) * n + j]);
        std::swap(num[size_t(k) * n + j], num[size_t(piv) * n + j]);
      }
    for (int i = k + 1; i < n; ++i) {
      const double f = den[size_t(i) * n + k] / den[size_t(k) * n + k];
      for (int j = k; j < n; ++j) den[size_t(i) * n + j] -= f * den[size_t(k) * n + j];
      for (int j = 0; j < n; ++j) num[size_t(i) * n + j] -= f * num[size_t(k) * n + j];
    }
  }
  for (int j = 0; j < n; ++j)
    for (int i = n - 1; i >= 0; --i) {
      double s = num[size_t(i) * n + j];
      for (int k = i + 1; k < n; ++k) s -= den[size_t(i) * n + k] * num[size_t(k) * n + j];
      num[size_t(i) * n + j] = s / den[size_t(i) * n + i];
    }
  for (int i = 0; i < sq; ++i) num = matmul(num, num, n);
  return num;
}

// ----------------------------------------------------------- gamma quantile
double regularized_gamma_p(double a, double x) {
  if (x <= 0.0) return 0.0;
  const double lga = std::lgamma(a);
  if (x < a + 1.0) {
    double term = 1.0 / a, sum = term, ap = a;
    for (int k = 0; k < 1000; ++k) {
      ap += 1.0;
      term *= x / ap;
      sum += term;
      if (std::fabs(term) < std::fabs(sum) * 1e-17) break;
    }
    return sum * std::exp(-x + a * std::log(x) - lga);
  }
  const double tiny = 1e-300;
  double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
  for (int k = 1; k < 1000; ++k) {
    const double an = -k * (k - a);
    b += 2.0;
    d = an * d + b;
    if (std::fabs(d) < tiny) d = tiny;
    c = b + an / c;
    if (std::fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    const double delta = d * c;
    h *= delta;
    if (std::fabs(delta - 1.0) < 1e-17) break;
  }
  return 1.0 - std::exp(-x + a * std::log(x) - lga) * h;
}

double gamma_quantile(double shape, double rate, double p) {
  double lo = 0.0, hi = 1.0;
  while (regularized_gamma_p(shape, hi * rate) < p) hi *= 2.0;
  for (int it = 0; it < 200 && hi - lo > 0.0; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    (regularized_gamma_p(shape, mid * rate) < p ? lo : hi) = mid;
  }
  return 0.5 * (lo + hi);
}


HostTransition::HostTransition(int m_, const std::vector<double>& q_, const std::vector<double>& pi_, int reversible)
    : m(m_), q(q_) {
  bool pos = true;
  for (double p : pi_) pos = pos && p > 0;
  if (reversible && pos) {
    std::vector<double> sym(static_cast<size_t>(m) * m), sp(static_cast<size_t>(m));
    for (int i = 0; i < m; ++i) sp[size_t(i)] = std::sqrt(pi_[size_t(i)]);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j)
        sym[size_t(i) * m + j] = 0.5 * (sp[size_t(i)] * q[size_t(i) * m + j] / sp[size_t(j)] +
                                        sp[size_t(j)] * q[size_t(j) * m + i] / sp[size_t(i)]);
    RowMat V;
    symmetric_eigen(sym, m, w, V);
    U.resize(size_t(m) * m);
    Ui.resize(size_t(m) * m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        U[size_t(i) * m + j] = V[size_t(i) * m + j] / sp[size_t(i)];
        Ui[size_t(i) * m + j] = V[size_t(j) * m + i] * sp[size_t(j)];
      }
    eig = true;
  }
}

std::vector<double> HostTransition::operator()(double t) const {
  std::vector<double> p(size_t(m) * m, 0.0);
  if (t == 0.0) {
    for (int i = 0; i < m; ++i) p[size_t(i) * m + i] = 1.0;
    return p;
  }
  if (eig) {
    for (int i = 0; i < m; ++i)
      for (int k = 0; k < m; ++k) {
        const double u = U[size_t(i) * m + k] * std::exp(w[size_t(k)] * t);
        for (int j = 0; j < m; ++j) p[size_t(i) * m + j] += u * Ui[size_t(k) * m + j];
      }
  } else {
    RowMat a(q);
    for (double& x : a) x *= t;
    p = expm_host(a, m);
  }
  for (double& x : p) x = std::max(x, 0.0);
  return p;
}

}  // namespace pg
