// =============================================================================
// TEST INFRASTRUCTURE ONLY — CPU parity oracle for the phylograd-b200 engine.
//
// A std-only C++20 restatement of the reference's hot path (phylograd,
// /root/reference/proj/include/phylograd/*.hpp).  The reference itself cannot
// be compiled here: it needs Eigen 3 and Boost.Math, neither of which exists in
// this image.  Every function below cites the reference
// file:line it restates.  Parity is PINNED by re-passing the reference's own
// known-answer tests (proj/tests/*.cpp) in tests/test_oracle_kats.py.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// arm may load this library — it is the checker, never the product path.
//
// Deviations from the reference (documented in DESIGN.md):
//  * Eigen's SelfAdjointEigenSolver is replaced by cyclic Jacobi; Eigen's
//    MatrixBase::exp() by the same Higham-2005 Pade scaling-and-squaring
//    algorithm written out; boost::math::gamma_p_inv by the reference test
//    oracle testutil.hpp:63-102 (regularized gamma + bisection).
//  * Tip data enter as integer codes (state index, -1 missing, or an
//    ambiguity class) and are expanded to the reference's dense tip partials.
//  * An engine may be split into contiguous pattern blocks evaluated on
//    std::threads (SPEC.md:303 admissible parallelism) with a fixed-order
//    reduction; one block reproduces the single-threaded reference exactly.
// =============================================================================
#include <algorithm>
#include <array>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <vector>

namespace orc {

using Vec = std::vector<double>;

// ---------------------------------------------------------------- dense math
// Column-major m x n matrix (matches Eigen's default storage used by the reference).
struct Mat {
  int r = 0, c = 0;
  Vec a;
  Mat() = default;
  Mat(int rows, int cols, double fill = 0.0) : r(rows), c(cols), a(size_t(rows) * cols, fill) {}
  double& operator()(int i, int j) { return a[size_t(j) * r + i]; }
  double operator()(int i, int j) const { return a[size_t(j) * r + i]; }
  static Mat identity(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

static Mat matmul(const Mat& x, const Mat& y) {
  Mat z(x.r, y.c);
  for (int j = 0; j < y.c; ++j)
    for (int k = 0; k < x.c; ++k) {
      const double v = y(k, j);
      for (int i = 0; i < x.r; ++i) z(i, j) += x(i, k) * v;
    }
  return z;
}
static Mat add(const Mat& x, const Mat& y, double sy = 1.0) {
  Mat z = x;
  for (size_t i = 0; i < z.a.size(); ++i) z.a[i] += sy * y.a[i];
  return z;
}
static Mat scale(const Mat& x, double s) {
  Mat z = x;
  for (double& v : z.a) v *= s;
  return z;
}

// Solve A X = B by LU with partial pivoting (Eigen partialPivLu, MatrixExponential.h).
static Mat lu_solve(Mat A, Mat B) {
  const int n = A.r;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A(i, k)) > std::abs(A(piv, k))) piv = i;
    if (piv != k) {
      for (int j = 0; j < n; ++j) std::swap(A(k, j), A(piv, j));
      for (int j = 0; j < B.c; ++j) std::swap(B(k, j), B(piv, j));
    }
    const double d = A(k, k);
    for (int i = k + 1; i < n; ++i) {
      const double f = A(i, k) / d;
      A(i, k) = f;
      for (int j = k + 1; j < n; ++j) A(i, j) -= f * A(k, j);
      for (int j = 0; j < B.c; ++j) B(i, j) -= f * B(k, j);
    }
  }
  for (int j = 0; j < B.c; ++j)
    for (int i = n - 1; i >= 0; --i) {
      double s = B(i, j);
      for (int k = i + 1; k < n; ++k) s -= A(i, k) * B(k, j);
      B(i, j) = s / A(i, i);
    }
  return B;
}

// Restates substitution.hpp:71-75 (Eigen MatrixBase::exp): Higham (2005)
// Pade scaling-and-squaring with degrees 3/5/7/9/13 selected on the L1 norm.
Mat expm(const Mat& arg) {
  for (double v : arg.a)
    if (!std::isfinite(v)) throw std::invalid_argument("matrix exponential: non-finite input");
  if (arg.r != arg.c) throw std::invalid_argument("matrix exponential: square input required");
  const int n = arg.r;
  double l1 = 0.0;
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += std::abs(arg(i, j));
    l1 = std::max(l1, s);
  }
  const Mat I = Mat::identity(n);
  Mat U, V;
  int squarings = 0;
  auto pade_low = [&](const Mat& A, const double* b, int deg) {
    Mat A2 = matmul(A, A);
    Mat tmpU = scale(I, b[1]), tmpV = scale(I, b[0]);
    Mat pw = A2;
    for (int k = 2; k <= deg; k += 2) {
      tmpU = add(tmpU, pw, b[k + 1]);
      tmpV = add(tmpV, pw, b[k]);
      if (k + 2 <= deg) pw = matmul(pw, A2);
    }
    U = matmul(A, tmpU);
    V = tmpV;
  };
  static const double b3[] = {120.0, 60.0, 12.0, 1.0};
  static const double b5[] = {30240.0, 15120.0, 3360.0, 420.0, 30.0, 1.0};
  static const double b7[] = {17297280.0, 8648640.0, 1995840.0, 277200.0, 25200.0, 1512.0, 56.0, 1.0};
  static const double b9[] = {17643225600.0, 8821612800.0, 2075673600.0, 302702400.0, 30270240.0,
                              2162160.0, 110880.0, 3960.0, 90.0, 1.0};
  if (l1 < 1.495585217958292e-002) {
    pade_low(arg, b3, 2);
  } else if (l1 < 2.539398330063230e-001) {
    pade_low(arg, b5, 4);
  } else if (l1 < 9.504178996162932e-001) {
    pade_low(arg, b7, 6);
  } else if (l1 < 2.097847961257068e+000) {
    pade_low(arg, b9, 8);
  } else {
    const double maxnorm = 5.371920351148152;
    std::frexp(l1 / maxnorm, &squarings);
    if (squarings < 0) squarings = 0;
    Mat A = arg;
    for (double& v : A.a) v = std::ldexp(v, -squarings);
    static const double b[] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                               1187353796428800.0,  129060195264000.0,   10559470521600.0,
                               670442572800.0,      33522128640.0,       1323241920.0,
                               40840800.0,          960960.0,            16380.0,
                               182.0,               1.0};
    Mat A2 = matmul(A, A), A4 = matmul(A2, A2), A6 = matmul(A4, A2);
    Mat t = add(add(scale(A6, b[13]), A4, b[11]), A2, b[9]);
    Mat tmp = matmul(A6, t);
    tmp = add(add(add(add(tmp, A6, b[7]), A4, b[5]), A2, b[3]), I, b[1]);
    U = matmul(A, tmp);
    t = add(add(scale(A6, b[12]), A4, b[10]), A2, b[8]);
    V = matmul(A6, t);
    V = add(add(add(add(V, A6, b[6]), A4, b[4]), A2, b[2]), I, b[0]);
  }
  Mat numer = add(U, V), denom = add(V, U, -1.0);
  Mat R = lu_solve(denom, numer);
  for (int i = 0; i < squarings; ++i) R = matmul(R, R);
  return R;
}

// Cyclic Jacobi eigensolver for a symmetric matrix (replaces Eigen's
// SelfAdjointEigenSolver used at substitution.hpp:202).  Returns eigenvalues
// and column eigenvectors (orthonormal).
static void jacobi_eigen(Mat S, Vec& values, Mat& vectors) {
  const int n = S.r;
  vectors = Mat::identity(n);
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += S(p, q) * S(p, q);
    if (off == 0.0) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = S(p, q);
        if (apq == 0.0) continue;
        const double app = S(p, p), aqq = S(q, q);
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double skp = S(k, p), skq = S(k, q);
          S(k, p) = c * skp - s * skq;
          S(k, q) = s * skp + c * skq;
        }
        for (int k = 0; k < n; ++k) {
          const double spk = S(p, k), sqk = S(q, k);
          S(p, k) = c * spk - s * sqk;
          S(q, k) = s * spk + c * sqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = vectors(k, p), vkq = vectors(k, q);
          vectors(k, p) = c * vkp - s * vkq;
          vectors(k, q) = s * vkp + c * vkq;
        }
      }
  }
  values.assign(n, 0.0);
  for (int i = 0; i < n; ++i) values[i] = S(i, i);
}

// ------------------------------------------------------------ rate categories
// testutil.hpp:63-92 restated: regularized lower incomplete gamma P(a, x).
double regularized_gamma_p(double a, double x) {
  if (x <= 0.0) return 0.0;
  const double lga = std::lgamma(a);
  if (x < a + 1.0) {
    double term = 1.0 / a, sum = term, ap = a;
    for (int k = 0; k < 500; ++k) {
      ap += 1.0;
      term *= x / ap;
      sum += term;
      if (std::abs(term) < std::abs(sum) * 1e-16) break;
    }
    return sum * std::exp(-x + a * std::log(x) - lga);
  }
  const double tiny = 1e-300;
  double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
  for (int k = 1; k < 500; ++k) {
    const double an = -k * (k - a);
    b += 2.0;
    d = an * d + b;
    if (std::abs(d) < tiny) d = tiny;
    c = b + an / c;
    if (std::abs(c) < tiny) c = tiny;
    d = 1.0 / d;
    const double delta = d * c;
    h *= delta;
    if (std::abs(delta - 1.0) < 1e-16) break;
  }
  return 1.0 - std::exp(-x + a * std::log(x) - lga) * h;
}

// testutil.hpp:94-102 restated (the reference tests pin gamma_p_inv to this at 1e-9).
double gamma_quantile(double shape, double rate, double p) {
  double lo = 0.0, hi = 1.0;
  while (regularized_gamma_p(shape, hi * rate) < p) hi *= 2.0;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    (regularized_gamma_p(shape, mid * rate) < p ? lo : hi) = mid;
  }
  return 0.5 * (lo + hi);
}

struct Categories {
  Vec rates, probs;
  int count() const { return int(rates.size()); }
};

// substitution.hpp:36-50 (RateCategories::make checks)
Categories make_categories(Vec rates, Vec probs) {
  if (rates.empty() || rates.size() != probs.size())
    throw std::invalid_argument("rate categories: need L >= 1 matched rates/probs");
  double ps = 0, mean = 0;
  for (size_t l = 0; l < rates.size(); ++l) {
    if (rates[l] <= 0.0) throw std::invalid_argument("rate categories: rates must be positive");
    ps += probs[l];
    mean += rates[l] * probs[l];
  }
  if (std::abs(ps - 1.0) > 1e-12) throw std::invalid_argument("rate categories: probabilities must sum to 1");
  if (std::abs(mean - 1.0) > 1e-10) throw std::invalid_argument("rate categories: mixture mean must be 1");
  return {std::move(rates), std::move(probs)};
}

// substitution.hpp:55-68: L equiprobable categories at gamma bin medians, mean one.
Categories discrete_gamma(double alpha, int count) {
  if (!(alpha > 0.0) || !std::isfinite(alpha))
    throw std::invalid_argument("discrete gamma: alpha must be positive and finite");
  if (count < 1) throw std::invalid_argument("discrete gamma: need at least one category");
  if (count == 1) return {{1.0}, {1.0}};
  Vec rates(count);
  double sum = 0.0;
  for (int l = 0; l < count; ++l) {
    const double p = (2.0 * l + 1.0) / (2.0 * count);
    // gamma_p_inv(alpha, p) / alpha == quantile of Gamma(shape alpha, rate alpha)
    rates[l] = gamma_quantile(alpha, 1.0, p) / alpha;
    sum += rates[l];
  }
  for (double& r : rates) r *= double(count) / sum;
  return make_categories(rates, Vec(count, 1.0 / count));
}

// ------------------------------------------------------------------- model
struct Model {
  int m = 0;
  Mat q;
  Vec pi;
  bool reversible = false;
  std::unordered_map<int, Mat> branch_q;
  bool have_eigen = false;
  Vec eig_values;
  Mat eig_u, eig_uinv;

  const Mat& generator(int branch) const {
    auto it = branch_q.find(branch);
    return it == branch_q.end() ? q : it->second;
  }
  bool homogeneous() const { return branch_q.empty(); }

  // substitution.hpp:168-180
  static void check_generator(const Mat& g) {
    for (double v : g.a)
      if (!std::isfinite(v)) throw std::invalid_argument("generator: non-finite entries");
    for (int i = 0; i < g.r; ++i) {
      double row = 0.0;
      for (int j = 0; j < g.c; ++j) {
        if (i != j && g(i, j) < 0.0) throw std::invalid_argument("generator: negative off-diagonal entry");
        row += g(i, j);
      }
      if (std::abs(row) > 1e-12) throw std::invalid_argument("generator: rows must sum to zero");
    }
  }

  // substitution.hpp:81-93 (raw constructor)
  Model(Mat qq, Vec p, bool rev) : m(qq.r), q(std::move(qq)), pi(std::move(p)), reversible(rev) {
    check_generator(q);
    if (int(pi.size()) != m) throw std::invalid_argument("model: pi length must match state count");
    double s = 0;
    for (double v : pi) {
      if (v < -1e-12) throw std::invalid_argument("model: pi must be a probability vector");
      s += v;
    }
    if (std::abs(s - 1.0) > 1e-12) throw std::invalid_argument("model: pi must be a probability vector");
    if (reversible) build_eigen_cache();
  }

  // substitution.hpp:196-208
  void build_eigen_cache() {
    for (double v : pi)
      if (v <= 0.0) return;
    Vec sp(m);
    for (int i = 0; i < m; ++i) sp[i] = std::sqrt(pi[i]);
    Mat sym(m, m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) sym(i, j) = sp[i] * q(i, j) / sp[j];
    Mat s2 = sym;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) s2(i, j) = 0.5 * (sym(i, j) + sym(j, i));
    Mat vecs;
    jacobi_eigen(s2, eig_values, vecs);
    eig_u = Mat(m, m);
    eig_uinv = Mat(m, m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        eig_u(i, j) = vecs(i, j) / sp[i];
        eig_uinv(i, j) = vecs(j, i) * sp[j];
      }
    have_eigen = true;
  }

  // substitution.hpp:138-143
  void set_branch_generator(int branch, Mat g) {
    if (g.r != m || g.c != m) throw std::invalid_argument("branch generator: wrong dimensions");
    check_generator(g);
    branch_q[branch] = std::move(g);
  }

  // substitution.hpp:147-160
  Mat transition_matrix(int branch, double b, double c = 1.0) const {
    if (b < 0.0) throw std::invalid_argument("transition matrix: negative branch length");
    if (!(c > 0.0)) throw std::invalid_argument("transition matrix: category rate must be positive");
    const double t = b * c;
    if (t == 0.0) return Mat::identity(m);
    Mat p;
    if (have_eigen && branch_q.find(branch) == branch_q.end()) {
      Mat ud(m, m);
      for (int j = 0; j < m; ++j) {
        const double e = std::exp(eig_values[j] * t);
        for (int i = 0; i < m; ++i) ud(i, j) = eig_u(i, j) * e;
      }
      p = matmul(ud, eig_uinv);
    } else {
      p = expm(scale(generator(branch), t));
    }
    for (double& v : p.a) v = std::max(v, 0.0);
    return p;
  }
};

// substitution.hpp:183-191
void finish_generator(Mat& q, const Vec& pi) {
  for (int i = 0; i < q.r; ++i) {
    q(i, i) = 0.0;
    double s = 0.0;
    for (int j = 0; j < q.c; ++j) s += q(i, j);
    q(i, i) = -s;
  }
  double rate = 0.0;
  for (int i = 0; i < q.r; ++i) rate -= pi[i] * q(i, i);
  for (double& v : q.a) v /= rate;
}

// substitution.hpp:109-124
Model gtr(const double* exch, const double* freqs) {
  for (int e = 0; e < 6; ++e)
    if (exch[e] <= 0.0) throw std::invalid_argument("gtr: exchangeabilities must be positive");
  double s = 0;
  for (int j = 0; j < 4; ++j) {
    if (freqs[j] <= 0.0) throw std::invalid_argument("frequencies must be positive and sum to 1");
    s += freqs[j];
  }
  if (std::abs(s - 1.0) > 1e-12) throw std::invalid_argument("frequencies must be positive and sum to 1");
  Mat q(4, 4);
  int e = 0;
  for (int i = 0; i < 4; ++i)
    for (int j = i + 1; j < 4; ++j, ++e) {
      q(i, j) = exch[e] * freqs[j];
      q(j, i) = exch[e] * freqs[i];
    }
  Vec pi(freqs, freqs + 4);
  finish_generator(q, pi);
  return Model(q, pi, true);
}

// --------------------------------------------------------------------- tree
struct NewickError : std::runtime_error {
  NewickError(const std::string& what, size_t pos)
      : std::runtime_error(what + " (at position " + std::to_string(pos) + ")"), position(pos) {}
  size_t position;
};

struct Tree {
  int tip_count = 0;
  std::vector<std::string> labels;
  std::vector<int> parent;
  std::vector<std::array<int, 2>> children;
  Vec branch_length, node_time;
  std::vector<int> post_order, pre_order;
  int node_count() const { return 2 * tip_count - 1; }
  int root() const { return node_count(); }
  int branch_count() const { return node_count() - 1; }
  bool is_tip(int n) const { return n >= 1 && n <= tip_count; }
  int sibling(int n) const {
    const int p = parent[n];
    return children[p][0] == n ? children[p][1] : children[p][0];
  }
};

// tree.hpp:60-77
void rebuild_traversals(Tree& t) {
  t.post_order.clear();
  std::vector<std::pair<int, bool>> stack{{t.root(), false}};
  while (!stack.empty()) {
    auto [node, expanded] = stack.back();
    stack.pop_back();
    if (expanded || t.is_tip(node)) {
      t.post_order.push_back(node);
    } else {
      stack.push_back({node, true});
      stack.push_back({t.children[node][1], false});
      stack.push_back({t.children[node][0], false});
    }
  }
  t.pre_order.assign(t.post_order.rbegin(), t.post_order.rend());
}

// tree.hpp:81-126
void validate_tree(const Tree& t) {
  if (t.tip_count < 2) throw std::invalid_argument("tree needs at least 2 tips");
  const int n = t.node_count();
  auto sized = [&](size_t s) { return s == size_t(n) + 1; };
  if (!sized(t.parent.size()) || !sized(t.children.size()) || !sized(t.labels.size()) ||
      !sized(t.branch_length.size()))
    throw std::invalid_argument("tree vectors not sized node_count()+1");
  if (t.parent[t.root()] != 0) throw std::invalid_argument("root must have no parent");
  for (int i = 1; i < n; ++i) {
    const int p = t.parent[i];
    if (p <= t.tip_count || p > n) throw std::invalid_argument("node " + std::to_string(i) + " has invalid parent");
    if (t.children[p][0] != i && t.children[p][1] != i)
      throw std::invalid_argument("parent/children maps inconsistent at node " + std::to_string(i));
    if (t.branch_length[i] < 0.0) throw std::invalid_argument("negative branch length at node " + std::to_string(i));
  }
  for (int i = t.tip_count + 1; i <= n; ++i)
    for (int c : t.children[i])
      if (c < 1 || c >= n || t.parent[c] != i)
        throw std::invalid_argument("bad child link at internal node " + std::to_string(i));
  for (int i = 1; i < n; ++i) {
    int hops = 0, node = i;
    while (node != t.root() && hops++ <= n) node = t.parent[node];
    if (hops > n) throw std::invalid_argument("parent links contain a cycle");
  }
  if (!t.node_time.empty()) {
    if (!sized(t.node_time.size())) throw std::invalid_argument("node_time not sized node_count()+1");
    for (int i = 1; i < n; ++i)
      if (!(t.node_time[i] > t.node_time[t.parent[i]]))
        throw std::invalid_argument("node_time must strictly increase from parent to child");
  }
  if (t.post_order.size() != size_t(n)) throw std::invalid_argument("post_order incomplete");
  std::vector<int> pos(n + 1, -1);
  for (int i = 0; i < n; ++i) pos[t.post_order[i]] = i;
  for (int i = 1; i < n; ++i)
    if (pos[i] < 0 || pos[i] >= pos[t.parent[i]])
      throw std::invalid_argument("post_order does not visit children before parents");
}

// tree.hpp:131-140
void assign_times_from_branch_lengths(Tree& t) {
  t.node_time.assign(t.node_count() + 1, 0.0);
  for (int node : t.pre_order) {
    if (node == t.root()) continue;
    if (t.branch_length[node] <= 0.0) throw std::invalid_argument("durations must be positive to assign node times");
    t.node_time[node] = t.node_time[t.parent[node]] + t.branch_length[node];
  }
}

// tree.hpp:144-282 (NewickParser)
struct NewickParser {
  std::string_view text;
  size_t pos = 0;
  struct Proto {
    std::string label;
    double length = 0.0;
    int left = -1, right = -1;
  };
  std::vector<Proto> proto;
  std::vector<int> tip_order, internal_order;

  [[noreturn]] void fail(const std::string& what) const { throw NewickError(what, pos); }
  void skip_ws() {
    while (pos < text.size() && std::isspace((unsigned char)text[pos])) ++pos;
  }
  char peek() {
    skip_ws();
    if (pos >= text.size()) fail("unexpected end of input");
    return text[pos];
  }
  void expect(char c) {
    if (peek() != c) fail(std::string("expected '") + c + "'");
    ++pos;
  }
  std::string parse_label() {
    skip_ws();
    const size_t start = pos;
    while (pos < text.size()) {
      const char c = text[pos];
      if (c == '(' || c == ')' || c == ',' || c == ':' || c == ';' || std::isspace((unsigned char)c)) break;
      ++pos;
    }
    return std::string(text.substr(start, pos - start));
  }
  double parse_length() {
    skip_ws();
    // std::from_chars(double) semantics: no leading '+', no whitespace.
    const char* b = text.data() + pos;
    const char* e = text.data() + text.size();
    double v = 0.0;
    auto [ptr, ec] = std::from_chars(b, e, v);
    if (ec != std::errc()) fail("expected a branch length");
    pos = size_t(ptr - text.data());
    if (v < 0.0) fail("negative branch length");
    return v;
  }
  int parse_subtree() {
    if (peek() == '(') {
      ++pos;
      std::vector<int> kids{parse_subtree()};
      while (peek() == ',') {
        ++pos;
        kids.push_back(parse_subtree());
      }
      expect(')');
      if (kids.size() == 1) fail("unifurcation: internal node with one child");
      if (kids.size() > 2) fail("polytomy: internal node with more than two children");
      const int idx = int(proto.size());
      proto.push_back({});
      proto[idx].left = kids[0];
      proto[idx].right = kids[1];
      skip_ws();
      if (pos < text.size() && text[pos] != ':' && text[pos] != ',' && text[pos] != ')' && text[pos] != ';')
        proto[idx].label = parse_label();
      skip_ws();
      if (pos < text.size() && text[pos] == ':') {
        ++pos;
        proto[idx].length = parse_length();
      }
      internal_order.push_back(idx);
      return idx;
    }
    std::string label = parse_label();
    if (label.empty()) fail("expected a tip label");
    const int idx = int(proto.size());
    proto.push_back({});
    proto[idx].label = std::move(label);
    skip_ws();
    if (pos < text.size() && text[pos] == ':') {
      ++pos;
      proto[idx].length = parse_length();
    }
    tip_order.push_back(idx);
    return idx;
  }
  Tree run() {
    const int root_idx = parse_subtree();
    expect(';');
    skip_ws();
    if (pos != text.size()) fail("trailing characters after ';'");
    if (proto[root_idx].left < 0) fail("a tree must have at least two tips");
    const int nt = int(tip_order.size());
    Tree t;
    t.tip_count = nt;
    const int n = t.node_count();
    t.labels.assign(n + 1, {});
    t.parent.assign(n + 1, 0);
    t.children.assign(n + 1, {0, 0});
    t.branch_length.assign(n + 1, 0.0);
    std::vector<int> id(proto.size(), 0);
    for (int k = 0; k < nt; ++k) id[tip_order[k]] = k + 1;
    for (size_t k = 0; k < internal_order.size(); ++k) id[internal_order[k]] = nt + 1 + int(k);
    for (size_t p = 0; p < proto.size(); ++p) {
      const int i = id[p];
      t.labels[i] = proto[p].label;
      t.branch_length[i] = proto[p].length;
      if (proto[p].left >= 0) {
        const int l = id[proto[p].left], r = id[proto[p].right];
        t.children[i] = {l, r};
        t.parent[l] = i;
        t.parent[r] = i;
      }
    }
    t.labels[t.root()].clear();
    t.branch_length[t.root()] = 0.0;
    for (int a = 1; a <= nt; ++a)
      for (int b = a + 1; b <= nt; ++b)
        if (t.labels[a] == t.labels[b]) throw NewickError("duplicate tip label '" + t.labels[a] + "'", 0);
    rebuild_traversals(t);
    return t;
  }
};

Tree parse_newick(std::string_view text) {
  NewickParser p{text, 0, {}, {}, {}};
  return p.run();
}

// tree.hpp:292-323
static void write_subtree(const Tree& t, int node, std::string& out) {
  if (t.is_tip(node)) {
    out += t.labels[node];
  } else {
    out += '(';
    write_subtree(t, t.children[node][0], out);
    out += ',';
    write_subtree(t, t.children[node][1], out);
    out += ')';
  }
  if (node != t.root()) {
    char buf[32];
    const int len = std::snprintf(buf, sizeof buf, "%.12g", t.branch_length[node]);
    out += ':';
    out.append(buf, size_t(len));
  }
}
std::string serialize_newick(const Tree& t) {
  std::string out;
  write_subtree(t, t.root(), out);
  out += ';';
  return out;
}

// validation.hpp:153-193
Tree random_coalescent_tree(int tips, std::mt19937_64& rng, double height_scale = 0.5) {
  if (tips < 2) throw std::invalid_argument("coalescent tree: need >= 2 tips");
  const int n = 2 * tips - 1;
  Tree t;
  t.tip_count = tips;
  t.labels.assign(n + 1, {});
  t.parent.assign(n + 1, 0);
  t.children.assign(n + 1, {0, 0});
  t.branch_length.assign(n + 1, 0.0);
  for (int k = 1; k <= tips; ++k) t.labels[k] = "t" + std::to_string(k);
  std::vector<int> active(tips);
  Vec height(n + 1, 0.0);
  for (int k = 0; k < tips; ++k) active[k] = k + 1;
  double clock = 0.0;
  std::exponential_distribution<double> exp_dist;
  for (int next = tips + 1; next <= n; ++next) {
    const int k = int(active.size());
    clock += exp_dist(rng) / (k * (k - 1) / 2.0);
    std::uniform_int_distribution<int> pick(0, k - 1);
    int a = pick(rng);
    int b = pick(rng);
    while (b == a) b = pick(rng);
    const int left = active[a], right = active[b];
    if (a > b) std::swap(a, b);
    active.erase(active.begin() + b);
    active.erase(active.begin() + a);
    active.push_back(next);
    height[next] = clock;
    t.children[next] = {left, right};
    t.parent[left] = t.parent[right] = next;
  }
  const double sc = height_scale / height[n];
  t.node_time.assign(n + 1, 0.0);
  for (int i = 1; i <= n; ++i) t.node_time[i] = (height[n] - height[i]) * sc;
  for (int i = 1; i < n; ++i) t.branch_length[i] = t.node_time[i] - t.node_time[t.parent[i]];
  rebuild_traversals(t);
  validate_tree(t);
  return t;
}

// testutil.hpp:20-27
Tree random_tree(int tips, std::mt19937_64& rng, double lo, double hi) {
  Tree t = random_coalescent_tree(tips, rng);
  t.node_time.clear();
  std::uniform_real_distribution<double> unif(lo, hi);
  for (int i = 1; i <= t.branch_count(); ++i) t.branch_length[i] = unif(rng);
  return t;
}

// testutil.hpp:31-48
std::vector<int> random_post_order(const Tree& t, std::mt19937_64& rng) {
  const int n = t.node_count();
  std::vector<int> pending(n + 1, 0), ready, order;
  for (int i = t.tip_count + 1; i <= n; ++i) pending[i] = 2;
  for (int i = 1; i <= t.tip_count; ++i) ready.push_back(i);
  while (!ready.empty()) {
    std::uniform_int_distribution<size_t> pick(0, ready.size() - 1);
    const size_t at = pick(rng);
    const int node = ready[at];
    ready.erase(ready.begin() + long(at));
    order.push_back(node);
    const int p = t.parent[node];
    if (p != 0 && --pending[p] == 0) ready.push_back(p);
  }
  return order;
}

// validation.hpp:196-202
Tree caterpillar_tree(int tips, double branch) {
  auto num = [](double v) { return std::to_string(v); };
  std::string nw = "(t1:" + num(branch) + ",t2:" + num(branch) + ")";
  for (int k = 3; k <= tips; ++k) nw = "(" + nw + ":" + num(branch) + ",t" + std::to_string(k) + ":" + num(branch) + ")";
  return parse_newick(nw + ";");
}

// --------------------------------------------------------------- alignment
// alignment.hpp:34-53
int nucleotide_mask(char c) {
  switch (c) {
    case 'A': return 1;
    case 'C': return 2;
    case 'G': return 4;
    case 'T': return 8;
    case 'R': return 1 | 4;
    case 'Y': return 2 | 8;
    case 'S': return 2 | 4;
    case 'W': return 1 | 8;
    case 'K': return 4 | 8;
    case 'M': return 1 | 2;
    case 'B': return 2 | 4 | 8;
    case 'D': return 1 | 4 | 8;
    case 'H': return 1 | 2 | 8;
    case 'V': return 1 | 2 | 4;
    case 'N': case '-': case '?': return 15;
    default: return 0;
  }
}

struct Alignment {
  int m = 4;
  std::vector<std::string> taxa;
  std::vector<long> weights;
  long site_count = 0;
  std::vector<Mat> tip_partials;               // per taxon: m x P
  std::vector<std::string> columns;            // compress() only
  std::vector<std::vector<int>> unique_columns; // from_codes() only
  int pattern_count() const { return int(weights.size()); }
  int taxon_index(const std::string& name) const {
    for (size_t i = 0; i < taxa.size(); ++i)
      if (taxa[i] == name) return int(i);
    return -1;
  }
};

// alignment.hpp:55-72 + :77-100 (FASTA reader; record checks)
void parse_fasta(std::string_view text, std::vector<std::string>& taxa, std::vector<std::string>& seqs) {
  std::string line;
  size_t i = 0;
  while (i <= text.size()) {
    size_t j = text.find('\n', i);
    if (j == std::string_view::npos) j = text.size();
    line.assign(text.substr(i, j - i));
    i = j + 1;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty() || line[0] == ';') {
      if (j == text.size()) break;
      continue;
    }
    if (line[0] == '>') {
      std::string name = line.substr(1);
      const size_t first = name.find_first_not_of(" \t");
      name = first == std::string::npos ? std::string() : name.substr(first);
      const size_t cut = name.find_first_of(" \t");
      if (cut != std::string::npos) name.resize(cut);
      if (name.empty()) throw std::invalid_argument("fasta: empty record name");
      taxa.push_back(name);
      seqs.emplace_back();
    } else {
      if (taxa.empty()) throw std::invalid_argument("fasta: sequence before first header");
      for (char c : line)
        if (!std::isspace((unsigned char)c)) seqs.back() += c;
    }
    if (j == text.size()) break;
  }
  if (taxa.empty()) throw std::invalid_argument("alignment: no records");
  for (size_t r = 0; r < taxa.size(); ++r) {
    for (size_t o = 0; o < r; ++o)
      if (taxa[o] == taxa[r]) throw std::invalid_argument("alignment: duplicate taxon name '" + taxa[r] + "'");
    if (seqs[r].size() != seqs[0].size()) throw std::invalid_argument("alignment: ragged record '" + taxa[r] + "'");
    for (char& c : seqs[r]) {
      c = char(std::toupper((unsigned char)c));
      if (nucleotide_mask(c) == 0)
        throw std::invalid_argument(std::string("alignment: unknown character '") + c + "' in record '" + taxa[r] + "'");
    }
  }
  if (seqs[0].empty()) throw std::invalid_argument("alignment: zero-length sequences");
}

// alignment.hpp:153-182
Alignment compress(const std::vector<std::string>& taxa, const std::vector<std::string>& seqs) {
  Alignment out;
  out.m = 4;
  out.taxa = taxa;
  out.site_count = long(seqs[0].size());
  const int nt = int(taxa.size());
  std::map<std::string, int> seen;
  for (long s = 0; s < out.site_count; ++s) {
    std::string col(size_t(nt), ' ');
    for (int r = 0; r < nt; ++r) col[size_t(r)] = seqs[size_t(r)][size_t(s)];
    auto [it, inserted] = seen.emplace(col, out.pattern_count());
    if (inserted) {
      out.columns.push_back(col);
      out.weights.push_back(1);
    } else {
      ++out.weights[size_t(it->second)];
    }
  }
  out.tip_partials.assign(size_t(nt), Mat(4, out.pattern_count()));
  for (int r = 0; r < nt; ++r)
    for (int p = 0; p < out.pattern_count(); ++p) {
      const int mask = nucleotide_mask(out.columns[size_t(p)][size_t(r)]);
      for (int j = 0; j < 4; ++j) out.tip_partials[size_t(r)](j, p) = (mask >> j) & 1 ? 1.0 : 0.0;
    }
  return out;
}

// alignment.hpp:186-229
Alignment from_codes(std::vector<std::string> taxa, const std::vector<std::vector<int>>& codes, int m) {
  if (m < 2) throw std::invalid_argument("alignment: state count must be >= 2");
  if (codes.size() != taxa.size()) throw std::invalid_argument("alignment: taxa/codes mismatch");
  Alignment out;
  out.m = m;
  out.taxa = std::move(taxa);
  const int nt = int(out.taxa.size());
  if (nt == 0) throw std::invalid_argument("alignment: no records");
  out.site_count = long(codes[0].size());
  std::map<std::vector<int>, int> seen;
  for (long s = 0; s < out.site_count; ++s) {
    std::vector<int> col(static_cast<size_t>(nt));
    for (int r = 0; r < nt; ++r) {
      if (codes[size_t(r)].size() != size_t(out.site_count)) throw std::invalid_argument("alignment: ragged code rows");
      const int c = codes[size_t(r)][size_t(s)];
      if (c < -1 || c >= m) throw std::invalid_argument("alignment: state code out of range");
      col[size_t(r)] = c;
    }
    auto [it, inserted] = seen.emplace(col, int(out.unique_columns.size()));
    if (inserted) {
      out.unique_columns.push_back(col);
      out.weights.push_back(1);
    } else {
      ++out.weights[size_t(it->second)];
    }
  }
  out.tip_partials.assign(size_t(nt), Mat(m, out.pattern_count()));
  for (int r = 0; r < nt; ++r)
    for (int p = 0; p < out.pattern_count(); ++p) {
      const int c = out.unique_columns[size_t(p)][size_t(r)];
      if (c < 0)
        for (int j = 0; j < m; ++j) out.tip_partials[size_t(r)](j, p) = 1.0;
      else
        out.tip_partials[size_t(r)](c, p) = 1.0;
    }
  return out;
}

// alignment.hpp:243-286 (draw order: per site, category first, then pre_order)
std::vector<std::vector<int>> simulate_states(const Tree& t, const Model& model, const Categories& cats,
                                              const Vec& blen, long sites, uint64_t seed) {
  if (sites < 1) throw std::invalid_argument("simulate: site_count must be >= 1");
  if (int(blen.size()) != t.branch_count()) throw std::invalid_argument("simulate: need one branch length per non-root node");
  const int L = cats.count();
  std::vector<std::vector<Mat>> trans(size_t(t.node_count() + 1));
  for (int i = 1; i <= t.branch_count(); ++i)
    for (int l = 0; l < L; ++l) trans[size_t(i)].push_back(model.transition_matrix(i, blen[size_t(i - 1)], cats.rates[size_t(l)]));
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  auto draw = [&](auto&& weight, int count) {
    const double u = unif(rng);
    double acc = 0.0;
    const int last = count - 1;
    for (int j = 0; j < last; ++j) {
      acc += weight(j);
      if (u < acc) return j;
    }
    return last;
  };
  std::vector<std::vector<int>> tips(size_t(t.tip_count), std::vector<int>(size_t(sites)));
  std::vector<int> state(size_t(t.node_count() + 1));
  for (long s = 0; s < sites; ++s) {
    const int l = draw([&](int j) { return cats.probs[size_t(j)]; }, L);
    for (int node : t.pre_order) {
      if (node == t.root())
        state[size_t(node)] = draw([&](int j) { return model.pi[size_t(j)]; }, model.m);
      else {
        const Mat& P = trans[size_t(node)][size_t(l)];
        const int from = state[size_t(t.parent[size_t(node)])];
        state[size_t(node)] = draw([&](int j) { return P(from, j); }, model.m);
      }
      if (t.is_tip(node)) tips[size_t(node - 1)][size_t(s)] = state[size_t(node)];
    }
  }
  return tips;
}

// ------------------------------------------------------------------ engine
struct EngineOptions {
  double threshold = 1e-150;
  bool force = false, disable = false;
};

// engine.hpp:47-438, restated over column-major m x P buffers (Mat) for one
// contiguous pattern block [p0, p0+P).
class Engine {
 public:
  Engine(const Tree& tree, const Alignment& aln, const Model& model, Categories cats, EngineOptions opt,
         int p0 = 0, int np = -1)
      : tree_(tree), model_(model), cats_(std::move(cats)), opt_(opt) {
    const int m = model_.m;
    if (aln.m != m) throw std::invalid_argument("engine: alignment/model state counts differ");
    if (int(aln.taxa.size()) != tree_.tip_count)
      throw std::invalid_argument("engine: alignment must carry exactly one record per tree tip");
    if (np < 0) np = aln.pattern_count() - p0;
    P_ = np;
    tip_partials_.resize(size_t(tree_.tip_count + 1));
    tip_codes_.resize(size_t(tree_.tip_count + 1));
    for (int t = 1; t <= tree_.tip_count; ++t) {
      const int row = aln.taxon_index(tree_.labels[size_t(t)]);
      if (row < 0) throw std::invalid_argument("engine: tree tip '" + tree_.labels[size_t(t)] + "' not found in alignment");
      Mat& tp = tip_partials_[size_t(t)];
      tp = Mat(m, P_);
      const Mat& src = aln.tip_partials[size_t(row)];
      for (int s = 0; s < P_; ++s)
        for (int j = 0; j < m; ++j) tp(j, s) = src(j, p0 + s);
      // engine.hpp:72-79: unit-indicator columns admit a gather
      tip_codes_[size_t(t)].assign(size_t(P_), -1);
      for (int s = 0; s < P_; ++s) {
        double sum = 0.0, mx = -INFINITY;
        int idx = -1;
        for (int j = 0; j < m; ++j) {
          sum += tp(j, s);
          if (tp(j, s) > mx) {
            mx = tp(j, s);
            idx = j;
          }
        }
        if (sum == 1.0 && mx == 1.0) tip_codes_[size_t(t)][size_t(s)] = idx;
      }
    }
    const int nodes = tree_.node_count(), L = cats_.count();
    auto grid = [&] { return std::vector<std::vector<Mat>>(size_t(nodes + 1), std::vector<Mat>(size_t(L))); };
    post_ = grid();
    pre_ = grid();
    edge_ = grid();
    trans_ = grid();
    for (int node = 1; node <= nodes; ++node)
      for (int l = 0; l < L; ++l) {
        if (!tree_.is_tip(node)) post_[size_t(node)][size_t(l)] = Mat(m, P_);
        pre_[size_t(node)][size_t(l)] = Mat(m, P_);
        if (node != tree_.root()) edge_[size_t(node)][size_t(l)] = Mat(m, P_);
      }
    scaler_post_.assign(size_t(nodes + 1), Vec(size_t(P_), 0.0));
    scaler_pre_.assign(size_t(nodes + 1), Vec(size_t(P_), 0.0));
    site_ll_.assign(size_t(P_), 0.0);
    weights_.resize(size_t(P_));
    for (int s = 0; s < P_; ++s) weights_[size_t(s)] = double(aln.weights[size_t(p0 + s)]);
    blen_.resize(size_t(tree_.branch_count()));
    for (int i = 1; i <= tree_.branch_count(); ++i) blen_[size_t(i - 1)] = tree_.branch_length[size_t(i)];
  }

  int patterns() const { return P_; }
  const Vec& branch_lengths() const { return blen_; }

  // engine.hpp:116-124
  void set_branch_lengths(const Vec& b) {
    if (b.size() != blen_.size()) throw std::invalid_argument("engine: branch length vector has wrong size");
    bool same = true;
    for (size_t i = 0; i < b.size(); ++i) {
      if (!std::isfinite(b[i]) || b[i] < 0.0) throw std::invalid_argument("engine: branch lengths must be finite and nonnegative");
      if (b[i] != blen_[i]) same = false;
    }
    if (same) return;
    blen_ = b;
    post_valid_ = pre_valid_ = hess_valid_ = ll_valid_ = false;
  }
  uint64_t node_visits() const { return visits_; }
  void reset_node_visits() { visits_ = 0; }
  void invalidate() { post_valid_ = pre_valid_ = hess_valid_ = ll_valid_ = false; }

  const Mat& post_partial(int node, int l) const { return post_matrix(node, l); }
  const Mat& pre_partial(int node, int l) const { return pre_[size_t(node)][size_t(l)]; }
  const Vec& post_scaler(int node) const { return scaler_post_[size_t(node)]; }
  const Vec& pre_scaler(int node) const { return scaler_pre_[size_t(node)]; }
  const Vec& site_ll() const { return site_ll_; }

  // engine.hpp:146-149
  double log_likelihood() {
    if (!ll_valid_) scratch_pass();
    return ll_;
  }
  // engine.hpp:151-162
  void branch_gradient(bool hess, double& ll, Vec& g, Vec& h) {
    post_order_pass();
    if (!pre_valid_ || (hess && !hess_valid_)) pre_order_pass(hess);
    ll = ll_;
    g = grad_;
    if (hess) h = hessd_;
  }

  // engine.hpp:168-180
  double log_likelihood_at_node(int node) {
    post_order_pass();
    if (!pre_valid_) pre_order_pass(false);
    const int m = model_.m;
    double total = 0.0;
    for (int s = 0; s < P_; ++s) {
      double mix = 0.0;
      for (int l = 0; l < cats_.count(); ++l) {
        const Mat& a = post_matrix(node, l);
        const Mat& b = pre_[size_t(node)][size_t(l)];
        double dot = 0.0;
        for (int j = 0; j < m; ++j) dot += a(j, s) * b(j, s);
        mix += cats_.probs[size_t(l)] * dot;
      }
      total += weights_[size_t(s)] * (std::log(mix) + scaler_post_[size_t(node)][size_t(s)] + scaler_pre_[size_t(node)][size_t(s)]);
    }
    return total;
  }

  // engine.hpp:182-221
  void post_order_pass() {
    if (post_valid_) return;
    const int L = cats_.count(), m = model_.m;
    for (int node : tree_.post_order) {
      ++visits_;
      if (!tree_.is_tip(node)) {
        const int c0 = tree_.children[size_t(node)][0], c1 = tree_.children[size_t(node)][1];
        for (int l = 0; l < L; ++l) {
          Mat& d = post_[size_t(node)][size_t(l)];
          const Mat& x = edge_[size_t(c0)][size_t(l)];
          const Mat& y = edge_[size_t(c1)][size_t(l)];
          for (size_t i = 0; i < d.a.size(); ++i) d.a[i] = x.a[i] * y.a[i];
        }
        Vec& sc = scaler_post_[size_t(node)];
        for (int s = 0; s < P_; ++s) sc[size_t(s)] = scaler_post_[size_t(c0)][size_t(s)] + scaler_post_[size_t(c1)][size_t(s)];
        rescale(post_[size_t(node)], sc);
      } else {
        std::fill(scaler_post_[size_t(node)].begin(), scaler_post_[size_t(node)].end(), 0.0);
      }
      if (node != tree_.root()) {
        const double b = blen_[size_t(node - 1)];
        for (int l = 0; l < L; ++l) {
          trans_[size_t(node)][size_t(l)] = model_.transition_matrix(node, b, cats_.rates[size_t(l)]);
          compute_edge(node, l);
        }
      }
    }
    const int root = tree_.root();
    ll_ = 0.0;
    for (int s = 0; s < P_; ++s) {
      double mix = 0.0;
      for (int l = 0; l < L; ++l) {
        const Mat& pr = post_[size_t(root)][size_t(l)];
        double dot = 0.0;
        for (int j = 0; j < m; ++j) dot += model_.pi[size_t(j)] * pr(j, s);
        mix += cats_.probs[size_t(l)] * dot;
      }
      if (!std::isfinite(mix)) throw std::runtime_error("engine: non-finite partial at pattern " + std::to_string(s + p0_report));
      if (mix <= 0.0) throw std::runtime_error("engine: site likelihood underflowed to zero at pattern " + std::to_string(s + p0_report));
      site_ll_[size_t(s)] = std::log(mix) + scaler_post_[size_t(root)][size_t(s)];
      ll_ += weights_[size_t(s)] * site_ll_[size_t(s)];
    }
    post_valid_ = ll_valid_ = true;
    pre_valid_ = hess_valid_ = false;
  }

  // engine.hpp:225-278
  void pre_order_pass(bool hess) {
    if (!post_valid_) throw std::logic_error("engine: pre-order pass requires a current post-order pass");
    const int L = cats_.count(), m = model_.m;
    grad_.assign(size_t(tree_.branch_count()), 0.0);
    gabs_.assign(size_t(tree_.branch_count()), 0.0);
    if (hess) hessd_.assign(size_t(tree_.branch_count()), 0.0);
    Mat buffer(m, P_), qp(m, P_);
    Vec u1(static_cast<size_t>(P_)), u2(static_cast<size_t>(P_)), r1(static_cast<size_t>(P_));
    Vec u1abs(static_cast<size_t>(P_));  // the same sums over absolute values (condition)
    for (int node : tree_.pre_order) {
      ++visits_;
      if (node == tree_.root()) {
        for (int l = 0; l < L; ++l) {
          Mat& q = pre_[size_t(node)][size_t(l)];
          for (int s = 0; s < P_; ++s)
            for (int j = 0; j < m; ++j) q(j, s) = model_.pi[size_t(j)];
        }
        std::fill(scaler_pre_[size_t(node)].begin(), scaler_pre_[size_t(node)].end(), 0.0);
        continue;
      }
      const int parent = tree_.parent[size_t(node)], sib = tree_.sibling(node);
      for (int l = 0; l < L; ++l) {
        const Mat& qk = pre_[size_t(parent)][size_t(l)];
        const Mat& es = edge_[size_t(sib)][size_t(l)];
        for (size_t i = 0; i < buffer.a.size(); ++i) buffer.a[i] = qk.a[i] * es.a[i];
        const Mat& T = trans_[size_t(node)][size_t(l)];
        Mat& out = pre_[size_t(node)][size_t(l)];
        for (int s = 0; s < P_; ++s)
          for (int j = 0; j < m; ++j) {
            double acc = 0.0;
            for (int i = 0; i < m; ++i) acc += T(i, j) * buffer(i, s);
            out(j, s) = acc;
          }
      }
      Vec& sc = scaler_pre_[size_t(node)];
      for (int s = 0; s < P_; ++s) sc[size_t(s)] = scaler_pre_[size_t(parent)][size_t(s)] + scaler_post_[size_t(sib)][size_t(s)];
      rescale(pre_[size_t(node)], sc);

      std::fill(u1.begin(), u1.end(), 0.0);
      std::fill(u1abs.begin(), u1abs.end(), 0.0);
      if (hess) std::fill(u2.begin(), u2.end(), 0.0);
      const Mat& Q = model_.generator(node);
      const Mat Q2 = hess ? q2_for(node) : Mat();
      for (int l = 0; l < L; ++l) {
        const double cl = cats_.rates[size_t(l)], wl = cats_.probs[size_t(l)];
        const Mat& pm = post_matrix(node, l);
        const Mat& q = pre_[size_t(node)][size_t(l)];
        for (int s = 0; s < P_; ++s) {
          double acc = 0.0, acc2 = 0.0, acca = 0.0;
          for (int i = 0; i < m; ++i) {
            double qpi = 0.0, q2pi = 0.0, qpa = 0.0;
            for (int j = 0; j < m; ++j) {
              qpi += Q(i, j) * pm(j, s);
              qpa += std::fabs(Q(i, j) * pm(j, s));
              if (hess) q2pi += Q2(i, j) * pm(j, s);
            }
            acc += qpi * q(i, s);
            acca += qpa * std::fabs(q(i, s));
            acc2 += q2pi * q(i, s);
          }
          u1[size_t(s)] += (cl * wl) * acc;
          u1abs[size_t(s)] += (cl * wl) * acca;
          if (hess) u2[size_t(s)] += (cl * cl * wl) * acc2;
        }
      }
      double g = 0.0, hd = 0.0, ga = 0.0;
      for (int s = 0; s < P_; ++s) {
        const double e = std::exp(scaler_post_[size_t(node)][size_t(s)] + scaler_pre_[size_t(node)][size_t(s)] - site_ll_[size_t(s)]);
        r1[size_t(s)] = u1[size_t(s)] * e;
        g += weights_[size_t(s)] * r1[size_t(s)];
        // condition of the component (test use): every product of the
        // per-pattern term taken in absolute value, so cancellation inside
        // Q e (rows of Q sum to zero) and across patterns both count
        ga += weights_[size_t(s)] * u1abs[size_t(s)] * e;
        if (hess) {
          const double r2 = u2[size_t(s)] * e;
          hd += weights_[size_t(s)] * (r2 - r1[size_t(s)] * r1[size_t(s)]);
        }
      }
      grad_[size_t(node - 1)] = g;
      gabs_[size_t(node - 1)] = ga;
      if (hess) hessd_[size_t(node - 1)] = hd;
    }
    pre_valid_ = true;
    hess_valid_ = hess;
  }

  int p0_report = 0;  // pattern offset added to error messages
  // sum_s w_s |term_{s,i}| of the last pre-order pass: the condition of each
  // gradient component (SURVEY.md §8d condition-aware parity)
  const Vec& gradient_abs() const { return gabs_; }

 private:
  // engine.hpp:284-361 (slot-pool likelihood-only route)
  void scratch_pass() {
    const int L = cats_.count(), m = model_.m;
    std::vector<int> slot_of(size_t(tree_.node_count() + 1), -1), free_slots;
    auto acquire = [&] {
      if (!free_slots.empty()) {
        const int s = free_slots.back();
        free_slots.pop_back();
        return s;
      }
      scratch_.emplace_back(size_t(L), Mat(m, P_));
      scratch_scaler_.emplace_back(size_t(P_), 0.0);
      return int(scratch_.size()) - 1;
    };
    Mat tmp(m, P_);
    int root_slot = -1;
    for (int node : tree_.post_order) {
      ++visits_;
      if (tree_.is_tip(node)) {
        const int slot = acquire();
        slot_of[size_t(node)] = slot;
        std::fill(scratch_scaler_[size_t(slot)].begin(), scratch_scaler_[size_t(slot)].end(), 0.0);
        const double b = blen_[size_t(node - 1)];
        for (int l = 0; l < L; ++l) {
          const Mat T = model_.transition_matrix(node, b, cats_.rates[size_t(l)]);
          tip_edge(node, T, scratch_[size_t(slot)][size_t(l)]);
        }
        continue;
      }
      const int left = slot_of[size_t(tree_.children[size_t(node)][0])];
      const int right = slot_of[size_t(tree_.children[size_t(node)][1])];
      for (int l = 0; l < L; ++l) {
        Mat& a = scratch_[size_t(left)][size_t(l)];
        const Mat& b = scratch_[size_t(right)][size_t(l)];
        for (size_t i = 0; i < a.a.size(); ++i) a.a[i] *= b.a[i];
      }
      for (int s = 0; s < P_; ++s) scratch_scaler_[size_t(left)][size_t(s)] += scratch_scaler_[size_t(right)][size_t(s)];
      free_slots.push_back(right);
      slot_of[size_t(node)] = left;
      rescale(scratch_[size_t(left)], scratch_scaler_[size_t(left)]);
      if (node != tree_.root()) {
        const double b = blen_[size_t(node - 1)];
        for (int l = 0; l < L; ++l) {
          const Mat T = model_.transition_matrix(node, b, cats_.rates[size_t(l)]);
          matvec_cols(T, scratch_[size_t(left)][size_t(l)], tmp);
          std::swap(scratch_[size_t(left)][size_t(l)].a, tmp.a);
        }
      } else {
        root_slot = left;
      }
    }
    ll_ = 0.0;
    for (int s = 0; s < P_; ++s) {
      double mix = 0.0;
      for (int l = 0; l < L; ++l) {
        const Mat& pr = scratch_[size_t(root_slot)][size_t(l)];
        double dot = 0.0;
        for (int j = 0; j < m; ++j) dot += model_.pi[size_t(j)] * pr(j, s);
        mix += cats_.probs[size_t(l)] * dot;
      }
      if (!std::isfinite(mix)) throw std::runtime_error("engine: non-finite partial at pattern " + std::to_string(s + p0_report));
      if (mix <= 0.0) throw std::runtime_error("engine: site likelihood underflowed to zero at pattern " + std::to_string(s + p0_report));
      site_ll_[size_t(s)] = std::log(mix) + scratch_scaler_[size_t(root_slot)][size_t(s)];
      ll_ += weights_[size_t(s)] * site_ll_[size_t(s)];
    }
    ll_valid_ = true;
  }

  static void matvec_cols(const Mat& T, const Mat& x, Mat& out) {
    const int m = T.r;
    for (int s = 0; s < x.c; ++s)
      for (int i = 0; i < m; ++i) {
        double acc = 0.0;
        for (int j = 0; j < m; ++j) acc += T(i, j) * x(j, s);
        out(i, s) = acc;
      }
  }

  void tip_edge(int node, const Mat& T, Mat& edge) const {
    const int m = model_.m;
    const std::vector<int>& codes = tip_codes_[size_t(node)];
    const Mat& part = tip_partials_[size_t(node)];
    for (int s = 0; s < P_; ++s) {
      const int c = codes[size_t(s)];
      if (c >= 0) {
        for (int i = 0; i < m; ++i) edge(i, s) = T(i, c);
      } else {
        for (int i = 0; i < m; ++i) {
          double acc = 0.0;
          for (int j = 0; j < m; ++j) acc += T(i, j) * part(j, s);
          edge(i, s) = acc;
        }
      }
    }
  }

  const Mat& post_matrix(int node, int l) const {
    return tree_.is_tip(node) ? tip_partials_[size_t(node)] : post_[size_t(node)][size_t(l)];
  }

  // engine.hpp:367-382
  void compute_edge(int node, int l) {
    const Mat& T = trans_[size_t(node)][size_t(l)];
    Mat& e = edge_[size_t(node)][size_t(l)];
    if (!tree_.is_tip(node)) {
      matvec_cols(T, post_[size_t(node)][size_t(l)], e);
      return;
    }
    tip_edge(node, T, e);
  }

  // engine.hpp:386-394
  Mat q2_for(int node) const {
    const Mat& q = model_.generator(node);
    return matmul(q, q);
  }

  // engine.hpp:396-414
  void rescale(std::vector<Mat>& parts, Vec& scaler) {
    if (opt_.disable) return;
    const int L = int(parts.size()), m = parts[0].r;
    peak_.assign(size_t(P_), 0.0);
    bool any = opt_.force;
    for (int s = 0; s < P_; ++s) {
      double pk = -INFINITY;
      for (int l = 0; l < L; ++l)
        for (int j = 0; j < m; ++j) pk = std::max(pk, parts[size_t(l)](j, s));
      // Eigen's maxCoeff propagates NaN like std::max with NaN in first slot is
      // not guaranteed; NaN columns are reported at the root either way.
      peak_[size_t(s)] = pk;
      if (!(pk >= opt_.threshold || pk <= 0.0)) any = true;
    }
    if (!any) return;
    for (int s = 0; s < P_; ++s) {
      const double pk = peak_[size_t(s)];
      if (pk <= 0.0) continue;
      if (opt_.force || pk < opt_.threshold) {
        for (int l = 0; l < L; ++l)
          for (int j = 0; j < m; ++j) parts[size_t(l)](j, s) /= pk;
        scaler[size_t(s)] += std::log(pk);
      }
    }
  }

  const Tree& tree_;
  const Model& model_;
  Categories cats_;
  EngineOptions opt_;
  int P_ = 0;
  std::vector<Mat> tip_partials_;
  std::vector<std::vector<int>> tip_codes_;
  std::vector<std::vector<Mat>> post_, pre_, edge_, trans_;
  std::vector<Vec> scaler_post_, scaler_pre_;
  Vec site_ll_, weights_, peak_, blen_, grad_, hessd_;
  std::vector<std::vector<Mat>> scratch_;
  std::vector<Vec> scratch_scaler_;
  double ll_ = 0.0;
  bool post_valid_ = false, pre_valid_ = false, hess_valid_ = false, ll_valid_ = false;
  Vec gabs_;
  uint64_t visits_ = 0;
};

// validation.hpp:27-78
double brute_force_log_likelihood(const Tree& t, const Alignment& aln, const Model& model, const Categories& cats,
                                  const Vec& blen) {
  const int nt = t.tip_count, m = model.m, ni = nt - 1;
  if (nt > 6 || std::pow(double(m), ni) > 2e6) throw std::invalid_argument("brute force: tree too large to enumerate");
  if (int(blen.size()) != t.branch_count()) throw std::invalid_argument("brute force: wrong branch length count");
  std::vector<int> row(size_t(nt + 1), -1);
  for (int k = 1; k <= nt; ++k) {
    row[size_t(k)] = aln.taxon_index(t.labels[size_t(k)]);
    if (row[size_t(k)] < 0) throw std::invalid_argument("brute force: unbound tip");
  }
  const int L = cats.count();
  std::vector<std::vector<Mat>> tr(size_t(t.node_count() + 1));
  for (int i = 1; i <= t.branch_count(); ++i)
    for (int l = 0; l < L; ++l) tr[size_t(i)].push_back(model.transition_matrix(i, blen[size_t(i - 1)], cats.rates[size_t(l)]));
  double total = 0.0;
  std::vector<int> assign(size_t(ni), 0);
  for (int p = 0; p < aln.pattern_count(); ++p) {
    double site = 0.0;
    for (int l = 0; l < L; ++l) {
      double csum = 0.0;
      std::fill(assign.begin(), assign.end(), 0);
      while (true) {
        auto st = [&](int node) { return assign[size_t(node - nt - 1)]; };
        double term = model.pi[size_t(st(t.root()))];
        for (int node = nt + 1; node < t.root() && term != 0.0; ++node)
          term *= tr[size_t(node)][size_t(l)](st(t.parent[size_t(node)]), st(node));
        for (int k = 1; k <= nt && term != 0.0; ++k) {
          const Mat& part = aln.tip_partials[size_t(row[size_t(k)])];
          const Mat& T = tr[size_t(k)][size_t(l)];
          const int from = st(t.parent[size_t(k)]);
          double dot = 0.0;
          for (int j = 0; j < m; ++j) dot += T(from, j) * part(j, p);
          term *= dot;
        }
        csum += term;
        int d = 0;
        while (d < ni && ++assign[size_t(d)] == m) assign[size_t(d++)] = 0;
        if (d == ni) break;
      }
      site += cats.probs[size_t(l)] * csum;
    }
    if (site <= 0.0) throw std::runtime_error("brute force: zero site likelihood");
    total += double(aln.weights[size_t(p)]) * std::log(site);
  }
  return total;
}

}  // namespace orc

// =============================================================================
// C-ABI for ctypes (tests / bench cpu leg only)
// =============================================================================
using namespace orc;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::logic_error*>(&e)) return 3;
  if (dynamic_cast<const NewickError*>(&e)) return 4;
  return 2;
}
#define ORC_TRY try {
#define ORC_CATCH \
  }               \
  catch (const std::exception& e) { return fail(e); }

Tree tree_from_arrays(int nt, const int* parent, const int* children, const double* blen, const int* post,
                      const char* const* labels) {
  Tree t;
  t.tip_count = nt;
  const int n = t.node_count();
  t.labels.assign(size_t(n + 1), {});
  t.parent.assign(parent, parent + n + 1);
  t.children.assign(size_t(n + 1), {0, 0});
  for (int i = 0; i <= n; ++i) t.children[size_t(i)] = {children[2 * i], children[2 * i + 1]};
  t.branch_length.assign(size_t(n + 1), 0.0);
  for (int i = 1; i < n; ++i) t.branch_length[size_t(i)] = blen[i - 1];
  if (post) {
    t.post_order.assign(post, post + n);
    t.pre_order.assign(t.post_order.rbegin(), t.post_order.rend());
  } else {
    rebuild_traversals(t);
  }
  for (int i = 1; i <= nt; ++i) t.labels[size_t(i)] = labels ? std::string(labels[i - 1]) : "t" + std::to_string(i);
  return t;
}

struct OTree {
  Tree t;
};
struct OModel {
  std::unique_ptr<Model> m;
};
struct OAln {
  Alignment a;
};

// A (possibly multi-block) engine.  Block b owns patterns [b0, b1).
struct OEngine {
  Tree tree;
  Alignment aln;
  std::unique_ptr<Model> model;
  std::vector<std::unique_ptr<Engine>> blocks;
};
}  // namespace

template <class F>
static void run_blocks(OEngine* h, F&& f) {
  const size_t nb = h->blocks.size();
  if (nb == 1) {
    f(0);
    return;
  }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> errs(nb);
  for (size_t b = 0; b < nb; ++b)
    th.emplace_back([&, b] {
      try {
        f(b);
      } catch (...) {
        errs[b] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// ---- rng (mirrors std::mt19937_64 sequences used by the reference tests)
void* orc_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void orc_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }
uint64_t orc_rng_next(void* r) { return (*static_cast<std::mt19937_64*>(r))(); }
double orc_rng_uniform(void* r, double lo, double hi) {
  std::uniform_real_distribution<double> u(lo, hi);
  return u(*static_cast<std::mt19937_64*>(r));
}

// ---- trees
int orc_tree_parse(const char* text, void** out) {
  ORC_TRY
  auto* h = new OTree{parse_newick(text)};
  *out = h;
  return 0;
  ORC_CATCH
}
int orc_newick_error_position(const char* text) {
  try {
    parse_newick(text);
  } catch (const NewickError& e) {
    return int(e.position);
  } catch (...) {
    return -2;
  }
  return -1;
}
int orc_tree_from_arrays(int nt, const int* parent, const int* children, const double* blen, const int* post,
                         void** out) {
  ORC_TRY
  auto* h = new OTree{tree_from_arrays(nt, parent, children, blen, post, nullptr)};
  *out = h;
  return 0;
  ORC_CATCH
}
int orc_tree_random(void* rng, int tips, double lo, double hi, int coalescent_times, void** out) {
  ORC_TRY
  auto& r = *static_cast<std::mt19937_64*>(rng);
  auto* h = new OTree{coalescent_times ? random_coalescent_tree(tips, r, hi) : random_tree(tips, r, lo, hi)};
  *out = h;
  return 0;
  ORC_CATCH
}
int orc_tree_caterpillar(int tips, double branch, void** out) {
  ORC_TRY
  *out = new OTree{caterpillar_tree(tips, branch)};
  return 0;
  ORC_CATCH
}
int orc_tree_random_post_order(void* tree, void* rng, int* out) {
  ORC_TRY
  auto v = random_post_order(static_cast<OTree*>(tree)->t, *static_cast<std::mt19937_64*>(rng));
  std::copy(v.begin(), v.end(), out);
  return 0;
  ORC_CATCH
}
void orc_tree_free(void* t) { delete static_cast<OTree*>(t); }
int orc_tree_tips(void* t) { return static_cast<OTree*>(t)->t.tip_count; }
// parent/children sized 2N (index 0 unused), blen sized 2N-2 (branch i-1), post/pre 2N-1,
// times 2N (empty -> not written; returns has_times)
int orc_tree_get(void* th, int* parent, int* children, double* blen, int* post, int* pre, double* times) {
  const Tree& t = static_cast<OTree*>(th)->t;
  const int n = t.node_count();
  for (int i = 0; i <= n; ++i) {
    parent[i] = t.parent[size_t(i)];
    children[2 * i] = t.children[size_t(i)][0];
    children[2 * i + 1] = t.children[size_t(i)][1];
  }
  for (int i = 1; i < n; ++i) blen[i - 1] = t.branch_length[size_t(i)];
  for (int i = 0; i < n; ++i) {
    post[i] = t.post_order[size_t(i)];
    pre[i] = t.pre_order[size_t(i)];
  }
  if (!t.node_time.empty() && times)
    for (int i = 0; i <= n; ++i) times[i] = t.node_time[size_t(i)];
  return t.node_time.empty() ? 0 : 1;
}
int orc_tree_label(void* th, int node, char* buf, int cap) {
  const std::string& s = static_cast<OTree*>(th)->t.labels[size_t(node)];
  std::snprintf(buf, size_t(cap), "%s", s.c_str());
  return int(s.size());
}
int orc_tree_serialize(void* th, char* buf, int cap) {
  const std::string s = serialize_newick(static_cast<OTree*>(th)->t);
  std::snprintf(buf, size_t(cap), "%s", s.c_str());
  return int(s.size());
}
int orc_tree_validate(int nt, const int* parent, const int* children, const double* blen, const int* post,
                      const double* times) {
  ORC_TRY
  Tree t = tree_from_arrays(nt, parent, children, blen, post, nullptr);
  // validate_tree checks raw branch lengths stored per node (index i)
  if (times) t.node_time.assign(times, times + t.node_count() + 1);
  validate_tree(t);
  return 0;
  ORC_CATCH
}
int orc_tree_assign_times(void* th, double* times) {
  ORC_TRY
  Tree& t = static_cast<OTree*>(th)->t;
  assign_times_from_branch_lengths(t);
  for (int i = 0; i <= t.node_count(); ++i) times[i] = t.node_time[size_t(i)];
  return 0;
  ORC_CATCH
}

// ---- categories / model
int orc_discrete_gamma(double alpha, int count, double* rates, double* probs) {
  ORC_TRY
  Categories c = discrete_gamma(alpha, count);
  std::copy(c.rates.begin(), c.rates.end(), rates);
  std::copy(c.probs.begin(), c.probs.end(), probs);
  return 0;
  ORC_CATCH
}
double orc_gamma_quantile(double shape, double rate, double p) { return gamma_quantile(shape, rate, p); }
int orc_categories_check(int L, const double* rates, const double* probs) {
  ORC_TRY
  make_categories(Vec(rates, rates + L), Vec(probs, probs + L));
  return 0;
  ORC_CATCH
}
// Builds a GTR generator (row-major out 4x4) with finish_generator normalisation.
int orc_gtr(const double* exch, const double* freqs, double* q_rowmajor) {
  ORC_TRY
  Model mdl = gtr(exch, freqs);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) q_rowmajor[i * 4 + j] = mdl.q(i, j);
  return 0;
  ORC_CATCH
}
// finish_generator on a row-major m x m matrix (diagonal reset + rate-1 normalisation)
void orc_finish_generator(int m, double* q_rowmajor, const double* pi) {
  Mat q(m, m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) q(i, j) = q_rowmajor[i * m + j];
  finish_generator(q, Vec(pi, pi + m));
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) q_rowmajor[i * m + j] = q(i, j);
}
static Mat from_rowmajor(int m, const double* a) {
  Mat q(m, m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) q(i, j) = a[i * m + j];
  return q;
}
int orc_model_new(int m, const double* q_rowmajor, const double* pi, int reversible, void** out) {
  ORC_TRY
  auto* h = new OModel{std::make_unique<Model>(from_rowmajor(m, q_rowmajor), Vec(pi, pi + m), reversible != 0)};
  *out = h;
  return 0;
  ORC_CATCH
}
int orc_model_set_branch_generator(void* mh, int branch, const double* q_rowmajor) {
  ORC_TRY
  Model& md = *static_cast<OModel*>(mh)->m;
  md.set_branch_generator(branch, from_rowmajor(md.m, q_rowmajor));
  return 0;
  ORC_CATCH
}
void orc_model_free(void* m) { delete static_cast<OModel*>(m); }
int orc_model_has_eigen(void* mh) { return static_cast<OModel*>(mh)->m->have_eigen ? 1 : 0; }
int orc_transition_matrix(void* mh, int branch, double b, double c, double* out_rowmajor) {
  ORC_TRY
  const Model& md = *static_cast<OModel*>(mh)->m;
  Mat p = md.transition_matrix(branch, b, c);
  for (int i = 0; i < md.m; ++i)
    for (int j = 0; j < md.m; ++j) out_rowmajor[i * md.m + j] = p(i, j);
  return 0;
  ORC_CATCH
}
int orc_expm(int m, const double* a_rowmajor, double* out_rowmajor) {
  ORC_TRY
  Mat r = expm(from_rowmajor(m, a_rowmajor));
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) out_rowmajor[i * m + j] = r(i, j);
  return 0;
  ORC_CATCH
}

// ---- alignments
// codes: ntax x sites int32 row-major (-1 missing).  Labels "t1".. unless given.
int orc_aln_from_codes(int ntax, long sites, const int* codes, int m, const char* const* labels, void** out) {
  ORC_TRY
  std::vector<std::string> taxa;
  std::vector<std::vector<int>> rows(static_cast<size_t>(ntax));
  for (int r = 0; r < ntax; ++r) {
    taxa.push_back(labels ? std::string(labels[r]) : "t" + std::to_string(r + 1));
    rows[size_t(r)].assign(codes + size_t(r) * size_t(sites), codes + size_t(r + 1) * size_t(sites));
  }
  *out = new OAln{from_codes(std::move(taxa), rows, m)};
  return 0;
  ORC_CATCH
}
int orc_aln_from_fasta(const char* text, void** out) {
  ORC_TRY
  std::vector<std::string> taxa, seqs;
  parse_fasta(text, taxa, seqs);
  *out = new OAln{compress(taxa, seqs)};
  return 0;
  ORC_CATCH
}
void orc_aln_free(void* a) { delete static_cast<OAln*>(a); }
int orc_aln_patterns(void* a) { return static_cast<OAln*>(a)->a.pattern_count(); }
int orc_aln_taxa(void* a) { return int(static_cast<OAln*>(a)->a.taxa.size()); }
int orc_aln_states(void* a) { return static_cast<OAln*>(a)->a.m; }
void orc_aln_weights(void* a, int64_t* out) {
  const auto& w = static_cast<OAln*>(a)->a.weights;
  for (size_t i = 0; i < w.size(); ++i) out[i] = w[i];
}
// unique columns as codes (from_codes) : out ntax x P row-major
void orc_aln_pattern_codes(void* a, int* out) {
  const Alignment& al = static_cast<OAln*>(a)->a;
  const int P = al.pattern_count(), nt = int(al.taxa.size());
  for (int r = 0; r < nt; ++r)
    for (int p = 0; p < P; ++p) out[size_t(r) * size_t(P) + size_t(p)] = al.unique_columns.empty() ? 0 : al.unique_columns[size_t(p)][size_t(r)];
}
// dense tip partial of taxon row: m x P column-major
void orc_aln_tip_partials(void* a, int taxon, double* out) {
  const Mat& t = static_cast<OAln*>(a)->a.tip_partials[size_t(taxon)];
  std::copy(t.a.begin(), t.a.end(), out);
}
int orc_aln_pattern_column(void* a, int p, char* buf, int cap) {
  const Alignment& al = static_cast<OAln*>(a)->a;
  const std::string s = al.columns.empty() ? std::string() : al.columns[size_t(p)];
  std::snprintf(buf, size_t(cap), "%s", s.c_str());
  return int(s.size());
}
int orc_aln_taxon_name(void* a, int r, char* buf, int cap) {
  const std::string& s = static_cast<OAln*>(a)->a.taxa[size_t(r)];
  std::snprintf(buf, size_t(cap), "%s", s.c_str());
  return int(s.size());
}
// Alignment directly from a compressed representation: codes ntax x P (state,
// -1 all-ones, or >= m meaning ambiguity class code-m with partial amb[(code-m)*m ..]).
int orc_aln_from_patterns(int ntax, int P, int m, const int* codes, int n_amb, const double* amb,
                          const int64_t* weights, const char* const* labels, void** out) {
  ORC_TRY
  Alignment al;
  al.m = m;
  for (int r = 0; r < ntax; ++r) al.taxa.push_back(labels ? std::string(labels[r]) : "t" + std::to_string(r + 1));
  al.weights.assign(weights, weights + P);
  al.site_count = 0;
  for (long w : al.weights) al.site_count += w;
  al.tip_partials.assign(size_t(ntax), Mat(m, P));
  for (int r = 0; r < ntax; ++r)
    for (int p = 0; p < P; ++p) {
      const int c = codes[size_t(r) * size_t(P) + size_t(p)];
      Mat& tp = al.tip_partials[size_t(r)];
      if (c == -1) {
        for (int j = 0; j < m; ++j) tp(j, p) = 1.0;
      } else if (c >= 0 && c < m) {
        tp(c, p) = 1.0;
      } else if (c >= m && c - m < n_amb) {
        for (int j = 0; j < m; ++j) tp(j, p) = amb[size_t(c - m) * size_t(m) + size_t(j)];
      } else {
        throw std::invalid_argument("alignment: state code out of range");
      }
    }
  *out = new OAln{std::move(al)};
  return 0;
  ORC_CATCH
}

int orc_simulate_states(void* tree, void* model, int L, const double* rates, const double* probs, const double* blen,
                        long sites, uint64_t seed, int* out) {
  ORC_TRY
  const Tree& t = static_cast<OTree*>(tree)->t;
  Categories cats{Vec(rates, rates + L), Vec(probs, probs + L)};
  auto st = simulate_states(t, *static_cast<OModel*>(model)->m, cats, Vec(blen, blen + t.branch_count()), sites, seed);
  for (int r = 0; r < t.tip_count; ++r)
    std::copy(st[size_t(r)].begin(), st[size_t(r)].end(), out + size_t(r) * size_t(sites));
  return 0;
  ORC_CATCH
}

// ---- engine
int orc_engine_new(void* tree, void* aln, void* model, int L, const double* rates, const double* probs,
                   double threshold, int force, int disable, int nblocks, void** out) {
  ORC_TRY
  auto* h = new OEngine;
  h->tree = static_cast<OTree*>(tree)->t;
  h->aln = static_cast<OAln*>(aln)->a;
  h->model = std::make_unique<Model>(*static_cast<OModel*>(model)->m);
  Categories cats = make_categories(Vec(rates, rates + L), Vec(probs, probs + L));
  EngineOptions opt{threshold, force != 0, disable != 0};
  const int P = h->aln.pattern_count();
  if (nblocks < 1) nblocks = 1;
  if (nblocks > P) nblocks = std::max(1, P);
  // block engines are built concurrently (their per-node grids dominate setup)
  h->blocks.resize(size_t(nblocks));
  run_blocks(h, [&](size_t b) {
    const int p0 = int(int64_t(P) * int64_t(b) / nblocks), p1 = int(int64_t(P) * int64_t(b + 1) / nblocks);
    h->blocks[b] = std::make_unique<Engine>(h->tree, h->aln, *h->model, cats, opt, p0, p1 - p0);
    h->blocks[b]->p0_report = p0;
  });
  *out = h;
  return 0;
  ORC_CATCH
}
void orc_engine_free(void* e) { delete static_cast<OEngine*>(e); }
int orc_engine_set_branch_lengths(void* eh, const double* b) {
  ORC_TRY
  auto* h = static_cast<OEngine*>(eh);
  Vec v(b, b + h->tree.branch_count());
  for (auto& blk : h->blocks) blk->set_branch_lengths(v);
  return 0;
  ORC_CATCH
}
void orc_engine_invalidate(void* eh) {
  for (auto& blk : static_cast<OEngine*>(eh)->blocks) blk->invalidate();
}
uint64_t orc_engine_node_visits(void* eh) { return static_cast<OEngine*>(eh)->blocks[0]->node_visits(); }
void orc_engine_reset_node_visits(void* eh) {
  for (auto& blk : static_cast<OEngine*>(eh)->blocks) blk->reset_node_visits();
}

int orc_engine_log_likelihood(void* eh, double* out) {
  ORC_TRY
  auto* h = static_cast<OEngine*>(eh);
  std::vector<double> part(h->blocks.size());
  run_blocks(h, [&](size_t b) { part[b] = h->blocks[b]->log_likelihood(); });
  double s = 0.0;
  for (double v : part) s += v;
  *out = s;
  return 0;
  ORC_CATCH
}
int orc_engine_post_order_pass(void* eh) {
  ORC_TRY
  auto* h = static_cast<OEngine*>(eh);
  run_blocks(h, [&](size_t b) { h->blocks[b]->post_order_pass(); });
  return 0;
  ORC_CATCH
}
int orc_engine_pre_order_pass(void* eh, int hess) {
  ORC_TRY
  auto* h = static_cast<OEngine*>(eh);
  run_blocks(h, [&](size_t b) { h->blocks[b]->pre_order_pass(hess != 0); });
  return 0;
  ORC_CATCH
}
int orc_engine_branch_gradient(void* eh, int hess, double* ll, double* grad, double* hd) {
  ORC_TRY
  auto* h = static_cast<OEngine*>(eh);
  const size_t nb = h->blocks.size(), B = size_t(h->tree.branch_count());
  std::vector<double> lls(nb);
  std::vector<Vec> gs(nb), hs(nb);
  run_blocks(h, [&](size_t b) { h->blocks[b]->branch_gradient(hess != 0, lls[b], gs[b], hs[b]); });
  *ll = 0.0;
  for (size_t i = 0; i < B; ++i) {
    grad[i] = 0.0;
    if (hess) hd[i] = 0.0;
  }
  for (size_t b = 0; b < nb; ++b) {
    *ll += lls[b];
    for (size_t i = 0; i < B; ++i) {
      grad[i] += gs[b][i];
      if (hess) hd[i] += hs[b][i];
    }
  }
  return 0;
  ORC_CATCH
}
int orc_engine_gradient_abs(void* eh, double* out) {
  ORC_TRY
  auto* h = static_cast<OEngine*>(eh);
  const size_t B = size_t(h->tree.branch_count());
  for (size_t i = 0; i < B; ++i) out[i] = 0.0;
  for (auto& blk : h->blocks) {
    const Vec& a = blk->gradient_abs();
    if (a.size() != B) throw std::logic_error("engine: no current gradient pass");
    for (size_t i = 0; i < B; ++i) out[i] += a[i];
  }
  return 0;
  ORC_CATCH
}
int orc_engine_log_likelihood_at_node(void* eh, int node, double* out) {
  ORC_TRY
  auto* h = static_cast<OEngine*>(eh);
  double s = 0.0;
  for (auto& blk : h->blocks) s += blk->log_likelihood_at_node(node);
  *out = s;
  return 0;
  ORC_CATCH
}
// m x P(block 0 only; tests use one block) column-major
int orc_engine_post_partial(void* eh, int node, int l, double* out) {
  ORC_TRY
  const Mat& mm = static_cast<OEngine*>(eh)->blocks[0]->post_partial(node, l);
  std::copy(mm.a.begin(), mm.a.end(), out);
  return 0;
  ORC_CATCH
}
int orc_engine_pre_partial(void* eh, int node, int l, double* out) {
  ORC_TRY
  const Mat& mm = static_cast<OEngine*>(eh)->blocks[0]->pre_partial(node, l);
  std::copy(mm.a.begin(), mm.a.end(), out);
  return 0;
  ORC_CATCH
}
int orc_engine_scalers(void* eh, int node, double* post, double* pre) {
  ORC_TRY
  auto& blk = static_cast<OEngine*>(eh)->blocks[0];
  std::copy(blk->post_scaler(node).begin(), blk->post_scaler(node).end(), post);
  std::copy(blk->pre_scaler(node).begin(), blk->pre_scaler(node).end(), pre);
  return 0;
  ORC_CATCH
}
int orc_engine_site_log_likelihoods(void* eh, double* out) {
  ORC_TRY
  auto* h = static_cast<OEngine*>(eh);
  size_t off = 0;
  for (auto& blk : h->blocks) {
    std::copy(blk->site_ll().begin(), blk->site_ll().end(), out + off);
    off += blk->site_ll().size();
  }
  return 0;
  ORC_CATCH
}

// validation.hpp:27-78
int orc_brute_force(void* tree, void* aln, void* model, int L, const double* rates, const double* probs,
                    const double* blen, double* out) {
  ORC_TRY
  const Tree& t = static_cast<OTree*>(tree)->t;
  Categories cats{Vec(rates, rates + L), Vec(probs, probs + L)};
  *out = brute_force_log_likelihood(t, static_cast<OAln*>(aln)->a, *static_cast<OModel*>(model)->m, cats,
                                    Vec(blen, blen + t.branch_count()));
  return 0;
  ORC_CATCH
}

}  // extern "C"
