// Host-side setup for phylograd-b200: the data formats either side of the hot
// path and seeded synthetic workloads.
//
//  * Newick parsing with the reference's integer numbering contract
//    (tree.hpp:144-289): tips 1..N in left-to-right order, internal nodes
//    N+1..2N-1 in completion order, root 2N-1.
//  * Pattern compression in first-occurrence order with integer weights
//    (alignment.hpp:186-229), hash-based and multithreaded instead of the
//    reference's std::map over column vectors; output order is identical.
//  * Discrete-gamma categories (substitution.hpp:55-68).
//  * Symmetric eigensolver used by the engine to form P(t) on the GPU.
//  * Synthetic workloads for BASELINE.json configs (Yule trees, model draws,
//    forward simulation) — input generation only, never on the timed path.
#include <algorithm>
#include <array>
#include <atomic>
#include <charconv>
#include <cstring>
#include <memory>
#include <random>
#include <string_view>
#include <thread>
#include <unordered_map>

#include "pg_common.hpp"

namespace pg {

namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& s) { g_last_error = s; }

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

// ------------------------------------------------------------------ newick
namespace {
struct Proto {
  std::string label;
  double length = 0.0;
  int left = -1, right = -1;
};

class NewickReader {
 public:
  explicit NewickReader(std::string_view t) : text_(t) {}

  void run() {
    const int root = subtree();
    expect(';');
    ws();
    if (pos_ != text_.size()) fail("trailing characters after ';'");
    if (nodes_[size_t(root)].left < 0) fail("a tree must have at least two tips");
    root_ = root;
  }
  int tips() const { return int(tip_ids_.size()); }

  void emit(int32_t* parent, int32_t* children, double* blen, int32_t* post, char* labels, int64_t cap) const {
    const int nt = tips(), n = 2 * nt - 1;
    std::vector<int> id(nodes_.size(), 0);
    for (int k = 0; k < nt; ++k) id[size_t(tip_ids_[size_t(k)])] = k + 1;
    for (size_t k = 0; k < done_.size(); ++k) id[size_t(done_[k])] = nt + 1 + int(k);
    std::fill(parent, parent + n + 1, 0);
    std::fill(children, children + 2 * (n + 1), 0);
    std::fill(blen, blen + n + 1, 0.0);
    for (size_t p = 0; p < nodes_.size(); ++p) {
      const int i = id[p];
      blen[i] = nodes_[p].length;
      if (nodes_[p].left >= 0) {
        const int l = id[size_t(nodes_[p].left)], r = id[size_t(nodes_[p].right)];
        children[2 * i] = l;
        children[2 * i + 1] = r;
        parent[l] = i;
        parent[r] = i;
      }
    }
    blen[n] = 0.0;
    // tree.hpp:60-77 left-child-first iterative post order
    int k = 0;
    std::vector<std::pair<int, bool>> st{{n, false}};
    while (!st.empty()) {
      auto [node, expanded] = st.back();
      st.pop_back();
      if (expanded || node <= nt) {
        post[k++] = node;
      } else {
        st.push_back({node, true});
        st.push_back({children[2 * node + 1], false});
        st.push_back({children[2 * node], false});
      }
    }
    if (labels) {
      int64_t off = 0;
      for (int t = 0; t < nt; ++t) {
        const std::string& s = nodes_[size_t(tip_ids_[size_t(t)])].label;
        if (off + int64_t(s.size()) + 1 > cap) throw std::invalid_argument("newick: label buffer too small");
        std::memcpy(labels + off, s.data(), s.size());
        off += int64_t(s.size());
        labels[off++] = '\0';
      }
    }
  }

 private:
  [[noreturn]] void fail(const std::string& w) const { throw NewickError(w, pos_); }
  void ws() {
    while (pos_ < text_.size() && std::isspace((unsigned char)text_[pos_])) ++pos_;
  }
  char peek() {
    ws();
    if (pos_ >= text_.size()) fail("unexpected end of input");
    return text_[pos_];
  }
  void expect(char c) {
    if (peek() != c) fail(std::string("expected '") + c + "'");
    ++pos_;
  }
  static bool is_delim(char c) {
    return c == '(' || c == ')' || c == ',' || c == ':' || c == ';' || std::isspace((unsigned char)c);
  }
  std::string label() {
    ws();
    const size_t b = pos_;
    while (pos_ < text_.size() && !is_delim(text_[pos_])) ++pos_;
    return std::string(text_.substr(b, pos_ - b));
  }
  double length() {
    ws();
    double v = 0.0;
    auto r = std::from_chars(text_.data() + pos_, text_.data() + text_.size(), v);
    if (r.ec != std::errc()) fail("expected a branch length");
    pos_ = size_t(r.ptr - text_.data());
    if (v < 0.0) fail("negative branch length");
    return v;
  }
  void maybe_length(int idx) {
    ws();
    if (pos_ < text_.size() && text_[pos_] == ':') {
      ++pos_;
      nodes_[size_t(idx)].length = length();
    }
  }
  int subtree() {
    if (peek() == '(') {
      ++pos_;
      std::vector<int> kids{subtree()};
      while (peek() == ',') {
        ++pos_;
        kids.push_back(subtree());
      }
      expect(')');
      if (kids.size() == 1) fail("unifurcation: internal node with one child");
      if (kids.size() > 2) fail("polytomy: internal node with more than two children");
      const int idx = int(nodes_.size());
      nodes_.push_back({});
      nodes_.back().left = kids[0];
      nodes_.back().right = kids[1];
      ws();
      if (pos_ < text_.size() && text_[pos_] != ':' && text_[pos_] != ',' && text_[pos_] != ')' && text_[pos_] != ';')
        label();  // internal labels are kept out of the numbering contract
      maybe_length(idx);
      done_.push_back(idx);
      return idx;
    }
    std::string lab = label();
    if (lab.empty()) fail("expected a tip label");
    const int idx = int(nodes_.size());
    nodes_.push_back({});
    nodes_.back().label = std::move(lab);
    maybe_length(idx);
    tip_ids_.push_back(idx);
    return idx;
  }

  std::string_view text_;
  size_t pos_ = 0;
  std::vector<Proto> nodes_;
  std::vector<int> tip_ids_, done_;
  int root_ = -1;

 public:
  void check_duplicates() const {
    std::unordered_map<std::string, int> seen;
    for (int t = 0; t < tips(); ++t) {
      const std::string& s = nodes_[size_t(tip_ids_[size_t(t)])].label;
      if (!seen.emplace(s, t).second) throw NewickError("duplicate tip label '" + s + "'", 0);
    }
  }
};
}  // namespace

// ------------------------------------------------------------ compression
namespace {
inline uint64_t mix64(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdull;
  return h ^ (h >> 33);
}

int hw_threads(int want) {
  if (want > 0) return want;
  const unsigned h = std::thread::hardware_concurrency();
  return h ? int(std::min(h, 256u)) : 1;
}

template <class F>
void parallel_for(int64_t n, int threads, F&& f) {
  threads = int(std::max<int64_t>(1, std::min<int64_t>(threads, n / 1024 + 1)));
  if (threads == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < threads; ++t) {
    const int64_t a = n * t / threads, b = n * (t + 1) / threads;
    th.emplace_back([&, a, b] { f(a, b); });
  }
  for (auto& x : th) x.join();
}

// First-occurrence compression of column vectors codes[r*sites + s] (r < ntax).
template <class T>
struct Compressed {
  std::vector<int64_t> rep;      // representative site of each pattern
  std::vector<int64_t> weights;
  std::vector<int32_t> site_to_pattern;
};

template <class T>
Compressed<T> compress_columns(const T* codes, int ntax, int64_t sites, int threads) {
  std::vector<uint64_t> h(size_t(sites), 0x1234567ull);
  parallel_for(sites, hw_threads(threads), [&](int64_t a, int64_t b) {
    for (int r = 0; r < ntax; ++r) {
      const T* row = codes + size_t(r) * size_t(sites);
      for (int64_t s = a; s < b; ++s) h[size_t(s)] = mix64(h[size_t(s)], uint64_t(int64_t(row[s]) + 2));
    }
  });
  Compressed<T> out;
  out.site_to_pattern.resize(size_t(sites));
  std::unordered_map<uint64_t, std::vector<int32_t>> buckets;
  buckets.reserve(size_t(sites));
  auto same = [&](int64_t s1, int64_t s2) {
    for (int r = 0; r < ntax; ++r)
      if (codes[size_t(r) * size_t(sites) + size_t(s1)] != codes[size_t(r) * size_t(sites) + size_t(s2)]) return false;
    return true;
  };
  for (int64_t s = 0; s < sites; ++s) {
    auto& bucket = buckets[h[size_t(s)]];
    int32_t found = -1;
    for (int32_t p : bucket)
      if (same(out.rep[size_t(p)], s)) {
        found = p;
        break;
      }
    if (found < 0) {
      found = int32_t(out.rep.size());
      out.rep.push_back(s);
      out.weights.push_back(0);
      bucket.push_back(found);
    }
    ++out.weights[size_t(found)];
    out.site_to_pattern[size_t(s)] = found;
  }
  return out;
}

struct CompressHandle {
  int ntax = 0;
  int64_t sites = 0;
  std::vector<int32_t> codes;
  Compressed<int32_t> c;
};

// ------------------------------------------------------------- synthetic
struct Synth {
  pg_synth_spec spec{};
  int N = 0, m = 4, L = 1;
  std::vector<int32_t> parent, children, post;
  std::vector<double> blen, dt, rates;
  std::vector<double> q, pi;
  int reversible = 1;
  std::vector<double> cat_rates, cat_probs;
  std::vector<int8_t> pcodes;  // [N][P]
  std::vector<int64_t> weights;
};

uint64_t splitmix(uint64_t& x) {
  uint64_t z = (x += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

std::vector<double> dirichlet(std::mt19937_64& rng, int k, double a) {
  std::gamma_distribution<double> g(a, 1.0);
  std::vector<double> v(static_cast<size_t>(k));
  double s = 0;
  for (auto& x : v) s += (x = g(rng));
  for (auto& x : v) x /= s;
  return v;
}

void finish_generator(std::vector<double>& q, const std::vector<double>& pi, int m) {
  for (int i = 0; i < m; ++i) {
    q[size_t(i) * m + i] = 0.0;
    double s = 0;
    for (int j = 0; j < m; ++j) s += q[size_t(i) * m + j];
    q[size_t(i) * m + i] = -s;
  }
  double rate = 0;
  for (int i = 0; i < m; ++i) rate -= pi[size_t(i)] * q[size_t(i) * m + i];
  for (auto& x : q) x /= rate;
}

// Yule (pure-birth) topology, numbered like parse_newick of its Newick text.
void yule_tree(Synth& S, std::mt19937_64& rng) {
  const int N = S.spec.tips;
  if (N < 2) throw std::invalid_argument("synth: need >= 2 tips");
  struct PN {
    int l = -1, r = -1;
  };
  std::vector<PN> pn(1);
  std::vector<int> leaves{0};
  while (int(leaves.size()) < N) {
    std::uniform_int_distribution<size_t> pick(0, leaves.size() - 1);
    const size_t at = pick(rng);
    const int v = leaves[at];
    const int a = int(pn.size()), b = a + 1;
    pn.push_back({});
    pn.push_back({});
    pn[size_t(v)].l = a;
    pn[size_t(v)].r = b;
    leaves[at] = a;
    leaves.push_back(b);
  }
  // numbering: tips in left-to-right order, internals in completion order
  const int n = 2 * N - 1;
  std::vector<int> id(pn.size(), 0);
  int next_tip = 1, next_int = N + 1;
  std::vector<std::pair<int, bool>> st{{0, false}};
  while (!st.empty()) {
    auto [v, exp] = st.back();
    st.pop_back();
    if (pn[size_t(v)].l < 0) {
      id[size_t(v)] = next_tip++;
    } else if (exp) {
      id[size_t(v)] = next_int++;
    } else {
      st.push_back({v, true});
      st.push_back({pn[size_t(v)].r, false});
      st.push_back({pn[size_t(v)].l, false});
    }
  }
  S.N = N;
  S.parent.assign(size_t(n + 1), 0);
  S.children.assign(size_t(2 * (n + 1)), 0);
  for (size_t v = 0; v < pn.size(); ++v)
    if (pn[v].l >= 0) {
      const int i = id[v], l = id[size_t(pn[v].l)], r = id[size_t(pn[v].r)];
      S.children[size_t(2 * i)] = l;
      S.children[size_t(2 * i + 1)] = r;
      S.parent[size_t(l)] = i;
      S.parent[size_t(r)] = i;
    }
  S.post.clear();
  std::vector<std::pair<int, bool>> st2{{n, false}};
  while (!st2.empty()) {
    auto [v, exp] = st2.back();
    st2.pop_back();
    if (exp || v <= N) {
      S.post.push_back(v);
    } else {
      st2.push_back({v, true});
      st2.push_back({S.children[size_t(2 * v + 1)], false});
      st2.push_back({S.children[size_t(2 * v)], false});
    }
  }
}

// The 61 sense codons of the standard genetic code (TCAG order) for GY94.
void gy94(Synth& S, std::mt19937_64& rng, double omega, double kappa) {
  static const char* aa = "FFLLSSSSYY**CC*WLLLLPPPPHHQQRRRRIIIMTTTTNNKKSSRRVVVVAAAADDEEGGGG";
  std::vector<int> sense;
  for (int c = 0; c < 64; ++c)
    if (aa[c] != '*') sense.push_back(c);
  const int m = int(sense.size());  // 61
  S.m = m;
  S.pi = dirichlet(rng, m, 2.0);
  S.q.assign(size_t(m) * m, 0.0);
  auto base = [](int c, int pos) { return (c >> (2 * (2 - pos))) & 3; };  // T=0 C=1 A=2 G=3
  auto transition = [](int x, int y) { return (x == 0 && y == 1) || (x == 1 && y == 0) || (x == 2 && y == 3) || (x == 3 && y == 2); };
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      if (i == j) continue;
      const int ci = sense[size_t(i)], cj = sense[size_t(j)];
      int diffs = 0, pos = -1;
      for (int k = 0; k < 3; ++k)
        if (base(ci, k) != base(cj, k)) {
          ++diffs;
          pos = k;
        }
      if (diffs != 1) continue;
      double r = S.pi[size_t(j)];
      if (transition(base(ci, pos), base(cj, pos))) r *= kappa;
      if (aa[ci] != aa[cj]) r *= omega;
      S.q[size_t(i) * m + j] = r;
    }
  finish_generator(S.q, S.pi, m);
  S.reversible = 1;
}

void draw_model(Synth& S, std::mt19937_64& rng) {
  const int kind = S.spec.model_kind;
  std::lognormal_distribution<double> ln05(0.0, 0.5), ln07(0.0, 0.7), ln1(0.0, 1.0);
  if (kind == 0 || kind == 1) {
    S.m = 4;
    double exch[6];
    std::vector<double> f;
    if (kind == 0) {
      const double k = 2.0;
      const double e[6] = {1.0, k, 1.0, 1.0, k, 1.0};
      std::copy(e, e + 6, exch);
      f = {0.3, 0.2, 0.2, 0.3};
    } else {
      for (double& x : exch) x = ln05(rng);
      f = dirichlet(rng, 4, 10.0);
    }
    S.q.assign(16, 0.0);
    int e = 0;
    for (int i = 0; i < 4; ++i)
      for (int j = i + 1; j < 4; ++j, ++e) {
        S.q[size_t(i) * 4 + j] = exch[e] * f[size_t(j)];
        S.q[size_t(j) * 4 + i] = exch[e] * f[size_t(i)];
      }
    S.pi = f;
    finish_generator(S.q, S.pi, 4);
    S.reversible = 1;
  } else if (kind == 2) {
    S.m = 4;
    S.q.assign(16, 0.0);
    for (int i = 0; i < 4; ++i) {
      double s = 0;
      for (int j = 0; j < 4; ++j)
        if (i != j) s += (S.q[size_t(i) * 4 + j] = ln07(rng));
      S.q[size_t(i) * 4 + i] = -s;
    }
    S.pi = dirichlet(rng, 4, 5.0);
    S.reversible = 0;
  } else if (kind == 3) {
    const int m = 20;
    S.m = m;
    std::vector<double> exch(190);
    for (double& x : exch) x = ln1(rng);
    S.pi = dirichlet(rng, m, 1.0);
    for (double& p : S.pi) p = std::max(p, 1e-12);  // keep pi > 0 for the eigen path
    double s = 0;
    for (double p : S.pi) s += p;
    for (double& p : S.pi) p /= s;
    S.q.assign(size_t(m) * m, 0.0);
    int e = 0;
    for (int i = 0; i < m; ++i)
      for (int j = i + 1; j < m; ++j, ++e) {
        S.q[size_t(i) * m + j] = exch[size_t(e)] * S.pi[size_t(j)];
        S.q[size_t(j) * m + i] = exch[size_t(e)] * S.pi[size_t(i)];
      }
    finish_generator(S.q, S.pi, m);
    S.reversible = 1;
  } else if (kind == 4) {
    gy94(S, rng, 0.3, 2.0);
  } else {
    throw std::invalid_argument("synth: unknown model kind");
  }
}

// Host P(t) for simulation: eigen path for reversible models, Pade otherwise.
struct HostP {
  int m;
  bool eig = false;
  std::vector<double> w, U, Ui;
  std::vector<double> q;
  HostP(const Synth& S) : m(S.m), q(S.q) {
    bool pos = true;
    for (double p : S.pi) pos = pos && p > 0;
    if (S.reversible && pos) {
      std::vector<double> sym(static_cast<size_t>(m) * m), sp(static_cast<size_t>(m));
      for (int i = 0; i < m; ++i) sp[size_t(i)] = std::sqrt(S.pi[size_t(i)]);
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
  std::vector<double> operator()(double t) const {
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
};

void simulate(Synth& S) {
  const int N = S.N, n = 2 * N - 1, m = S.m, L = S.L;
  const int64_t sites = S.spec.sites;
  HostP hp(S);
  // cumulative rows per (node, category)
  std::vector<double> cdf(size_t(n + 1) * L * m * m);
  for (int v = 1; v < n; ++v)
    for (int l = 0; l < L; ++l) {
      auto p = hp(S.blen[size_t(v - 1)] * S.cat_rates[size_t(l)]);
      for (int i = 0; i < m; ++i) {
        double acc = 0;
        for (int j = 0; j < m; ++j) {
          acc += p[size_t(i) * m + j];
          cdf[((size_t(v) * L + l) * m + i) * m + j] = acc;
        }
      }
    }
  std::vector<double> root_cdf(static_cast<size_t>(m)), cat_cdf(static_cast<size_t>(L));
  double acc = 0;
  for (int j = 0; j < m; ++j) root_cdf[size_t(j)] = (acc += S.pi[size_t(j)]);
  acc = 0;
  for (int l = 0; l < L; ++l) cat_cdf[size_t(l)] = (acc += S.cat_probs[size_t(l)]);
  std::vector<int> pre(S.post.rbegin(), S.post.rend());

  std::vector<int8_t> codes(size_t(N) * size_t(sites));
  const int64_t block = 4096;
  const int64_t nblocks = (sites + block - 1) / block;
  std::atomic<int64_t> next{0};
  auto worker = [&] {
    std::vector<int> state(size_t(n + 1));
    for (;;) {
      const int64_t bi = next.fetch_add(1);
      if (bi >= nblocks) break;
      uint64_t sm = S.spec.seed * 0x9E3779B97F4A7C15ull + uint64_t(bi) + 1;
      std::mt19937_64 rng(splitmix(sm));
      auto unif = [&] { return double(rng() >> 11) * 0x1.0p-53; };
      auto pick = [&](const double* c, int k) {
        const double u = unif() * c[k - 1];
        int j = 0;
        while (j < k - 1 && !(u < c[j])) ++j;
        return j;
      };
      std::bernoulli_distribution gap(S.spec.gap_fraction > 0 ? S.spec.gap_fraction : 0.0);
      const int64_t s0 = bi * block, s1 = std::min(sites, s0 + block);
      for (int64_t s = s0; s < s1; ++s) {
        const int l = pick(cat_cdf.data(), L);
        for (int v : pre) {
          if (v == n)
            state[size_t(v)] = pick(root_cdf.data(), m);
          else
            state[size_t(v)] = pick(&cdf[((size_t(v) * L + l) * m + state[size_t(S.parent[size_t(v)])]) * m], m);
          if (v <= N) codes[size_t(v - 1) * size_t(sites) + size_t(s)] = int8_t(state[size_t(v)]);
        }
        if (S.spec.gap_fraction > 0)
          for (int t = 0; t < N; ++t)
            if (gap(rng)) codes[size_t(t) * size_t(sites) + size_t(s)] = -1;
      }
    }
  };
  const int T = hw_threads(S.spec.threads);
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) th.emplace_back(worker);
  for (auto& x : th) x.join();

  auto c = compress_columns(codes.data(), N, sites, T);
  const int64_t P = int64_t(c.rep.size());
  S.weights = c.weights;
  S.pcodes.resize(size_t(N) * size_t(P));
  parallel_for(N, T, [&](int64_t a, int64_t b) {
    for (int64_t t = a; t < b; ++t)
      for (int64_t p = 0; p < P; ++p)
        S.pcodes[size_t(t) * size_t(P) + size_t(p)] = codes[size_t(t) * size_t(sites) + size_t(c.rep[size_t(p)])];
  });
}
}  // namespace

}  // namespace pg

using namespace pg;

extern "C" {

const char* pg_last_error(void) { return g_last_error.c_str(); }

int pg_newick_parse(const char* text, int* tip_count, int32_t* parent, int32_t* children, double* branch_length,
                    int32_t* post_order, char* label_buf, int64_t label_cap) {
  return guarded([&] {
    if (!text) throw std::invalid_argument("newick: null text");
    NewickReader r{std::string_view(text)};
    r.run();
    r.check_duplicates();
    *tip_count = r.tips();
    if (parent) r.emit(parent, children, branch_length, post_order, label_buf, label_cap);
  });
}

int pg_compress_codes(int ntax, int64_t sites, const int32_t* codes, int state_count, void** handle,
                      int* pattern_count) {
  return guarded([&] {
    if (state_count < 2) throw std::invalid_argument("alignment: state count must be >= 2");
    if (ntax <= 0) throw std::invalid_argument("alignment: no records");
    auto* h = new CompressHandle;
    std::unique_ptr<CompressHandle> guard(h);
    h->ntax = ntax;
    h->sites = sites;
    h->codes.assign(codes, codes + size_t(ntax) * size_t(sites));
    for (int32_t c : h->codes)
      if (c < -1 || c >= state_count) throw std::invalid_argument("alignment: state code out of range");
    h->c = compress_columns(h->codes.data(), ntax, sites, 0);
    *pattern_count = int(h->c.rep.size());
    *handle = guard.release();
  });
}

int pg_compress_result(void* handle, int32_t* pattern_codes, int64_t* weights, int32_t* site_to_pattern) {
  return guarded([&] {
    auto* h = static_cast<CompressHandle*>(handle);
    const size_t P = h ? h->c.rep.size() : 0;
    if (!h) throw std::invalid_argument("alignment: null compression handle");
    if (pattern_codes)
      for (int r = 0; r < h->ntax; ++r)
        for (size_t p = 0; p < P; ++p)
          pattern_codes[size_t(r) * P + p] = h->codes[size_t(r) * size_t(h->sites) + size_t(h->c.rep[p])];
    if (weights) std::copy(h->c.weights.begin(), h->c.weights.end(), weights);
    if (site_to_pattern) std::copy(h->c.site_to_pattern.begin(), h->c.site_to_pattern.end(), site_to_pattern);
  });
}

void pg_compress_free(void* handle) { delete static_cast<CompressHandle*>(handle); }

int pg_discrete_gamma(double alpha, int count, double* rates, double* probs) {
  return guarded([&] {
    if (!(alpha > 0.0) || !std::isfinite(alpha))
      throw std::invalid_argument("discrete gamma: alpha must be positive and finite");
    if (count < 1) throw std::invalid_argument("discrete gamma: need at least one category");
    if (count == 1) {
      rates[0] = probs[0] = 1.0;
      return;
    }
    double s = 0;
    for (int l = 0; l < count; ++l) {
      rates[l] = gamma_quantile(alpha, 1.0, (2.0 * l + 1.0) / (2.0 * count)) / alpha;
      s += rates[l];
    }
    for (int l = 0; l < count; ++l) {
      rates[l] *= double(count) / s;
      probs[l] = 1.0 / count;
    }
  });
}

int pg_synth_create(const pg_synth_spec* spec, void** handle, int* pattern_count, int* state_count) {
  return guarded([&] {
    auto S = std::make_unique<Synth>();
    S->spec = *spec;
    uint64_t sm = spec->seed;
    std::mt19937_64 tree_rng(splitmix(sm)), param_rng(splitmix(sm)), len_rng(splitmix(sm));
    yule_tree(*S, tree_rng);
    draw_model(*S, param_rng);
    const int B = 2 * S->N - 2;
    S->blen.assign(size_t(B), 0.0);
    S->dt.assign(size_t(B), 0.0);
    S->rates.assign(size_t(B), 0.0);
    if (spec->clock) {
      std::exponential_distribution<double> ex(1.0 / spec->dt_mean);
      std::normal_distribution<double> z(0.0, 1.0);
      for (int i = 0; i < B; ++i) {
        S->dt[size_t(i)] = ex(len_rng);
        S->rates[size_t(i)] = spec->rate_scale * std::exp(spec->rate_sd * z(len_rng));
        S->blen[size_t(i)] = S->rates[size_t(i)] * S->dt[size_t(i)];
      }
    } else {
      std::exponential_distribution<double> ex(1.0 / spec->branch_mean);
      for (int i = 0; i < B; ++i) S->blen[size_t(i)] = ex(len_rng);
    }
    S->L = std::max(1, spec->categories);
    S->cat_rates.assign(size_t(S->L), 1.0);
    S->cat_probs.assign(size_t(S->L), 1.0 / S->L);
    if (S->L > 1) {
      const int rc = pg_discrete_gamma(spec->gamma_alpha, S->L, S->cat_rates.data(), S->cat_probs.data());
      if (rc) throw std::invalid_argument(g_last_error);
    }
    simulate(*S);
    *pattern_count = int(S->weights.size());
    *state_count = S->m;
    *handle = S.release();
  });
}

int pg_synth_tree(void* handle, int32_t* parent, int32_t* children, int32_t* post_order, double* branch_lengths,
                  double* durations, double* rates) {
  return guarded([&] {
    auto* S = static_cast<Synth*>(handle);
    std::copy(S->parent.begin(), S->parent.end(), parent);
    std::copy(S->children.begin(), S->children.end(), children);
    std::copy(S->post.begin(), S->post.end(), post_order);
    std::copy(S->blen.begin(), S->blen.end(), branch_lengths);
    if (durations) std::copy(S->dt.begin(), S->dt.end(), durations);
    if (rates) std::copy(S->rates.begin(), S->rates.end(), rates);
  });
}

int pg_synth_model(void* handle, double* q, double* pi, int* reversible, double* cat_rates, double* cat_probs) {
  return guarded([&] {
    auto* S = static_cast<Synth*>(handle);
    std::copy(S->q.begin(), S->q.end(), q);
    std::copy(S->pi.begin(), S->pi.end(), pi);
    *reversible = S->reversible;
    std::copy(S->cat_rates.begin(), S->cat_rates.end(), cat_rates);
    std::copy(S->cat_probs.begin(), S->cat_probs.end(), cat_probs);
  });
}

int pg_synth_patterns(void* handle, int8_t* codes, int64_t* weights) {
  return guarded([&] {
    auto* S = static_cast<Synth*>(handle);
    std::copy(S->pcodes.begin(), S->pcodes.end(), codes);
    std::copy(S->weights.begin(), S->weights.end(), weights);
  });
}

void pg_synth_free(void* handle) { delete static_cast<Synth*>(handle); }

}  // extern "C"
