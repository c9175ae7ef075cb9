// The reference-type adapter (include/phylograd_b200/reference_adapter.hpp)
// compiled against stand-ins that carry the reference's own member names and
// accessors (tree.hpp:27-50, alignment.hpp:129-238 with dense m x P tip
// partials, substitution.hpp:23-51/:126-134) — Eigen is not in this image, so
// the stand-ins provide the operator()(i, j) / operator[] / rows() / cols()
// surface the adapter reads.  Reads an instance in tests/cpp/facade_config.cpp's
// format, builds the reference-shaped objects, runs make_engine +
// branch_gradient and writes f64 logL, grad[2N-2], int32 shard_count.
//
//   adapter_test in.bin out.bin
#include <array>
#include <cstdio>
#include <string>
#include <unordered_map>
#include <vector>

#include "phylograd_b200/reference_adapter.hpp"

namespace phylograd {  // reference-shaped stand-ins
struct Vec {
  std::vector<double> v;
  double operator[](int i) const { return v[size_t(i)]; }
  long size() const { return long(v.size()); }
};
struct Mat {  // column-major like Eigen::MatrixXd
  int r = 0, c = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(int rows, int cols) : r(rows), c(cols), v(size_t(rows) * size_t(cols), 0.0) {}
  double operator()(int i, int j) const { return v[size_t(j) * size_t(r) + size_t(i)]; }
  double& operator()(int i, int j) { return v[size_t(j) * size_t(r) + size_t(i)]; }
  int rows() const { return r; }
  int cols() const { return c; }
};
struct Tree {
  int tip_count = 0;
  std::vector<std::string> labels;
  std::vector<int> parent;
  std::vector<std::array<int, 2>> children;
  std::vector<double> branch_length;
  std::vector<double> node_time;
  std::vector<int> post_order, pre_order;
  int node_count() const { return 2 * tip_count - 1; }
  int branch_count() const { return node_count() - 1; }
};
class SitePatternAlignment {
 public:
  int state_count() const { return m_; }
  int pattern_count() const { return int(weights_.size()); }
  const std::vector<std::string>& taxa() const { return taxa_; }
  const std::vector<long>& weights() const { return weights_; }
  const Mat& tip_partials(int taxon_index) const { return tip_partials_[size_t(taxon_index)]; }
  int m_ = 4;
  std::vector<std::string> taxa_;
  std::vector<long> weights_;
  std::vector<Mat> tip_partials_;
};
class SubstitutionModel {
 public:
  int state_count() const { return m_; }
  const Vec& root_distribution() const { return pi_; }
  bool reversible() const { return rev_; }
  const Mat& generator(int branch) const {
    auto it = branch_q_.find(branch);
    return it == branch_q_.end() ? q_ : it->second;
  }
  int m_ = 4;
  Mat q_;
  Vec pi_;
  bool rev_ = true;
  std::unordered_map<int, Mat> branch_q_;
};
struct RateCategories {
  Vec rates, probs;
  int count() const { return int(rates.size()); }
};
}  // namespace phylograd

template <class T>
static void rd(FILE* f, T* p, size_t n) {
  if (n && std::fread(p, sizeof(T), n, f) != n) throw std::runtime_error("adapter_test: short input");
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  try {
    FILE* f = std::fopen(argv[1], "rb");
    if (!f) throw std::runtime_error("adapter_test: cannot open input");
    int32_t hdr[6];
    rd(f, hdr, 6);
    const int N = hdr[0], m = hdr[1], L = hdr[2], P = hdr[3];
    const int n = 2 * N - 1, B = n - 1;
    phylograd::Tree tree;
    tree.tip_count = N;
    tree.parent.resize(size_t(n + 1));
    std::vector<int32_t> ch(size_t(2 * (n + 1)));
    tree.post_order.resize(size_t(n));
    rd(f, tree.parent.data(), tree.parent.size());
    rd(f, ch.data(), ch.size());
    rd(f, tree.post_order.data(), tree.post_order.size());
    tree.children.resize(size_t(n + 1));
    for (int i = 0; i <= n; ++i) tree.children[size_t(i)] = {ch[size_t(2 * i)], ch[size_t(2 * i + 1)]};
    tree.branch_length.assign(size_t(n + 1), 0.0);
    rd(f, tree.branch_length.data() + 1, size_t(B));
    tree.labels.assign(size_t(n + 1), "");
    for (int t = 1; t <= N; ++t) tree.labels[size_t(t)] = "t" + std::to_string(t);
    phylograd::SubstitutionModel model;
    model.m_ = m;
    model.q_ = phylograd::Mat(m, m);
    std::vector<double> q(size_t(m) * m);
    rd(f, q.data(), q.size());
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) model.q_(i, j) = q[size_t(i) * m + j];
    model.pi_.v.resize(size_t(m));
    rd(f, model.pi_.v.data(), size_t(m));
    model.rev_ = hdr[4] != 0;
    phylograd::RateCategories cats;
    cats.rates.v.resize(size_t(L));
    cats.probs.v.resize(size_t(L));
    rd(f, cats.rates.v.data(), size_t(L));
    rd(f, cats.probs.v.data(), size_t(L));
    // reference alignment: taxa in REVERSED order (binding by label, engine.hpp:66-71),
    // dense 0/1 tip partials, all-ones for missing
    phylograd::SitePatternAlignment aln;
    aln.m_ = m;
    aln.taxa_.resize(size_t(N));
    aln.tip_partials_.assign(size_t(N), phylograd::Mat(m, P));
    std::vector<int8_t> row(static_cast<size_t>(P));
    for (int t = 0; t < N; ++t) {
      rd(f, row.data(), size_t(P));
      const size_t r = size_t(N - 1 - t);
      aln.taxa_[r] = "t" + std::to_string(t + 1);
      for (int p = 0; p < P; ++p)
        for (int j = 0; j < m; ++j)
          aln.tip_partials_[r](j, p) = row[size_t(p)] < 0 ? 1.0 : (row[size_t(p)] == j ? 1.0 : 0.0);
    }
    std::vector<int64_t> w(static_cast<size_t>(P));
    rd(f, w.data(), size_t(P));
    aln.weights_.assign(w.begin(), w.end());
    std::fclose(f);

    auto engine = phylograd_b200::make_engine(tree, aln, model, cats);
    const auto rep = engine->branch_gradient();
    FILE* o = std::fopen(argv[2], "wb");
    std::fwrite(&rep.log_likelihood, 8, 1, o);
    std::fwrite(rep.branch_gradient.data(), 8, size_t(B), o);
    const int32_t shards = engine->shard_count();
    std::fwrite(&shards, 4, 1, o);
    std::fclose(o);
    std::printf("adapter_test: %d tips, %d patterns, logL %.12f\n", N, P, rep.log_likelihood);
  } catch (const std::exception& e) {
    std::printf("FAIL: %s\n", e.what());
    return 1;
  }
  return 0;
}
