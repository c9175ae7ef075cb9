// phylograd-b200 C++ facade: the reference's LikelihoodEngine surface
// (/root/reference/proj/include/phylograd/engine.hpp:33-438) rebuilt on the
// C-ABI in include/phylograd_b200.h.  A phylograd user swaps
//     #include "phylograd/engine.hpp"        -> #include "phylograd_b200/engine.hpp"
//     phylograd::LikelihoodEngine            -> phylograd_b200::LikelihoodEngine
// and keeps the call pattern: construct from tree / alignment / model /
// categories, set_branch_lengths, log_likelihood, branch_gradient(with_hessian).
// Setup types are plain structs (no Eigen): vectors of doubles / ints with the
// reference's numbering (tips 1..N, root 2N-1, branch index node-1).
// Errors are rethrown as the reference's exception types with its messages.
#pragma once

#include <algorithm>
#include <cmath>
#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../phylograd_b200.h"

namespace phylograd_b200 {

struct NewickError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == PG_OK) return;
  const std::string msg = pg_last_error();
  switch (rc) {
    case PG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case PG_ERR_LOGIC: throw std::logic_error(msg);
    case PG_ERR_NEWICK: throw NewickError(msg);
    case PG_ERR_NOT_SUPPORTED: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// tree.hpp:27-50
struct Tree {
  int tip_count = 0;
  std::vector<std::string> labels;           // [2N], tips 1..N
  std::vector<int32_t> parent;               // [2N], parent[root] = 0
  std::vector<std::array<int32_t, 2>> children;  // [2N]
  std::vector<double> branch_length;         // [2N], [root] unused
  std::vector<int32_t> post_order;           // [2N-1]
  int node_count() const { return 2 * tip_count - 1; }
  int root() const { return node_count(); }
  int branch_count() const { return node_count() - 1; }
  bool is_tip(int n) const { return n >= 1 && n <= tip_count; }
};

// tree.hpp:284-289
inline Tree parse_newick(const std::string& text) {
  int nt = 0;
  check(pg_newick_parse(text.c_str(), &nt, nullptr, nullptr, nullptr, nullptr, nullptr, 0));
  Tree t;
  t.tip_count = nt;
  const int n = 2 * nt - 1;
  std::vector<int32_t> ch(size_t(2 * (n + 1)));
  t.parent.resize(size_t(n + 1));
  t.branch_length.resize(size_t(n + 1));
  t.post_order.resize(size_t(n));
  std::string buf(text.size() + size_t(nt) + 16, '\0');
  check(pg_newick_parse(text.c_str(), &nt, t.parent.data(), ch.data(), t.branch_length.data(), t.post_order.data(),
                        buf.data(), int64_t(buf.size())));
  t.children.resize(size_t(n + 1));
  for (int i = 0; i <= n; ++i) t.children[size_t(i)] = {ch[size_t(2 * i)], ch[size_t(2 * i + 1)]};
  t.labels.assign(size_t(n + 1), "");
  size_t off = 0;
  for (int i = 1; i <= nt; ++i) {
    t.labels[size_t(i)] = std::string(buf.c_str() + off);
    off += t.labels[size_t(i)].size() + 1;
  }
  return t;
}

// alignment.hpp:129-238 in compact form: per taxon, int8 codes per pattern
// (state, -1 missing, m+a ambiguity class a), integer weights.
struct SitePatternAlignment {
  int state_count = 4;
  std::vector<std::string> taxa;
  std::vector<std::vector<int8_t>> codes;  // [taxon][pattern]
  std::vector<int64_t> weights;
  std::vector<double> ambiguity;           // [A][m]
  int pattern_count() const { return int(weights.size()); }
  int taxon_index(const std::string& name) const {
    for (size_t i = 0; i < taxa.size(); ++i)
      if (taxa[i] == name) return int(i);
    return -1;
  }

  // alignment.hpp:186-229 (first-occurrence order, bit-exact)
  static SitePatternAlignment from_codes(std::vector<std::string> taxa, const std::vector<std::vector<int>>& codes,
                                         int state_count) {
    if (codes.size() != taxa.size()) throw std::invalid_argument("alignment: taxa/codes mismatch");
    if (taxa.empty()) throw std::invalid_argument("alignment: no records");
    const int64_t sites = int64_t(codes[0].size());
    std::vector<int32_t> flat(taxa.size() * size_t(sites));
    for (size_t r = 0; r < taxa.size(); ++r) {
      if (int64_t(codes[r].size()) != sites) throw std::invalid_argument("alignment: ragged code rows");
      for (int64_t s = 0; s < sites; ++s) flat[r * size_t(sites) + size_t(s)] = codes[r][size_t(s)];
    }
    void* h = nullptr;
    int P = 0;
    check(pg_compress_codes(int(taxa.size()), sites, flat.data(), state_count, &h, &P));
    std::vector<int32_t> pc(taxa.size() * size_t(P));
    SitePatternAlignment out;
    out.weights.resize(size_t(P));
    const int rc = pg_compress_result(h, pc.data(), out.weights.data(), nullptr);
    pg_compress_free(h);
    check(rc);
    out.state_count = state_count;
    out.taxa = std::move(taxa);
    out.codes.assign(out.taxa.size(), std::vector<int8_t>(size_t(P)));
    for (size_t r = 0; r < out.taxa.size(); ++r)
      for (int p = 0; p < P; ++p) out.codes[r][size_t(p)] = int8_t(pc[r * size_t(P) + size_t(p)]);
    return out;
  }

  // The same compression on GPU `device` (pg_compress_codes_gpu), for
  // alignments too large for the host path; bit-identical result.  codes is
  // row-major [taxa][sites] int8 (-1 missing).
  static SitePatternAlignment from_codes_gpu(std::vector<std::string> taxa, const std::vector<int8_t>& codes,
                                             int64_t sites, int state_count, int device = 0) {
    if (taxa.empty()) throw std::invalid_argument("alignment: no records");
    if (int64_t(codes.size()) != int64_t(taxa.size()) * sites)
      throw std::invalid_argument("alignment: taxa/codes mismatch");
    void* h = nullptr;
    int P = 0;
    check(pg_compress_codes_gpu(int(taxa.size()), sites, codes.data(), 0, state_count, device, &h, &P));
    std::vector<int8_t> pc(taxa.size() * size_t(P));
    SitePatternAlignment out;
    out.weights.resize(size_t(P));
    const int rc = pg_compress_result_gpu(h, pc.data(), out.weights.data(), nullptr, nullptr);
    pg_compress_free_gpu(h);
    check(rc);
    out.state_count = state_count;
    out.taxa = std::move(taxa);
    out.codes.assign(out.taxa.size(), std::vector<int8_t>(size_t(P)));
    for (size_t r = 0; r < out.taxa.size(); ++r)
      std::copy(pc.begin() + std::ptrdiff_t(r * size_t(P)), pc.begin() + std::ptrdiff_t((r + 1) * size_t(P)),
                out.codes[r].begin());
    return out;
  }
};

// substitution.hpp:23-51
struct RateCategories {
  std::vector<double> rates{1.0}, probs{1.0};
  int count() const { return int(rates.size()); }
  static RateCategories single() { return {}; }
};

// substitution.hpp:55-68
inline RateCategories discrete_gamma_categories(double alpha, int count) {
  RateCategories c;
  c.rates.assign(size_t(count > 0 ? count : 1), 0.0);
  c.probs.assign(c.rates.size(), 0.0);
  check(pg_discrete_gamma(alpha, count, c.rates.data(), c.probs.data()));
  return c;
}

// substitution.hpp:77-219 (generators; P(t) is formed on the GPU)
struct SubstitutionModel {
  int state_count = 4;
  std::vector<double> q;   // row-major m x m
  std::vector<double> pi;  // root distribution
  bool reversible = true;
  std::map<int, std::vector<double>> branch_q;
  void set_branch_generator(int branch, std::vector<double> g) { branch_q[branch] = std::move(g); }
};

// engine.hpp:33-37
struct EngineOptions {
  double rescaling_threshold = 1e-150;
  bool force_rescaling = false;
  bool disable_rescaling = false;
  int device = 0;
  bool capture_partials = false;  // keep per-node partials for the engine.hpp:134-141 accessors (debug)
  // Multi-GPU from one process (pg_create_multi): non-empty -> patterns shard
  // contiguously over these devices, one reduction of [logL, g, h] per
  // evaluation: PG_REDUCE_NCCL (ncclAllReduce) or PG_REDUCE_FIXED_ORDER
  // (rank-order sum on the first device, bit-reproducible).
  std::vector<int> devices;
  int reduce_mode = PG_REDUCE_NCCL;
};

// clock.hpp:140-152 (likelihood part of the unconstrained gradient) and
// clock.hpp:199-213 (node_time_gradient)
struct ClockGradient {
  double log_likelihood = 0.0;
  double dlog_mu = 0.0;                // sum_i b_i g_i
  std::vector<double> dlog_epsilon;    // b_i g_i, entry node-1
  std::vector<double> node_time;       // d logL / d t_k, k = N+1..2N-1 at entry k-N-1
};

// engine.hpp:39-45
struct GradientReport {
  double log_likelihood = 0.0;
  std::vector<double> branch_gradient;   // entry node-1
  std::vector<double> hessian_diagonal;  // empty unless requested
  int pattern_count = 0;
  int category_count = 0;
};

// engine.hpp:47-438
class LikelihoodEngine {
 public:
  LikelihoodEngine(const Tree& tree, const SitePatternAlignment& alignment, const SubstitutionModel& model,
                   RateCategories categories, EngineOptions options = {})
      : tree_(tree), categories_(std::move(categories)) {
    const int m = model.state_count;
    if (alignment.state_count != m) throw std::invalid_argument("engine: alignment/model state counts differ");
    if (int(alignment.taxa.size()) != tree.tip_count)
      throw std::invalid_argument("engine: alignment must carry exactly one record per tree tip");
    std::vector<int8_t> codes(size_t(tree.tip_count) * size_t(alignment.pattern_count()));
    for (int t = 1; t <= tree.tip_count; ++t) {
      const int row = alignment.taxon_index(tree.labels[size_t(t)]);
      if (row < 0) throw std::invalid_argument("engine: tree tip '" + tree.labels[size_t(t)] + "' not found in alignment");
      std::copy(alignment.codes[size_t(row)].begin(), alignment.codes[size_t(row)].end(),
                codes.begin() + long(size_t(t - 1) * size_t(alignment.pattern_count())));
    }
    pg_options o;
    pg_default_options(&o);
    o.rescaling_threshold = options.rescaling_threshold;
    o.force_rescaling = options.force_rescaling;
    o.disable_rescaling = options.disable_rescaling;
    o.device = options.device;
    o.capture_partials = options.capture_partials ? 1 : 0;
    // the handle is owned by a guard until construction finishes, so a
    // setter that throws does not leak the engine and its device buffers
    pg_engine* raw = nullptr;
    if (options.devices.empty())
      check(pg_create(&o, &raw));
    else
      check(pg_create_multi(&o, int(options.devices.size()), options.devices.data(), options.reduce_mode, &raw));
    std::unique_ptr<pg_engine, void (*)(pg_engine*)> guard(raw, pg_destroy);
    h_ = raw;
    std::vector<int32_t> ch(size_t(2 * (tree.node_count() + 1)));
    for (int i = 0; i <= tree.node_count(); ++i) {
      ch[size_t(2 * i)] = tree.children[size_t(i)][0];
      ch[size_t(2 * i + 1)] = tree.children[size_t(i)][1];
    }
    check(pg_set_topology(h_, tree.tip_count, tree.parent.data(), ch.data(), tree.post_order.data()));
    check(pg_set_patterns(h_, m, alignment.pattern_count(), codes.data(),
                          int(alignment.ambiguity.size() / size_t(m)), alignment.ambiguity.data(),
                          alignment.weights.data()));
    check(pg_set_model(h_, m, model.q.data(), model.pi.data(), model.reversible));
    for (const auto& [br, g] : model.branch_q) check(pg_set_branch_generator(h_, br, g.data()));
    check(pg_set_categories(h_, categories_.count(), categories_.rates.data(), categories_.probs.data()));
    std::vector<double> b(tree.branch_length.begin() + 1, tree.branch_length.begin() + tree.node_count());
    set_branch_lengths(b);
    guard.release();
    patterns_ = alignment.pattern_count();
    states_ = m;
    tip_codes_ = std::move(codes);
    ambiguity_ = alignment.ambiguity;
    weights_ = alignment.weights;
  }
  ~LikelihoodEngine() { pg_destroy(h_); }
  LikelihoodEngine(const LikelihoodEngine&) = delete;
  LikelihoodEngine& operator=(const LikelihoodEngine&) = delete;

  const Tree& tree() const { return tree_; }
  const RateCategories& categories() const { return categories_; }
  std::vector<double> branch_lengths() const {
    std::vector<double> b(size_t(tree_.branch_count()));
    check(pg_get_branch_lengths(h_, b.data()));
    return b;
  }
  void set_branch_lengths(const std::vector<double>& b) {
    if (int(b.size()) != tree_.branch_count()) throw std::invalid_argument("engine: branch length vector has wrong size");
    check(pg_set_branch_lengths(h_, b.data()));
  }
  void set_clock_durations(const std::vector<double>& dt) { check(pg_set_clock_durations(h_, dt.data())); }
  std::uint64_t node_visits() const { return pg_node_visits(h_); }
  void reset_node_visits() { pg_reset_node_visits(h_); }
  void invalidate_caches() { pg_invalidate_caches(h_); }

  double log_likelihood() { return eval(PG_EVAL_LOGL).log_likelihood; }
  void post_order_pass() { eval(PG_EVAL_LOGL | PG_EVAL_POST_PASS); }
  void pre_order_pass(bool with_hessian_diagonal = false) {
    eval(PG_EVAL_GRAD | PG_EVAL_REQUIRE_POST | (with_hessian_diagonal ? PG_EVAL_HESS : 0));
  }
  GradientReport branch_gradient(bool with_hessian_diagonal = false) {
    return eval(PG_EVAL_GRAD | (with_hessian_diagonal ? PG_EVAL_HESS : 0));
  }
  std::vector<double> hessian_diagonal() { return branch_gradient(true).hessian_diagonal; }
  // clock.hpp:146-152 / cli.hpp:437-438: d logL / d r_i = dt_i g_i
  GradientReport rate_gradient(bool with_hessian_diagonal = false) {
    return eval(PG_EVAL_RATE_GRAD | (with_hessian_diagonal ? PG_EVAL_HESS : 0));
  }
  // The relaxed-clock chain rule on the GPU at the current lengths
  // b_i = r_i dt_i; rates r_i = mu eps_i (nullptr: b_i / dt_i from the
  // clock durations).
  ClockGradient clock_gradient(const std::vector<double>* rates = nullptr) {
    ClockGradient c;
    c.dlog_epsilon.assign(size_t(tree_.branch_count()), 0.0);
    c.node_time.assign(size_t(tree_.tip_count - 1), 0.0);
    if (rates && int(rates->size()) != tree_.branch_count()) throw std::invalid_argument("clock: need one rate per branch");
    check(pg_clock_gradient(h_, rates ? rates->data() : nullptr, &c.log_likelihood, &c.dlog_mu, c.dlog_epsilon.data(),
                            c.node_time.data()));
    return c;
  }
  int shard_count() const {
    int n = 1;
    check(pg_group_info(h_, &n, nullptr, nullptr));
    return n;
  }
  pg_engine* handle() { return h_; }

  // engine.hpp:134-141 (needs EngineOptions::capture_partials): partials as
  // column-major m x P (entry (s, p) at p * m + s), log scalers per pattern.
  // Tips: their 0/1 (or ambiguity) partials and zero scalers, like the reference.
  std::vector<double> post_partial(int node, int category) {
    if (node >= 1 && node <= tree_.tip_count) return tip_partial(node);
    return partials(node, category).post;
  }
  std::vector<double> pre_partial(int node, int category) { return partials(node, category).pre; }
  std::vector<double> post_scaler(int node) {
    if (node >= 1 && node <= tree_.tip_count) return std::vector<double>(size_t(patterns_), 0.0);
    return partials(node, 0).post_scaler;
  }
  std::vector<double> pre_scaler(int node) { return partials(node, 0).pre_scaler; }
  // engine.hpp:168-180: logL from the partials meeting at `node` (Eq. 8)
  double log_likelihood_at_node(int node) {
    const std::vector<int64_t>& weights = weights_;
    branch_gradient();
    const int m = states_, P = patterns_;
    std::vector<double> mix(size_t(P), 0.0);
    for (int l = 0; l < categories_.count(); ++l) {
      const auto a = post_partial(node, l), b = pre_partial(node, l);
      for (int p = 0; p < P; ++p) {
        double d = 0.0;
        for (int i = 0; i < m; ++i) d += a[size_t(p) * m + i] * b[size_t(p) * m + i];
        mix[size_t(p)] += categories_.probs[size_t(l)] * d;
      }
    }
    const auto sa = post_scaler(node), sb = pre_scaler(node);
    double ll = 0.0;
    for (int p = 0; p < P; ++p)
      ll += double(weights[size_t(p)]) * (std::log(mix[size_t(p)]) + sa[size_t(p)] + sb[size_t(p)]);
    return ll;
  }

 private:
  struct NodePartials {
    std::vector<double> post, pre, post_scaler, pre_scaler;
  };
  NodePartials partials(int node, int category) {
    NodePartials r;
    const size_t mp = size_t(states_) * size_t(patterns_);
    r.post.resize(mp);
    r.pre.resize(mp);
    r.post_scaler.resize(size_t(patterns_));
    r.pre_scaler.resize(size_t(patterns_));
    check(pg_get_partials(h_, node, category, r.post.data(), r.pre.data(), r.post_scaler.data(),
                          r.pre_scaler.data()));
    return r;
  }
  std::vector<double> tip_partial(int tip) const {
    const int m = states_, P = patterns_;
    std::vector<double> v(size_t(m) * size_t(P), 0.0);
    for (int p = 0; p < P; ++p) {
      const int c = tip_codes_[size_t(tip - 1) * size_t(P) + size_t(p)];
      for (int i = 0; i < m; ++i)
        v[size_t(p) * m + i] = c < 0 ? 1.0 : c < m ? (i == c ? 1.0 : 0.0) : ambiguity_[size_t(c - m) * m + i];
    }
    return v;
  }

  GradientReport eval(int flags) {
    GradientReport r;
    r.branch_gradient.assign(size_t(tree_.branch_count()), 0.0);
    std::vector<double> h(size_t(tree_.branch_count()), 0.0);
    check(pg_evaluate(h_, flags, &r.log_likelihood, r.branch_gradient.data(), h.data()));
    if (flags & PG_EVAL_HESS) r.hessian_diagonal = std::move(h);
    if (!(flags & (PG_EVAL_GRAD | PG_EVAL_RATE_GRAD))) r.branch_gradient.clear();
    r.pattern_count = patterns_;
    r.category_count = categories_.count();
    return r;
  }

  Tree tree_;
  RateCategories categories_;
  pg_engine* h_ = nullptr;
  int patterns_ = 0, states_ = 0;
  std::vector<int8_t> tip_codes_;  // [tip][pattern] (for the tip partial accessors)
  std::vector<double> ambiguity_;  // [class][m]
  std::vector<int64_t> weights_;   // pattern multiplicities
};

}  // namespace phylograd_b200
