// Host-side setup for phylograd-b200: the data formats either side of the hot
// path.
//
//  * Newick parsing with the reference's integer numbering contract
//    (tree.hpp:144-289): tips 1..N in left-to-right order, internal nodes
//    N+1..2N-1 in completion order, root 2N-1.
//  * Pattern compression in first-occurrence order with integer weights
//    (alignment.hpp:186-229), hash-based and multithreaded instead of the
//    reference's std::map over column vectors; output order is identical.
//  * Discrete-gamma categories (substitution.hpp:55-68).
// The dense linear algebra lives in pg_linalg.cpp; the seeded synthetic
// workloads (input generation only) in workloads/ — a separate library.
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
#include "pg_hostutil.hpp"

namespace pg {

namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& s) { g_last_error = s; }

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
using namespace hostutil;

struct CompressHandle {
  int ntax = 0;
  int64_t sites = 0;
  std::vector<int32_t> codes;
  Compressed<int32_t> c;
};

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


}  // extern "C"
