// phylograd-b200: build the engine straight from the reference's OWN setup
// objects (phylograd::Tree, SitePatternAlignment, SubstitutionModel,
// RateCategories — tree.hpp:27-50, alignment.hpp:129-238,
// substitution.hpp:23-51/:77-219), so a caller that already holds them swaps
// only the engine type (engine.hpp:49-51):
//
//     #include "phylograd/engine.hpp"                 // the reference types
//     #include "phylograd_b200/reference_adapter.hpp"
//     auto engine = phylograd_b200::make_engine(tree, alignment, model, cats);
//     engine->set_branch_lengths(b);  auto rep = engine->branch_gradient();
//
// The adapters are templates over the reference types and read them only
// through their public members and accessors; the Eigen members are read with
// operator()(i, j) / operator[](i) / rows() / cols() / size(), so the header
// itself needs no Eigen (tests/cpp/adapter_test.cpp compiles it against
// stand-ins with the reference's member names).
//
// Tip partials become compact codes with the reference's own rule
// (engine.hpp:72-79): a column with sum 1 and max 1 is a state index, an
// all-ones column is "missing" (-1), any other column is an ambiguity class
// (distinct columns deduplicated in first-occurrence order).  Per-branch
// generators are carried over by asking generator(i) for every branch and
// keeping those that differ from generator(0) (substitution.hpp:131-134).
#pragma once

#include <map>
#include <memory>
#include <vector>

#include "engine.hpp"

namespace phylograd_b200 {

template <class RefTree>
Tree from_reference_tree(const RefTree& t) {
  Tree out;
  out.tip_count = t.tip_count;
  out.labels.assign(t.labels.begin(), t.labels.end());
  out.parent.assign(t.parent.begin(), t.parent.end());
  out.children.resize(t.children.size());
  for (size_t i = 0; i < t.children.size(); ++i) out.children[i] = {int32_t(t.children[i][0]), int32_t(t.children[i][1])};
  out.branch_length.assign(t.branch_length.begin(), t.branch_length.end());
  out.post_order.assign(t.post_order.begin(), t.post_order.end());
  return out;
}

template <class RefAln>
SitePatternAlignment from_reference_alignment(const RefAln& a) {
  SitePatternAlignment out;
  const int m = a.state_count(), P = a.pattern_count();
  out.state_count = m;
  out.taxa.assign(a.taxa().begin(), a.taxa().end());
  out.weights.assign(a.weights().begin(), a.weights().end());
  std::map<std::vector<double>, int> classes;  // ambiguity column -> class index
  out.codes.assign(out.taxa.size(), std::vector<int8_t>(size_t(P), 0));
  std::vector<double> col(static_cast<size_t>(m));
  for (size_t r = 0; r < out.taxa.size(); ++r) {
    const auto& tp = a.tip_partials(int(r));  // m x P
    for (int p = 0; p < P; ++p) {
      double sum = 0.0, mx = -1.0;
      int arg = -1;
      bool all_ones = true;
      for (int j = 0; j < m; ++j) {
        const double v = tp(j, p);
        col[size_t(j)] = v;
        sum += v;
        if (v > mx) {
          mx = v;
          arg = j;
        }
        all_ones = all_ones && v == 1.0;
      }
      int code;
      if (sum == 1.0 && mx == 1.0) {
        code = arg;  // engine.hpp:77: unit indicator column
      } else if (all_ones) {
        code = -1;   // alignment.hpp:223-224: missing / gap
      } else {
        auto it = classes.find(col);
        if (it == classes.end()) {
          it = classes.emplace(col, int(classes.size())).first;
          out.ambiguity.insert(out.ambiguity.end(), col.begin(), col.end());
        }
        code = m + it->second;
        if (code > 127) throw std::invalid_argument("alignment: too many ambiguity classes");
      }
      out.codes[r][size_t(p)] = int8_t(code);
    }
  }
  return out;
}

template <class RefModel>
SubstitutionModel from_reference_model(const RefModel& model, int branch_count) {
  SubstitutionModel out;
  const int m = model.state_count();
  out.state_count = m;
  out.reversible = model.reversible();
  auto flat = [&](const auto& q) {
    std::vector<double> v(size_t(m) * m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) v[size_t(i) * m + j] = q(i, j);
    return v;
  };
  out.q = flat(model.generator(0));
  out.pi.resize(size_t(m));
  for (int i = 0; i < m; ++i) out.pi[size_t(i)] = model.root_distribution()[i];
  for (int b = 1; b <= branch_count; ++b) {
    std::vector<double> g = flat(model.generator(b));
    if (g != out.q) out.set_branch_generator(b, std::move(g));
  }
  return out;
}

template <class RefCats>
RateCategories from_reference_categories(const RefCats& c) {
  RateCategories out;
  out.rates.resize(size_t(c.count()));
  out.probs.resize(size_t(c.count()));
  for (int l = 0; l < c.count(); ++l) {
    out.rates[size_t(l)] = c.rates[l];
    out.probs[size_t(l)] = c.probs[l];
  }
  return out;
}

// engine.hpp:49-51 with the reference's own argument types.
template <class RefTree, class RefAln, class RefModel, class RefCats>
std::unique_ptr<LikelihoodEngine> make_engine(const RefTree& tree, const RefAln& alignment, const RefModel& model,
                                              const RefCats& categories, EngineOptions options = {}) {
  return std::make_unique<LikelihoodEngine>(from_reference_tree(tree), from_reference_alignment(alignment),
                                            from_reference_model(model, tree.branch_count()),
                                            from_reference_categories(categories), options);
}

}  // namespace phylograd_b200
