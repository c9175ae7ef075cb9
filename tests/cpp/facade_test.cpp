// C++ drop-in check: the reference's canonical call pattern (README.md
// "Library sketch"; test_engine.cpp:24-35, :189-204) through the
// phylograd_b200 facade.  Exit code 0 = pass.  Needs a GPU at run time.
#include <cmath>
#include <cstdio>

#include "phylograd_b200/engine.hpp"

using namespace phylograd_b200;

static int failures = 0;
static void expect(bool ok, const char* what) {
  std::printf("%s: %s\n", ok ? "PASS" : "FAIL", what);
  if (!ok) ++failures;
}

int main() {
  Tree tree = parse_newick("(A:0.1,B:0.2);");
  SubstitutionModel jc;
  jc.q.assign(16, 1.0 / 3.0);
  for (int i = 0; i < 4; ++i) jc.q[size_t(i * 4 + i)] = -1.0;
  jc.pi.assign(4, 0.25);
  auto aln = SitePatternAlignment::from_codes({"A", "B"}, {{0}, {1}}, 4);
  {
    // GPU compression through the facade: bit-identical to the host path
    const std::vector<std::vector<int>> cols = {{0, 1, 0, 2, -1, 1, 0}, {3, 3, 3, 1, 2, 3, 3}};
    std::vector<int8_t> flat;
    for (const auto& row : cols)
      for (int c : row) flat.push_back(int8_t(c));
    auto host = SitePatternAlignment::from_codes({"x", "y"}, cols, 4);
    auto dev = SitePatternAlignment::from_codes_gpu({"x", "y"}, flat, 7, 4);
    expect(host.weights == dev.weights && host.codes == dev.codes, "GPU compression matches the host");
  }
  LikelihoodEngine engine(tree, aln, jc, RateCategories::single());
  const double same = 0.25 + 0.75 * std::exp(-4.0 * 0.3 / 3.0);
  const double site = 0.25 * (1.0 - same) / 3.0;
  expect(std::fabs(engine.log_likelihood() - std::log(site)) < 1e-14, "two-taxon JC logL");
  GradientReport r = engine.branch_gradient(true);
  const double g = std::exp(-0.4) / (0.75 * (1.0 - std::exp(-0.4)));
  expect(std::fabs(r.branch_gradient[0] - g) < 1e-12 * g, "two-taxon JC gradient (branch 1)");
  expect(std::fabs(r.branch_gradient[1] - g) < 1e-12 * g, "two-taxon JC gradient (branch 2)");
  expect(r.hessian_diagonal.size() == 2, "hessian requested");
  engine.reset_node_visits();
  engine.invalidate_caches();
  engine.branch_gradient();
  expect(engine.node_visits() == 6, "node visits 2(2N-1)");
  bool threw = false;
  try {
    engine.set_branch_lengths({-0.1, 0.2});
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  expect(threw, "negative length rejected with std::invalid_argument");
  threw = false;
  try {
    Tree other = parse_newick("(A:0.1,Mismatch:0.2);");
    LikelihoodEngine bad(other, aln, jc, RateCategories::single());
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()).find("not found") != std::string::npos;
  }
  expect(threw, "unbound tip -> 'not found'");
  {
    // engine.hpp:134-141 accessors + Eq. 8 node invariance (test_engine.cpp:133-147)
    Tree t5 = parse_newick("((A:0.1,B:0.2):0.05,(C:0.3,(D:0.1,E:0.15):0.2):0.1);");
    auto a5 = SitePatternAlignment::from_codes({"A", "B", "C", "D", "E"},
                                               {{0, 1, 2, 3, -1, 0}, {0, 1, 2, 2, 1, 0}, {1, 1, 2, 3, 0, 3},
                                                {0, 3, 2, 3, 1, 0}, {0, 1, 0, 3, 1, 2}},
                                               4);
    EngineOptions opts;
    opts.capture_partials = true;
    LikelihoodEngine e5(t5, a5, jc, discrete_gamma_categories(0.7, 3), opts);
    const double ll = e5.log_likelihood();
    bool ok = true;
    for (int k = 1; k <= t5.node_count(); ++k)
      ok = ok && std::fabs(e5.log_likelihood_at_node(k) - ll) < 1e-11 * std::fabs(ll);
    expect(ok, "log_likelihood_at_node equals logL at every node");
    expect(e5.post_partial(1, 0).size() == size_t(4 * a5.pattern_count()), "post_partial is m x P");
  }
  auto cats = discrete_gamma_categories(0.5, 4);
  expect(cats.count() == 4 && std::fabs(cats.rates[0] - 0.0290777) < 1e-6, "discrete gamma(0.5, 4)");
  return failures == 0 ? 0 : 1;
}
