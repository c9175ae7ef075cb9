// Seeded synthetic workloads (input generation only; see pg_workloads.h).
// Yule trees numbered like parse_newick (tree.hpp:144-289), model draws as the
// BASELINE.json configs state, forward simulation (alignment.hpp:243-286) and
// first-occurrence compression (alignment.hpp:186-229).  Built into its own
// library, workloads/_build/libpg_workloads.so, with hidden visibility except
// for the pgw_* entry points.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../paper_1905_12146_b200/csrc/pg_common.hpp"
#include "../paper_1905_12146_b200/csrc/pg_hostutil.hpp"
#include "../paper_1905_12146_b200/csrc/pg_simulate.hpp"
#include "pg_workloads.h"

#define PGW_API __attribute__((visibility("default")))

namespace pg {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& s) { g_last_error = s; }

namespace {
using namespace hostutil;

// substitution.hpp:55-68: L equiprobable categories at the bin medians of
// Gamma(alpha, alpha), rescaled to mean one.
void discrete_gamma(double alpha, int count, double* rates, double* probs) {
  double s = 0;
  for (int l = 0; l < count; ++l) {
    rates[l] = gamma_quantile(alpha, 1.0, (2.0 * l + 1.0) / (2.0 * count)) / alpha;
    s += rates[l];
  }
  for (int l = 0; l < count; ++l) {
    rates[l] *= double(count) / s;
    probs[l] = 1.0 / count;
  }
}

struct Synth {
  pgw_spec spec{};
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

// Host P(t) for simulation (pg_linalg.cpp): shared with the GPU simulator.
struct HostP : HostTransition {
  explicit HostP(const Synth& S) : HostTransition(S.m, S.q, S.pi, S.reversible) {}
  HostP(int m_, const std::vector<double>& q_, const std::vector<double>& pi_, int reversible)
      : HostTransition(m_, q_, pi_, reversible) {}
};

void simulate_blocked(Synth& S);

// First-occurrence compression of the simulated columns into S.pcodes / S.weights.
void compress_into(Synth& S, const std::vector<int8_t>& codes, int T) {
  const int N = S.N;
  const int64_t sites = S.spec.sites;
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

// alignment.hpp:243-286 in the reference's draw order: one mt19937_64(seed)
// stream, uniform_real_distribution<double>(0, 1), the category drawn first
// (draw(categories.probs)), then every node in pre-order (reverse of the
// post-order, tree.hpp:76): the root from pi, the rest from the row of
// P(b_node c_l) of the parent's state, each by the linear cumulative scan of
// alignment.hpp:258-266 (acc += w_j; u < acc; the last index otherwise).
// The per-(node, category) P(t) follows substitution.hpp:147-160 (t = b c,
// t = 0 -> I, eigen or Pade, clamp >= 0).  A state differs from the
// reference's only if u falls within rounding of a cumulative boundary.
void simulate_reference(int N, const int32_t* parent, const int32_t* post, int m, const HostP& hp, int L,
                        const double* cat_rates, const double* cat_probs, const double* pi, const double* blen,
                        int64_t sites, uint64_t seed, int8_t* out /* [N][sites] */) {
  const int n = 2 * N - 1;
  std::vector<std::vector<double>> P(size_t(n + 1) * L);
  for (int v = 1; v < n; ++v)
    for (int l = 0; l < L; ++l) P[size_t(v) * L + l] = hp(blen[v - 1] * cat_rates[l]);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  auto draw = [&](const double* w, int k) {
    const double u = unif(rng);
    double acc = 0.0;
    for (int j = 0; j < k - 1; ++j) {
      acc += w[j];
      if (u < acc) return j;
    }
    return k - 1;
  };
  std::vector<int> state(size_t(n + 1), 0);
  for (int64_t s = 0; s < sites; ++s) {
    const int l = draw(cat_probs, L);
    for (int k = n - 1; k >= 0; --k) {
      const int v = post[k];
      if (v == n) state[size_t(v)] = draw(pi, m);
      else state[size_t(v)] = draw(&P[size_t(v) * L + l][size_t(state[size_t(parent[v])]) * m], m);
      if (v <= N) out[size_t(v - 1) * size_t(sites) + size_t(s)] = int8_t(state[size_t(v)]);
    }
  }
}

// Counter-based per-site stream (pg_simulate.hpp): the CPU twin of
// pg_simulate_states_gpu.  out: [N][sites].
void simulate_counter(int N, const int32_t* parent, const int32_t* post, int m, const HostTransition& P, int L,
                      const double* cat_rates, const double* cat_probs, const double* pi, const double* blen,
                      int64_t sites, uint64_t seed, double gap, int threads, int8_t* out) {
  const int n = 2 * N - 1;
  std::vector<double> cdf, root, cat;
  build_sim_tables(N, m, L, P, cat_rates, cat_probs, pi, blen, cdf, root, cat);
  const uint64_t D = sim::draws_per_site(N);
  parallel_for(sites, hw_threads(threads), [&](int64_t a, int64_t b) {
    std::vector<int> state(size_t(n + 1), 0);
    for (int64_t s = a; s < b; ++s) {
      const int l = sim::pick(cat.data(), L, sim::unit(seed, uint64_t(s), D, 0));
      for (int j = 0; j < n; ++j) {
        const int v = post[n - 1 - j];
        const double u = sim::unit(seed, uint64_t(s), D, uint64_t(1 + j));
        state[size_t(v)] = v == n ? sim::pick(root.data(), m, u)
                                  : sim::pick(&cdf[((size_t(v) * L + l) * m + size_t(state[size_t(parent[v])])) * m], m, u);
        if (v <= N) out[size_t(v - 1) * size_t(sites) + size_t(s)] = int8_t(state[size_t(v)]);
      }
      if (gap > 0.0)
        for (int t = 0; t < N; ++t)
          if (sim::unit(seed, uint64_t(s), D, uint64_t(1 + n + t)) < gap) out[size_t(t) * size_t(sites) + size_t(s)] = -1;
    }
  });
}

void simulate(Synth& S) {
  if (S.spec.sim == PGW_SIM_NONE) return;
  if (S.spec.sim == PGW_SIM_COUNTER) {
    const int N = S.N, T = hw_threads(S.spec.threads);
    const int64_t sites = S.spec.sites;
    HostP hp(S);
    std::vector<int8_t> codes(size_t(N) * size_t(sites));
    simulate_counter(N, S.parent.data(), S.post.data(), S.m, hp, S.L, S.cat_rates.data(), S.cat_probs.data(),
                     S.pi.data(), S.blen.data(), sites, S.spec.seed, S.spec.gap_fraction, T, codes.data());
    compress_into(S, codes, T);
    return;
  }
  if (S.spec.sim == PGW_SIM_REFERENCE) {
    const int N = S.N, T = hw_threads(S.spec.threads);
    const int64_t sites = S.spec.sites;
    HostP hp(S);
    std::vector<int8_t> codes(size_t(N) * size_t(sites));
    simulate_reference(N, S.parent.data(), S.post.data(), S.m, hp, S.L, S.cat_rates.data(), S.cat_probs.data(),
                       S.pi.data(), S.blen.data(), sites, S.spec.seed, codes.data());
    if (S.spec.gap_fraction > 0) {
      // gaps from their own sequential stream, column by column
      uint64_t sm = S.spec.seed ^ 0x6761707366726163ull;
      std::mt19937_64 grng(splitmix(sm));
      std::bernoulli_distribution gap(S.spec.gap_fraction);
      for (int64_t s = 0; s < sites; ++s)
        for (int t = 0; t < N; ++t)
          if (gap(grng)) codes[size_t(t) * size_t(sites) + size_t(s)] = -1;
    }
    compress_into(S, codes, T);
    return;
  }
  simulate_blocked(S);
}

// Independent mt19937_64 streams per block of 4096 sites (deterministic for
// any thread count).
void simulate_blocked(Synth& S) {

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

  compress_into(S, codes, T);
}
}  // namespace
}  // namespace pg

using namespace pg;

extern "C" {

PGW_API const char* pgw_last_error(void) { return g_last_error.c_str(); }

PGW_API int pgw_create(const pgw_spec* spec, void** handle, int* pattern_count, int* state_count) {
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
      discrete_gamma(spec->gamma_alpha, S->L, S->cat_rates.data(), S->cat_probs.data());
    }
    simulate(*S);
    *pattern_count = int(S->weights.size());
    *state_count = S->m;
    *handle = S.release();
  });
}

PGW_API int pgw_tree(void* handle, int32_t* parent, int32_t* children, int32_t* post_order, double* branch_lengths,
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

PGW_API int pgw_model(void* handle, double* q, double* pi, int* reversible, double* cat_rates, double* cat_probs) {
  return guarded([&] {
    auto* S = static_cast<Synth*>(handle);
    std::copy(S->q.begin(), S->q.end(), q);
    std::copy(S->pi.begin(), S->pi.end(), pi);
    *reversible = S->reversible;
    std::copy(S->cat_rates.begin(), S->cat_rates.end(), cat_rates);
    std::copy(S->cat_probs.begin(), S->cat_probs.end(), cat_probs);
  });
}

PGW_API int pgw_patterns(void* handle, int8_t* codes, int64_t* weights) {
  return guarded([&] {
    auto* S = static_cast<Synth*>(handle);
    std::copy(S->pcodes.begin(), S->pcodes.end(), codes);
    std::copy(S->weights.begin(), S->weights.end(), weights);
  });
}

PGW_API void pgw_free(void* handle) { delete static_cast<Synth*>(handle); }

PGW_API int pgw_simulate_states(int tip_count, const int32_t* parent, const int32_t* post_order, int state_count,
                                const double* q, const double* pi, int reversible, int category_count,
                                const double* cat_rates, const double* cat_probs, const double* branch_lengths,
                                int64_t sites, uint64_t seed, int8_t* states) {
  return guarded([&] {
    if (sites < 1) throw std::invalid_argument("simulate: site_count must be >= 1");
    if (tip_count < 2 || state_count < 2 || category_count < 1) throw std::invalid_argument("simulate: bad sizes");
    for (int i = 0; i < 2 * tip_count - 2; ++i)
      if (!(branch_lengths[i] >= 0.0)) throw std::invalid_argument("transition matrix: negative branch length");
    const int m = state_count;
    HostP hp(m, std::vector<double>(q, q + size_t(m) * m), std::vector<double>(pi, pi + m), reversible);
    simulate_reference(tip_count, parent, post_order, m, hp, category_count, cat_rates, cat_probs, pi,
                       branch_lengths, sites, seed, states);
  });
}

PGW_API int pgw_simulate_states_counter(int tip_count, const int32_t* parent, const int32_t* post_order,
                                        int state_count, const double* q, const double* pi, int reversible,
                                        int category_count, const double* cat_rates, const double* cat_probs,
                                        const double* branch_lengths, int64_t sites, uint64_t seed,
                                        double gap_fraction, int threads, int8_t* states) {
  return guarded([&] {
    if (sites < 1) throw std::invalid_argument("simulate: site_count must be >= 1");
    if (tip_count < 2 || state_count < 2 || state_count > 127 || category_count < 1)
      throw std::invalid_argument("simulate: bad sizes");
    if (!(gap_fraction >= 0.0 && gap_fraction < 1.0)) throw std::invalid_argument("simulate: gap fraction in [0, 1)");
    for (int i = 0; i < 2 * tip_count - 2; ++i)
      if (!(branch_lengths[i] >= 0.0)) throw std::invalid_argument("transition matrix: negative branch length");
    const int m = state_count;
    HostTransition P(m, std::vector<double>(q, q + size_t(m) * m), std::vector<double>(pi, pi + m), reversible);
    simulate_counter(tip_count, parent, post_order, m, P, category_count, cat_rates, cat_probs, pi, branch_lengths,
                     sites, seed, gap_fraction, threads, states);
  });
}

}  // extern "C"
