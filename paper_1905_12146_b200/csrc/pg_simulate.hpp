// Counter-based forward simulation of alignment columns (alignment.hpp:243-286
// semantics: per site a rate category, then the root state from pi and every
// other node from the row of P(b_node c_l) selected by its parent's state, in
// pre-order).  The reference draws everything from ONE sequential
// mt19937_64 stream, which no parallel machine can reproduce; here draw k of
// site s is splitmix64 at counter s * D + k of the seed (D = 1 + (2N-1) + N
// draws per site: category, nodes in pre-order, per-taxon gap), so every site
// is independent.  The same inline helpers run on the host (workloads/, the
// CPU twin) and on the GPU (pg_simulate.cu), over the same host-built
// cumulative tables, so the two give bit-identical columns.
#pragma once

#include <cstdint>
#include <vector>

#ifdef __CUDACC__
#define PG_SIM_HD __host__ __device__ __forceinline__
#else
#define PG_SIM_HD inline
#endif

namespace pg {
namespace sim {

PG_SIM_HD uint64_t splitmix_at(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ull * (counter + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// uniform in [0, 1) with 53 random bits
PG_SIM_HD double unit(uint64_t seed, uint64_t site, uint64_t per_site, uint64_t k) {
  return double(splitmix_at(seed, site * per_site + k) >> 11) * 0x1.0p-53;
}
// index of the first cumulative entry above u * total (alignment.hpp:258-266 scan)
PG_SIM_HD int pick(const double* c, int k, double u) {
  const double v = u * c[k - 1];
  int j = 0;
  while (j < k - 1 && !(v < c[j])) ++j;
  return j;
}
// draws per site: category, 2N-1 nodes, N gaps
PG_SIM_HD uint64_t draws_per_site(int N) { return uint64_t(1 + (2 * N - 1) + N); }

}  // namespace sim

// Host tables: cumulative rows of P(b_v c_l) per (node v = 1..2N-2, category,
// parent state) -> cdf[((v L + l) m + i) m + j]; root and category CDFs.
template <class PT>
inline void build_sim_tables(int N, int m, int L, const PT& P, const double* cat_rates, const double* cat_probs,
                             const double* pi, const double* blen, std::vector<double>& cdf, std::vector<double>& root,
                             std::vector<double>& cat) {
  const int n = 2 * N - 1;
  cdf.assign(size_t(n + 1) * L * m * m, 0.0);
  for (int v = 1; v < n; ++v)
    for (int l = 0; l < L; ++l) {
      const std::vector<double> p = P(blen[v - 1] * cat_rates[l]);
      for (int i = 0; i < m; ++i) {
        double acc = 0.0;
        for (int j = 0; j < m; ++j) {
          acc += p[size_t(i) * m + j];
          cdf[((size_t(v) * L + l) * m + i) * m + j] = acc;
        }
      }
    }
  root.assign(size_t(m), 0.0);
  double acc = 0.0;
  for (int j = 0; j < m; ++j) root[size_t(j)] = (acc += pi[j]);
  cat.assign(size_t(L), 0.0);
  acc = 0.0;
  for (int l = 0; l < L; ++l) cat[size_t(l)] = (acc += cat_probs[l]);
}

}  // namespace pg
