// Host helpers shared by the setup C-ABI (pg_setup.cpp) and the workload
// generator (workloads/pg_workloads.cpp): a small thread pool loop and the
// first-occurrence column compressor (alignment.hpp:186-229 order).
#pragma once

#include <algorithm>
#include <cstdint>
#include <thread>
#include <unordered_map>
#include <vector>

namespace pg {
namespace hostutil {

inline uint64_t mix64(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdull;
  return h ^ (h >> 33);
}

inline int hw_threads(int want) {
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


}  // namespace hostutil
}  // namespace pg
