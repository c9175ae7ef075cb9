// Config-scale evaluation through the C++ drop-in facade
// (include/phylograd_b200/engine.hpp): the reference's call pattern —
// construct LikelihoodEngine(tree, alignment, model, categories, options),
// branch_gradient(), and for clock workloads the relaxed-clock chain rule
// (clock.hpp:140-152, :199-213) — on an instance written by the test
// (tests/test_cpp_facade.py), optionally sharded over a device list.
//
//   facade_config in.bin out.bin [--devices 0,0] [--fixed]
//
// in.bin  (little endian): int32 N, m, L, P, reversible, clock;
//         int32 parent[2N], children[2N*2], post_order[2N-1];
//         f64 branch_length[2N-2], q[m*m], pi[m], rates[L], probs[L];
//         int8 codes[N*P] (tip-major, -1 missing); int64 weights[P];
//         f64 durations[2N-2] (clock only)
// out.bin: f64 logL, grad[2N-2]; clock: f64 dlog_mu, dlog_eps[2N-2],
//         node_time[N-1]; int32 shard_count
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "phylograd_b200/engine.hpp"

using namespace phylograd_b200;

template <class T>
static void rd(FILE* f, T* p, size_t n) {
  if (n && std::fread(p, sizeof(T), n, f) != n) throw std::runtime_error("facade_config: short input");
}
template <class T>
static void wr(FILE* f, const T* p, size_t n) {
  if (n && std::fwrite(p, sizeof(T), n, f) != n) throw std::runtime_error("facade_config: short write");
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: facade_config in.bin out.bin [--devices 0,1] [--fixed]\n");
    return 2;
  }
  EngineOptions opt;
  for (int a = 3; a < argc; ++a) {
    if (!std::strcmp(argv[a], "--fixed")) opt.reduce_mode = PG_REDUCE_FIXED_ORDER;
    if (!std::strcmp(argv[a], "--devices") && a + 1 < argc) {
      std::string s = argv[++a];
      size_t pos = 0;
      while (pos < s.size()) {
        const size_t c = s.find(',', pos);
        opt.devices.push_back(std::stoi(s.substr(pos, c - pos)));
        pos = c == std::string::npos ? s.size() : c + 1;
      }
    }
  }
  try {
    FILE* f = std::fopen(argv[1], "rb");
    if (!f) throw std::runtime_error("facade_config: cannot open input");
    int32_t hdr[6];
    rd(f, hdr, 6);
    const int N = hdr[0], m = hdr[1], L = hdr[2], P = hdr[3], rev = hdr[4], clk = hdr[5];
    const int n = 2 * N - 1, B = n - 1;
    Tree tree;
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
    SubstitutionModel model;
    model.state_count = m;
    model.q.resize(size_t(m) * m);
    model.pi.resize(size_t(m));
    rd(f, model.q.data(), model.q.size());
    rd(f, model.pi.data(), model.pi.size());
    model.reversible = rev != 0;
    RateCategories cats;
    cats.rates.resize(size_t(L));
    cats.probs.resize(size_t(L));
    rd(f, cats.rates.data(), size_t(L));
    rd(f, cats.probs.data(), size_t(L));
    SitePatternAlignment aln;
    aln.state_count = m;
    aln.codes.assign(size_t(N), std::vector<int8_t>(size_t(P)));
    for (int t = 0; t < N; ++t) {
      aln.taxa.push_back("t" + std::to_string(t + 1));
      rd(f, aln.codes[size_t(t)].data(), size_t(P));
    }
    aln.weights.resize(size_t(P));
    rd(f, aln.weights.data(), size_t(P));
    std::vector<double> dt;
    if (clk) {
      dt.resize(size_t(B));
      rd(f, dt.data(), size_t(B));
    }
    std::fclose(f);

    LikelihoodEngine engine(tree, aln, model, cats, opt);
    GradientReport rep = engine.branch_gradient();
    FILE* o = std::fopen(argv[2], "wb");
    if (!o) throw std::runtime_error("facade_config: cannot open output");
    wr(o, &rep.log_likelihood, 1);
    wr(o, rep.branch_gradient.data(), size_t(B));
    if (clk) {
      engine.set_clock_durations(dt);
      ClockGradient cg = engine.clock_gradient();
      wr(o, &cg.dlog_mu, 1);
      wr(o, cg.dlog_epsilon.data(), size_t(B));
      wr(o, cg.node_time.data(), size_t(N - 1));
    }
    const int32_t shards = engine.shard_count();
    wr(o, &shards, 1);
    std::fclose(o);
    std::printf("facade_config: %d tips, %d patterns, %d states, %d categories, %d shard(s), logL %.12f\n", N, P, m, L,
                shards, rep.log_likelihood);
  } catch (const std::exception& e) {
    std::printf("FAIL: %s\n", e.what());
    return 1;
  }
  return 0;
}
