// GPU forward simulation of alignment columns (the
// setup path at scale): alignment.hpp:243-286 semantics with the
// counter-based per-site stream of pg_simulate.hpp, bit-identical with the
// CPU twin in workloads/ (PGW_SIM_COUNTER).  One thread per site walks the
// nodes in pre-order; internal-node states live in a [N-1][sites] int8
// scratch (coalesced over sites), tip states go straight to the output
// [tips][sites].  The cumulative transition rows are built on the host with
// the same code as the CPU twin and uploaded (small: (2N) L m^2 doubles).
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "pg_common.hpp"
#include "pg_simulate.hpp"

namespace {

#define PG_SIM_CUDA(call)                                                                              \
  do {                                                                                                 \
    cudaError_t e_ = (call);                                                                           \
    if (e_ != cudaSuccess) throw pg::CudaError(std::string("cuda: ") + #call + ": " + cudaGetErrorString(e_)); \
  } while (0)

__global__ void __launch_bounds__(256) simulate_kernel(const double* __restrict__ cdf, const double* __restrict__ root_cdf,
                                                       const double* __restrict__ cat_cdf, const int* __restrict__ pre,
                                                       const int* __restrict__ parent, int N, int m, int L,
                                                       long long sites, unsigned long long seed, double gap,
                                                       int8_t* __restrict__ tips, int8_t* __restrict__ inner) {
  const int n = 2 * N - 1;
  const uint64_t D = pg::sim::draws_per_site(N);
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < sites;
       s += (long long)gridDim.x * blockDim.x) {
    const int l = pg::sim::pick(cat_cdf, L, pg::sim::unit(seed, uint64_t(s), D, 0));
    for (int j = 0; j < n; ++j) {
      const int v = pre[j];
      int st;
      const double u = pg::sim::unit(seed, uint64_t(s), D, uint64_t(1 + j));
      if (v == n) {
        st = pg::sim::pick(root_cdf, m, u);
      } else {
        const int ps = inner[size_t(parent[v] - N - 1) * size_t(sites) + size_t(s)];
        st = pg::sim::pick(cdf + ((size_t(v) * L + l) * m + ps) * m, m, u);
      }
      if (v <= N) tips[size_t(v - 1) * size_t(sites) + size_t(s)] = int8_t(st);
      else inner[size_t(v - N - 1) * size_t(sites) + size_t(s)] = int8_t(st);
    }
    if (gap > 0.0)
      for (int t = 0; t < N; ++t)
        if (pg::sim::unit(seed, uint64_t(s), D, uint64_t(1 + n + t)) < gap) tips[size_t(t) * size_t(sites) + size_t(s)] = -1;
  }
}

template <class T>
struct DevArr {
  T* p = nullptr;
  explicit DevArr(size_t n) { PG_SIM_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
  ~DevArr() {
    if (p) cudaFree(p);
  }
  DevArr(const DevArr&) = delete;
  DevArr& operator=(const DevArr&) = delete;
};

}  // namespace

extern "C" int pg_simulate_states_gpu(int tip_count, const int32_t* parent, const int32_t* post_order, int state_count,
                                      const double* q, const double* pi, int reversible, int category_count,
                                      const double* cat_rates, const double* cat_probs, const double* branch_lengths,
                                      int64_t sites, uint64_t seed, double gap_fraction, int device, int8_t* states,
                                      int states_on_device, float* device_ms) {
  return pg::guarded([&] {
    if (sites < 1) throw std::invalid_argument("simulate: site_count must be >= 1");
    if (tip_count < 2 || state_count < 2 || state_count > 127 || category_count < 1)
      throw std::invalid_argument("simulate: bad sizes");
    if (!(gap_fraction >= 0.0 && gap_fraction < 1.0)) throw std::invalid_argument("simulate: gap fraction in [0, 1)");
    const int N = tip_count, n = 2 * N - 1, m = state_count, L = category_count;
    for (int i = 0; i < n - 1; ++i)
      if (!(branch_lengths[i] >= 0.0)) throw std::invalid_argument("transition matrix: negative branch length");
    pg::HostTransition P(m, std::vector<double>(q, q + size_t(m) * m), std::vector<double>(pi, pi + m), reversible);
    std::vector<double> cdf, root, cat;
    pg::build_sim_tables(N, m, L, P, cat_rates, cat_probs, pi, branch_lengths, cdf, root, cat);
    std::vector<int> pre(static_cast<size_t>(n)), par(parent, parent + n + 1);
    for (int j = 0; j < n; ++j) pre[size_t(j)] = post_order[n - 1 - j];  // tree.hpp:76
    PG_SIM_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    PG_SIM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::unique_ptr<CUstream_st, void (*)(cudaStream_t)> sguard(st, [](cudaStream_t x) { cudaStreamDestroy(x); });
    DevArr<double> d_cdf(cdf.size()), d_root(root.size()), d_cat(cat.size());
    DevArr<int> d_pre(pre.size()), d_par(par.size());
    DevArr<int8_t> d_inner(size_t(N - 1) * size_t(sites));
    std::unique_ptr<DevArr<int8_t>> d_tips;
    int8_t* tips = states;
    if (!states_on_device) {
      d_tips = std::make_unique<DevArr<int8_t>>(size_t(N) * size_t(sites));
      tips = d_tips->p;
    }
    PG_SIM_CUDA(cudaMemcpyAsync(d_cdf.p, cdf.data(), cdf.size() * 8, cudaMemcpyHostToDevice, st));
    PG_SIM_CUDA(cudaMemcpyAsync(d_root.p, root.data(), root.size() * 8, cudaMemcpyHostToDevice, st));
    PG_SIM_CUDA(cudaMemcpyAsync(d_cat.p, cat.data(), cat.size() * 8, cudaMemcpyHostToDevice, st));
    PG_SIM_CUDA(cudaMemcpyAsync(d_pre.p, pre.data(), pre.size() * 4, cudaMemcpyHostToDevice, st));
    PG_SIM_CUDA(cudaMemcpyAsync(d_par.p, par.data(), par.size() * 4, cudaMemcpyHostToDevice, st));
    cudaEvent_t e0, e1;
    PG_SIM_CUDA(cudaEventCreate(&e0));
    PG_SIM_CUDA(cudaEventCreate(&e1));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const long long blocks = std::min<long long>((sites + 255) / 256, (long long)sms * 16);
    PG_SIM_CUDA(cudaEventRecord(e0, st));
    simulate_kernel<<<unsigned(blocks), 256, 0, st>>>(d_cdf.p, d_root.p, d_cat.p, d_pre.p, d_par.p, N, m, L, sites,
                                                    seed, gap_fraction, tips, d_inner.p);
    PG_SIM_CUDA(cudaGetLastError());
    PG_SIM_CUDA(cudaEventRecord(e1, st));
    if (!states_on_device)
      PG_SIM_CUDA(cudaMemcpyAsync(states, tips, size_t(N) * size_t(sites), cudaMemcpyDeviceToHost, st));
    PG_SIM_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    PG_SIM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (device_ms) *device_ms = ms;
  });
}
