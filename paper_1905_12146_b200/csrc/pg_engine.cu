// phylograd-b200 engine: host orchestration of the sm_100a kernels behind the
// C-ABI in include/phylograd_b200.h.  Mirrors phylograd::LikelihoodEngine
// (/root/reference/proj/include/phylograd/engine.hpp:47-438): same setup
// contract, cache semantics (engine.hpp:116-130, :146-162), node-visit
// instrumentation and error messages; the arithmetic runs on the GPU only.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is dlopen()ed by pg_create_multi

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "pg_common.hpp"
#include "pg_kernels.cuh"
#include "pg_walk.cuh"
#include "pg_walkl.cuh"

void* pg_walk4_kernel_lc4(bool homog, bool hess, int nc);
void* pg_walk4_kernel_lc2(bool homog, bool hess, int nc);
void* pg_walk4_kernel_l12(bool homog, bool hess, int nc, int L);
// L = 4: lcv 4 (one lane per pattern) or 2 (two lanes); L = 1, 2: one lane
void* pg_walk4s_kernel(bool homog, bool hess, int nc);
void* pg_walk4t_kernel(bool hess, int nc);
size_t pg_walk4t_smem(int nc);
size_t pg_walk4s_smem(int nc);
void* pg_walk4s_cherry_kernel(bool homog, bool hess, int nc);
void pg_cherry_tables(const int4* cherries, int ncherry, int N, int nc, const double* tc, const double* qtc, double* ct,
                      cudaStream_t stream);
size_t pg_walk4s_cherry_smem();
void pg_cherry_codes(const int4* cherries, int ncherry, int N, long long Pc, int nc, const uint8_t* codes, uint8_t* cc,
                     cudaStream_t stream);
static void* pg_walk4_kernel(bool homog, bool hess, int nc, int lcv, int L) {
  if (L != 4) return pg_walk4_kernel_l12(homog, hess, nc, L);
  return lcv == 4 ? pg_walk4_kernel_lc4(homog, hess, nc) : pg_walk4_kernel_lc2(homog, hess, nc);
}
int pg_walk4_nc(int nc);
void* pg_walkl_kernel(int L, bool homog, bool hess);
void* pg_walkm_kernel(int mp, bool hess, bool fast);
bool pg_walkm_fast_tables_fit(int mp, int nc);
size_t pg_walkm_smem(int mp);
int pg_walkm_wpc(int mp);

void* pg_walk_kernel_small(int MP, int LC);
void* pg_walk_kernel_mid(int MP, int LC);
void* pg_walk_kernel_large(int MP, int LC);

namespace pg {
namespace {

// tip column indices: states stay, class columns move from old_mp + a to new_mp + a
__global__ void pg_recode_kernel(uint8_t* codes, int64_t n, int old_mp, int new_mp) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int c = codes[i];
    if (c >= old_mp) codes[i] = uint8_t(c - old_mp + new_mp);
  }
}

#define PG_CUDA(call)                                                                                  \
  do {                                                                                                 \
    cudaError_t e_ = (call);                                                                           \
    if (e_ != cudaSuccess) throw CudaError(std::string("cuda: ") + #call + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void ensure(size_t count) {
    if (count <= n && p) return;
    release();
    PG_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    n = count;
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    ensure(count);
    if (count) PG_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

int pow2ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace
}  // namespace pg

using namespace pg;

struct pg_engine {
  pg_options opt{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;

  // topology (reference numbering)
  int N = 0;
  std::vector<int> parent, children;  // [2N], [2N*2]
  std::vector<int4> post_steps, pre_steps;
  // walk4s cherry tables (pg_walk4s.cuh): {k, a, b, 0} per cherry, the step
  // lists with the children's cherry flags (post: without the cherries' steps)
  bool use_cherry = false;
  // 4-state data without ambiguity classes (NC = 4; with missing characters
  // NC = 5) through walk4s on a tree with a cherry (any binary tree of more
  // than two tips); PG_WALK4S_CHERRY=0 turns the tables off, for A/B
  bool cherry_wanted() const {
    return use_walk4 && use_walk4s && (NC == 4 || (NC == 5 && A == 1)) && m == 4 && N > 2 &&
           !(std::getenv("PG_WALK4S_CHERRY") && std::atoi(std::getenv("PG_WALK4S_CHERRY")) == 0);
  }
  std::vector<int4> cherries, post_steps_ch, pre_steps_ch, pre_steps_fused;
  // patterns
  int m_aln = 0, P = 0, A = 0;
  bool classes_used = true;  // some tip code is missing (-1) or an ambiguity class
  int64_t Pc = 0;  // device row stride of the tip codes
  bool has_patterns = false;
  std::vector<double> amb;  // [A][m]
  // model
  int m = 0;
  bool has_model = false, reversible = false, have_eigen = false;
  std::vector<double> q, pi, eig_u, eig_ui, eig_w;
  std::map<int, std::vector<double>> branch_q;
  // categories
  int L = 0;
  std::vector<double> rates, probs;
  // lengths
  std::vector<double> blen, dt;
  bool has_dt = false, blen_host_stale = false;
  // per-evaluation CUDA events around the walk kernel and the whole evaluation
  bool timing = false;
  std::vector<cudaEvent_t> tev;  // 3 per evaluation: start, walk begin, walk end
  size_t tev_used = 0;

  // geometry
  int MP = 0, LC = 0, G = 0, NC = 0, TW = 0, ntiles = 0, accw = 0;
  bool use_walk4 = false;
  bool use_walkl = false;   // level-scheduled 4-state traversal (pg_walkl.cuh): small P
  // P up to this x SMs: level-scheduled (PG_WALKL=0/1 forces).  Measured on C2
  // (512 taxa, GTR+G4): 1,250 patterns 0.30 vs 1.83 ms, 2,500 0.43 vs 2.37 ms,
  // 5,000 0.69 vs 0.83 ms, 10,000 1.25 vs 0.98 ms, 20,000 2.14 vs 1.22 ms
  int walkl_max_patterns_per_sm = 48;
  int walkl_npost = 0, walkl_npre = 0, walkl_grid = 0;
  DevBuf<int> d_lvl_nodes, d_lvl_off, d_Sx;
  DevBuf<unsigned> d_bar;
  bool use_walkm = false;  // DMMA large-state kernel (pg_walkm.cuh)
  int codes_mp = 0;        // MP the device tip codes' class columns are encoded for
  int walkm_wpc = 4;       // warps per CTA in walkm
  int walk4_lcv = 4;  // categories per lane of the 4-state kernel
  bool use_walk4t = false;  // tensor-core (DMMA) variant (L = 4, one lane per pattern state)
  bool use_walk4s = false;  // single-buffered variant (L = 4, one lane per pattern): 16 warps per SM
  size_t walk_smem = 0;
  bool geometry_dirty = true, model_dirty = true, tc_dirty = true, patterns_dirty = true;

  // device state
  DevBuf<uint8_t> d_codes;
  DevBuf<double> d_qtc, d_fpp, d_fpt, d_fq, d_f4post, d_f4pre;
  DevBuf<double> d_weights, d_tc, d_qtab, d_pi, d_rates, d_probs, d_blen, d_dt, d_eu, d_eui, d_ew, d_amb;
  DevBuf<int> d_qidx, d_err, d_qexp;
  DevBuf<int4> d_post, d_pre, d_pre_fused, d_cherries;
  DevBuf<double> d_ct;
  DevBuf<uint8_t> d_ccodes;
  DevBuf<double> d_escr, d_qscr, d_acc, d_out, d_site_ll;
  DevBuf<double> d_cap_post, d_cap_pre;
  DevBuf<int> d_cap_post_exp, d_cap_pre_exp;
  double* h_out = nullptr;  // pinned
  int* h_err = nullptr;     // pinned [3]
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;

  // caches (engine.hpp:436)
  bool post_valid = false, pre_valid = false, hess_valid = false, ll_valid = false, rate_grad = false;
  double logl = 0.0;
  std::vector<double> grad, hess;
  uint64_t visits = 0;
  int last_launches = 0;
  float last_walk_ms = 0.f, last_total_ms = 0.f;
  int pending_flags = 0;
  bool err_armed = false;  // d_err holds the flags of evaluations not yet checked

  ~pg_engine() {
    destroy_group();
    for (cudaEvent_t ev : tev) cudaEventDestroy(ev);
    if (h_out) cudaFreeHost(h_out);
    if (h_err) cudaFreeHost(h_err);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev2) cudaEventDestroy(ev2);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }

  int B() const { return 2 * N - 2; }
  void invalidate() { post_valid = pre_valid = hess_valid = ll_valid = false; }

  void set_device() { PG_CUDA(cudaSetDevice(device)); }

  // ---------------------------------------------------------------- setup
  void set_topology(int nt, const int32_t* par, const int32_t* ch, const int32_t* post) {
    if (nt < 2) throw std::invalid_argument("tree needs at least 2 tips");
    const int n = 2 * nt - 1;
    std::vector<int> pa(par, par + n + 1), cc(ch, ch + 2 * (n + 1));
    // tree.hpp:81-126 validate_tree (structural part)
    if (pa[size_t(n)] != 0) throw std::invalid_argument("root must have no parent");
    for (int i = 1; i < n; ++i) {
      const int p = pa[size_t(i)];
      if (p <= nt || p > n) throw std::invalid_argument("node " + std::to_string(i) + " has invalid parent");
      if (cc[size_t(2 * p)] != i && cc[size_t(2 * p + 1)] != i)
        throw std::invalid_argument("parent/children maps inconsistent at node " + std::to_string(i));
    }
    for (int i = nt + 1; i <= n; ++i)
      for (int k = 0; k < 2; ++k) {
        const int c = cc[size_t(2 * i + k)];
        if (c < 1 || c >= n || pa[size_t(c)] != i)
          throw std::invalid_argument("bad child link at internal node " + std::to_string(i));
      }
    for (int i = 1; i <= nt; ++i)
      if (cc[size_t(2 * i)] != 0 || cc[size_t(2 * i + 1)] != 0)
        throw std::invalid_argument("bad child link at tip " + std::to_string(i));
    for (int i = 1; i < n; ++i) {
      int hops = 0, v = i;
      while (v != n && hops++ <= n) v = pa[size_t(v)];
      if (hops > n) throw std::invalid_argument("parent links contain a cycle");
    }
    if (post) {
      std::vector<int> pos(size_t(n + 1), -1);
      for (int k = 0; k < n; ++k) {
        const int v = post[k];
        if (v < 1 || v > n || pos[size_t(v)] >= 0) throw std::invalid_argument("post_order incomplete");
        pos[size_t(v)] = k;
      }
      for (int i = 1; i < n; ++i)
        if (pos[size_t(i)] >= pos[size_t(pa[size_t(i)])])
          throw std::invalid_argument("post_order does not visit children before parents");
    }
    N = nt;
    parent = pa;
    children = cc;
    build_schedule();
    blen.assign(size_t(B()), 0.0);
    dt.clear();
    has_dt = false;
    geometry_dirty = model_dirty = tc_dirty = true;
    invalidate();
  }

  // Heavy-child-first post order over internal nodes (Sethi-Ullman-like): the
  // arithmetic at each node is order independent, so this only changes which
  // edge messages are still on chip when their parent needs them.
  void build_schedule() {
    const int n = 2 * N - 1;
    std::vector<int> size(size_t(n + 1), 1);
    // children have smaller completion index only in the reference numbering's
    // internal block; compute sizes by explicit post traversal.
    std::vector<int> order;
    order.reserve(size_t(n));
    std::vector<std::pair<int, bool>> st{{n, false}};
    while (!st.empty()) {
      auto [v, ex] = st.back();
      st.pop_back();
      if (v <= N || ex) {
        order.push_back(v);
      } else {
        st.push_back({v, true});
        st.push_back({children[size_t(2 * v + 1)], false});
        st.push_back({children[size_t(2 * v)], false});
      }
    }
    for (int v : order)
      if (v > N) size[size_t(v)] = size[size_t(children[size_t(2 * v)])] + size[size_t(children[size_t(2 * v + 1)])];
    post_steps.clear();
    st.push_back({n, false});
    while (!st.empty()) {
      auto [v, ex] = st.back();
      st.pop_back();
      if (v <= N) continue;
      const int c0 = children[size_t(2 * v)], c1 = children[size_t(2 * v + 1)];
      if (ex) {
        post_steps.push_back(make_int4(v, c0, c1, 0));
        continue;
      }
      st.push_back({v, true});
      const bool c0_heavy = size[size_t(c0)] >= size[size_t(c1)];
      const int heavy = c0_heavy ? c0 : c1, light = c0_heavy ? c1 : c0;
      st.push_back({light, false});
      st.push_back({heavy, false});  // popped first
    }
    pre_steps.assign(post_steps.rbegin(), post_steps.rend());
    for (size_t i = 0; i < pre_steps.size(); ++i) {
      int next = 0;
      if (i + 1 < pre_steps.size()) {
        const int nx = pre_steps[i + 1].x;
        if (parent[size_t(nx)] == pre_steps[i].x) next = nx;
      }
      pre_steps[i].w = next;
    }
  }

  // Level lists of the level-scheduled traversal (pg_walkl.cuh): internal
  // nodes by height (post-order levels: a node needs only its children) and
  // by depth (pre-order levels: a node needs only its parent).
  void build_levels() {
    const int n = 2 * N - 1;
    std::vector<int> height(size_t(n + 1), 0), depth(size_t(n + 1), 0);
    for (const int4& st : post_steps) height[size_t(st.x)] = 1 + std::max(height[size_t(st.y)], height[size_t(st.z)]);
    for (const int4& st : pre_steps) {
      depth[size_t(st.y)] = depth[size_t(st.x)] + 1;
      depth[size_t(st.z)] = depth[size_t(st.x)] + 1;
    }
    int H = 0, D = 0;
    for (const int4& st : post_steps) {
      H = std::max(H, height[size_t(st.x)]);
      D = std::max(D, depth[size_t(st.x)]);
    }
    std::vector<std::vector<int>> by_h(size_t(H + 1)), by_d(size_t(D + 1));
    for (const int4& st : post_steps) {
      by_h[size_t(height[size_t(st.x)])].push_back(st.x);
      by_d[size_t(depth[size_t(st.x)])].push_back(st.x);
    }
    std::vector<int> nodes, off;
    off.push_back(0);
    for (int h = 1; h <= H; ++h) {
      nodes.insert(nodes.end(), by_h[size_t(h)].begin(), by_h[size_t(h)].end());
      off.push_back(int(nodes.size()));
    }
    walkl_npost = H;
    off.push_back(int(nodes.size()));
    for (int d = 0; d <= D; ++d) {
      nodes.insert(nodes.end(), by_d[size_t(d)].begin(), by_d[size_t(d)].end());
      off.push_back(int(nodes.size()));
    }
    walkl_npre = D + 1;
    d_lvl_nodes.upload(nodes.data(), nodes.size(), stream);
    d_lvl_off.upload(off.data(), off.size(), stream);
  }

  void set_patterns(int mm, int np, const int8_t* codes, int na, const double* ambig, const int64_t* w) {
    if (N == 0) throw std::logic_error("engine: set the topology before the patterns");
    if (mm < 2) throw std::invalid_argument("alignment: state count must be >= 2");
    if (mm > 64) throw NotSupported("engine: at most 64 states are supported");
    if (np < 0) throw std::invalid_argument("alignment: negative pattern count");
    if (mm + na + 1 > 127) throw std::invalid_argument("alignment: too many ambiguity classes");
    // MP depends on m; column index encoding: state s -> s, class a -> MP + a,
    // missing -> MP + na (an extra all-ones class, alignment.hpp:223-224).
    const int mp = mm <= 4 ? 4 : mm <= 8 ? 8 : mm <= 20 ? 20 : mm <= 32 ? 32 : 64;
    // device layout: tip-major rows padded to whole 32-pattern tiles so a
    // warp tile's codes of one tip are 32 aligned bytes (cp.async staging)
    const int64_t pc = (int64_t(np) + 31) / 32 * 32;
    std::vector<uint8_t> col(size_t(N) * size_t(std::max<int64_t>(pc, 32)), 0);
    bool cls = false;
    for (int t = 0; t < N; ++t)
      for (int s = 0; s < np; ++s) {
        const int c = codes[size_t(t) * size_t(np) + size_t(s)];
        if (c < -1 || c >= mm + na) throw std::invalid_argument("alignment: state code out of range");
        cls = cls || c < 0 || c >= mm;
        col[size_t(t) * size_t(pc) + size_t(s)] = uint8_t(c < 0 ? mp + na : c < mm ? c : mp + (c - mm));
      }
    std::vector<double> ambv(size_t(na + 1) * mm, 1.0);
    for (int a = 0; a < na; ++a)
      for (int j = 0; j < mm; ++j) ambv[size_t(a) * mm + j] = ambig[size_t(a) * mm + j];
    std::vector<double> wd(static_cast<size_t>(np));
    for (int s = 0; s < np; ++s) {
      if (w[s] < 0) throw std::invalid_argument("alignment: negative pattern weight");
      wd[size_t(s)] = double(w[s]);
    }
    set_device();
    d_codes.upload(col.data(), col.size(), stream);
    d_weights.upload(wd.data(), wd.size(), stream);
    d_amb.upload(ambv.data(), ambv.size(), stream);
    PG_CUDA(cudaStreamSynchronize(stream));
    m_aln = mm;
    codes_mp = mp;
    P = np;
    Pc = int64_t(std::max<int64_t>(pc, 32));
    A = na + 1;
    classes_used = cls;
    amb = ambv;
    has_patterns = true;
    geometry_dirty = tc_dirty = true;
    invalidate();
  }

  static void check_generator(const double* g, int mm) {
    for (int i = 0; i < mm * mm; ++i)
      if (!std::isfinite(g[i])) throw std::invalid_argument("generator: non-finite entries");
    for (int i = 0; i < mm; ++i) {
      double row = 0.0;
      for (int j = 0; j < mm; ++j) {
        if (i != j && g[i * mm + j] < 0.0) throw std::invalid_argument("generator: negative off-diagonal entry");
        row += g[i * mm + j];
      }
      if (std::fabs(row) > 1e-12) throw std::invalid_argument("generator: rows must sum to zero");
    }
  }

  void set_model(int mm, const double* qq, const double* pp, int rev) {
    if (mm < 2 || mm > 64) throw std::invalid_argument("model: state count must be in 2..64");
    check_generator(qq, mm);
    double s = 0;
    for (int i = 0; i < mm; ++i) {
      if (pp[i] < -1e-12) throw std::invalid_argument("model: pi must be a probability vector");
      s += pp[i];
    }
    if (std::fabs(s - 1.0) > 1e-12) throw std::invalid_argument("model: pi must be a probability vector");
    m = mm;
    q.assign(qq, qq + mm * mm);
    pi.assign(pp, pp + mm);
    reversible = rev != 0;
    branch_q.clear();
    // substitution.hpp:196-208: symmetric similarity transform
    have_eigen = false;
    bool positive = true;
    for (double v : pi) positive = positive && v > 0.0;
    if (reversible && positive) {
      std::vector<double> sp(static_cast<size_t>(mm)), sym(static_cast<size_t>(mm) * mm);
      for (int i = 0; i < mm; ++i) sp[size_t(i)] = std::sqrt(pi[size_t(i)]);
      for (int i = 0; i < mm; ++i)
        for (int j = 0; j < mm; ++j) {
          const double a = sp[size_t(i)] * q[size_t(i) * mm + j] / sp[size_t(j)];
          const double b = sp[size_t(j)] * q[size_t(j) * mm + i] / sp[size_t(i)];
          sym[size_t(i) * mm + j] = 0.5 * (a + b);
        }
      std::vector<double> V;
      symmetric_eigen(sym, mm, eig_w, V);
      eig_u.assign(size_t(mm) * mm, 0.0);
      eig_ui.assign(size_t(mm) * mm, 0.0);
      for (int i = 0; i < mm; ++i)
        for (int j = 0; j < mm; ++j) {
          eig_u[size_t(i) * mm + j] = V[size_t(i) * mm + j] / sp[size_t(i)];
          eig_ui[size_t(i) * mm + j] = V[size_t(j) * mm + i] * sp[size_t(j)];
        }
      have_eigen = true;
    }
    has_model = true;
    model_dirty = tc_dirty = geometry_dirty = true;
    invalidate();
  }

  void set_branch_generator(int branch, const double* qq) {
    if (!has_model) throw std::logic_error("engine: set the model before branch generators");
    if (branch < 1 || branch > B()) throw std::invalid_argument("branch generator: branch out of range");
    check_generator(qq, m);
    if (branch_q.empty()) geometry_dirty = true;  // kernel variant (and its occupancy) changes
    branch_q[branch] = std::vector<double>(qq, qq + m * m);
    model_dirty = tc_dirty = true;
    invalidate();
  }

  void set_categories(int nl, const double* r, const double* pr) {
    if (nl < 1) throw std::invalid_argument("rate categories: need L >= 1 matched rates/probs");
    double ps = 0, mean = 0;
    for (int l = 0; l < nl; ++l) {
      if (!(r[l] > 0.0)) throw std::invalid_argument("rate categories: rates must be positive");
      ps += pr[l];
      mean += r[l] * pr[l];
    }
    if (std::fabs(ps - 1.0) > 1e-12) throw std::invalid_argument("rate categories: probabilities must sum to 1");
    if (std::fabs(mean - 1.0) > 1e-10) throw std::invalid_argument("rate categories: mixture mean must be 1");
    if (nl > 128) throw NotSupported("engine: at most 128 rate categories");
    L = nl;
    rates.assign(r, r + nl);
    probs.assign(pr, pr + nl);
    set_device();
    d_rates.upload(rates.data(), size_t(L), stream);
    d_probs.upload(probs.data(), size_t(L), stream);
    PG_CUDA(cudaStreamSynchronize(stream));
    geometry_dirty = tc_dirty = true;
    invalidate();
  }

  void sync_host_blen() {
    if (!blen_host_stale) return;
    PG_CUDA(cudaMemcpyAsync(blen.data(), d_blen.p, sizeof(double) * size_t(B()), cudaMemcpyDeviceToHost, stream));
    PG_CUDA(cudaStreamSynchronize(stream));
    blen_host_stale = false;
  }

  void set_branch_lengths(const double* b) {
    if (N == 0) throw std::logic_error("engine: set the topology first");
    sync_host_blen();
    bool same = true;
    for (int i = 0; i < B(); ++i) {
      if (!std::isfinite(b[i]) || b[i] < 0.0)
        throw std::invalid_argument("engine: branch lengths must be finite and nonnegative");
      if (b[i] != blen[size_t(i)]) same = false;
    }
    if (same && !tc_dirty) return;  // caches stay valid (engine.hpp:121)
    std::copy(b, b + B(), blen.begin());
    set_device();
    d_blen.upload(blen.data(), blen.size(), stream);
    tc_dirty = true;
    invalidate();
  }

  void set_branch_lengths_device(const double* b) {
    if (N == 0) throw std::logic_error("engine: set the topology first");
    set_device();
    d_blen.ensure(size_t(B()));
    PG_CUDA(cudaMemcpyAsync(d_blen.p, b, sizeof(double) * size_t(B()), cudaMemcpyDeviceToDevice, stream));
    blen_host_stale = true;
    tc_dirty = true;
    invalidate();
  }

  void set_durations(const double* d) {
    if (N == 0) throw std::logic_error("engine: set the topology first");
    for (int i = 0; i < B(); ++i)
      if (!std::isfinite(d[i]) || d[i] < 0.0) throw std::invalid_argument("clock: durations must be finite and nonnegative");
    dt.assign(d, d + B());
    has_dt = true;
    set_device();
    d_dt.upload(dt.data(), dt.size(), stream);
    PG_CUDA(cudaStreamSynchronize(stream));
    invalidate();
  }

  // ------------------------------------------------------------ prepare
  void check_ready() {
    if (N == 0) throw std::logic_error("engine: topology not set");
    if (!has_patterns) throw std::logic_error("engine: patterns not set");
    if (!has_model) throw std::logic_error("engine: model not set");
    if (L == 0) throw std::logic_error("engine: rate categories not set");
    if (m_aln != m) throw std::invalid_argument("engine: alignment/model state counts differ");
  }

  void upload_model() {
    std::vector<double> qt(size_t(1 + branch_q.size()) * MP * MP, 0.0), pipad(size_t(MP), 0.0);
    std::vector<int> qidx(size_t(2 * N), 0);
    auto put = [&](int slot, const std::vector<double>& g) {
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) qt[size_t(slot) * MP * MP + size_t(i) * MP + j] = g[size_t(i) * m + j];
    };
    put(0, q);
    int slot = 1;
    for (auto& [br, g] : branch_q) {
      put(slot, g);
      qidx[size_t(br)] = slot++;
    }
    for (int i = 0; i < m; ++i) pipad[size_t(i)] = pi[size_t(i)];
    d_qtab.upload(qt.data(), qt.size(), stream);
    if (use_walkm) {
      // generators in mma.m8n8k4 B-fragment order (y = Q x), see tc_kernel
      const int nq = int(1 + branch_q.size()), KK = MP / 4, NT = (KK + 1) / 2, frag = KK * NT * 32;
      std::vector<double> fq(size_t(nq) * frag, 0.0);
      for (int g = 0; g < nq; ++g)
        for (int e = 0; e < frag; ++e) {
          const int lane = e & 31, f = e >> 5, ki = f / NT, ni = f % NT;
          const int k = 4 * ki + (lane & 3), gq = lane >> 2, n = 4 * (2 * ni + (gq & 1)) + (gq >> 1);
          if (n < MP) fq[size_t(g) * frag + pgk::frag_pos(f, lane, KK * NT)] = qt[size_t(g) * MP * MP + size_t(n) * MP + k];
        }
      d_fq.upload(fq.data(), fq.size(), stream);
    }
    d_qidx.upload(qidx.data(), qidx.size(), stream);
    d_pi.upload(pipad.data(), pipad.size(), stream);
    if (have_eigen) {
      d_eu.upload(eig_u.data(), eig_u.size(), stream);
      d_eui.upload(eig_ui.data(), eig_ui.size(), stream);
      d_ew.upload(eig_w.data(), eig_w.size(), stream);
    } else {
      d_eu.ensure(1);
      d_eui.ensure(1);
      d_ew.ensure(1);
    }
    model_dirty = false;
  }

  int walk_max_blocks_per_sm();
  int walk_max_blocks_per_sm_occ();

  void prepare_geometry() {
    // DMMA kernel for every state space above 4 (m = 5..8 on walkm<8>: 1.8x
    // the generic kernel, scripts/m_scale.py)
    use_walkm = m > 4 && !opt.capture_partials && std::getenv("PG_NO_WALKM") == nullptr;
    if (use_walkm) {
      MP = m <= 8 ? 8 : m <= 16 ? 16 : m <= 20 ? 20 : m <= 24 ? 24 : m <= 32 ? 32 : 64;
      // walkm indexes its tables (TC / QTC columns and the P / P^T fragment
      // tables, ((node-1) L + l) * max(FRAG, (MP+A) MP)) and its CTA-major
      // scratch ([node][category][warp][8 MP + 8 exponents]) with 32-bit offsets
      const int64_t lim = int64_t(1) << 31;
      const int64_t KK = MP / 4, frag = KK * ((KK + 1) / 2) * 32;  // WalkMGeom<MP>::FRAG
      const int64_t table = std::max<int64_t>(frag, int64_t(MP + A) * MP);
      if (int64_t(B()) * L * table >= lim || int64_t(N) * L * (MP * 8 + 4) * pg_walkm_wpc(MP) >= lim)
        use_walkm = false;
    }
    if (!use_walkm) MP = m <= 4 ? 4 : m <= 8 ? 8 : m <= 20 ? 20 : m <= 32 ? 32 : 64;
    NC = MP + A;
    if (codes_mp != MP) {
      // class columns (ambiguity / missing) were encoded as codes_mp + a at
      // set_patterns; the chosen kernel pads the states to MP instead
      const int64_t n = int64_t(N) * Pc;
      pg_recode_kernel<<<unsigned(std::min<int64_t>((n + 255) / 256, 4096)), 256, 0, stream>>>(d_codes.p, n, codes_mp,
                                                                                            MP);
      PG_CUDA(cudaGetLastError());
      codes_mp = MP;
    }
    int nc4 = 0;
    const int maxLC = MP == 4 ? 4 : MP == 8 ? 2 : 1;
    LC = std::min(maxLC, pow2ceil(L));
    // Prefer more, smaller tiles when the pattern count cannot fill the GPU.
    while (LC > 1 && (int64_t(P) * pow2ceil((L + LC - 1) / LC)) / 32 < int64_t(num_sms)) LC >>= 1;
    G = pow2ceil((L + LC - 1) / LC);
    if (G > 32) throw NotSupported("engine: too many rate categories for the lane layout");
    const int TP = 32 / G;
    ntiles = (P + TP - 1) / TP;
    // specialised pipelined 4-state kernel (pg_walk4.cuh)
    nc4 = MP == 4 ? pg_walk4_nc(NC) : 0;
    // pipelined 4-state kernel: 4 categories (one or two lanes per pattern) or
    // 1 / 2 categories (one lane per pattern)
    {
      // L = 4 keeps its own lane split below; L = 1..3 use one lane per
      // pattern, L = 8 two; every variant needs about one warp tile per SM
      const int64_t tp = L == 8 ? 16 : 32;
      use_walk4 = MP == 4 && !opt.capture_partials && nc4 > 0 && std::getenv("PG_NO_WALK4") == nullptr &&
                  (L == 4 ? (LC == 4 && G == 1)
                          : (L == 1 || ((L == 2 || L == 3 || L == 8) && int64_t(P) / tp >= int64_t(num_sms))));
    }
    walk_smem = 0;
    // level-scheduled traversal when the pattern tiles cannot fill the GPU:
    // walk4's unit is a 16- or 32-pattern tile walking ~2N dependent steps,
    // so with fewer than ~2 tiles per SM (C2 on 8 GPUs: ~2,500 patterns)
    // node-level parallelism pays (PG_WALKL=0/1 forces the choice)
    {
      const char* wl = std::getenv("PG_WALKL");
      const bool want = wl ? std::atoi(wl) != 0 : int64_t(P) <= int64_t(walkl_max_patterns_per_sm) * num_sms;
      use_walkl = MP == 4 && !opt.capture_partials && P > 0 && (L == 1 || L == 2 || L == 4 || L == 8) && want &&
                  pg_walkl_kernel(L, branch_q.empty(), false) != nullptr;
    }
    if (use_walkl) use_walk4 = false;
    if (use_walk4) {
      NC = nc4;  // TC blocks padded with zero columns to the instantiated width
      // one lane per pattern unless that leaves fewer than ~2 tiles per
      // resident warp slot (measured: C3 153 ms LCV=4 vs 180 ms LCV=2;
      // C2 1.72 ms vs 1.55 ms)
      if (L == 4) {
        walk4_lcv = (int64_t(P) / 32 >= int64_t(num_sms) * 8 * 2) ? 4 : 2;
        if (const char* v = std::getenv("PG_WALK4_LCV")) walk4_lcv = std::atoi(v) == 4 ? 4 : 2;
      } else {
        walk4_lcv = L == 8 ? 4 : L;  // one lane per pattern holds every category (L = 8: two lanes)
      }
      G = L / walk4_lcv;
      ntiles = (P + 32 / G - 1) / (32 / G);
      // one lane per pattern: the single-buffered walk4s (default; C3 walk
      // 145-147 ms vs walk4's 149-150 ms on the same boxes), PG_WALK4S=0: walk4
      const bool lane1 = L == 4 && walk4_lcv == 4;
      use_walk4s = lane1 && pg_walk4s_kernel(true, false, NC) != nullptr;
      // (measured also on C3 slices, the shard sizes of 2-8 GPUs: 116,972
      // patterns 19.4 vs 22.8 ms, 458,456 patterns 72.0 vs 76.2 ms)
      if (const char* v = std::getenv("PG_WALK4S")) use_walk4s = lane1 && std::atoi(v) != 0;
      use_walk4t = lane1 && pg_walk4t_kernel(false, NC) != nullptr && std::getenv("PG_WALK4T") != nullptr &&
                   std::atoi(std::getenv("PG_WALK4T")) != 0;
      if (use_walk4t) use_walk4s = false;
      // no missing / ambiguous tip codes (C3): TC blocks of the 4 state
      // columns only, one 16-byte chunk per lane (PG_WALK4S_NC5=1 keeps 5)
      if (use_walk4s && !classes_used && m == 4 && std::getenv("PG_WALK4S_NC5") == nullptr) NC = 4;
      walk_smem = use_walk4t   ? pg_walk4t_smem(NC)
                  : use_walk4s ? pg_walk4s_smem(NC)
                             : size_t(pgk::kWarpsPerBlock) * 2 * pgk::walk4_stage_d2(walk4_lcv, L, NC) * sizeof(double2);
      if (cherry_wanted() && NC == 4) walk_smem = std::max(walk_smem, pg_walk4s_cherry_smem());
    }
    if (use_walkl) {
      G = L;
      ntiles = (P + 32 / L - 1) / (32 / L);  // accumulator rows: one per pattern tile
      build_levels();
    }
    if (use_walkm) {
      use_walk4 = use_walkl = false;
      LC = 1;
      G = 4;  // a quad of lanes per pattern (DMMA fragment layout)
      walkm_wpc = pg_walkm_wpc(MP);
      ntiles = (P + 8 * walkm_wpc - 1) / (8 * walkm_wpc);  // CTA tiles of 8 patterns per warp
      walk_smem = pg_walkm_smem(MP);
    }
    const int maxw = walk_max_blocks_per_sm() * num_sms * (use_walkm ? walkm_wpc : pgk::kWarpsPerBlock);
    // walkm slot per (node, category): 8 patterns x MP doubles + 8 int exponents;
    const size_t vec = use_walkm ? size_t(L) * (8 * MP + 4) : size_t(32) * LC * MP;
    if (use_walkl) {
      // every internal node's e and q for all patterns; one accumulator row per tile
      TW = ntiles;
      walkl_grid = maxw / pgk::kWarpsPerBlock;  // all co-resident CTAs (cooperative launch)
      accw = 1 + 2 * B();
      const size_t all = size_t(std::max(N - 1, 1)) * size_t(P) * size_t(L) * 4;
      d_escr.ensure(all);
      d_qscr.ensure(all);
      d_Sx.ensure(size_t(std::max(N - 1, 1)) * size_t(P));
      if (d_bar.n < 2) {
        d_bar.ensure(2);
        PG_CUDA(cudaMemsetAsync(d_bar.p, 0, 2 * sizeof(unsigned), stream));
      }
      d_children.upload(children.data(), children.size(), stream);
    }
    const size_t per_warp = size_t(std::max(N - 1, 1)) * vec * sizeof(double) * 2;
    // The grid (and with it the fixed-order reduction over warp rows) must
    // not depend on the run-time memory state, or results would not be
    // bit-reproducible: the scratch budget is a fixed share of
    // the device's total memory, not of what happens to be free.
    size_t total_b = 0;
    {
      cudaDeviceProp prop{};
      PG_CUDA(cudaGetDeviceProperties(&prop, device));
      total_b = prop.totalGlobalMem;
    }
    const size_t budget = size_t(double(total_b) * 0.6);
    int cap = int(std::max<size_t>(1, budget / per_warp));
    if (use_walkl) {
      // set above
    } else if (use_walkm) {
      // CTA tiles: 4 warps per tile
      int ctas = std::max(1, std::min({maxw / walkm_wpc, std::max(ntiles, 1), std::max(cap / walkm_wpc, 1)}));
      TW = ctas * walkm_wpc;
    } else {
      TW = std::max(1, std::min({maxw, std::max(ntiles, 1), cap}));
      TW = (TW + pgk::kWarpsPerBlock - 1) / pgk::kWarpsPerBlock * pgk::kWarpsPerBlock;
    }
    accw = 1 + 2 * B();
    if (!use_walkl) {
      d_escr.ensure(size_t(TW) * size_t(std::max(N - 1, 1)) * vec);
      d_qscr.ensure(size_t(TW) * size_t(std::max(N - 1, 1)) * vec);
    }
    if (use_walk4 && use_walk4s) d_qexp.ensure(size_t(TW) * size_t(std::max(N - 1, 1)) * 32);
    if (use_walk4 && use_walk4t) {
      d_f4post.ensure(size_t(B()) * L * 32);
      d_f4pre.ensure(size_t(B()) * (L + 1) * 32);
    }
    d_acc.ensure(size_t(TW) * size_t(accw));
    d_out.ensure(size_t(accw));
    d_site_ll.ensure(size_t(std::max(P, 1)));
    d_err.ensure(3);
    d_tc.ensure(size_t(B()) * L * NC * MP);
    // Q P column tables: tip Q e in walkm, and in walk4's pre-order pass
    if (use_walkm || use_walk4 || use_walkl) d_qtc.ensure(size_t(B()) * L * NC * MP);
    if (use_walkm) {
      const size_t frag = size_t(MP / 4) * ((MP / 4 + 1) / 2) * 32;  // WalkMGeom<MP>::FRAG
      d_fpp.ensure(size_t(B()) * L * frag);
      d_fpt.ensure(size_t(B()) * L * frag);
    }
    // cherry tables: walk4s with the 4 state columns only (no missing or
    // ambiguous codes), an internal non-root node with two tip children
    // (PG_WALK4S_CHERRY=0 turns them off, for A/B)
    use_cherry = false;
    cherries.clear();
    if (cherry_wanted()) {
      std::vector<char> is_ch(size_t(2 * N), 0);
      for (const int4& st : post_steps)
        if (st.x != 2 * N - 1 && st.y <= N && st.z <= N) {
          is_ch[size_t(st.x)] = 1;
          cherries.push_back(make_int4(st.x, st.y, st.z, 0));
        }
      use_cherry = !cherries.empty();
      if (use_cherry) {
        auto flagged = [&](int4 st) {
          if (st.y > N && is_ch[size_t(st.y)]) st.x |= pgk::kCherryY;
          if (st.z > N && is_ch[size_t(st.z)]) st.x |= pgk::kCherryZ;
          return st;
        };
        post_steps_ch.clear();
        pre_steps_ch.clear();
        for (const int4& st : post_steps)
          if (!is_ch[size_t(st.x)]) post_steps_ch.push_back(flagged(st));
        for (const int4& st : pre_steps) pre_steps_ch.push_back(flagged(st));
        // one shared generator: the cherries' pre-order steps are fused into
        // their parents' (reverse of the filtered post order; the hand-off
        // target is the following step's node when it is a child)
        pre_steps_fused.assign(post_steps_ch.rbegin(), post_steps_ch.rend());
        for (size_t i = 0; i < pre_steps_fused.size(); ++i) {
          int next = 0;
          if (i + 1 < pre_steps_fused.size()) {
            const int nx = pre_steps_fused[i + 1].x & pgk::kNodeMask;
            if (parent[size_t(nx)] == (pre_steps_fused[i].x & pgk::kNodeMask)) next = nx;
          }
          pre_steps_fused[i].w = next;
        }
        d_pre_fused.upload(pre_steps_fused.data(), pre_steps_fused.size(), stream);
        d_cherries.upload(cherries.data(), cherries.size(), stream);
        d_ct.ensure(size_t(N - 1) * 2 * pgk::kCherryBlk);
        d_ccodes.ensure(size_t(N - 1) * size_t(Pc));
        pg_cherry_codes(d_cherries.p, int(cherries.size()), N, Pc, NC, d_codes.p, d_ccodes.p, stream);
        PG_CUDA(cudaGetLastError());
      }
    }
    if (use_cherry) {
      d_post.upload(post_steps_ch.data(), post_steps_ch.size(), stream);
      d_pre.upload(pre_steps_ch.data(), pre_steps_ch.size(), stream);
    } else {
      d_post.upload(post_steps.data(), post_steps.size(), stream);
      d_pre.upload(pre_steps.data(), pre_steps.size(), stream);
    }
    if (!h_out) {
      PG_CUDA(cudaMallocHost(&h_err, 3 * sizeof(int)));
      PG_CUDA(cudaEventCreate(&ev0));
      PG_CUDA(cudaEventCreate(&ev1));
      PG_CUDA(cudaEventCreate(&ev2));
    }
    if (h_out) cudaFreeHost(h_out);
    PG_CUDA(cudaMallocHost(&h_out, size_t(accw) * sizeof(double)));
    if (opt.capture_partials) {
      const size_t nn = size_t(2 * N);
      d_cap_post.ensure(nn * L * size_t(P) * MP);
      d_cap_pre.ensure(nn * L * size_t(P) * MP);
      d_cap_post_exp.ensure(nn * size_t(P));
      d_cap_pre_exp.ensure(nn * size_t(P));
      PG_CUDA(cudaMemsetAsync(d_cap_post.p, 0, d_cap_post.n * sizeof(double), stream));
      PG_CUDA(cudaMemsetAsync(d_cap_pre.p, 0, d_cap_pre.n * sizeof(double), stream));
      PG_CUDA(cudaMemsetAsync(d_cap_post_exp.p, 0, d_cap_post_exp.n * sizeof(int), stream));
      PG_CUDA(cudaMemsetAsync(d_cap_pre_exp.p, 0, d_cap_pre_exp.n * sizeof(int), stream));
    }
    if (d_blen.n < size_t(B())) d_blen.upload(blen.data(), blen.size(), stream);
    geometry_dirty = false;
    model_dirty = true;
  }

  void launch_tc();
  void launch_walk(bool do_pre, bool do_hess);

  // ------------------------------------------------------------ evaluate
  // Enqueues the evaluation; results land in d_out (or out_device).
  void enqueue(int flags, double* out_device) {
    check_ready();
    set_device();
    // a forced evaluation rebuilds P(t) like the reference's post pass, which
    // recomputes trans_ every time (engine.hpp:197-201)
    if (flags & PG_EVAL_FORCE) tc_dirty = true;
    if (geometry_dirty) prepare_geometry();
    if (model_dirty) upload_model();
    const bool want_grad = flags & (PG_EVAL_GRAD | PG_EVAL_HESS | PG_EVAL_RATE_GRAD);
    const bool want_hess = flags & PG_EVAL_HESS;
    if ((flags & PG_EVAL_RATE_GRAD) && !has_dt) throw std::logic_error("engine: rate gradient needs clock durations");
    int launches = 0;
    // Error flags are sticky until read: several device-side evaluations
    // (pg_evaluate_device) enqueued back to back report a failure of ANY of
    // them at the next pg_check_errors, not only of the last one.
    if (!err_armed) {
      PG_CUDA(cudaMemsetAsync(d_err.p, 0x7f, 3 * sizeof(int), stream));  // INT_MAX-ish sentinel
      err_armed = true;
    }
    PG_CUDA(cudaEventRecord(ev0, stream));
    cudaEvent_t* te = nullptr;
    if (timing) {
      if (tev_used + 3 > tev.size())
        for (int k = 0; k < 3; ++k) {
          cudaEvent_t ev;
          PG_CUDA(cudaEventCreate(&ev));
          tev.push_back(ev);
        }
      te = &tev[tev_used];
      tev_used += 3;
      PG_CUDA(cudaEventRecord(te[0], stream));
    }
    if (tc_dirty) {
      launch_tc();
      ++launches;
      if (use_cherry) {
        pg_cherry_tables(d_cherries.p, int(cherries.size()), N, NC, d_tc.p, d_qtc.p, d_ct.p, stream);
        PG_CUDA(cudaGetLastError());
        ++launches;
      }
      tc_dirty = false;
    }
    PG_CUDA(cudaEventRecord(ev1, stream));
    if (te) PG_CUDA(cudaEventRecord(te[1], stream));
    launch_walk(want_grad, want_hess);
    ++launches;
    PG_CUDA(cudaEventRecord(ev2, stream));
    if (te) PG_CUDA(cudaEventRecord(te[2], stream));
    const int width = want_hess ? accw : 1 + B();
    double* out = out_device ? out_device : d_out.p;
    pgk::reduce_kernel<<<(width + 31) / 32, 32 * pgk::kReduceGroups, 0, stream>>>(
        d_acc.p, TW, accw, width, out, (flags & PG_EVAL_RATE_GRAD) ? d_dt.p : nullptr, B());
    PG_CUDA(cudaGetLastError());
    ++launches;
    last_launches = launches;
    PG_CUDA(cudaMemcpyAsync(h_err, d_err.p, 3 * sizeof(int), cudaMemcpyDeviceToHost, stream));
    pending_flags = flags;
  }

  void check_errors() {
    PG_CUDA(cudaStreamSynchronize(stream));
    err_armed = false;  // the next evaluation starts a fresh error window
    PG_CUDA(cudaEventElapsedTime(&last_walk_ms, ev1, ev2));
    PG_CUDA(cudaEventElapsedTime(&last_total_ms, ev0, ev2));
    if (h_err[2] == 1) throw std::invalid_argument("transition matrix: negative branch length");
    const int nf = h_err[0], uf = h_err[1];
    const int sentinel = 0x7f7f7f7f;
    if (nf != sentinel || uf != sentinel) {
      // pattern_offset: index of this shard's first pattern in a multi-device group
      if (nf <= uf)
        throw std::runtime_error("engine: non-finite partial at pattern " + std::to_string(int64_t(nf) + pattern_offset));
      throw std::runtime_error("engine: site likelihood underflowed to zero at pattern " +
                               std::to_string(int64_t(uf) + pattern_offset));
    }
  }

  // Cache test of engine.hpp:146-162 (after the FORCE / REQUIRE_POST rules).
  bool begin_evaluate(int flags) {
    if ((flags & PG_EVAL_REQUIRE_POST) && !post_valid)
      throw std::logic_error("engine: pre-order pass requires a current post-order pass");
    if (flags & PG_EVAL_FORCE) {
      invalidate();
      tc_dirty = true;
    }
    const bool want_grad = flags & (PG_EVAL_GRAD | PG_EVAL_HESS | PG_EVAL_RATE_GRAD);
    const bool want_hess = flags & PG_EVAL_HESS;
    const bool rate = flags & PG_EVAL_RATE_GRAD;
    const bool post_pass = flags & PG_EVAL_POST_PASS;
    return want_grad ? (pre_valid && post_valid && (!want_hess || hess_valid) && rate == rate_grad)
                     : (post_pass ? post_valid : ll_valid);
  }
  static int out_width(int flags, int B) {
    const bool want_grad = flags & (PG_EVAL_GRAD | PG_EVAL_HESS | PG_EVAL_RATE_GRAD);
    return (flags & PG_EVAL_HESS) ? 1 + 2 * B : (want_grad ? 1 + B : 1);
  }
  // Waits for an enqueued evaluation, raises its errors and moves the cache
  // flags / visit counters like the reference's passes; `res` (host) holds
  // [logL, g, h] of the evaluation (for a group shard: the reduced result).
  void finish_evaluate(int flags, const double* res) {
    const bool want_grad = flags & (PG_EVAL_GRAD | PG_EVAL_HESS | PG_EVAL_RATE_GRAD);
    const bool want_hess = flags & PG_EVAL_HESS;
    try {
      check_errors();
    } catch (...) {
      invalidate();
      throw;
    }
    if (res) {
      logl = res[0];
      if (want_grad) grad.assign(res + 1, res + 1 + B());
      if (want_hess) hess.assign(res + 1 + B(), res + 1 + 2 * B());
    }
    ll_valid = true;
    if (want_grad) {
      // reference: post visits only when the post cache was stale
      visits += uint64_t(post_valid ? 0 : 2 * N - 1) + uint64_t(2 * N - 1);
      post_valid = pre_valid = true;
      hess_valid = want_hess;
      rate_grad = flags & PG_EVAL_RATE_GRAD;
    } else if (flags & PG_EVAL_POST_PASS) {
      visits += uint64_t(2 * N - 1);  // post_order_pass (engine.hpp:188)
      post_valid = true;
      pre_valid = hess_valid = false;
    } else {
      visits += uint64_t(2 * N - 1);  // scratch likelihood route (engine.hpp:308-309)
    }
  }
  void copy_out(int flags, double* ll_out, double* g_out, double* h_out_) const {
    const bool want_grad = flags & (PG_EVAL_GRAD | PG_EVAL_HESS | PG_EVAL_RATE_GRAD);
    if (ll_out) *ll_out = logl;
    if (want_grad && g_out) std::copy(grad.begin(), grad.end(), g_out);
    if ((flags & PG_EVAL_HESS) && h_out_) std::copy(hess.begin(), hess.end(), h_out_);
  }

  void evaluate(int flags, double* ll_out, double* g_out, double* h_out_) {
    if (!shards.empty()) {
      group_evaluate(flags);  // every shard caches the reduced result
      shards[0]->copy_out(flags, ll_out, g_out, h_out_);
      return;
    }
    if (!begin_evaluate(flags)) {
      enqueue(flags, nullptr);
      PG_CUDA(cudaMemcpyAsync(h_out, d_out.p, size_t(out_width(flags, B())) * sizeof(double), cudaMemcpyDeviceToHost,
                              stream));
      finish_evaluate(flags, h_out);
    }
    copy_out(flags, ll_out, g_out, h_out_);
  }

  // ------------------------------------------------ multi-device group
  // pg_create_multi: this object only holds the group; the work runs on one
  // single-device engine per entry of the device list, each owning a
  // contiguous block of patterns, and one reduction of
  // [logL, g, h] per evaluation (NCCL all-reduce, or a fixed rank-order sum).
  std::vector<std::unique_ptr<pg_engine>> shards;
  std::vector<int> shard_p0;
  int reduce_mode = PG_REDUCE_NCCL;
  int64_t pattern_offset = 0;
  std::vector<void*> nccl_comms;  // ncclComm_t per shard
  std::vector<DevBuf<double>> shard_out;  // per shard: [1 + 2B] on its device
  DevBuf<double> d_gather;                // fixed-order mode: G x (1 + 2B) on shard 0's device
  std::vector<double> group_res;
  bool is_group() const { return !shards.empty(); }
  void group_evaluate(int flags);
  void destroy_group();

  // ------------------------------------------------ clock chain rule
  DevBuf<int> d_children;
  DevBuf<double> d_clk, d_cg, d_crates;
  void clock_gradient(const double* rates, double* ll, double* dlog_mu, double* dlog_eps, double* dnode);
};

namespace {

void* select_walk(int MP, int LC) {
  void* f = pg_walk_kernel_small(MP, LC);
  if (!f) f = pg_walk_kernel_mid(MP, LC);
  if (!f) f = pg_walk_kernel_large(MP, LC);
  if (!f) throw NotSupported("engine: no kernel for this state/category layout");
  return f;
}

}  // namespace

int pg_engine::walk_max_blocks_per_sm() {
  // PG_WALK_MAXB caps the resident CTAs per SM (occupancy experiments)
  const int cap = std::getenv("PG_WALK_MAXB") ? std::max(1, std::atoi(std::getenv("PG_WALK_MAXB"))) : INT_MAX;
  return std::min(cap, walk_max_blocks_per_sm_occ());
}

int pg_engine::walk_max_blocks_per_sm_occ() {
  int nb = 0;
  if (use_walkm) {
    for (int h = 0; h < 3; ++h) {
      const void* fn = pg_walkm_kernel(MP, h == 1, h == 2);
      PG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(walk_smem)));
      int b = 0;
      PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, 32 * walkm_wpc, walk_smem));
      nb = h == 0 ? b : std::min(nb, b);
    }
    return std::max(nb, 1);
  }
  if (use_walkl) {
    for (int v = 0; v < 2; ++v) {
      int b = 0;
      PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, pg_walkl_kernel(L, branch_q.empty(), v & 1), 256, 0));
      nb = v == 0 ? b : std::min(nb, b);
    }
    return std::max(nb, 1);
  }
  if (use_walk4) {
    // occupancy of the model's variants (with and without the Hessian) bounds the grid
    for (int v = 0; v < 2; ++v) {
      const void* fn = use_walk4t   ? pg_walk4t_kernel(v & 1, NC)
                       : use_walk4s ? pg_walk4s_kernel(branch_q.empty(), v & 1, NC)
                                    : pg_walk4_kernel(branch_q.empty(), v & 1, NC, walk4_lcv, L);
      PG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(walk_smem)));
      int b = 0;
      PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, pgk::kWarpsPerBlock * 32, walk_smem));
      nb = v == 0 ? b : std::min(nb, b);
      if (cherry_wanted()) {
        // the cherry-table instances (3 CTAs per SM) set the grid
        const void* fc = pg_walk4s_cherry_kernel(branch_q.empty(), v & 1, NC);
        PG_CUDA(cudaFuncSetAttribute(fc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(walk_smem)));
        PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fc, pgk::kWarpsPerBlock * 32, walk_smem));
        nb = std::min(nb, b);
      }
    }
  } else {
    PG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, select_walk(MP, LC), pgk::kWarpsPerBlock * 32, 0));
  }
  return std::max(nb, 1);
}

void pg_engine::launch_tc() {
  pgk::TcParams p{};
  p.blen = d_blen.p;
  p.rates = d_rates.p;
  p.qtab = d_qtab.p;
  p.qidx = d_qidx.p;
  p.eig_u = d_eu.p;
  p.eig_ui = d_eui.p;
  p.eig_w = d_ew.p;
  p.amb = d_amb.p;
  p.tc = d_tc.p;
  p.qtc = (use_walkm || use_walk4 || use_walkl) ? d_qtc.p : nullptr;
  p.fpp = use_walkm ? d_fpp.p : nullptr;
  p.fpt = use_walkm ? d_fpt.p : nullptr;
  p.f4post = (use_walk4 && use_walk4t) ? d_f4post.p : nullptr;
  p.f4pre = (use_walk4 && use_walk4t) ? d_f4pre.p : nullptr;
  p.err = d_err.p;
  p.m = m;
  p.MP = MP;
  p.NC = NC;
  p.A = A;
  p.L = L;
  p.have_eigen = have_eigen ? 1 : 0;
  const size_t smem = (size_t(7) * m * m + m) * sizeof(double);
  if (smem > 48 * 1024)
    PG_CUDA(cudaFuncSetAttribute(pgk::tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  dim3 grid{unsigned(B()), unsigned(L), 1u};
  pgk::tc_kernel<<<grid, m > 24 ? 512 : 128, smem, stream>>>(p);  // codon blocks: one per SM (smem), more threads
  PG_CUDA(cudaGetLastError());
}

void pg_engine::launch_walk(bool do_pre, bool do_hess) {
  pgk::WalkParams p{};
  p.codes = d_codes.p;
  p.weights = d_weights.p;
  p.tc = d_tc.p;
  p.qtc = (use_walkm || use_walk4 || use_walkl) ? d_qtc.p : nullptr;
  p.qtab = d_qtab.p;
  p.qidx = d_qidx.p;
  p.pi = d_pi.p;
  p.rates = d_rates.p;
  p.probs = d_probs.p;
  p.post = d_post.p;
  p.pre = d_pre.p;
  p.escr = d_escr.p;
  p.qscr = d_qscr.p;
  p.acc = d_acc.p;
  p.err = d_err.p;
  p.site_ll = d_site_ll.p;
  if (opt.capture_partials) {
    p.cap_post = d_cap_post.p;
    p.cap_pre = d_cap_pre.p;
    p.cap_post_exp = d_cap_post_exp.p;
    p.cap_pre_exp = d_cap_pre_exp.p;
  }
  p.N = N;
  p.P = P;
  p.Pc = Pc;
  p.L = L;
  p.G = G;
  p.NC = NC;
  p.nsteps = int(post_steps.size());
  p.ntiles = ntiles;
  p.accw = accw;
  p.B = B();
  p.thr = opt.rescaling_threshold;
  p.force = opt.force_rescaling;
  p.disable = opt.disable_rescaling;
  p.do_pre = do_pre ? 1 : 0;
  p.hess = do_hess ? 1 : 0;
  if (use_walkm) {
    pgk::WalkMParams pm{};
    pm.p = p;
    pm.fpp = d_fpp.p;
    pm.fpt = d_fpt.p;
    pm.fq = d_fq.p;
    pm.homogeneous = branch_q.empty() ? 1 : 0;
    // the compile-time-folded gradient kernel when its assumptions hold
    // (PG_WALKM_FAST=0 keeps the general one, for A/B)
    static const bool fast_env = !(std::getenv("PG_WALKM_FAST") && std::atoi(std::getenv("PG_WALKM_FAST")) == 0);
    const bool fast = fast_env && !do_hess && branch_q.empty() && !opt.disable_rescaling && L == 4 &&
                      pg_walkm_fast_tables_fit(MP, NC);
    void* fn = pg_walkm_kernel(MP, do_hess, fast);
    void* args[] = {&pm};
    PG_CUDA(cudaLaunchKernel(fn, dim3(unsigned(TW / walkm_wpc)), dim3(32 * walkm_wpc), args, walk_smem, stream));
    return;
  }
  if (use_walkl) {
    pgk::WalkLParams pl{};
    pl.p = p;
    for (int i = 0; i < 4; ++i) {
      pl.pi[i] = i < m ? pi[size_t(i)] : 0.0;
      for (int j = 0; j < 4; ++j) pl.q[i * 4 + j] = (i < m && j < m) ? q[size_t(i) * m + j] : 0.0;
    }
    pl.lvl_nodes = d_lvl_nodes.p;
    pl.lvl_off = d_lvl_off.p;
    pl.npost = walkl_npost;
    pl.npre = walkl_npre;
    pl.children = d_children.p;
    pl.E = d_escr.p;
    pl.Qp = d_qscr.p;
    pl.Sx = d_Sx.p;
    pl.bar = d_bar.p;
    pl.ntp = ntiles;
    void* fn = pg_walkl_kernel(L, branch_q.empty(), do_hess);
    // every CTA resident (grid barrier between levels): cooperative launch
    const int grid = walkl_grid;
    void* args[] = {&pl};
    PG_CUDA(cudaLaunchCooperativeKernel(fn, dim3(unsigned(grid)), dim3(256), args, 0, stream));
    return;
  }
  if (use_walk4) {
    pgk::Walk4Params p4{};
    p4.p = p;
    for (int i = 0; i < 4; ++i) {
      p4.pi[i] = i < m ? pi[size_t(i)] : 0.0;
      for (int j = 0; j < 4; ++j) p4.q[i * 4 + j] = (i < m && j < m) ? q[size_t(i) * m + j] : 0.0;
    }
    if (use_walk4s || use_walk4t) {
      pgk::Walk4SParams ps{};
      ps.w = p4;
      for (int l = 0; l < 4; ++l) {
        const double w = l < L ? probs[size_t(l)] : 0.0, r = l < L ? rates[size_t(l)] : 0.0;
        ps.cw[l] = w;
        ps.crw[l] = r * w;
        ps.cr2w[l] = r * r * w;
      }
      ps.qexp = d_qexp.p;
      if (use_walk4t) {
        pgk::Walk4TParams pt{};
        pt.s = ps;
        pt.f4post = d_f4post.p;
        pt.f4pre = d_f4pre.p;
        void* fn = pg_walk4t_kernel(do_hess, NC);
        void* args[] = {&pt};
        PG_CUDA(cudaLaunchKernel(fn, dim3(unsigned(TW / pgk::kWarpsPerBlock)), dim3(pgk::kWarpsPerBlock * 32), args,
                                 walk_smem, stream));
        return;
      }
      ps.ct = use_cherry ? d_ct.p : nullptr;
      ps.ccodes = use_cherry ? d_ccodes.p : nullptr;
      ps.npost = use_cherry ? int(post_steps_ch.size()) : int(post_steps.size());
      // fused cherry steps: the gradient instances (W tables) and the one-generator Hessian ones
      if (use_cherry && NC == 4 && (!do_hess || branch_q.empty())) ps.w.p.pre = d_pre_fused.p;
      void* fn = use_cherry ? pg_walk4s_cherry_kernel(branch_q.empty(), do_hess, NC)
                            : pg_walk4s_kernel(branch_q.empty(), do_hess, NC);
      void* args[] = {&ps};
      PG_CUDA(cudaLaunchKernel(fn, dim3(unsigned(TW / pgk::kWarpsPerBlock)), dim3(pgk::kWarpsPerBlock * 32), args,
                               walk_smem, stream));
      return;
    }
    void* fn = pg_walk4_kernel(branch_q.empty(), do_hess, NC, walk4_lcv, L);
    void* args[] = {&p4};
    PG_CUDA(cudaLaunchKernel(fn, dim3(unsigned(TW / pgk::kWarpsPerBlock)), dim3(pgk::kWarpsPerBlock * 32), args,
                             walk_smem, stream));
    return;
  }
  void* fn = select_walk(MP, LC);
  void* args[] = {&p};
  PG_CUDA(cudaLaunchKernel(fn, dim3(unsigned(TW / pgk::kWarpsPerBlock)), dim3(pgk::kWarpsPerBlock * 32), args, 0,
                           stream));
}


// ======================================================= NCCL (dlopen)
namespace {
struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  int version = 0;
};
NcclApi& nccl() {
  static NcclApi api;
  if (api.so) return api;
  // the process may already hold torch's copy (same soname): dlopen returns it
  void* so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!so) so = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!so) throw NcclError(std::string("nccl: cannot load libnccl.so.2: ") + dlerror());
  auto sym = [&](const char* n) {
    void* f = dlsym(so, n);
    if (!f) throw NcclError(std::string("nccl: missing symbol ") + n);
    return f;
  };
  api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(sym("ncclCommInitAll"));
  api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
  api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
  api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
  api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
  api.get_version = reinterpret_cast<decltype(api.get_version)>(sym("ncclGetVersion"));
  api.get_version(&api.version);
  api.so = so;
  return api;
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string("nccl: ") + what + ": " + nccl().error_string(r));
}
}  // namespace

void pg_engine::destroy_group() {
  for (void* c : nccl_comms)
    if (c) nccl().comm_destroy(static_cast<ncclComm_t>(c));
  nccl_comms.clear();
  shard_out.clear();
  shards.clear();
}

void pg_engine::group_evaluate(int flags) {
  const int G = int(shards.size());
  bool all_cached = true;
  for (auto& sh : shards) {
    sh->set_device();
    all_cached = sh->begin_evaluate(flags) && all_cached;
  }
  if (all_cached) return;  // every shard caches the reduced result
  const int Bn = shards[0]->B();
  const int width = out_width(flags, Bn);
  for (int r = 0; r < G; ++r) {
    pg_engine& sh = *shards[size_t(r)];
    sh.set_device();
    shard_out[size_t(r)].ensure(size_t(1 + 2 * Bn));
    sh.enqueue(flags | PG_EVAL_FORCE, shard_out[size_t(r)].p);
  }
  pg_engine& s0 = *shards[0];
  if (reduce_mode == PG_REDUCE_NCCL) {
    NcclApi& api = nccl();
    nccl_check(api.group_start(), "ncclGroupStart");
    for (int r = 0; r < G; ++r) {
      pg_engine& sh = *shards[size_t(r)];
      sh.set_device();
      nccl_check(api.all_reduce(shard_out[size_t(r)].p, shard_out[size_t(r)].p, size_t(width), ncclFloat64, ncclSum,
                                static_cast<ncclComm_t>(nccl_comms[size_t(r)]), sh.stream),
                 "ncclAllReduce");
    }
    nccl_check(api.group_end(), "ncclGroupEnd");
    s0.set_device();
    PG_CUDA(cudaMemcpyAsync(s0.h_out, shard_out[0].p, size_t(width) * sizeof(double), cudaMemcpyDeviceToHost,
                            s0.stream));
  } else {
    // fixed rank-order sum on the first device: bit-reproducible
    s0.set_device();
    d_gather.ensure(size_t(G) * size_t(width));
    for (int r = 0; r < G; ++r) {
      pg_engine& sh = *shards[size_t(r)];
      sh.set_device();
      PG_CUDA(cudaMemcpyPeerAsync(d_gather.p + size_t(r) * width, s0.device, shard_out[size_t(r)].p, sh.device,
                                  size_t(width) * sizeof(double), sh.stream));
      if (r > 0) {
        cudaEvent_t ev;
        PG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        PG_CUDA(cudaEventRecord(ev, sh.stream));
        s0.set_device();
        PG_CUDA(cudaStreamWaitEvent(s0.stream, ev, 0));
        PG_CUDA(cudaEventDestroy(ev));  // released once the wait has been satisfied
      }
    }
    s0.set_device();
    pgk::shard_sum_kernel<<<(width + 255) / 256, 256, 0, s0.stream>>>(d_gather.p, G, width, s0.d_out.p);
    PG_CUDA(cudaGetLastError());
    PG_CUDA(cudaMemcpyAsync(s0.h_out, s0.d_out.p, size_t(width) * sizeof(double), cudaMemcpyDeviceToHost, s0.stream));
  }
  // wait for every shard, raise the first error, cache the reduced result
  std::exception_ptr first;
  s0.set_device();
  try {
    PG_CUDA(cudaStreamSynchronize(s0.stream));
  } catch (...) {
    first = std::current_exception();
  }
  group_res.assign(s0.h_out, s0.h_out + width);
  for (auto& sh : shards) {
    try {
      sh->set_device();
      sh->finish_evaluate(flags, group_res.data());
    } catch (...) {
      if (!first) first = std::current_exception();
    }
  }
  if (first) {
    for (auto& sh : shards) sh->invalidate();
    std::rethrow_exception(first);
  }
}

void pg_engine::clock_gradient(const double* r_host, double* ll_out, double* dlog_mu, double* dlog_eps,
                               double* dnode) {
  pg_engine& pe = is_group() ? *shards[0] : *this;
  if (!r_host && !pe.has_dt) throw std::logic_error("engine: clock gradient needs rates or clock durations");
  evaluate(PG_EVAL_GRAD, ll_out, nullptr, nullptr);
  const int Bn = pe.B(), Nn = pe.N;
  pe.set_device();
  d_children.upload(pe.children.data(), pe.children.size(), pe.stream);
  d_cg.upload(pe.grad.data(), pe.grad.size(), pe.stream);
  if (r_host) {
    for (int i = 0; i < Bn; ++i)
      if (!std::isfinite(r_host[i])) throw std::invalid_argument("clock: rates must be finite");
    d_crates.upload(r_host, size_t(Bn), pe.stream);
  }
  d_clk.ensure(size_t(1 + Bn + Nn - 1));
  pgk::clock_kernel<<<1, pgk::kClockThreads, 0, pe.stream>>>(d_cg.p, pe.d_blen.p, r_host ? d_crates.p : nullptr,
                                                             pe.d_dt.p, d_children.p, Nn, d_clk.p);
  PG_CUDA(cudaGetLastError());
  std::vector<double> h(size_t(1 + Bn + Nn - 1));
  PG_CUDA(cudaMemcpyAsync(h.data(), d_clk.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, pe.stream));
  PG_CUDA(cudaStreamSynchronize(pe.stream));
  if (dlog_mu) *dlog_mu = h[0];
  if (dlog_eps) std::copy(h.begin() + 1, h.begin() + 1 + Bn, dlog_eps);
  if (dnode) std::copy(h.begin() + 1 + Bn, h.end(), dnode);
}

namespace {
template <class F>
void each(pg_engine* e, F&& f) {
  if (e->is_group())
    for (auto& sh : e->shards) f(sh.get());
  else
    f(e);
}
pg_engine* primary(pg_engine* e) { return e->is_group() ? e->shards[0].get() : e; }
const pg_engine* primary(const pg_engine* e) { return e->is_group() ? e->shards[0].get() : e; }
void single_only(const pg_engine* e, const char* what) {
  if (e->is_group()) throw NotSupported(std::string(what) + ": not supported on a multi-device group");
}
}  // namespace

// ============================================================== C-ABI
extern "C" {

void pg_default_options(pg_options* opt) {
  std::memset(opt, 0, sizeof(*opt));
  opt->rescaling_threshold = 1e-150;
}

int pg_create(const pg_options* opt, pg_engine** out) {
  return guarded([&] {
    auto e = std::make_unique<pg_engine>();
    if (opt) e->opt = *opt;
    else pg_default_options(&e->opt);
    e->device = e->opt.device;
    int count = 0;
    PG_CUDA(cudaGetDeviceCount(&count));
    if (e->device < 0 || e->device >= count) throw CudaError("engine: CUDA device not available");
    e->set_device();
    PG_CUDA(cudaDeviceGetAttribute(&e->num_sms, cudaDevAttrMultiProcessorCount, e->device));
    PG_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    e->own_stream = true;
    *out = e.release();
  });
}

void pg_destroy(pg_engine* e) { delete e; }

int pg_create_multi(const pg_options* opt, int device_count, const int* devices, int reduce_mode, pg_engine** out) {
  return guarded([&] {
    if (device_count < 1 || !devices) throw std::invalid_argument("engine: need at least one device");
    if (reduce_mode != PG_REDUCE_NCCL && reduce_mode != PG_REDUCE_FIXED_ORDER)
      throw std::invalid_argument("engine: unknown reduce mode");
    std::vector<int> devs(devices, devices + device_count);
    if (reduce_mode == PG_REDUCE_NCCL) {
      std::vector<int> sorted = devs;
      std::sort(sorted.begin(), sorted.end());
      if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
        throw std::invalid_argument("engine: the NCCL reduction needs distinct devices (use PG_REDUCE_FIXED_ORDER)");
    }
    auto g = std::make_unique<pg_engine>();
    if (opt) g->opt = *opt;
    else pg_default_options(&g->opt);
    if (g->opt.capture_partials) throw NotSupported("engine: partial capture is not supported on a multi-device group");
    g->reduce_mode = reduce_mode;
    g->device = devs[0];
    for (int d : devs) {
      pg_options o = g->opt;
      o.device = d;
      pg_engine* sh = nullptr;
      if (pg_create(&o, &sh) != PG_OK) throw CudaError(pg_last_error());
      g->shards.emplace_back(sh);
    }
    g->shard_out.resize(devs.size());
    if (reduce_mode == PG_REDUCE_NCCL) {
      g->nccl_comms.assign(devs.size(), nullptr);
      std::vector<ncclComm_t> comms(devs.size());
      nccl_check(nccl().comm_init_all(comms.data(), device_count, devs.data()), "ncclCommInitAll");
      for (size_t i = 0; i < comms.size(); ++i) g->nccl_comms[i] = comms[i];
    } else {
      // peer access lets the gather copies go over NVLink directly
      for (int d : devs)
        for (int d2 : devs)
          if (d != d2) {
            int ok = 0;
            cudaDeviceCanAccessPeer(&ok, d, d2);
            if (ok) {
              cudaSetDevice(d);
              const cudaError_t r = cudaDeviceEnablePeerAccess(d2, 0);
              if (r != cudaSuccess && r != cudaErrorPeerAccessAlreadyEnabled) PG_CUDA(r);
              cudaGetLastError();
            }
          }
    }
    *out = g.release();
  });
}

int pg_group_info(const pg_engine* e, int* shard_count, int* nccl_version, int* reduce_mode) {
  return guarded([&] {
    if (shard_count) *shard_count = e->is_group() ? int(e->shards.size()) : 1;
    if (nccl_version) *nccl_version = (e->is_group() && e->reduce_mode == PG_REDUCE_NCCL) ? nccl().version : 0;
    if (reduce_mode) *reduce_mode = e->reduce_mode;
  });
}

int pg_clock_gradient(pg_engine* e, const double* rates, double* log_likelihood, double* dlog_mu, double* dlog_eps,
                      double* dnode_time) {
  return guarded([&] { e->clock_gradient(rates, log_likelihood, dlog_mu, dlog_eps, dnode_time); });
}

int pg_set_topology(pg_engine* e, int tip_count, const int32_t* parent, const int32_t* children,
                    const int32_t* post_order) {
  return guarded([&] { each(e, [&](pg_engine* x) { x->set_topology(tip_count, parent, children, post_order); }); });
}

int pg_set_patterns(pg_engine* e, int state_count, int pattern_count, const int8_t* codes, int ambiguity_count,
                    const double* ambiguity, const int64_t* weights) {
  return guarded([&] {
    if (!e->is_group()) {
      e->set_patterns(state_count, pattern_count, codes, ambiguity_count, ambiguity, weights);
      return;
    }
    // contiguous pattern blocks, shard r: [floor(r P / G), floor((r+1) P / G))
    const int G = int(e->shards.size());
    const int N = e->shards[0]->N;
    if (pattern_count < 0) throw std::invalid_argument("alignment: negative pattern count");
    for (int r = 0; r < G; ++r) {
      const int p0 = int(int64_t(pattern_count) * r / G), p1 = int(int64_t(pattern_count) * (r + 1) / G);
      std::vector<int8_t> c(size_t(N) * size_t(p1 - p0));
      for (int t = 0; t < N; ++t)
        std::copy(codes + size_t(t) * size_t(pattern_count) + size_t(p0),
                  codes + size_t(t) * size_t(pattern_count) + size_t(p1), c.begin() + ptrdiff_t(size_t(t) * (p1 - p0)));
      e->shards[size_t(r)]->set_patterns(state_count, p1 - p0, c.data(), ambiguity_count, ambiguity, weights + p0);
      e->shards[size_t(r)]->pattern_offset = p0;
    }
  });
}

int pg_set_model(pg_engine* e, int state_count, const double* q, const double* pi, int reversible) {
  return guarded([&] { each(e, [&](pg_engine* x) { x->set_model(state_count, q, pi, reversible); }); });
}

int pg_set_branch_generator(pg_engine* e, int branch, const double* q) {
  return guarded([&] { each(e, [&](pg_engine* x) { x->set_branch_generator(branch, q); }); });
}

int pg_set_categories(pg_engine* e, int category_count, const double* rates, const double* probs) {
  return guarded([&] { each(e, [&](pg_engine* x) { x->set_categories(category_count, rates, probs); }); });
}

int pg_set_branch_lengths(pg_engine* e, const double* b) {
  return guarded([&] { each(e, [&](pg_engine* x) { x->set_branch_lengths(b); }); });
}

int pg_set_branch_lengths_device(pg_engine* e, const double* b_device) {
  return guarded([&] {
    single_only(e, "pg_set_branch_lengths_device");
    e->set_branch_lengths_device(b_device);
  });
}

int pg_get_branch_lengths(pg_engine* e, double* b) {
  return guarded([&] {
    pg_engine* x = primary(e);
    x->set_device();
    x->sync_host_blen();
    std::copy(x->blen.begin(), x->blen.end(), b);
  });
}

int pg_set_clock_durations(pg_engine* e, const double* dt) {
  return guarded([&] { each(e, [&](pg_engine* x) { x->set_durations(dt); }); });
}

int pg_evaluate(pg_engine* e, int flags, double* log_likelihood, double* grad, double* hess) {
  return guarded([&] {
    if ((flags & (PG_EVAL_GRAD | PG_EVAL_RATE_GRAD)) && !grad)
      throw std::invalid_argument("pg_evaluate: gradient requested without an output buffer");
    if ((flags & PG_EVAL_HESS) && !hess)
      throw std::invalid_argument("pg_evaluate: Hessian requested without an output buffer");
    e->evaluate(flags, log_likelihood, grad, hess);
  });
}

int pg_evaluate_device(pg_engine* e, int flags, double* out_device) {
  return guarded([&] {
    single_only(e, "pg_evaluate_device");
    if (!out_device) throw std::invalid_argument("pg_evaluate_device: null output");
    e->invalidate();
    e->enqueue(flags | PG_EVAL_FORCE, out_device);
  });
}

int pg_check_errors(pg_engine* e) {
  return guarded([&] {
    single_only(e, "pg_check_errors");
    const bool grad = e->pending_flags & (PG_EVAL_GRAD | PG_EVAL_HESS | PG_EVAL_RATE_GRAD);
    e->check_errors();
    e->visits += uint64_t(grad ? 2 : 1) * uint64_t(2 * e->N - 1);
  });
}

int pg_set_stream(pg_engine* e, void* s) {
  return guarded([&] {
    single_only(e, "pg_set_stream");
    if (e->own_stream && e->stream) {
      PG_CUDA(cudaStreamSynchronize(e->stream));
      PG_CUDA(cudaStreamDestroy(e->stream));
    }
    e->stream = static_cast<cudaStream_t>(s);
    e->own_stream = false;
  });
}

int pg_get_partials(pg_engine* e, int node, int category, double* post, double* pre, double* post_scaler,
                    double* pre_scaler) {
  return guarded([&] {
    single_only(e, "pg_get_partials");
    if (!e->opt.capture_partials) throw std::logic_error("engine: partial capture is disabled");
    if (!e->pre_valid) throw std::logic_error("engine: no current gradient pass to read partials from");
    const int n = 2 * e->N - 1;
    if (node < 1 || node > n || category < 0 || category >= e->L)
      throw std::invalid_argument("engine: node or category out of range");
    e->set_device();
    const int P = e->P, MP = e->MP, m = e->m;
    const size_t nn = size_t(2 * e->N);
    std::vector<double> cp(nn * e->L * size_t(P) * MP), cq(cp.size());
    std::vector<int> ep(nn * size_t(P)), eq(ep.size());
    PG_CUDA(cudaMemcpy(cp.data(), e->d_cap_post.p, cp.size() * 8, cudaMemcpyDeviceToHost));
    PG_CUDA(cudaMemcpy(cq.data(), e->d_cap_pre.p, cq.size() * 8, cudaMemcpyDeviceToHost));
    PG_CUDA(cudaMemcpy(ep.data(), e->d_cap_post_exp.p, ep.size() * 4, cudaMemcpyDeviceToHost));
    PG_CUDA(cudaMemcpy(eq.data(), e->d_cap_pre_exp.p, eq.size() * 4, cudaMemcpyDeviceToHost));
    // reconstruct per-node log scalers (engine.hpp:192, :252) from own exponents
    std::vector<long> spost(nn * size_t(P), 0), spre(nn * size_t(P), 0);
    // post: children before parents -> iterate the schedule
    for (const int4& st : e->post_steps)
      for (int s = 0; s < P; ++s)
        spost[size_t(st.x) * P + s] =
            spost[size_t(st.y) * P + s] + spost[size_t(st.z) * P + s] + ep[size_t(st.x) * P + s];
    for (const int4& st : e->pre_steps)
      for (int side = 0; side < 2; ++side) {
        const int x = side ? st.z : st.y, y = side ? st.y : st.z;
        for (int s = 0; s < P; ++s)
          spre[size_t(x) * P + s] = spre[size_t(st.x) * P + s] + spost[size_t(y) * P + s] + eq[size_t(x) * P + s];
      }
    // Present values like the reference (engine.hpp:396-414): unscaled when the
    // true partial's peak is >= the rescaling threshold, otherwise normalised
    // with the remaining log scaler (true = value * exp(scaler)).
    const double ln2 = 0.6931471805599453;
    const double thr = e->opt.rescaling_threshold;
    const int L = e->L;
    auto emit = [&](const std::vector<double>& cap, long E, int s, double* out, double* scaler, bool is_pre) {
      double pk = 0.0;
      for (int l = 0; l < L; ++l)
        for (int j = 0; j < m; ++j) pk = std::max(pk, cap[((size_t(node) * L + l) * P + s) * MP + j]);
      const double true_pk = std::ldexp(pk, int(std::max<long>(std::min<long>(E, 4000), -4000)));
      const bool fold = e->opt.disable_rescaling || pk == 0.0 || (true_pk >= thr && std::isfinite(true_pk));
      long keepE = 0;
      if (!fold) {
        int ex;
        std::frexp(pk, &ex);
        keepE = E + ex;  // normalise peak into [0.5, 1)
      }
      for (int j = 0; j < m; ++j) {
        const double v = cap[((size_t(node) * L + category) * P + s) * MP + j];
        if (out) out[size_t(s) * m + j] = std::ldexp(v, int(std::max<long>(std::min<long>(E - keepE, 4000), -4000)));
      }
      if (scaler) *scaler = double(keepE) * ln2;
      (void)is_pre;
    };
    for (int s = 0; s < P; ++s) {
      if (node <= e->N) {
        if (post)
          for (int j = 0; j < m; ++j) post[size_t(s) * m + j] = std::numeric_limits<double>::quiet_NaN();
        if (post_scaler) post_scaler[s] = 0.0;
      } else {
        emit(cp, spost[size_t(node) * P + s], s, post, post_scaler ? post_scaler + s : nullptr, false);
      }
      if (node == n) {
        if (pre)
          for (int j = 0; j < m; ++j) pre[size_t(s) * m + j] = e->pi[size_t(j)];
        if (pre_scaler) pre_scaler[s] = 0.0;
      } else {
        emit(cq, spre[size_t(node) * P + s], s, pre, pre_scaler ? pre_scaler + s : nullptr, true);
      }
    }
  });
}

int pg_get_site_log_likelihoods(pg_engine* e, double* out) {
  return guarded([&] {
    int64_t off = 0;
    each(e, [&](pg_engine* x) {  // shards in pattern order
      if (!x->ll_valid) throw std::logic_error("engine: no current evaluation");
      x->set_device();
      PG_CUDA(cudaMemcpy(out + off, x->d_site_ll.p, size_t(x->P) * sizeof(double), cudaMemcpyDeviceToHost));
      off += x->P;
    });
  });
}

uint64_t pg_node_visits(const pg_engine* e) { return primary(e)->visits; }
void pg_reset_node_visits(pg_engine* e) {
  each(e, [](pg_engine* x) { x->visits = 0; });
}
void pg_invalidate_caches(pg_engine* e) {
  each(e, [](pg_engine* x) {
    x->invalidate();
    x->tc_dirty = true;  // the reference recomputes trans_ in every post pass (engine.hpp:197-201)
  });
}

int pg_engine_info(const pg_engine* e, int* launches, int* total_warps, int* lanes_per_pattern, int* padded_states) {
  return guarded([&] {
    e = primary(e);
    if (launches) *launches = e->last_launches;
    if (total_warps) *total_warps = e->TW;
    if (lanes_per_pattern) *lanes_per_pattern = e->G;
    if (padded_states) *padded_states = e->MP;
  });
}

int pg_timing(pg_engine* e, int enable, int* evaluations, double* walk_ms_total, double* eval_ms_total) {
  return guarded([&] {
    if (e->is_group())
      for (size_t i = 1; i < e->shards.size(); ++i) {  // shard 0 reports below
        pg_engine* x = e->shards[i].get();
        x->set_device();
        PG_CUDA(cudaStreamSynchronize(x->stream));
        x->tev_used = 0;
        x->timing = enable != 0;
      }
    e = primary(e);
    e->set_device();
    PG_CUDA(cudaStreamSynchronize(e->stream));
    const int n = int(e->tev_used / 3);
    double w = 0.0, t = 0.0;
    for (int i = 0; i < n; ++i) {
      float a = 0.f, b = 0.f;
      PG_CUDA(cudaEventElapsedTime(&a, e->tev[size_t(3 * i + 1)], e->tev[size_t(3 * i + 2)]));
      PG_CUDA(cudaEventElapsedTime(&b, e->tev[size_t(3 * i)], e->tev[size_t(3 * i + 2)]));
      w += a;
      t += b;
    }
    if (evaluations) *evaluations = n;
    if (walk_ms_total) *walk_ms_total = w;
    if (eval_ms_total) *eval_ms_total = t;
    e->tev_used = 0;
    e->timing = enable != 0;
  });
}

int pg_engine_variant(const pg_engine* e) {
  e = primary(e);
  return e->use_walkm ? 2 : e->use_walkl ? 3 : e->use_walk4 ? (e->use_walk4t ? 5 : e->use_walk4s ? 4 : 1) : 0;
}

int pg_last_walk_ms(const pg_engine* e, float* walk_ms, float* total_ms) {
  return guarded([&] {
    e = primary(e);
    if (walk_ms) *walk_ms = e->last_walk_ms;
    if (total_ms) *total_ms = e->last_total_ms;
  });
}

}  // extern "C"
