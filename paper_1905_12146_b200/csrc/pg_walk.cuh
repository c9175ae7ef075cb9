// phylograd-b200 device code (sm_100a, fp64).
//
// Three kernel families replace LikelihoodEngine's hot loops
// (/root/reference/proj/include/phylograd/engine.hpp):
//
//  K1 tc_kernel     — P(t) = e^{Q b c} per (branch, category) from the
//                     symmetric eigensystem (substitution.hpp:147-160, :196-208)
//                     or Pade scaling-and-squaring (substitution.hpp:71-75),
//                     clamp >= 0, t == 0 -> I; stored as columns, followed by
//                     P * (ambiguity partial) columns so every tip edge is a
//                     gather (engine.hpp:367-382).
//  K2 walk_kernel   — per-warp pattern tile walks the whole tree:
//                     post-order pruning p_k = e_c0 o e_c1 with per-pattern
//                     rescaling (engine.hpp:182-221, :396-414) and edge
//                     messages e_k = P_k p_k, then the pre-order pass
//                     q_c = P_c^T (q_k o e_sib) (engine.hpp:225-253) with the
//                     gradient (and Hessian diagonal) fused in
//                     (engine.hpp:255-274) using the self-normalised ratio
//                     top^T Q e / top^T e (Eq. 8 node invariance).
//  K3 reduce_kernel — fixed-order sum of the per-warp accumulators, then the
//                     clock chain rule d/dr = dt * d/db (clock.hpp:146-152).
#pragma once
// K2 lives here; K1/K3 are in pg_kernels.cuh.

#include <cstdint>
#include <cuda_runtime.h>

namespace pgk {

constexpr int kWarpsPerBlock = 4;

// mbarrier + 1-D bulk copy (TMA engine) helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* mb, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(mb)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* mb) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(mb))
      : "memory");
}
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// the same with an L2 cache-policy hint (e.g. evict-first for read-once data)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, uint64_t* mb,
                                              unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(mb)), "l"(pol)
      : "memory");
}
// order this thread's generic-proxy global stores before later async-proxy
// (bulk copy) reads issued by other threads after a barrier
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}


constexpr unsigned kFull = 0xffffffffu;

// Storage position of B fragment f = ki * NT + ni (of F = K * NT) for `lane`
// in the walkm matrix tables.  Codon-size tables (F >= kFragPairMin) store the
// fragments in pairs, (2h, 2h+1) adjacent per lane, so one 16-byte
// shared-memory load feeds two DMMAs (C5 413 -> 397 ms); an odd last fragment
// follows the pairs lane-contiguously.  Smaller tables keep one fragment per
// 256-byte row (C4: 144.6 vs 146.3 ms paired).
constexpr int kFragPairMin = 64;
__host__ __device__ __forceinline__ int frag_pos(int f, int lane, int F) {
  if (F < kFragPairMin) return f * 32 + lane;
  return f < (F & ~1) ? (((f >> 1) * 32 + lane) * 2 + (f & 1)) : ((F >> 1) * 64 + lane);
}

struct WalkParams {
  const uint8_t* codes;  // [N][Pc] tip column index into the TC table (rows padded to 32)
  const double* weights; // [P]
  const double* tc;      // [B][L][NC][MP]: column c of P (c < MP) or P*ambiguity (c >= MP)
  const double* qtc;     // same table for Q*P (walkm tips), may be null
  const double* qtab;    // [nq][MP][MP] row-major generators
  const int* qidx;       // [2N] node -> generator index
  const double* pi;      // [MP]
  const double* rates;   // [L]
  const double* probs;   // [L]
  const int4* post;      // [nsteps] {k, c0, c1, 0} internal nodes, heavy-child-first post order
  const int4* pre;       // [nsteps] {k, c0, c1, next} reverse of post; next = following step's node if a child of k
  double* escr;          // [TW][N-1][VEC] edge messages e_k of internal non-root nodes (walkm: + exponents per slot)
  double* qscr;          // [TW][N-1][VEC] pre-order partials of deferred internal nodes
  double* acc;           // [TW][accw]: [0] logL, [x] grad of branch x, [B+x] hess
  int* err;              // [2] first non-finite pattern, first underflowed pattern
  double* site_ll;       // [P] optional
  double* cap_post;      // optional debug capture [(2N)][L][P][MP]
  double* cap_pre;
  int* cap_post_exp;     // [(2N)][P]
  int* cap_pre_exp;
  int N, P, L, G, NC, nsteps, ntiles, accw, B;
  long long Pc;  // row stride of codes (P rounded up to 32)
  double thr;
  int force, disable, do_pre, hess;
};

// Parameters of the pipelined 4-state kernel (pg_walk4.cuh).
struct Walk4Params {
  WalkParams p;
  double q[16];  // homogeneous generator (row-major), constant-bank operands
  double pi[4];
};

// cherry flags of a step's children in its descriptor's x (pg_walk4s.cuh, CH instances)
constexpr int kCherryY = 1 << 29, kCherryZ = 1 << 30, kNodeMask = kCherryY - 1;
// double2 per cherry block: e_k table [0,128) | TC_u [128,160) | TC_v [160,192) | tip ids [192] | pad |
// W_u [200,328) | W_v [328,456)
constexpr int kCherryBlk = 456;

// Parameters of the single-buffered 4-state kernel (pg_walk4s.cuh).
struct Walk4SParams {
  Walk4Params w;
  double cw[4], crw[4], cr2w[4];  // category weights w_l, c_l w_l, c_l^2 w_l (constant-bank operands)
  int* qexp;                       // [TW][N-1][32] normalisation exponents of the deferred pre-partials
  // cherry tables (pg_walk4s.cuh, CH instances)
  const double* ct;       // [N-1][4][16][4] e_k per (category, code pair) of cherry node k, by k - N - 1
  const uint8_t* ccodes;  // [N-1][Pc] combined code rows 4 ca + cb, by k - N - 1
  int npost;              // post-order steps without the cherries' own
};

// Parameters of the tensor-core 4-state kernel (pg_walk4t.cuh).
struct Walk4TParams {
  Walk4SParams s;
  const double* f4post;  // [B][L][32] B fragments of e = P x
  const double* f4pre;   // [B][L+1][32] B fragments of (P^T t | Q^T t), [L]: (Q^2)^T t
};

// Parameters of the DMMA large-state kernel (pg_walkm.cuh).
struct WalkMParams {
  WalkParams p;
  const double* fpp;  // [B][L][MP*MP] P in B-fragment order (y = P x)
  const double* fpt;  // [B][L][MP*MP] (y = P^T x)
  const double* fq;   // [nQ][MP*MP] generators in B-fragment order (y = Q x)
  int homogeneous;  // stage the shared generator in shared memory
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
// sums of a over the warp in lane 0 and of b in lane 16 (one butterfly for
// two values: the first level exchanges halves)
__device__ __forceinline__ double warp_sum2(double a, double b) {
  const bool lo = (threadIdx.x & 16) == 0;
  double v = (lo ? a : b) + __shfl_xor_sync(kFull, lo ? b : a, 16);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ double group_sum(double v, int G) {
  for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ double group_max(double v, int G) {
  for (int o = 1; o < G; o <<= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// One lane holds LC categories x MP states of one pattern.  Slot layout is
// [LC*MP/2][32 lanes] double2 so every warp access is 512 contiguous bytes.
template <int MP, int LC>
__device__ __forceinline__ void load_slot(const double* base, int lane, double (&v)[LC][MP]) {
  const double2* src = reinterpret_cast<const double2*>(base);
#pragma unroll
  for (int q = 0; q < LC * MP / 2; ++q) {
    const double2 d = __ldcg(src + q * 32 + lane);
    v[(2 * q) / MP][(2 * q) % MP] = d.x;
    v[(2 * q + 1) / MP][(2 * q + 1) % MP] = d.y;
  }
}
template <int MP, int LC>
__device__ __forceinline__ void store_slot(double* base, int lane, const double (&v)[LC][MP]) {
  double2* dst = reinterpret_cast<double2*>(base);
#pragma unroll
  for (int q = 0; q < LC * MP / 2; ++q) {
    double2 d;
    d.x = v[(2 * q) / MP][(2 * q) % MP];
    d.y = v[(2 * q + 1) / MP][(2 * q + 1) % MP];
    __stcg(dst + q * 32 + lane, d);
  }
}

// Tip edge message: gather column `code` of P (or of P * ambiguity partial).
template <int MP, int LC>
__device__ __forceinline__ void gather_tip(const WalkParams& p, int node, int sc, const int (&lc)[LC],
                                           double (&v)[LC][MP]) {
  const int col = p.codes[size_t(node - 1) * size_t(p.Pc) + sc];
#pragma unroll
  for (int j = 0; j < LC; ++j) {
    const double2* src =
        reinterpret_cast<const double2*>(p.tc + ((size_t(node - 1) * p.L + lc[j]) * p.NC + col) * MP);
#pragma unroll
    for (int h = 0; h < MP / 2; ++h) {
      const double2 d = __ldg(src + h);
      v[j][2 * h] = d.x;
      v[j][2 * h + 1] = d.y;
    }
  }
}

// Exact power-of-two normalisation of one pattern's LC x MP block (group max
// over the G lanes of the pattern brought into [0.5, 1)).  Returns the
// exponent removed.  Post-order partials are normalised at every internal
// node (the reference rescales by the peak only below 1e-150, engine.hpp:
// 396-414; scaling by 2^k is exact, so values differ from the reference only
// by that bookkeeping, which logL = log(mix) + S ln 2 undoes).  Pre-order
// partials are normalised when produced: the gradient ratio is invariant to
// it, and keeping q ~ 1 keeps q o e_a o e_b away from the subnormal range.
template <int MP, int LC>
__device__ __forceinline__ int normalize(double (&v)[LC][MP], int G) {
  double pk = 0.0;
#pragma unroll
  for (int j = 0; j < LC; ++j)
#pragma unroll
    for (int i = 0; i < MP; ++i) pk = fmax(pk, v[j][i]);
  pk = group_max(pk, G);
  const long long bits = __double_as_longlong(pk);
  const int biased = int((bits >> 52) & 0x7ff);
  if (pk <= 0.0 || biased == 0x7ff) return 0;  // zero, inf or NaN: leave alone
  int ex;
  if (biased == 0) {  // subnormal peak
    frexp(pk, &ex);
#pragma unroll
    for (int j = 0; j < LC; ++j)
#pragma unroll
      for (int i = 0; i < MP; ++i) v[j][i] = ldexp(v[j][i], -ex);
    return ex;
  }
  ex = biased - 1022;
  if (ex == 0) return 0;
  const double sc = __longlong_as_double((long long)(1023 - ex) << 52);
  if (1023 - ex <= 0 || 1023 - ex >= 2047) {
#pragma unroll
    for (int j = 0; j < LC; ++j)
#pragma unroll
      for (int i = 0; i < MP; ++i) v[j][i] = ldexp(v[j][i], -ex);
    return ex;
  }
#pragma unroll
  for (int j = 0; j < LC; ++j)
#pragma unroll
    for (int i = 0; i < MP; ++i) v[j][i] *= sc;
  return ex;
}

template <int MP, int LC>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) walk_kernel(const __grid_constant__ WalkParams p) {
  const int lane = threadIdx.x & 31;
  const int warp = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int TW = gridDim.x * kWarpsPerBlock;
  const int G = p.G, TP = 32 / G;
  const int g = lane & (G - 1), pl = lane / G;
  const int root = 2 * p.N - 1;

  int lc[LC];
  double cw[LC], crw[LC], cr2w[LC];
  bool creal[LC];
#pragma unroll
  for (int j = 0; j < LC; ++j) {
    const int l = g * LC + j;
    creal[j] = l < p.L;
    lc[j] = creal[j] ? l : p.L - 1;
    const double w = creal[j] ? p.probs[lc[j]] : 0.0, r = p.rates[lc[j]];
    cw[j] = w;
    crw[j] = r * w;
    cr2w[j] = r * r * w;
  }
  constexpr size_t VEC = size_t(32) * LC * MP;
  double* E = p.escr + size_t(warp) * size_t(p.N - 1) * VEC;
  double* Qs = p.qscr + size_t(warp) * size_t(p.N - 1) * VEC;
  double* A = p.acc + size_t(warp) * p.accw;
  for (int i = lane; i < p.accw; i += 32) A[i] = 0.0;
  __syncwarp();

  for (int t = warp; t < p.ntiles; t += TW) {
    const int s = t * TP + pl;
    const bool valid = s < p.P;
    const int sc = valid ? s : p.P - 1;
    const double w = valid ? p.weights[sc] : 0.0;
    const bool owner = valid && g == 0;

    // ------------------------------------------------ post-order pass (a)
    int S = 0;  // accumulated power-of-two rescale exponent of this pattern
    double keep[LC][MP];
    int last = -1;
    for (int i = 0; i < p.nsteps; ++i) {
      const int4 st = p.post[i];
      const int k = st.x;
      double x[LC][MP], y[LC][MP];
      if (st.y <= p.N) gather_tip<MP, LC>(p, st.y, sc, lc, x);
      else if (st.y == last) {
#pragma unroll
        for (int j = 0; j < LC; ++j)
#pragma unroll
          for (int q = 0; q < MP; ++q) x[j][q] = keep[j][q];
      } else load_slot<MP, LC>(E + size_t(st.y - p.N - 1) * VEC, lane, x);
      if (st.z <= p.N) gather_tip<MP, LC>(p, st.z, sc, lc, y);
      else if (st.z == last) {
#pragma unroll
        for (int j = 0; j < LC; ++j)
#pragma unroll
          for (int q = 0; q < MP; ++q) y[j][q] = keep[j][q];
      } else load_slot<MP, LC>(E + size_t(st.z - p.N - 1) * VEC, lane, y);

#pragma unroll
      for (int j = 0; j < LC; ++j)
#pragma unroll
        for (int q = 0; q < MP; ++q) x[j][q] *= y[j][q];
      const int ex = p.disable ? 0 : normalize<MP, LC>(x, G);
      S += ex;
      if (p.cap_post && valid) {
#pragma unroll
        for (int j = 0; j < LC; ++j)
          if (creal[j])
            for (int q = 0; q < MP; ++q) p.cap_post[((size_t(k) * p.L + lc[j]) * p.P + s) * MP + q] = x[j][q];
        if (g == 0) p.cap_post_exp[size_t(k) * p.P + s] = ex;
      }
      if (k == root) {
        double mix = 0.0;
#pragma unroll
        for (int j = 0; j < LC; ++j) {
          double d = 0.0;
#pragma unroll
          for (int q = 0; q < MP; ++q) d = fma(p.pi[q], x[j][q], d);
          mix = fma(cw[j], d, mix);
        }
        mix = group_sum(mix, G);
        const double ll = log(mix) + double(S) * 0.6931471805599453;
        if (owner) {
          if (!isfinite(mix)) atomicMin(&p.err[0], s);
          else if (mix <= 0.0) atomicMin(&p.err[1], s);
          if (p.site_ll) p.site_ll[s] = ll;
        }
        const double v = warp_sum(owner ? w * ll : 0.0);
        if (lane == 0) A[0] += v;
      } else {
        // edge message e_k = P_k p_k (engine.hpp:367-372)
#pragma unroll
        for (int j = 0; j < LC; ++j) {
          const double2* T =
              reinterpret_cast<const double2*>(p.tc + (size_t(k - 1) * p.L + lc[j]) * p.NC * MP);
          double e[MP];
#pragma unroll
          for (int q = 0; q < MP; ++q) e[q] = 0.0;
#pragma unroll
          for (int c = 0; c < MP; ++c) {
            const double xc = x[j][c];
#pragma unroll
            for (int h = 0; h < MP / 2; ++h) {
              const double2 col = __ldg(T + c * (MP / 2) + h);
              e[2 * h] = fma(col.x, xc, e[2 * h]);
              e[2 * h + 1] = fma(col.y, xc, e[2 * h + 1]);
            }
          }
#pragma unroll
          for (int q = 0; q < MP; ++q) keep[j][q] = e[q];
        }
        store_slot<MP, LC>(E + size_t(k - p.N - 1) * VEC, lane, keep);
        last = k;
      }
    }
    if (!p.do_pre) continue;

    // ----------------------------------- pre-order pass + gradient (b)+(c)
    double qreg[LC][MP];
    int qnode = -1;
    for (int i = 0; i < p.nsteps; ++i) {
      const int4 st = p.pre[i];
      const int k = st.x;
      double q[LC][MP];
      if (k == root) {
#pragma unroll
        for (int j = 0; j < LC; ++j)
#pragma unroll
          for (int r = 0; r < MP; ++r) q[j][r] = p.pi[r];
      } else if (k == qnode) {
#pragma unroll
        for (int j = 0; j < LC; ++j)
#pragma unroll
          for (int r = 0; r < MP; ++r) q[j][r] = qreg[j][r];
      } else {
        load_slot<MP, LC>(Qs + size_t(k - p.N - 1) * VEC, lane, q);
      }
      double ea[LC][MP], eb[LC][MP];
      if (st.y <= p.N) gather_tip<MP, LC>(p, st.y, sc, lc, ea);
      else load_slot<MP, LC>(E + size_t(st.y - p.N - 1) * VEC, lane, ea);
      if (st.z <= p.N) gather_tip<MP, LC>(p, st.z, sc, lc, eb);
      else load_slot<MP, LC>(E + size_t(st.z - p.N - 1) * VEC, lane, eb);

      // denominator L_s e^{-S}: identical for both children (Eq. 8)
      double den = 0.0;
#pragma unroll
      for (int j = 0; j < LC; ++j) {
        double d = 0.0;
#pragma unroll
        for (int r = 0; r < MP; ++r) d = fma(q[j][r] * ea[j][r], eb[j][r], d);
        den = fma(cw[j], d, den);
      }
      den = group_sum(den, G);

      auto child = [&](const int x, const double(&ex_)[LC][MP], const double(&ey)[LC][MP]) {
        const bool need_q = x > p.N || p.cap_pre != nullptr;
        const double* Qm = p.qtab + size_t(p.qidx[x]) * MP * MP;
        double num = 0.0, num2 = 0.0;
        double qx[LC][MP];
#pragma unroll
        for (int j = 0; j < LC; ++j) {
          double top[MP];
#pragma unroll
          for (int r = 0; r < MP; ++r) top[r] = q[j][r] * ey[j][r];
          double qe[MP];
#pragma unroll
          for (int r = 0; r < MP; ++r) {
            double a = 0.0;
#pragma unroll
            for (int c = 0; c < MP; ++c) a = fma(__ldg(Qm + r * MP + c), ex_[j][c], a);
            qe[r] = a;
          }
          double d1 = 0.0;
#pragma unroll
          for (int r = 0; r < MP; ++r) d1 = fma(top[r], qe[r], d1);
          num = fma(crw[j], d1, num);
          if (p.hess) {
            double d2 = 0.0;
#pragma unroll
            for (int r = 0; r < MP; ++r) {
              double a = 0.0;
#pragma unroll
              for (int c = 0; c < MP; ++c) a = fma(__ldg(Qm + r * MP + c), qe[c], a);
              d2 = fma(top[r], a, d2);
            }
            num2 = fma(cr2w[j], d2, num2);
          }
          if (need_q) {
            // q_x = P_x^T top (engine.hpp:249-250): column c of P dotted with top
            const double2* T =
                reinterpret_cast<const double2*>(p.tc + (size_t(x - 1) * p.L + lc[j]) * p.NC * MP);
#pragma unroll
            for (int c = 0; c < MP; ++c) {
              double a = 0.0;
#pragma unroll
              for (int h = 0; h < MP / 2; ++h) {
                const double2 col = __ldg(T + c * (MP / 2) + h);
                a = fma(col.x, top[2 * h], a);
                a = fma(col.y, top[2 * h + 1], a);
              }
              qx[j][c] = a;
            }
          }
        }
        num = group_sum(num, G);
        const double r1 = num / den;
        const double gv = warp_sum(owner ? w * r1 : 0.0);
        if (lane == 0) A[x] += gv;
        if (p.hess) {
          num2 = group_sum(num2, G);
          const double r2 = num2 / den;
          const double hv = warp_sum(owner ? w * (r2 - r1 * r1) : 0.0);
          if (lane == 0) A[p.B + x] += hv;
        }
        if (need_q) {
          // normalise q_x by an exact power of two (the gradient ratio is
          // invariant to it); the exponent is recorded for the debug capture
          const int exq = normalize<MP, LC>(qx, G);
          if (p.cap_pre && valid) {
#pragma unroll
            for (int j = 0; j < LC; ++j)
              if (creal[j])
                for (int r = 0; r < MP; ++r) p.cap_pre[((size_t(x) * p.L + lc[j]) * p.P + s) * MP + r] = qx[j][r];
            if (g == 0) p.cap_pre_exp[size_t(x) * p.P + s] = exq;
          }
          if (x > p.N) {
            if (x == st.w) {
#pragma unroll
              for (int j = 0; j < LC; ++j)
#pragma unroll
                for (int r = 0; r < MP; ++r) qreg[j][r] = qx[j][r];
              qnode = x;
            } else {
              store_slot<MP, LC>(Qs + size_t(x - p.N - 1) * VEC, lane, qx);
            }
          }
        }
      };
      child(st.y, ea, eb);
      child(st.z, eb, ea);
    }
  }
}

}  // namespace pgk
