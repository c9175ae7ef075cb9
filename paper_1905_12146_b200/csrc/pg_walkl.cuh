// K2e: level-scheduled 4-state traversal for the small-P regime.
//
// The persistent walks (walk4 / walkm) give every warp whole tiles of
// patterns and walk the whole tree per tile, so their parallelism is the
// number of pattern tiles: with few patterns per GPU (C2 at 8 GPUs: ~2,500
// patterns = 78 tiles of 32 for 148 SMs) most SMs idle and each tile's
// ~2N dependent steps are latency-bound.  Here the parallelism is
// (independent nodes of one tree level) x (pattern tiles), as the north star
// sketches ("level-scheduled launches so that independent nodes of one tree
// depth run concurrently"): the post-order pass runs level by level in node
// height (a node only needs its children: height(k) = 1 + max over children),
// the pre-order pass level by level in node depth, with a grid-wide barrier
// between levels inside one persistent cooperative launch (no per-level
// launch latency).  A warp unit is one node x TP = 32 / L patterns, lane
// (pattern, category); cross-category quantities (normalisation peak, root
// mixture, gradient ratio terms) are L-lane shuffles.
//
// Every edge message e_k and pre-partial q_k lives in global memory
// ([internal node][pattern][category][4] doubles, with the per-pattern
// cumulative post exponent S_k), which at small P stays in L2.  The gradient
// of branch x from pattern tile t is written once to accumulator row t
// (single writer), and K3 sums the rows in fixed order: deterministic.
// Same arithmetic as walk4 per (pattern, category); category sums are
// shuffle trees instead of sequential fma chains.
#pragma once

#include "pg_walk4.cuh"

namespace pgk {

struct WalkLParams {
  WalkParams p;
  double q[16];           // homogeneous generator (row-major, constant-bank operands)
  double pi[4];
  const int* lvl_nodes;   // post levels (internal nodes by height), then pre levels (by depth)
  const int* lvl_off;     // [npost + 1 + npre + 1] offsets into lvl_nodes
  int npost, npre;
  const int* children;    // [2N][2]
  double* E;              // [N-1][P][L][4] edge messages of internal nodes (index node-N-1)
  double* Qp;             // [N-1][P][L][4] pre-partials of internal nodes
  int* Sx;                // [N-1][P] cumulative post exponents
  unsigned* bar;          // grid barrier {arrivals, generation}
  int ntp;                // pattern tiles of TP = 32 / L patterns
};

// Grid-wide barrier for a cooperative (co-resident) grid: the last arriving
// CTA resets the count and bumps the generation; writes before the barrier
// are visible to every CTA after it.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

template <int L, bool HOMOG, bool HESS>
__global__ void __launch_bounds__(256) walkl_kernel(const __grid_constant__ WalkLParams PL) {
  constexpr int TP = 32 / L;  // patterns per warp unit
  const WalkParams& p = PL.p;
  const int lane = threadIdx.x & 31, pl = lane / L, c = lane % L;
  const int gw = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nw = int((gridDim.x * blockDim.x) >> 5);
  const int N = p.N, root = 2 * N - 1, P = p.P, NC = p.NC, B = p.B;
  const long long accw = p.accw;
  const double cw = p.probs[c], crw = p.rates[c] * cw, cr2w = p.rates[c] * crw;
  auto gmaxi = [&](int v) {
#pragma unroll
    for (int o = 1; o < L; o <<= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
    return v;
  };
  auto gsum = [&](double v) {
#pragma unroll
    for (int o = 1; o < L; o <<= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
  };
  auto ld4 = [](const double* src, double (&v)[4]) {
    const double2 a = __ldcg(reinterpret_cast<const double2*>(src)), b = __ldcg(reinterpret_cast<const double2*>(src) + 1);
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  };
  auto st4 = [](double* dst, const double (&v)[4], double s) {
    __stcg(reinterpret_cast<double2*>(dst), make_double2(v[0] * s, v[1] * s));
    __stcg(reinterpret_cast<double2*>(dst) + 1, make_double2(v[2] * s, v[3] * s));
  };
  // column `code` of category c of node x's [L][NC][4] table (P columns, then P * ambiguity)
  auto col = [&](const double* tab, int x, int code, double (&v)[4]) {
    const double2* s2 = reinterpret_cast<const double2*>(tab + ((size_t(x - 1) * L + c) * NC + code) * 4);
    const double2 a = __ldg(s2), b = __ldg(s2 + 1);
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  };
  auto qm = [&](int x, int r, int cc) -> double {
    if constexpr (HOMOG) return PL.q[r * 4 + cc];
    else return __ldg(p.qtab + size_t(p.qidx[x]) * 16 + r * 4 + cc);
  };
  auto slot = [&](double* base, int node, int s) { return base + ((size_t(node - N - 1) * P + s) * L + c) * 4; };

  // ------------------------------------------------------- post levels
  for (int lv = 0; lv < PL.npost; ++lv) {
    const int o0 = PL.lvl_off[lv], o1 = PL.lvl_off[lv + 1];
    const long long units = (long long)(o1 - o0) * PL.ntp;
    for (long long u = gw; u < units; u += nw) {
      const int k = PL.lvl_nodes[o0 + int(u / PL.ntp)], tile = int(u % PL.ntp);
      const int s = tile * TP + pl;
      const bool valid = s < P;
      const int sc = valid ? s : P - 1;
      const int y = PL.children[2 * k], z = PL.children[2 * k + 1];
      double a[4], b[4], x[4];
      int S = 0;
      if (y <= N) col(p.tc, y, p.codes[size_t(y - 1) * size_t(p.Pc) + sc], a);
      else {
        ld4(slot(PL.E, y, sc), a);
        S += __ldcg(PL.Sx + size_t(y - N - 1) * P + sc);
      }
      if (z <= N) col(p.tc, z, p.codes[size_t(z - 1) * size_t(p.Pc) + sc], b);
      else {
        ld4(slot(PL.E, z, sc), b);
        S += __ldcg(PL.Sx + size_t(z - N - 1) * P + sc);
      }
      int hm = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        x[r] = a[r] * b[r];
        hm = max(hm, __double2hiint(x[r]));
      }
      if (!p.disable) {
        const int ex = peak_exponent(gmaxi(hm));
        if (ex != 0) {
          S += ex;
          if (ex <= 1022) {
            const double sc2 = pow2_neg(ex);
#pragma unroll
            for (int r = 0; r < 4; ++r) x[r] *= sc2;
          } else {
#pragma unroll
            for (int r = 0; r < 4; ++r) x[r] = ldexp(x[r], -ex);
          }
        }
      }
      if (k == root) {
        double dd = 0.0;
#pragma unroll
        for (int r = 0; r < 4; ++r) dd = fma(PL.pi[r], x[r], dd);
        const double mix = gsum(cw * dd);
        const double ll = log(mix) + double(S) * 0.6931471805599453;
        const bool owner = valid && c == 0;
        if (owner) {
          if (!isfinite(mix)) atomicMin(&p.err[0], s);
          else if (mix <= 0.0) atomicMin(&p.err[1], s);
          if (p.site_ll) p.site_ll[s] = ll;
        }
        const double v = warp_sum(owner ? p.weights[s] * ll : 0.0);
        if (lane == 0) p.acc[size_t(tile) * accw] = v;
      } else {
        // e_k = P_k p_k (engine.hpp:367-372)
        const double2* T = reinterpret_cast<const double2*>(p.tc + (size_t(k - 1) * L + c) * NC * 4);
        double e[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const double2 u0 = __ldg(T + 2 * cc), u1 = __ldg(T + 2 * cc + 1);
          e[0] = fma(u0.x, x[cc], e[0]);
          e[1] = fma(u0.y, x[cc], e[1]);
          e[2] = fma(u1.x, x[cc], e[2]);
          e[3] = fma(u1.y, x[cc], e[3]);
        }
        if (valid) {
          st4(slot(PL.E, k, s), e, 1.0);
          if (c == 0) __stcg(PL.Sx + size_t(k - N - 1) * P + s, S);
        }
      }
    }
    grid_barrier(PL.bar);
  }

  // -------------------------------------------------------- pre levels
  if (!p.do_pre) return;
  const int* poff = PL.lvl_off + PL.npost + 1;
  for (int lv = 0; lv < PL.npre; ++lv) {
    const int o0 = poff[lv], o1 = poff[lv + 1];
    const long long units = (long long)(o1 - o0) * PL.ntp;
    for (long long u = gw; u < units; u += nw) {
      const int k = PL.lvl_nodes[o0 + int(u / PL.ntp)], tile = int(u % PL.ntp);
      const int s = tile * TP + pl;
      const bool valid = s < P;
      const int sc = valid ? s : P - 1;
      const int y = PL.children[2 * k], z = PL.children[2 * k + 1];
      const bool a_int = y > N, b_int = z > N;
      double q[4], ea[4], eb[4];
      if (k == root) {
#pragma unroll
        for (int r = 0; r < 4; ++r) q[r] = PL.pi[r];
      } else {
        ld4(slot(PL.Qp, k, sc), q);
      }
      int code0 = 0, code1 = 0;
      if (a_int) ld4(slot(PL.E, y, sc), ea);
      else {
        code0 = p.codes[size_t(y - 1) * size_t(p.Pc) + sc];
        col(p.tc, y, code0, ea);
      }
      if (b_int) ld4(slot(PL.E, z, sc), eb);
      else {
        code1 = p.codes[size_t(z - 1) * size_t(p.Pc) + sc];
        col(p.tc, z, code1, eb);
      }
      double ta[4], tb[4], dd = 0.0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        ta[r] = q[r] * eb[r];
        tb[r] = q[r] * ea[r];
        dd = fma(ta[r], ea[r], dd);
      }
      double qea[4], qeb[4];
      if (a_int || !p.qtc) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double v = 0.0;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) v = fma(qm(y, r, cc), ea[cc], v);
          qea[r] = v;
        }
      } else {
        col(p.qtc, y, code0, qea);
      }
      if (b_int || !p.qtc) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double v = 0.0;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) v = fma(qm(z, r, cc), eb[cc], v);
          qeb[r] = v;
        }
      } else {
        col(p.qtc, z, code1, qeb);
      }
      double d1a = 0.0, d1b = 0.0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        d1a = fma(ta[r], qea[r], d1a);
        d1b = fma(tb[r], qeb[r], d1b);
      }
      const double den = gsum(cw * dd), na = gsum(crw * d1a), nb = gsum(crw * d1b);
      const double inv = 1.0 / den;
      const double r1a = na * inv, r1b = nb * inv;
      const bool owner = valid && c == 0;
      const double w = owner ? p.weights[s] : 0.0;
      const double ga = warp_sum(w * r1a), gb = warp_sum(w * r1b);
      double* row = p.acc + size_t(tile) * accw;
      if (lane == 0) {
        row[y] = ga;
        row[z] = gb;
      }
      if constexpr (HESS) {
        double d2a = 0.0, d2b = 0.0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double u = 0.0, v = 0.0;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            u = fma(qm(y, r, cc), qea[cc], u);
            v = fma(qm(z, r, cc), qeb[cc], v);
          }
          d2a = fma(ta[r], u, d2a);
          d2b = fma(tb[r], v, d2b);
        }
        const double na2 = gsum(cr2w * d2a), nb2 = gsum(cr2w * d2b);
        const double ha2 = warp_sum(w * (na2 * inv - r1a * r1a)), hb2 = warp_sum(w * (nb2 * inv - r1b * r1b));
        if (lane == 0) {
          row[B + y] = ha2;
          row[B + z] = hb2;
        }
      }
      // outgoing pre-partials q_x = P_x^T top (engine.hpp:249-250), normalised
      auto emit = [&](int xn, const double (&t)[4]) {
        const double2* T = reinterpret_cast<const double2*>(p.tc + (size_t(xn - 1) * L + c) * NC * 4);
        double qx[4];
        int h = 0;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const double2 u0 = __ldg(T + 2 * cc), u1 = __ldg(T + 2 * cc + 1);
          qx[cc] = fma(u0.x, t[0], fma(u0.y, t[1], fma(u1.x, t[2], u1.y * t[3])));
          h = max(h, __double2hiint(qx[cc]));
        }
        const int ex = peak_exponent(gmaxi(h));
        const double scl = (ex != 0 && ex <= 1022) ? pow2_neg(ex) : 1.0;
        if (valid) st4(slot(PL.Qp, xn, s), qx, scl);
      };
      if (a_int) emit(y, ta);
      if (b_int) emit(z, tb);
    }
    if (lv + 1 < PL.npre) grid_barrier(PL.bar);
  }
}

}  // namespace pgk
