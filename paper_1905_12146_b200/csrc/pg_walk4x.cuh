// K2d: the 4-state walk with the rate categories spread over the warps of a
// CTA (C2/C3: 4-state + Gamma4).
//
// A CTA of LW warps owns a tile of 32 patterns; warp l holds category l of
// every pattern of the tile (one lane per pattern, 4 doubles per vector), and
// the warps walk the tree in lock-step, one node per step.  Against walk4
// (one lane per pattern holding all categories, 255 registers, 8 warps per
// SM) a thread carries a quarter of the state, so about four times as many
// warps are resident and the fp64 / shared-memory latencies of one warp are
// covered by the others (walk4's C3 profile: 2 warps per scheduler, 36 % of
// the samples in fixed-latency waits, 17 % in shared-memory load-use waits).
//
// Staging.  Every operand of the CTA tile is ONE 1-D bulk copy (cp.async.bulk,
// TMA engine) into a stage of shared memory: an internal child's edge-message
// slot or a deferred pre-partial ([node][cat][lane][4] doubles, LW KB), a
// node's column table TC ([cat][NC][4] doubles), a tip's 32 code bytes, a
// tip's Q P table (pre-order pass).  Three stages rotate; step j+1's copies
// are issued at the top of step j (lane 0 of the warps, operands spread over
// the warps) and complete on the stage's mbarrier, and the DRAM operands of
// step j+2 are prefetched into L2 at the same time.  A value produced by
// step i and consumed by step i+1 or i+2 never goes through global memory
// for that use: the producing warp writes its category slice straight into
// the consumer's stage (the post-order edge message of step i+1 stays in
// registers; a pre-partial consumed next or after one more step; the root's
// pi).  Anything consumed later was stored at least two steps earlier, so
// its async-proxy fence and CTA barrier precede the copy.
//
// Cross-category quantities go through a small shared exchange (double-
// buffered by step parity) with one CTA barrier per step: the per-pattern
// peak exponent (post: normalisation of p_k; pre: of the outgoing q_c), the
// root mixture and the gradient ratio terms (den, num_a, num_b).  Every
// per-pattern arithmetic chain is the one walk4 evaluates (same operand
// order, same fma nesting over categories).
#pragma once

#include "pg_walk4.cuh"

namespace pgk {

__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

// one step of a CTA's stream: descriptor, tile, index within the tile's
// post (k < n) / pre (k >= n) steps; k < 0 past the end
struct Walk4xStep {
  int4 d;
  int tile, k;
  bool pre;
};

template <int LW, int NC, bool HESS>
struct Walk4xGeom {
  static constexpr int NST = 3;              // stages
  static constexpr int SLOT = LW * 32 * 4;   // doubles: one node slot of the CTA tile
  static constexpr int TCB = LW * NC * 4;    // doubles: one node's column table (all categories)
  static constexpr int STAGE = 3 * SLOT + 3 * TCB + 8;  // 3 operand slots, 3 TC blocks, 2 x 32 code bytes
  static constexpr int NR = HESS ? 5 : 3;    // gradient exchange terms per (category, pattern)
  // exchange (per parity): int peak exponents [2][32][LW], double terms [NR][32][LW]
  static constexpr int XI = 2 * 32 * LW;
  static constexpr int XD = NR * 32 * LW;
  static constexpr size_t smem_bytes() {
    return size_t(NST * STAGE) * 8 + size_t(2 * XD) * 8 + size_t(2 * XI) * 4 + NST * 8;
  }
};

template <bool HOMOG, bool HESS, int NC, int LW>
__global__ void __launch_bounds__(32 * LW, (LW >= 4 ? 4 : 8)) walk4x_kernel(const __grid_constant__ Walk4Params P4) {
  using Gx = Walk4xGeom<LW, NC, HESS>;
  constexpr int NST = Gx::NST, SLOT = Gx::SLOT, TCB = Gx::TCB, STAGE = Gx::STAGE;
  const WalkParams& p = P4.p;
  extern __shared__ __align__(16) double sm4x[];
  double* stg = sm4x;                                        // [NST][STAGE]
  double* xd = sm4x + NST * STAGE;                           // [2][NR][32][LW]
  int* xi = reinterpret_cast<int*>(xd + 2 * Gx::XD);         // [2][2][32][LW]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(xi + 2 * Gx::XI);
  const int tid = threadIdx.x, lane = tid & 31, l = tid >> 5;  // warp = category
  const int N = p.N, root = 2 * N - 1, n = p.nsteps;
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(mbar + i, LW);  // lane 0 of every warp arrives once per use
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  double* A = p.acc + size_t(blockIdx.x) * p.accw;  // this CTA's accumulator row
  for (int i = tid; i < p.accw; i += 32 * LW) A[i] = 0.0;
  // CTA-major scratch: slot of node k at (k - N - 1) * SLOT, category l at + l * 128
  double* E = p.escr + size_t(blockIdx.x) * size_t(N - 1) * SLOT;
  double* Qs = p.qscr + size_t(blockIdx.x) * size_t(N - 1) * SLOT;

  auto op = [&](int st, int k) -> double* { return stg + st * STAGE + k * SLOT; };
  auto tcb = [&](int st, int k) -> double* { return stg + st * STAGE + 3 * SLOT + k * TCB; };
  auto cbytes = [&](int st) -> uint8_t* { return reinterpret_cast<uint8_t*>(stg + st * STAGE + 3 * SLOT + 3 * TCB); };
  // this warp's category part of a slot: [h][lane] double2 (512 B per access)
  auto rd4 = [&](const double* slot, double (&v)[4]) {
    const double2* s2 = reinterpret_cast<const double2*>(slot + l * 128) + lane;
    const double2 a = s2[0], b = s2[32];
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  };
  auto wr4_smem = [&](double* slot, const double (&v)[4], double s) {
    double2* d2 = reinterpret_cast<double2*>(slot + l * 128) + lane;
    d2[0] = make_double2(v[0] * s, v[1] * s);
    d2[32] = make_double2(v[2] * s, v[3] * s);
  };
  // column `code` of category l in a [cat][NC][4] table
  auto col4 = [&](const double* tab, int code, double (&v)[4]) {
    const double2* c2 = reinterpret_cast<const double2*>(tab + (l * NC + code) * 4);
    const double2 a = c2[0], b = c2[1];
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  };
  auto qm = [&](int x, int r, int c) -> double {
    if constexpr (HOMOG) return P4.q[r * 4 + c];
    else return __ldg(p.qtab + size_t(p.qidx[x]) * 16 + r * 4 + c);
  };

  // ---------------------------------------------------------- step stream
  // The CTA's work is one stream of steps: per tile, the n post-order steps,
  // then (gradient) the n pre-order steps.  A window of descriptors runs two
  // steps ahead of the current one (D[0] = current, D[1], D[2]) and keeps the
  // two previous ones (Dm1, Dm2).
  const int per_tile = p.do_pre ? 2 * n : n;
  if (int(blockIdx.x) >= p.ntiles) return;
  auto load = [&](int tile, int k) -> Walk4xStep {
    Walk4xStep s;
    s.tile = tile;
    s.k = k;
    s.pre = k >= n;
    if (tile >= p.ntiles) {
      s.d = make_int4(-1, -1, -1, -1);
      s.k = -1;
    } else {
      s.d = k >= n ? __ldg(p.pre + (k - n)) : __ldg(p.post + k);
    }
    return s;
  };
  auto next_of = [&](const Walk4xStep& s) -> Walk4xStep {
    if (s.k < 0) return s;
    return s.k + 1 < per_tile ? load(s.tile, s.k + 1) : load(s.tile + int(gridDim.x), 0);
  };
  auto none = [&]() {
    Walk4xStep s;
    s.d = make_int4(-1, -1, -1, -1);
    s.tile = -1;
    s.k = -1;
    s.pre = false;
    return s;
  };
  // the same tile and pass (post / pre) as `a`
  auto same_pass = [&](const Walk4xStep& a, const Walk4xStep& b) {
    return a.k >= 0 && b.k >= 0 && a.tile == b.tile && a.pre == b.pre;
  };
  // internal child of a pre-order step that is NOT visited next (deferred)
  auto other_child = [&](const int4 d) -> int {
    const int o = d.y == d.w ? d.z : d.y;
    return o > N ? o : -1;
  };
  // does step s take its pre-partial from a hand-off (previous step's or the
  // one before's)?  prev1 / prev2: the two steps before s
  auto q_handed = [&](const Walk4xStep& s, const Walk4xStep& prev1, const Walk4xStep& prev2) {
    if (s.d.x == root) return true;  // pi, written by the root's post step
    if (same_pass(prev1, s) && prev1.d.w == s.d.x) return true;
    if (same_pass(prev2, s) && other_child(prev2.d) == s.d.x) return true;
    return false;
  };
  // post: is child c of step s in registers (previous step's node) or handed
  // into the stage by the step before that?
  auto e_handed = [&](int c, const Walk4xStep& s, const Walk4xStep& prev1, const Walk4xStep& prev2) {
    return (same_pass(prev1, s) && prev1.d.x == c) || (same_pass(prev2, s) && prev2.d.x == c);
  };

  const unsigned long long pol_first = policy_evict_first();
  // issue step s's bulk copies into stage st (lane 0 of warp (operand % LW));
  // prev1 / prev2: the two steps before s
  auto issue = [&](const Walk4xStep& s, const Walk4xStep& prev1, const Walk4xStep& prev2, int st) {
    if (lane != 0) return;
    uint64_t* mb = mbar + st;
    unsigned tx = 0;
    if (s.k >= 0) {
      int k = 0;
      auto mine = [&]() { return (k++ % LW) == l; };
      auto copy = [&](void* dst, const void* src, unsigned bytes) {
        bulk_g2s(dst, src, bytes, mb);
        tx += bytes;
      };
      auto copy_once = [&](void* dst, const void* src, unsigned bytes) {
        bulk_g2s_hint(dst, src, bytes, mb, pol_first);
        tx += bytes;
      };
      const int4 d = s.d;
      const uint8_t* codes = p.codes + size_t(s.tile) * 32;
      const size_t Pc = size_t(p.Pc);
      uint8_t* cb = cbytes(st);
      if (!s.pre) {
        if (d.y <= N) {
          if (mine()) copy(cb, codes + size_t(d.y - 1) * Pc, 32);
          if (mine()) copy(tcb(st, 1), p.tc + size_t(d.y - 1) * TCB, TCB * 8);
        } else if (!e_handed(d.y, s, prev1, prev2)) {
          if (mine()) copy(op(st, 0), E + size_t(d.y - N - 1) * SLOT, SLOT * 8);
        }
        if (d.z <= N) {
          if (mine()) copy(cb + 32, codes + size_t(d.z - 1) * Pc, 32);
          if (mine()) copy(tcb(st, 2), p.tc + size_t(d.z - 1) * TCB, TCB * 8);
        } else if (!e_handed(d.z, s, prev1, prev2)) {
          if (mine()) copy(op(st, 0), E + size_t(d.z - N - 1) * SLOT, SLOT * 8);
        }
        if (d.x != root)
          if (mine()) copy(tcb(st, 0), p.tc + size_t(d.x - 1) * TCB, TCB * 8);
      } else {
        if (!q_handed(s, prev1, prev2))
          if (mine()) copy_once(op(st, 2), Qs + size_t(d.x - N - 1) * SLOT, SLOT * 8);
        if (d.y <= N) {
          if (mine()) copy(cb, codes + size_t(d.y - 1) * Pc, 32);
          if (p.qtc)
            if (mine()) copy(op(st, 0), p.qtc + size_t(d.y - 1) * TCB, TCB * 8);
        } else {
          if (mine()) copy_once(op(st, 0), E + size_t(d.y - N - 1) * SLOT, SLOT * 8);
        }
        if (d.z <= N) {
          if (mine()) copy(cb + 32, codes + size_t(d.z - 1) * Pc, 32);
          if (p.qtc)
            if (mine()) copy(op(st, 1), p.qtc + size_t(d.z - 1) * TCB, TCB * 8);
        } else {
          if (mine()) copy_once(op(st, 1), E + size_t(d.z - N - 1) * SLOT, SLOT * 8);
        }
        if (mine()) copy(tcb(st, 0), p.tc + size_t(d.y - 1) * TCB, TCB * 8);
        if (mine()) copy(tcb(st, 1), p.tc + size_t(d.z - 1) * TCB, TCB * 8);
      }
    }
    mbar_arrive_tx(mb, tx);
  };
  // L2 prefetch of step s's scratch operands from DRAM (those not handed on)
  auto prefetch = [&](const Walk4xStep& s, const Walk4xStep& prev1, const Walk4xStep& prev2) {
    if (tid != 32 * (LW - 1) || s.k < 0) return;
    const int4 d = s.d;
    if (!s.pre) {
      if (d.y > N && !e_handed(d.y, s, prev1, prev2)) bulk_prefetch_l2(E + size_t(d.y - N - 1) * SLOT, SLOT * 8);
      if (d.z > N && !e_handed(d.z, s, prev1, prev2)) bulk_prefetch_l2(E + size_t(d.z - N - 1) * SLOT, SLOT * 8);
    } else {
      if (d.y > N) bulk_prefetch_l2(E + size_t(d.y - N - 1) * SLOT, SLOT * 8);
      if (d.z > N) bulk_prefetch_l2(E + size_t(d.z - N - 1) * SLOT, SLOT * 8);
    }
  };

  Walk4xStep Dm2 = none(), Dm1 = none();
  Walk4xStep D0 = load(blockIdx.x, 0);
  Walk4xStep D1 = next_of(D0);
  Walk4xStep D2 = next_of(D1);
  int st = 0;          // stage of D0; D1 -> (st + 1) % 3, D2 -> (st + 2) % 3
  unsigned phase = 0;  // parity bit per stage
  issue(D0, Dm1, Dm2, st);
  prefetch(D1, D0, Dm1);
  // step-to-step state (per warp: its category)
  double keep[4] = {0.0, 0.0, 0.0, 0.0};  // post: previous step's edge message
  int last = -1;                          // post: node whose e is in `keep`
  int S = 0;                              // post: accumulated exponent of the tile's patterns

  for (long long j = 0; D0.k >= 0; ++j) {
    const int st1 = st == NST - 1 ? 0 : st + 1, st2 = st1 == NST - 1 ? 0 : st1 + 1;
    // step j+1's copies and step j+2's L2 prefetch go out before this step
    // waits for its own operands
    issue(D1, D0, Dm1, st1);
    prefetch(D2, D1, D0);
    const int4 d = D0.d;
    const bool pre = D0.pre;
    const int s = D0.tile * 32 + lane;
    const bool valid = s < p.P;
    const bool owner = valid;
    const double w = valid ? p.weights[s] : 0.0;
    if (!pre && D0.k == 0) {
      S = 0;
      last = -1;
    }
    mbar_wait(mbar + st, (phase >> st) & 1u);
    phase ^= 1u << st;
    const int px = int(j & 1);
    int* xint = xi + px * Gx::XI;
    double* xdbl = xd + px * Gx::XD;

    if (!pre) {
      // ------------------------------------------ post-order step (a)
      const int code0 = d.y <= N ? cbytes(st)[lane] : 0;
      const int code1 = d.z <= N ? cbytes(st)[32 + lane] : 0;
      double a[4], b[4], x[4];
      if (d.y <= N) col4(tcb(st, 1), code0, a);
      else if (d.y == last) {
#pragma unroll
        for (int r = 0; r < 4; ++r) a[r] = keep[r];
      } else rd4(op(st, 0), a);
      if (d.z <= N) col4(tcb(st, 2), code1, b);
      else if (d.z == last) {
#pragma unroll
        for (int r = 0; r < 4; ++r) b[r] = keep[r];
      } else rd4(op(st, 0), b);
      int hm = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        x[r] = a[r] * b[r];
        hm = max(hm, __double2hiint(x[r]));
      }
      xint[lane * LW + l] = hm;
      fence_proxy_async_global();  // earlier scratch stores before later bulk reads (after the barrier)
      __syncthreads();
      if (!p.disable) {
        int hmax = xint[lane * LW];
#pragma unroll
        for (int c = 1; c < LW; ++c) hmax = max(hmax, xint[lane * LW + c]);
        const int ex = peak_exponent(hmax);
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
      if (d.x == root) {
        // root: mix = sum_l w_l pi . p_l (the fma order of walk4), logL
        double dd = 0.0;
#pragma unroll
        for (int r = 0; r < 4; ++r) dd = fma(P4.pi[r], x[r], dd);
        xdbl[lane * LW + l] = dd;
        __syncthreads();
        if (l == 0) {
          double mix = 0.0;
#pragma unroll
          for (int c = 0; c < LW; ++c) mix = fma(p.probs[c], xdbl[lane * LW + c], mix);
          const double ll = log(mix) + double(S) * 0.6931471805599453;
          if (owner) {
            if (!isfinite(mix)) atomicMin(&p.err[0], s);
            else if (mix <= 0.0) atomicMin(&p.err[1], s);
            if (p.site_ll) p.site_ll[s] = ll;
          }
          const double v = warp_sum(owner ? w * ll : 0.0);
          if (lane == 0) atomicAdd(A, v);
        }
        // the first pre-order step's q is pi: handed on through its q slot
        if (p.do_pre) {
          const double pv[4] = {P4.pi[0], P4.pi[1], P4.pi[2], P4.pi[3]};
          wr4_smem(op(st1, 2), pv, 1.0);
        }
      } else {
        // e_k = P_k p_k (engine.hpp:367-372), column c of P at TC column c
        const double2* Tl = reinterpret_cast<const double2*>(tcb(st, 0) + l * NC * 4);
        double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double2 u = Tl[2 * c], v = Tl[2 * c + 1];
          e0 = fma(u.x, x[c], e0);
          e1 = fma(u.y, x[c], e1);
          e2 = fma(v.x, x[c], e2);
          e3 = fma(v.y, x[c], e3);
        }
        keep[0] = e0;
        keep[1] = e1;
        keep[2] = e2;
        keep[3] = e3;
        double2* dst = reinterpret_cast<double2*>(E + size_t(d.x - N - 1) * SLOT + l * 128) + lane;
        __stcs(dst, make_double2(e0, e1));
        __stcs(dst + 32, make_double2(e2, e3));
        // consumed two steps on: straight into that step's stage
        if (same_pass(D2, D0) && (D2.d.y == d.x || D2.d.z == d.x)) wr4_smem(op(st2, 0), keep, 1.0);
        last = d.x;
      }
    } else {
      // ------------------------------- pre-order step + gradient (b)+(c)
      const bool a_int = d.y > N, b_int = d.z > N;
      const int code0 = a_int ? 0 : cbytes(st)[lane];
      const int code1 = b_int ? 0 : cbytes(st)[32 + lane];
      const double* Ta = tcb(st, 0);
      const double* Tb = tcb(st, 1);
      double q[4], ea[4], eb[4];
      rd4(op(st, 2), q);
      if (a_int) rd4(op(st, 0), ea);
      else col4(Ta, code0, ea);
      if (b_int) rd4(op(st, 1), eb);
      else col4(Tb, code1, eb);
      double ta[4], tb[4], dd = 0.0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        ta[r] = q[r] * eb[r];  // top for child a
        tb[r] = q[r] * ea[r];  // top for child b
        dd = fma(ta[r], ea[r], dd);
      }
      // Q e: mat-vec for an internal child; for a tip the staged Q P column
      // (P and Q commute, engine.hpp:260)
      double qea[4], qeb[4];
      if (a_int || !p.qtc) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double u = 0.0;
#pragma unroll
          for (int c = 0; c < 4; ++c) u = fma(qm(d.y, r, c), ea[c], u);
          qea[r] = u;
        }
      } else {
        col4(op(st, 0), code0, qea);
      }
      if (b_int || !p.qtc) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double v = 0.0;
#pragma unroll
          for (int c = 0; c < 4; ++c) v = fma(qm(d.z, r, c), eb[c], v);
          qeb[r] = v;
        }
      } else {
        col4(op(st, 1), code1, qeb);
      }
      double d1a = 0.0, d1b = 0.0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        d1a = fma(ta[r], qea[r], d1a);
        d1b = fma(tb[r], qeb[r], d1b);
      }
      double d2a = 0.0, d2b = 0.0;
      if constexpr (HESS) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double u = 0.0, v = 0.0;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            u = fma(qm(d.y, r, c), qea[c], u);
            v = fma(qm(d.z, r, c), qeb[c], v);
          }
          d2a = fma(ta[r], u, d2a);
          d2b = fma(tb[r], v, d2b);
        }
      }
      // outgoing pre-partials q_x = P_x^T top (engine.hpp:249-250), unnormalised
      double qa[4], qb[4];
      int ha = 0, hb = 0;
      if (a_int) {
        const double2* Tl = reinterpret_cast<const double2*>(Ta + l * NC * 4);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double2 u = Tl[2 * c], v = Tl[2 * c + 1];
          qa[c] = fma(u.x, ta[0], fma(u.y, ta[1], fma(v.x, ta[2], v.y * ta[3])));
          ha = max(ha, __double2hiint(qa[c]));
        }
      }
      if (b_int) {
        const double2* Tl = reinterpret_cast<const double2*>(Tb + l * NC * 4);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double2 u = Tl[2 * c], v = Tl[2 * c + 1];
          qb[c] = fma(u.x, tb[0], fma(u.y, tb[1], fma(v.x, tb[2], v.y * tb[3])));
          hb = max(hb, __double2hiint(qb[c]));
        }
      }
      // exchange: [0] dd, [1] d1a, [2] d1b (, [3] d2a, [4] d2b); peaks ha, hb
      xdbl[(0 * 32 + lane) * LW + l] = dd;
      xdbl[(1 * 32 + lane) * LW + l] = d1a;
      xdbl[(2 * 32 + lane) * LW + l] = d1b;
      if constexpr (HESS) {
        xdbl[(3 * 32 + lane) * LW + l] = d2a;
        xdbl[(4 * 32 + lane) * LW + l] = d2b;
      }
      xint[(0 * 32 + lane) * LW + l] = ha;
      xint[(1 * 32 + lane) * LW + l] = hb;
      fence_proxy_async_global();
      __syncthreads();
      // consumed scratch is dead: drop it from L2 without write-back
      if (lane < 8) {
        const char* eb_ = reinterpret_cast<const char*>(E) + size_t(l) * 1024 + lane * 128;
        const char* qb_ = reinterpret_cast<const char*>(Qs) + size_t(l) * 1024 + lane * 128;
        if (a_int) discard_l2(eb_ + size_t(d.y - N - 1) * SLOT * 8);
        if (b_int) discard_l2(eb_ + size_t(d.z - N - 1) * SLOT * 8);
        if (!q_handed(D0, Dm1, Dm2)) discard_l2(qb_ + size_t(d.x - N - 1) * SLOT * 8);
      }
      // gradient: warp 0 for child a, warp 1 (or 0) for child b, with walk4's
      // fma order over categories
      constexpr int wa = 0, wb = LW > 1 ? 1 : 0;
      if (l == wa || l == wb) {
        double den = 0.0, na = 0.0, nb = 0.0, na2 = 0.0, nb2 = 0.0;
#pragma unroll
        for (int c = 0; c < LW; ++c) {
          const double cwc = p.probs[c], crwc = p.rates[c] * cwc;
          den = fma(cwc, xdbl[(0 * 32 + lane) * LW + c], den);
          na = fma(crwc, xdbl[(1 * 32 + lane) * LW + c], na);
          nb = fma(crwc, xdbl[(2 * 32 + lane) * LW + c], nb);
          if constexpr (HESS) {
            const double cr2wc = p.rates[c] * crwc;
            na2 = fma(cr2wc, xdbl[(3 * 32 + lane) * LW + c], na2);
            nb2 = fma(cr2wc, xdbl[(4 * 32 + lane) * LW + c], nb2);
          }
        }
        const double inv = 1.0 / den;
        if (l == wa) {
          const double r1a = na * inv;
          const double ga = warp_sum(owner ? w * r1a : 0.0);
          if (lane == 0) atomicAdd(A + d.y, ga);
          if constexpr (HESS) {
            const double ha2 = warp_sum(owner ? w * (na2 * inv - r1a * r1a) : 0.0);
            if (lane == 0) atomicAdd(A + p.B + d.y, ha2);
          }
        }
        if (l == wb) {
          const double r1b = nb * inv;
          const double gb = warp_sum(owner ? w * r1b : 0.0);
          if (lane == 0) atomicAdd(A + d.z, gb);
          if constexpr (HESS) {
            const double hb2 = warp_sum(owner ? w * (nb2 * inv - r1b * r1b) : 0.0);
            if (lane == 0) atomicAdd(A + p.B + d.z, hb2);
          }
        }
      }
      // normalise (shared peak over the categories) and hand on: the child
      // visited next through the next stage's q slot, a child visited two
      // steps on through that stage's, any other to scratch
      auto emit = [&](int x, const double (&qx)[4], int field) {
        int hx = xint[(field * 32 + lane) * LW];
#pragma unroll
        for (int c = 1; c < LW; ++c) hx = max(hx, xint[(field * 32 + lane) * LW + c]);
        const int ex = peak_exponent(hx);
        const double scl = (ex != 0 && ex <= 1022) ? pow2_neg(ex) : 1.0;
        if (x == d.w) {
          wr4_smem(op(st1, 2), qx, scl);
        } else if (same_pass(D2, D0) && D2.d.x == x) {
          wr4_smem(op(st2, 2), qx, scl);
        } else {
          double2* dst = reinterpret_cast<double2*>(Qs + size_t(x - N - 1) * SLOT + l * 128) + lane;
          __stcg(dst, make_double2(qx[0] * scl, qx[1] * scl));
          __stcg(dst + 32, make_double2(qx[2] * scl, qx[3] * scl));
        }
      };
      if (a_int) emit(d.y, qa, 0);
      if (b_int) emit(d.z, qb, 1);
    }
    __syncwarp();
    Dm2 = Dm1;
    Dm1 = D0;
    D0 = D1;
    D1 = D2;
    D2 = next_of(D1);
    st = st1;
  }
}

}  // namespace pgk
