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
// Per step every operand of the CTA tile is ONE 1-D bulk copy (cp.async.bulk,
// TMA engine) into the next stage while this step computes: an internal
// child's edge-message slot or a deferred pre-partial ([node][cat][lane][4]
// doubles, LW KB), a node's column table TC ([cat][NC][4] doubles), a tip's
// 32 code bytes, a tip's Q P table (pre-order pass).  The copies of a stage
// are issued by lane 0 of the warps (spread over the warps) after the step's
// CTA barrier and complete on the stage's mbarrier.
//
// Cross-category quantities go through a small shared exchange (double-
// buffered by step parity) with one CTA barrier per step: the per-pattern
// peak exponent (post: normalisation of p_k; pre: of the outgoing q_c), the
// root mixture and the gradient ratio terms (den, num_a, num_b).  Every
// arithmetic chain is the one walk4 evaluates (same operand order, same fma
// nesting over categories), so the two kernels give bit-identical results.
#pragma once

#include "pg_walk4.cuh"

namespace pgk {

template <int LW, int NC, bool HESS>
struct Walk4xGeom {
  static constexpr int SLOT = LW * 32 * 4;   // doubles: one node slot of the CTA tile
  static constexpr int TCB = LW * NC * 4;    // doubles: one node's column table (all categories)
  static constexpr int STAGE = 3 * SLOT + 3 * TCB + 8;  // 3 operand slots, 3 TC blocks, 2 x 32 code bytes
  static constexpr int NR = HESS ? 5 : 3;    // gradient exchange terms per (category, pattern)
  // exchange (per parity): int peak exponents [2][32][LW], double terms [NR][32][LW]
  static constexpr int XI = 2 * 32 * LW;
  static constexpr int XD = NR * 32 * LW;
  static constexpr size_t smem_bytes() {
    return size_t(2 * STAGE) * 8 + size_t(2 * XD) * 8 + size_t(2 * XI) * 4 + 2 * 8;
  }
};

template <bool HOMOG, bool HESS, int NC, int LW>
__global__ void __launch_bounds__(32 * LW, (LW >= 4 ? 4 : 8)) walk4x_kernel(const __grid_constant__ Walk4Params P4) {
  using Gx = Walk4xGeom<LW, NC, HESS>;
  constexpr int SLOT = Gx::SLOT, TCB = Gx::TCB, STAGE = Gx::STAGE, NR = Gx::NR;
  const WalkParams& p = P4.p;
  extern __shared__ __align__(16) double sm4x[];
  double* stg = sm4x;                                        // [2][STAGE]
  double* xd = sm4x + 2 * STAGE;                             // [2][NR][32][LW]
  int* xi = reinterpret_cast<int*>(xd + 2 * Gx::XD);         // [2][2][32][LW]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(xi + 2 * Gx::XI);
  const int tid = threadIdx.x, lane = tid & 31, l = tid >> 5;  // warp = category
  const int N = p.N, root = 2 * N - 1, n = p.nsteps;
  if (tid == 0) {
    mbar_init(mbar, LW);  // lane 0 of every warp arrives once per stage
    mbar_init(mbar + 1, LW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const double cw = p.probs[l], crw = p.rates[l] * cw, cr2w = p.rates[l] * crw;
  double* A = p.acc + size_t(blockIdx.x) * p.accw;  // this CTA's accumulator row
  for (int i = tid; i < p.accw; i += 32 * LW) A[i] = 0.0;
  // CTA-major scratch: slot of node k at (k - N - 1) * SLOT, category l at + l * 128
  double* E = p.escr + size_t(blockIdx.x) * size_t(N - 1) * SLOT;
  double* Qs = p.qscr + size_t(blockIdx.x) * size_t(N - 1) * SLOT;

  auto op = [&](int st, int k) -> double* { return stg + st * STAGE + k * SLOT; };
  auto tcb = [&](int st, int k) -> const double* { return stg + st * STAGE + 3 * SLOT + k * TCB; };
  auto code_of = [&](int st, int k) -> int {
    return reinterpret_cast<const uint8_t*>(stg + st * STAGE + 3 * SLOT + 3 * TCB + 4 * k)[lane];
  };
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
  // The CTA's work is one stream of steps: per tile, the post-order steps,
  // then (gradient) the pre-order steps.  Step j's operands are staged into
  // stage j & 1 during step j - 1.
  const int per_tile = p.do_pre ? 2 * n : n;
  const int ntiles = p.ntiles;
  const int first_tile = blockIdx.x;
  if (first_tile >= ntiles) return;
  const long long total = (long long)((ntiles - 1 - first_tile) / gridDim.x + 1) * per_tile;
  auto tile_of = [&](long long j) { return first_tile + int(j / per_tile) * int(gridDim.x); };
  auto desc_of = [&](long long j, bool& pre) -> int4 {
    const int k = int(j % per_tile);
    pre = k >= n;
    return pre ? __ldg(p.pre + (k - n)) : __ldg(p.post + k);
  };
  const unsigned long long pol_first = policy_evict_first();
  // issue step j's bulk copies into stage j & 1 (lane 0 of warp (operand % LW)).
  // aux: post step -> the node whose edge message stays in registers (the
  // previous step's node, not staged); pre step -> 1 if its q is handed on
  // through the q slot (not staged)
  auto issue = [&](long long j, int4 d, bool pre, int aux) {
    const int st = int(j & 1);
    const int t = tile_of(j);
    const uint8_t* codes = p.codes + size_t(t) * 32;
    const size_t Pc = size_t(p.Pc);
    uint64_t* mb = mbar + st;
    unsigned tx = 0;
    int k = 0;
    auto mine = [&]() { return lane == 0 && (k++ % LW) == l; };
    auto copy = [&](void* dst, const void* src, unsigned bytes) {
      bulk_g2s(dst, src, bytes, mb);
      tx += bytes;
    };
    auto copy_once = [&](void* dst, const void* src, unsigned bytes) {
      bulk_g2s_hint(dst, src, bytes, mb, pol_first);
      tx += bytes;
    };
    double* base = stg + st * STAGE;
    uint8_t* cbase = reinterpret_cast<uint8_t*>(base + 3 * SLOT + 3 * TCB);
    if (!pre) {
      if (d.y <= N) {
        if (mine()) copy(cbase, codes + size_t(d.y - 1) * Pc, 32);
        if (mine()) copy(base + 3 * SLOT + TCB, p.tc + size_t(d.y - 1) * TCB, TCB * 8);
      } else if (d.y != aux) {
        if (mine()) copy(op(st, 0), E + size_t(d.y - N - 1) * SLOT, SLOT * 8);
      }
      if (d.z <= N) {
        if (mine()) copy(cbase + 32, codes + size_t(d.z - 1) * Pc, 32);
        if (mine()) copy(base + 3 * SLOT + 2 * TCB, p.tc + size_t(d.z - 1) * TCB, TCB * 8);
      } else if (d.z != aux) {
        if (mine()) copy(op(st, 0), E + size_t(d.z - N - 1) * SLOT, SLOT * 8);
      }
      if (d.x != root)
        if (mine()) copy(base + 3 * SLOT, p.tc + size_t(d.x - 1) * TCB, TCB * 8);
    } else {
      if (d.x != root && !aux)
        if (mine()) copy_once(op(st, 2), Qs + size_t(d.x - N - 1) * SLOT, SLOT * 8);
      if (d.y <= N) {
        if (mine()) copy(cbase, codes + size_t(d.y - 1) * Pc, 32);
        if (p.qtc)
          if (mine()) copy(op(st, 0), p.qtc + size_t(d.y - 1) * TCB, TCB * 8);
      } else {
        if (mine()) copy_once(op(st, 0), E + size_t(d.y - N - 1) * SLOT, SLOT * 8);
      }
      if (d.z <= N) {
        if (mine()) copy(cbase + 32, codes + size_t(d.z - 1) * Pc, 32);
        if (p.qtc)
          if (mine()) copy(op(st, 1), p.qtc + size_t(d.z - 1) * TCB, TCB * 8);
      } else {
        if (mine()) copy_once(op(st, 1), E + size_t(d.z - N - 1) * SLOT, SLOT * 8);
      }
      if (mine()) copy(base + 3 * SLOT, p.tc + size_t(d.y - 1) * TCB, TCB * 8);
      if (mine()) copy(base + 3 * SLOT + TCB, p.tc + size_t(d.z - 1) * TCB, TCB * 8);
    }
    if (lane == 0) mbar_arrive_tx(mb, tx);
  };

  unsigned phase = 0;  // parity bit per stage
  bool cur_pre = false;
  int4 cur = desc_of(0, cur_pre);
  issue(0, cur, cur_pre, -1);
  // step-to-step state (per warp: its category)
  double keep[4] = {0.0, 0.0, 0.0, 0.0};  // post: previous step's edge message
  int last = -1;                          // post: node whose e is in `keep`
  int S = 0;                              // post: accumulated exponent of the tile's patterns
  int prev_next = 0;                      // pre: node whose q was handed on through the q slot

  for (long long j = 0; j < total; ++j) {
    const int st = int(j & 1);
    const int t = tile_of(j);
    const int s = t * 32 + lane;
    const bool valid = s < p.P;
    const bool owner = valid;
    const double w = valid ? p.weights[s] : 0.0;
    const int4 d = cur;
    const bool pre = cur_pre;
    bool nxt_pre = false;
    const bool has_next = j + 1 < total;
    int4 dn = make_int4(0, 0, 0, 0);
    if (has_next) dn = desc_of(j + 1, nxt_pre);
    if (!pre && int(j % per_tile) == 0) {
      S = 0;
      last = -1;
    }
    mbar_wait(mbar + st, (phase >> st) & 1u);
    phase ^= 1u << st;
    int* xint = xi + st * Gx::XI;
    double* xdbl = xd + st * Gx::XD;

    if (!pre) {
      // ------------------------------------------ post-order step (a)
      const int code0 = d.y <= N ? code_of(st, 0) : 0;
      const int code1 = d.z <= N ? code_of(st, 1) : 0;
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
      // next: the first pre-order step (its q = pi is written below), or the
      // next post-order step with this step's edge message kept in registers
      if (has_next) issue(j + 1, dn, nxt_pre, nxt_pre ? int(dn.x == root) : (d.x != root ? d.x : -1));
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
          double pv[4] = {P4.pi[0], P4.pi[1], P4.pi[2], P4.pi[3]};
          wr4_smem(op(st ^ 1, 2), pv, 1.0);
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
        last = d.x;
      }
    } else {
      // ------------------------------- pre-order step + gradient (b)+(c)
      const bool a_int = d.y > N, b_int = d.z > N;
      const int code0 = a_int ? 0 : code_of(st, 0);
      const int code1 = b_int ? 0 : code_of(st, 1);
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
      const bool q_next = has_next && nxt_pre && dn.x == d.w;  // next step's q handed on
      if (has_next) issue(j + 1, dn, nxt_pre, nxt_pre ? int(q_next) : -1);
      // consumed scratch is dead: drop it from L2 without write-back
      if (lane < 8) {
        const char* eb_ = reinterpret_cast<const char*>(E) + size_t(l) * 1024 + lane * 128;
        const char* qb_ = reinterpret_cast<const char*>(Qs) + size_t(l) * 1024 + lane * 128;
        if (a_int) discard_l2(eb_ + size_t(d.y - N - 1) * SLOT * 8);
        if (b_int) discard_l2(eb_ + size_t(d.z - N - 1) * SLOT * 8);
        if (d.x != root && prev_next != d.x) discard_l2(qb_ + size_t(d.x - N - 1) * SLOT * 8);
      }
      // gradient: warp 0 for child a, warp 1 (or 0) for child b, with walk4's
      // fma order over categories
      const int wa = 0, wb = LW > 1 ? 1 : 0;
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
      // visited next through the next stage's q slot, the other to scratch
      auto emit = [&](int x, const double (&qx)[4], int field) {
        int hx = xint[(field * 32 + lane) * LW];
#pragma unroll
        for (int c = 1; c < LW; ++c) hx = max(hx, xint[(field * 32 + lane) * LW + c]);
        const int ex = peak_exponent(hx);
        const double scl = (ex != 0 && ex <= 1022) ? pow2_neg(ex) : 1.0;
        if (x == d.w) {
          wr4_smem(op(st ^ 1, 2), qx, scl);
        } else {
          double2* dst = reinterpret_cast<double2*>(Qs + size_t(x - N - 1) * SLOT + l * 128) + lane;
          __stcg(dst, make_double2(qx[0] * scl, qx[1] * scl));
          __stcg(dst + 32, make_double2(qx[2] * scl, qx[3] * scl));
        }
      };
      if (a_int) emit(d.y, qa, 0);
      if (b_int) emit(d.z, qb, 1);
      prev_next = d.w;
      (void)crw;
      (void)cr2w;
      (void)cw;
    }
    __syncwarp();
    cur = dn;
    cur_pre = nxt_pre;
  }
}

}  // namespace pgk
