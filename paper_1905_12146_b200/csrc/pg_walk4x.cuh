// K2d: the 4-state walk with the rate categories spread over the warps of a
// CTA (C2/C3: 4-state + Gamma4), warp-specialised.
//
// A CTA owns a tile of 32 patterns.  LW consumer warps hold one rate
// category each (one lane per pattern, 4 doubles per vector) and walk the
// tree in lock-step, one node per step; a producer warp stages every step's
// operands ahead of them.  Against walk4 (one lane per pattern holding all
// categories, 255 registers, 8 warps per SM) a consumer thread carries a
// quarter of the state, so twice as many warps are resident and the
// fp64 / shared-memory latencies of one warp are covered by the others
// (walk4's C3 profile: 2 warps per scheduler, 36 % of the samples in
// fixed-latency waits, 17 % in shared-memory load-use waits).
//
// Staging (producer warp).  The host precomputes, per post- and pre-order
// step, a header (descriptor + hand-off flags) and the list of that step's
// operand copies (Walk4xCopy: table, source offset, stage offset, bytes).
// The producer walks the same step stream, waits until a stage is free
// (`empty` mbarrier, one arrival per consumer warp), posts the byte count on
// the stage's `full` mbarrier and issues the copies as 1-D bulk copies
// (cp.async.bulk, TMA engine), one per lane: an internal child's edge-message
// slot or a deferred pre-partial ([node][cat][lane][4] doubles, LW KB), a
// node's column table TC ([cat][NC][4] doubles), a tip's 32 code bytes, a
// tip's Q P table, and the header itself.  Four stages give three steps of
// lookahead; the scratch operands two steps on are also prefetched into L2.
//
// Hand-offs (consumer warps).  A value produced by step i and consumed by
// step i+1..i+3 of the same pass (the producer may run that far ahead)
// never goes through global memory for that use: the producing warp writes
// its category slice straight into the consumer's stage (post: the edge
// message of step i+1 stays in registers; pre: the child's pre-partial; the
// root's pi for the first pre-order step).  Anything consumed later was
// stored at least four steps before its copy is issued; its writer fenced it
// (fence.proxy.async) before arriving on the stage's `empty` barrier that the
// producer waited on.
//
// Cross-category quantities go through a small shared exchange (double-
// buffered by step parity) with one consumer barrier per step: the
// per-pattern peak exponent (post: normalisation of p_k; pre: of the
// outgoing q_c), the root mixture and the gradient ratio terms (den, num_a,
// num_b).  Every per-pattern arithmetic chain is the one walk4 evaluates
// (same operand order, same fma nesting over categories).
#pragma once

#include "pg_walk4.cuh"
#include "pg_walk4x_tables.hpp"

namespace pgk {

__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(mb)) : "memory");
}
__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}

// Step headers and copy lists: pg_walk4x_tables.hpp (built on the host).
// Header flags: hand-off distances and the pre-order q source (see there).
// Copy kinds: 0 edge-message scratch (CTA base), 1 pre-partial scratch (CTA
// base), 2 TC, 3 QTC, 4 tip codes (tile base), 5 step headers.

template <int LW, int NC, bool HESS>
struct Walk4xGeom {
  static constexpr int NST = kW4xHand + 1;   // stages: kW4xHand steps of lookahead
  static constexpr int SLOT = LW * 32 * 4;   // doubles: one node slot of the CTA tile
  static constexpr int TCB = LW * NC * 4;    // doubles: one node's column table (all categories)
  // stage (doubles): header, 3 operand slots, 3 TC blocks, 2 x 32 code bytes
  static constexpr int HDR = 0, OP0 = 4, TC0 = 4 + 3 * SLOT, CODES = TC0 + 3 * TCB;
  static constexpr int STAGE = CODES + 8;
  static constexpr int NR = HESS ? 5 : 3;    // gradient exchange terms per (category, pattern)
  // exchange (per parity): int peak exponents [2][32][LW], double terms [NR][32][LW]
  static constexpr int XI = 2 * 32 * LW;
  static constexpr int XD = NR * 32 * LW;
  static constexpr int THREADS = 32 * (LW + 1);  // LW consumer warps + 1 producer warp
  static constexpr size_t smem_bytes() {
    return size_t(NST * STAGE) * 8 + size_t(2 * XD) * 8 + size_t(2 * XI) * 4 + 2 * NST * 8;
  }
};

template <bool HOMOG, bool HESS, int NC, int LW>
__global__ void __launch_bounds__(32 * (LW + 1), (LW >= 4 ? 3 : 8))
    walk4x_kernel(const __grid_constant__ Walk4xParams PX) {
  using Gx = Walk4xGeom<LW, NC, HESS>;
  constexpr int NST = Gx::NST, SLOT = Gx::SLOT, TCB = Gx::TCB, STAGE = Gx::STAGE;
  constexpr int CT = 32 * LW;  // consumer threads
  const Walk4Params& P4 = PX.p4;
  const WalkParams& p = P4.p;
  extern __shared__ __align__(16) double sm4x[];
  double* stg = sm4x;                                        // [NST][STAGE]
  double* xd = sm4x + NST * STAGE;                           // [2][NR][32][LW]
  int* xi = reinterpret_cast<int*>(xd + 2 * Gx::XD);         // [2][2][32][LW]
  uint64_t* full = reinterpret_cast<uint64_t*>(xi + 2 * Gx::XI);
  uint64_t* empty = full + NST;
  const int tid = threadIdx.x, lane = tid & 31, l = tid >> 5;  // warp l < LW: category l; l == LW: producer
  const int N = p.N, root = 2 * N - 1, n = p.nsteps;
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(full + i, 1);    // the producer's expect_tx arrival (+ the copies' bytes)
      mbar_init(empty + i, LW);  // lane 0 of every consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (int(blockIdx.x) >= p.ntiles) return;
  const int per_tile = p.do_pre ? 2 * n : n;
  const int my_tiles = (p.ntiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1;
  // CTA-major scratch: slot of node k at (k - N - 1) * SLOT, category l at + l * 128
  double* E = p.escr + size_t(blockIdx.x) * size_t(N - 1) * SLOT;
  double* Qs = p.qscr + size_t(blockIdx.x) * size_t(N - 1) * SLOT;

  if (l == LW) {
    // ======================================================== producer
    // Lane c < ncopy issues copy c of a step; the copy entry (lanes 0..7) and
    // the step's {ncopy, tx} (lane 8) are loaded three steps ahead into
    // registers, so no global load sits between a free stage and its copies.
    auto entry = [&](int k, Walk4xCopy& c, int2& h) {
      if (lane < kW4xMaxCopies) c = PX.cpy[size_t(k) * kW4xMaxCopies + lane];
      else if (lane == 8) h = make_int2(__ldg(&PX.hdr[k].ncopy), __ldg(&PX.hdr[k].tx));
    };
    Walk4xCopy c0{}, c1{}, c2{}, c3{};
    int2 h0 = make_int2(0, 0), h1 = h0, h2 = h0, h3 = h0;
    // iterator three steps ahead: (tile index ti3, step k3)
    int ti3 = 0, k3 = 0;
    auto advance3 = [&]() {
      if (++k3 == per_tile) {
        k3 = 0;
        ++ti3;
      }
    };
    entry(0, c0, h0);
    advance3();
    if (ti3 < my_tiles) entry(k3, c1, h1);
    advance3();
    if (ti3 < my_tiles) entry(k3, c2, h2);
    advance3();
    int st = 0;
    unsigned ephase = 0;
    long long j = 0;
    for (int ti = 0; ti < my_tiles; ++ti) {
      const int tile = int(blockIdx.x) + ti * int(gridDim.x);
      for (int k = 0; k < per_tile; ++k, ++j) {
        c3 = Walk4xCopy{};
        if (ti3 < my_tiles) entry(k3, c3, h3);  // three steps on (consumed next iterations)
        // L2 prefetch of the scratch operands two steps on (entry loaded last iteration)
        if (lane < kW4xMaxCopies) {
          const int kind = c2.kb >> 24;
          if (kind <= 1 && (c2.kb & 0xffffff) != 0)
            bulk_prefetch_l2((kind == 0 ? E : Qs) + c2.src, unsigned(c2.kb & 0xffffff));
        }
        if (j >= NST) {
          mbar_wait(empty + st, (ephase >> st) & 1u);
          ephase ^= 1u << st;
        }
        const int ncopy = __shfl_sync(kFull, h0.x, 8), tx = __shfl_sync(kFull, h0.y, 8);
        if (lane == 0) mbar_arrive_tx(full + st, unsigned(tx));
        __syncwarp();
        double* sb = stg + st * STAGE;
        if (lane < ncopy) {
          const int kind = c0.kb >> 24, bytes = c0.kb & 0xffffff;
          const void* src;
          switch (kind) {
            case 0: src = E + c0.src; break;
            case 1: src = Qs + c0.src; break;
            case 2: src = p.tc + c0.src; break;
            case 3: src = p.qtc + c0.src; break;
            case 4: src = p.codes + c0.src + size_t(tile) * 32; break;
            default: src = reinterpret_cast<const char*>(PX.hdr) + c0.src; break;
          }
          bulk_g2s(reinterpret_cast<char*>(sb) + c0.dst, src, unsigned(bytes), full + st);
        }
        c0 = c1;
        c1 = c2;
        c2 = c3;
        h0 = h1;
        h1 = h2;
        h2 = h3;
        if (ti3 < my_tiles) advance3();
        st = st == NST - 1 ? 0 : st + 1;
      }
    }
    return;
  }

  // ========================================================== consumers
  double* A = p.acc + size_t(blockIdx.x) * p.accw;  // this CTA's accumulator row
  for (int i = tid; i < p.accw; i += CT) A[i] = 0.0;
  consumer_sync(CT);

  auto op = [&](int st, int k) -> double* { return stg + st * STAGE + Gx::OP0 + k * SLOT; };
  auto tcb = [&](int st, int k) -> const double* { return stg + st * STAGE + Gx::TC0 + k * TCB; };
  auto cbytes = [&](int st) -> const uint8_t* {
    return reinterpret_cast<const uint8_t*>(stg + st * STAGE + Gx::CODES);
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

  int st = 0;
  unsigned fphase = 0;
  double keep[4] = {0.0, 0.0, 0.0, 0.0};  // post: previous step's edge message
  int last = -1;                          // post: node whose e is in `keep`
  long long j = 0;
  for (int ti = 0; ti < my_tiles; ++ti) {
    const int tile = int(blockIdx.x) + ti * int(gridDim.x);
    const int s = tile * 32 + lane;
    const bool owner = s < p.P;
    const double w = owner ? p.weights[s] : 0.0;
    int S = 0;  // post: accumulated exponent of the tile's patterns
    last = -1;
    for (int k = 0; k < per_tile; ++k, ++j) {
      const int st1 = st == NST - 1 ? 0 : st + 1;
      // stage of the step `dist` on (hand-offs)
      auto stage_on = [&](int dist) { return st + dist >= NST ? st + dist - NST : st + dist; };
      mbar_wait(full + st, (fphase >> st) & 1u);
      fphase ^= 1u << st;
      const Walk4xHdr& H = *reinterpret_cast<const Walk4xHdr*>(stg + st * STAGE + Gx::HDR);
      const int4 d = H.d;
      const int flags = H.flags;
      const int px = int(j & 1);
      int* xint = xi + px * Gx::XI;
      double* xdbl = xd + px * Gx::XD;

      if (k < n) {
        // ---------------------------------------- post-order step (a)
        double a[4], b[4], x[4];
        if (d.y <= N) col4(tcb(st, 1), cbytes(st)[lane], a);
        else if (d.y == last) {
#pragma unroll
          for (int r = 0; r < 4; ++r) a[r] = keep[r];
        } else rd4(op(st, 0), a);
        if (d.z <= N) col4(tcb(st, 2), cbytes(st)[32 + lane], b);
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
        consumer_sync(CT);
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
          consumer_sync(CT);
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
          if ((flags & 3) >= 2) wr4_smem(op(stage_on(flags & 3), 0), keep, 1.0);
          last = d.x;
        }
      } else {
        // ----------------------------- pre-order step + gradient (b)+(c)
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
        consumer_sync(CT);
        // consumed scratch is dead: drop it from L2 without write-back
        if (lane < 8) {
          const char* eb_ = reinterpret_cast<const char*>(E) + size_t(l) * 1024 + lane * 128;
          const char* qb_ = reinterpret_cast<const char*>(Qs) + size_t(l) * 1024 + lane * 128;
          if (a_int) discard_l2(eb_ + size_t(d.y - N - 1) * SLOT * 8);
          if (b_int) discard_l2(eb_ + size_t(d.z - N - 1) * SLOT * 8);
          if (flags & kW4xPreQGlobal) discard_l2(qb_ + size_t(d.x - N - 1) * SLOT * 8);
        }
        // gradient: warp 0 for child a, warp 1 (or 0) for child b, with
        // walk4's fma order over categories
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
        auto emit = [&](int x, const double (&qx)[4], int field, int dist) {
          int hx = xint[(field * 32 + lane) * LW];
#pragma unroll
          for (int c = 1; c < LW; ++c) hx = max(hx, xint[(field * 32 + lane) * LW + c]);
          const int ex = peak_exponent(hx);
          const double scl = (ex != 0 && ex <= 1022) ? pow2_neg(ex) : 1.0;
          if (x == d.w) {
            wr4_smem(op(st1, 2), qx, scl);
          } else if (dist >= 2) {
            wr4_smem(op(stage_on(dist), 2), qx, scl);
          } else {
            double2* dst = reinterpret_cast<double2*>(Qs + size_t(x - N - 1) * SLOT + l * 128) + lane;
            __stcg(dst, make_double2(qx[0] * scl, qx[1] * scl));
            __stcg(dst + 32, make_double2(qx[2] * scl, qx[3] * scl));
          }
        };
        if (a_int) emit(d.y, qa, 0, (flags >> 1) & 3);
        if (b_int) emit(d.z, qb, 1, (flags >> 3) & 3);
      }
      // this step's stage is consumed: its scratch stores are fenced for the
      // async proxy (bulk copies issued after the producer sees `empty`)
      fence_proxy_async_global();
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
      st = st1;
    }
  }
}

}  // namespace pgk
