// K2a (tensor) — the 4-state, 4-category walk with its 4x4 mat-vecs on the
// fp64 tensor cores (mma.sync m8n8k4 f64 -> DMMA).
//
// Layout: a warp owns 32 patterns in 4 groups of 8; lane t holds state
// kq = t%4 of pattern 8g + t/4 of every group g and every category l (16
// doubles per vector, like walk4_kernel).  That is the A-fragment layout of
// m8n8k4 (row = pattern, column = state), and with the B fragments built by
// K1 (pg_kernels.cuh, f4post / f4pre) the D fragment's even column 2c lands
// on the lane of state c: one DMMA per (group, category) computes
//  * post order: e = P x (odd columns unused);
//  * pre order, per child: q_c = P_c^T top in the even columns and
//    u = Q^T top in the odd ones, so the gradient numerator
//    top.(Q e_c) = u.e_c (engine.hpp:258-262) is a lane-local product summed
//    over the quad -- no separate Q e mat-vec;
//  * with the Hessian, (Q^2)^T top from a second fragment.
// Chained steps need no shuffles.  walk4/walk4s spend most of their
// instructions and shared-memory wavefronts on the mat-vecs' P-block
// broadcast loads (8 LDS.128 per category per mat-vec); here a mat-vec is
// 4 DMMAs per category over the warp's 32 patterns and one 8-byte fragment
// load per lane.  Per-pattern quantities (normalisation peak, the gradient
// denominator and numerators, the root mixture) are quad reductions.
//
// Measured (C3 full size, profiles/r23_walk4t_C3_100k*): 215.6 ms at 168
// registers (3 CTAs/SM, spilling: 754 M local loads per evaluation), 185.3 ms
// at 255 (2 CTAs/SM, the default here) vs walk4s's 138 ms, parity exact --
// 7.4 G vs 6.5 G instructions per 10^5 columns: the
// quad reductions (normalisation peak, denominator, numerators, root
// mixture), the zero-initialised DMMA accumulators and the per-group
// normalisation add back more than the mat-vecs save, and DMMA is 4 % of the
// issued instructions.  Opt-in (PG_WALK4T=1).
//
// Staging as walk4s_kernel: one shared-memory stage per warp (children's
// edge messages, a deferred pre-partial, tip TC blocks, fragment blocks, code
// rows) filled once the previous step has consumed it; the hand-offs (the
// previous step's edge message, the pre-partial of the child visited next)
// stay in registers.
#pragma once

#include "pg_walk4s.cuh"

#ifndef PG_WALK4T_MINB
#define PG_WALK4T_MINB 2
#endif

namespace pgk {

__device__ __forceinline__ void dmma4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NC>
struct Walk4TGeom {
  static constexpr int L = 4;
  static constexpr int TCB = L * NC * 4;  // doubles per TC block
  static constexpr int VEC = 32 * L * 4;  // doubles per node slot of one warp
  static constexpr int SD2 = VEC / 2;     // double2 per node slot
  static constexpr int FB = (L + 1) * 32; // doubles per fragment block
  // per warp (doubles): slots A, B, Q; TC blocks 0, 1; fragment blocks 0, 1; code rows
  static constexpr int OFF_A = 0, OFF_B = VEC, OFF_Q = 2 * VEC, OFF_T0 = 3 * VEC, OFF_T1 = OFF_T0 + TCB,
                       OFF_F0 = OFF_T1 + TCB, OFF_F1 = OFF_F0 + FB, OFF_C = OFF_F1 + FB;
  static constexpr int WARP = (OFF_C + 8 + 15) & ~15;  // doubles, 128-byte aligned
};

template <bool HESS, int NC>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, PG_WALK4T_MINB)
    walk4t_kernel(const __grid_constant__ Walk4TParams PT) {
  using Gm = Walk4TGeom<NC>;
  constexpr int L = 4, VEC = Gm::VEC, SD2 = Gm::SD2, TCB = Gm::TCB;
  const Walk4SParams& PS = PT.s;
  const Walk4Params& P4 = PS.w;
  const WalkParams& p = P4.p;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int warp = blockIdx.x * kWarpsPerBlock + wib;
  const int TW = gridDim.x * kWarpsPerBlock;
  const int N = p.N, root = 2 * N - 1;
  const int kq = lane & 3, i8 = lane >> 2;  // state, pattern within a group
  double* const wsm = reinterpret_cast<double*>(smem_raw) + size_t(wib) * Gm::WARP;
  double2* const sA = reinterpret_cast<double2*>(wsm + Gm::OFF_A);
  double2* const sB = reinterpret_cast<double2*>(wsm + Gm::OFF_B);
  double2* const sQ = reinterpret_cast<double2*>(wsm + Gm::OFF_Q);
  double* const sT0 = wsm + Gm::OFF_T0;
  double* const sT1 = wsm + Gm::OFF_T1;
  double* const sF0 = wsm + Gm::OFF_F0;
  double* const sF1 = wsm + Gm::OFF_F1;
  unsigned char* const sC = reinterpret_cast<unsigned char*>(wsm + Gm::OFF_C);  // 2 x 32 code bytes

  const size_t wbase = size_t(warp) * size_t(N - 1);
  // slot element (g, l) of a lane: double2 (2g + l/2) * 32 + lane, component l%2
  const double2* Eb = reinterpret_cast<const double2*>(p.escr + wbase * VEC) + lane - size_t(SD2) * size_t(N + 1);
  double2* Ew = reinterpret_cast<double2*>(p.escr + wbase * VEC) + lane - size_t(SD2) * size_t(N + 1);
  double2* Qw = reinterpret_cast<double2*>(p.qscr + wbase * VEC) + lane - size_t(SD2) * size_t(N + 1);
  double* A = p.acc + size_t(warp) * p.accw;
  for (int i = lane; i < p.accw; i += 32) A[i] = 0.0;
  __syncwarp();

  const unsigned long long pol_first = policy_evict_first();
  auto stage_slot = [&](double2* slot, const double2* gs) {
#pragma unroll
    for (int q = 0; q < 8; ++q) cp16_cg(slot + lane + q * 32, gs + q * 32);
  };
  auto stage_slot_once = [&](double2* slot, const double2* gs) {
#pragma unroll
    for (int q = 0; q < 8; ++q) cp16_cg_hint(slot + lane + q * 32, gs + q * 32, pol_first);
  };
  auto stage_blk = [&](double* d, const double* src, int nd) {  // nd doubles (multiple of 2), 16-byte chunks
    const double2* gs = reinterpret_cast<const double2*>(src);
    double2* dd = reinterpret_cast<double2*>(d);
    for (int c = lane; c < nd / 2; c += 32) cp16_ca(dd + c, gs + c);
  };
  const size_t Pc = size_t(p.Pc);
  auto shfl_d = [&](double v, int m) -> double { return __shfl_xor_sync(kFull, v, m); };
  // quad (4 states of a pattern) max of an int
  auto quad_maxi = [&](int v) {
    v = max(v, __shfl_xor_sync(kFull, v, 1));
    return max(v, __shfl_xor_sync(kFull, v, 2));
  };
  // reduce-scatter over the quad: v[g] are partial sums of group g; returns
  // the total of group kq (the lane's own pattern 8 kq + i8)
  auto quad_rs = [&](const double (&v)[4]) -> double {
    const bool hi = kq >= 2;
    const double r0 = (hi ? v[2] : v[0]) + shfl_d(hi ? v[0] : v[2], 2);
    const double r1 = (hi ? v[3] : v[1]) + shfl_d(hi ? v[1] : v[3], 2);
    const bool odd = kq & 1;
    return (odd ? r1 : r0) + shfl_d(odd ? r0 : r1, 1);
  };
  // the 4 categories of group g of a staged slot: two 16-byte loads
  auto slot_grp = [&](const double2* slot, int g, double (&v)[L]) {
    const double2 a = slot[(2 * g) * 32 + lane], b = slot[(2 * g + 1) * 32 + lane];
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  };
  // tip edge message of group g: the lane's state of the code's TC column per
  // category (base = the TC block + 4 code + state, category stride 4 NC)
  auto tip_grp = [&](const double* base, double (&v)[L]) {
#pragma unroll
    for (int l = 0; l < L; ++l) v[l] = base[l * NC * 4];
  };
  auto shfl4 = [&](const int4 v, int src) -> int4 {
    int4 o;
    o.x = __shfl_sync(kFull, v.x, src);
    o.y = __shfl_sync(kFull, v.y, src);
    o.z = __shfl_sync(kFull, v.z, src);
    o.w = __shfl_sync(kFull, v.w, src);
    return o;
  };

  const int n = p.nsteps;
  for (int t = warp; t < p.ntiles; t += TW) {
    // the lane's own pattern (reductions land there): 8 kq + i8
    const int s = t * 32 + 8 * kq + i8;
    const bool valid = s < p.P;
    const int sc = valid ? s : p.P - 1;
    const double w = valid ? p.weights[sc] : 0.0;
    const uint8_t* codes = p.codes + size_t(t) * 32;  // tile base; row stride Pc
    auto code_row = [&](unsigned char* d, int tip) {
      if (lane < 2) cp16_ca(d + 16 * lane, codes + size_t(tip - 1) * Pc + 16 * lane);
    };

    // ------------------------------------------------ post-order pass (a)
    {
      int S[4] = {0, 0, 0, 0};  // per group (quad-uniform) accumulated exponents
      double keep[4][L];
      auto issue = [&](const int4 d, int last) {
        if (d.y <= N) {
          code_row(sC, d.y);
          stage_blk(sT0, p.tc + size_t(d.y - 1) * TCB, TCB);
        } else if (d.y != last) {
          stage_slot(sA, Eb + size_t(d.y) * SD2);
        }
        if (d.z <= N) {
          code_row(sC + 32, d.z);
          stage_blk(sT1, p.tc + size_t(d.z - 1) * TCB, TCB);
        } else if (d.z != last) {
          stage_slot(sA, Eb + size_t(d.z) * SD2);
        }
        if (d.x != root) stage_blk(sF0, PT.f4post + size_t(d.x - 1) * L * 32, L * 32);
      };
      int4 win = lane < n ? p.post[lane] : make_int4(0, 0, 0, 0);
      int4 winn = 32 + lane < n ? p.post[32 + lane] : make_int4(0, 0, 0, 0);
      int4 d = shfl4(win, 0);
      issue(d, -1);
      cp_commit();
      int last = -1;
      for (int i = 0; i < n; ++i) {
        int4 dn = make_int4(0, 0, 0, 0);
        if (i + 1 < n) {
          const int li = (i + 1) & 31;
          if (li == 0) {
            win = winn;
            winn = i + 33 + lane < n ? p.post[i + 33 + lane] : make_int4(0, 0, 0, 0);
          }
          dn = shfl4(win, li);
        }
        cpa_wait_all();
        __syncwarp();
        // operand kinds: 0 tip, 1 the previous step's node (registers), 2
        // slot A; in the heavy-child-first order only (T,T), (T,K), (K,T),
        // (K,S), (S,K) occur -- each compiled straight-line
        const int ka = d.y <= N ? 0 : d.y == last ? 1 : 2;
        const int kb = d.z <= N ? 0 : d.z == last ? 1 : 2;
        double x[4][L];
        int hm[4] = {0, 0, 0, 0};
        auto operand = [&](auto K, const unsigned char* crow, const double* T, int g, double (&v)[L]) {
          constexpr int k = decltype(K)::value;
          if constexpr (k == 0) tip_grp(T + 4 * int(crow[8 * g + i8]) + kq, v);
          else if constexpr (k == 1) {
#pragma unroll
            for (int l = 0; l < L; ++l) v[l] = keep[g][l];
          } else {
            slot_grp(sA, g, v);
          }
        };
        auto product = [&](auto KA, auto KB) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            double a[L], b[L];
            operand(KA, sC, sT0, g, a);
            operand(KB, sC + 32, sT1, g, b);
#pragma unroll
            for (int l = 0; l < L; ++l) {
              x[g][l] = a[l] * b[l];
              hm[g] = max(hm[g], __double2hiint(x[g][l]));
            }
          }
        };
        using K0 = std::integral_constant<int, 0>;
        using K1 = std::integral_constant<int, 1>;
        using K2 = std::integral_constant<int, 2>;
        if (ka == 0) {
          if (kb == 0) product(K0{}, K0{});
          else if (kb == 1) product(K0{}, K1{});
          else product(K0{}, K2{});
        } else if (ka == 1) {
          if (kb == 0) product(K1{}, K0{});
          else product(K1{}, K2{});
        } else {
          if (kb == 0) product(K2{}, K0{});
          else product(K2{}, K1{});
        }
        if (!p.disable) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int ex = peak_exponent(quad_maxi(hm[g]));
            if (ex != 0) {
              S[g] += ex;
              if (ex <= 1022) {
                const double sc2 = pow2_neg(ex);
#pragma unroll
                for (int l = 0; l < L; ++l) x[g][l] *= sc2;
              } else {
#pragma unroll
                for (int l = 0; l < L; ++l) x[g][l] = ldexp(x[g][l], -ex);
              }
            }
          }
        }
        if (d.x == root) {
          double part[4];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            double m0 = 0.0;
#pragma unroll
            for (int l = 0; l < L; ++l) m0 = fma(PS.cw[l], x[g][l], m0);
            part[g] = P4.pi[kq] * m0;
          }
          const double mix = quad_rs(part);
          const int Sown = kq == 0 ? S[0] : kq == 1 ? S[1] : kq == 2 ? S[2] : S[3];
          const double ll = log(mix) + double(Sown) * 0.6931471805599453;
          if (valid) {
            if (!isfinite(mix)) atomicMin(&p.err[0], s);
            else if (mix <= 0.0) atomicMin(&p.err[1], s);
            if (p.site_ll) p.site_ll[s] = ll;
          }
          const double v = warp_sum(valid ? w * ll : 0.0);
          if (lane == 0) atomicAdd(A, v);
        } else {
          double fr[L];
#pragma unroll
          for (int l = 0; l < L; ++l) fr[l] = sF0[l * 32 + lane];
          double2* dst = Ew + size_t(d.x) * SD2;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
#pragma unroll
            for (int l = 0; l < L; ++l) {
              double e0 = 0.0, e1 = 0.0;
              dmma4(e0, e1, x[g][l], fr[l]);
              keep[g][l] = e0;
            }
            __stcs(dst + (2 * g) * 32, make_double2(keep[g][0], keep[g][1]));
            __stcs(dst + (2 * g + 1) * 32, make_double2(keep[g][2], keep[g][3]));
          }
          last = d.x;
        }
        __syncwarp();
        if (i + 1 < n) issue(dn, d.x);
        cp_commit();
        d = dn;
      }
      cpa_wait_all();
      __syncwarp();
    }
    if (!p.do_pre) continue;

    // ----------------------------------- pre-order pass + gradient (b)+(c)
    {
      auto issue = [&](const int4 d, int handed) {
        if (d.x != root && handed != d.x) stage_slot(sQ, Qw + size_t(d.x) * SD2);
        if (d.y <= N) {
          code_row(sC, d.y);
          stage_blk(sT0, p.tc + size_t(d.y - 1) * TCB, TCB);
        } else {
          stage_slot_once(sA, Eb + size_t(d.y) * SD2);
        }
        if (d.z <= N) {
          code_row(sC + 32, d.z);
          stage_blk(sT1, p.tc + size_t(d.z - 1) * TCB, TCB);
        } else {
          stage_slot_once(sB, Eb + size_t(d.z) * SD2);
        }
        const int nf = HESS ? (L + 1) * 32 : L * 32;
        stage_blk(sF0, PT.f4pre + size_t(d.y - 1) * (L + 1) * 32, nf);
        stage_blk(sF1, PT.f4pre + size_t(d.z - 1) * (L + 1) * 32, nf);
      };
      const char* base_e = reinterpret_cast<const char*>(p.escr + wbase * VEC);
      const char* base_q = reinterpret_cast<const char*>(p.qscr + wbase * VEC);
      int4 win = lane < n ? p.pre[lane] : make_int4(0, 0, 0, 0);
      int4 winn = 32 + lane < n ? p.pre[32 + lane] : make_int4(0, 0, 0, 0);
      int4 d = shfl4(win, 0);
      issue(d, 0);
      cp_commit();
      double q[4][L];  // the step's pre-partial when handed on (registers)
      int handed = 0;
      for (int i = 0; i < n; ++i) {
        int4 dn = make_int4(0, 0, 0, 0);
        if (i + 1 < n) {
          const int li = (i + 1) & 31;
          if (li == 0) {
            win = winn;
            winn = i + 33 + lane < n ? p.pre[i + 33 + lane] : make_int4(0, 0, 0, 0);
          }
          dn = shfl4(win, li);
        }
        cpa_wait_all();
        __syncwarp();
        // the step's pre-partial into registers: pi at the root, already there
        // when handed on, else from slot Q
        const int qsrc = d.x == root ? 0 : handed == d.x ? 1 : 2;
        if (qsrc == 0) {
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int l = 0; l < L; ++l) q[g][l] = P4.pi[kq];
        } else if (qsrc == 2) {
#pragma unroll
          for (int g = 0; g < 4; ++g) slot_grp(sQ, g, q[g]);
        }
        const bool a_int = d.y > N, b_int = d.z > N;
        double fa[L], fb[L], fa2 = 0.0, fb2 = 0.0;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          fa[l] = sF0[l * 32 + lane];
          fb[l] = sF1[l * 32 + lane];
        }
        if constexpr (HESS) {
          fa2 = sF0[L * 32 + lane];
          fb2 = sF1[L * 32 + lane];
        }
        double dd[4], na[4], nb[4], na2[4], nb2[4];
        const bool next_a = d.y == d.w, next_b = d.z == d.w;
        double2* qa_dst = Qw + size_t(d.y) * SD2;  // lane offset included
        double2* qb_dst = Qw + size_t(d.z) * SD2;
        // normalise an internal child's pre-partial (per pattern = per quad)
        // and hand it on in place or store it to its scratch slot
        auto emit = [&](double (&o)[L], int h, bool next, double2* dst, int g) {
          const int ex = peak_exponent(quad_maxi(h));
          const double scl = (ex != 0 && ex <= 1022) ? pow2_neg(ex) : 1.0;
#pragma unroll
          for (int l = 0; l < L; ++l) o[l] *= scl;
          if (next) {
#pragma unroll
            for (int l = 0; l < L; ++l) q[g][l] = o[l];
          } else {
            __stcg(dst + (2 * g) * 32, make_double2(o[0], o[1]));
            __stcg(dst + (2 * g + 1) * 32, make_double2(o[2], o[3]));
          }
        };
        // child kinds (internal / tip) compiled straight-line
        auto body = [&](auto AI, auto BI) {
          constexpr bool ai = decltype(AI)::value, bi = decltype(BI)::value;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            double av[L], bv[L];
            if constexpr (ai) slot_grp(sA, g, av);
            else tip_grp(sT0 + 4 * int(sC[8 * g + i8]) + kq, av);
            if constexpr (bi) slot_grp(sB, g, bv);
            else tip_grp(sT1 + 4 * int(sC[32 + 8 * g + i8]) + kq, bv);
            double oa[L], ob[L];
            int ha = 0, hb = 0;
            double ddg = 0.0, nag = 0.0, nbg = 0.0, na2g = 0.0, nb2g = 0.0;
#pragma unroll
            for (int l = 0; l < L; ++l) {
              const double ta = q[g][l] * bv[l], tb = q[g][l] * av[l];  // tops of children a and b
              ddg = fma(PS.cw[l] * ta, av[l], ddg);
              double qa = 0.0, ua = 0.0, qb = 0.0, ub = 0.0;
              dmma4(qa, ua, ta, fa[l]);  // q_a = P_a^T top_a (even columns), u_a = Q^T top_a (odd)
              dmma4(qb, ub, tb, fb[l]);
              nag = fma(PS.crw[l] * ua, av[l], nag);
              nbg = fma(PS.crw[l] * ub, bv[l], nbg);
              if constexpr (HESS) {
                double va = 0.0, xa = 0.0, vb = 0.0, xb = 0.0;
                dmma4(va, xa, ta, fa2);  // (Q^2)^T top_a
                dmma4(vb, xb, tb, fb2);
                na2g = fma(PS.cr2w[l] * va, av[l], na2g);
                nb2g = fma(PS.cr2w[l] * vb, bv[l], nb2g);
              }
              oa[l] = qa;
              ob[l] = qb;
              if constexpr (ai) ha = max(ha, __double2hiint(qa));
              if constexpr (bi) hb = max(hb, __double2hiint(qb));
            }
            dd[g] = ddg;
            na[g] = nag;
            nb[g] = nbg;
            na2[g] = na2g;
            nb2[g] = nb2g;
            // (the group's q is consumed: in-place hand-off is safe)
            if constexpr (ai) emit(oa, ha, next_a, qa_dst, g);
            if constexpr (bi) emit(ob, hb, next_b, qb_dst, g);
          }
        };
        using T_ = std::true_type;
        using F_ = std::false_type;
        if (a_int) {
          if (b_int) body(T_{}, T_{});
          else body(T_{}, F_{});
        } else {
          if (b_int) body(F_{}, T_{});
          else body(F_{}, F_{});
        }
        __syncwarp();
        // the stage is consumed: the next step's operands
        if (i + 1 < n) issue(dn, d.w);
        cp_commit();
        // consumed scratch is dead: drop it from L2 without write-back
        if (lane < VEC / 16) {
          if (a_int) discard_l2(base_e + size_t(d.y - N - 1) * (VEC * 8) + lane * 128);
          if (b_int) discard_l2(base_e + size_t(d.z - N - 1) * (VEC * 8) + lane * 128);
          if (qsrc == 2) discard_l2(base_q + size_t(d.x - N - 1) * (VEC * 8) + lane * 128);
        }
        // per-pattern denominator and numerators (quad reduce-scatter onto
        // the lane's own pattern), gradient contributions
        const double den = quad_rs(dd);
        const double inv = 1.0 / den;
        const double r1a = quad_rs(na) * inv, r1b = quad_rs(nb) * inv;
        const double ga = warp_sum(valid ? w * r1a : 0.0);
        const double gb = warp_sum(valid ? w * r1b : 0.0);
        if (lane == 0) {
          atomicAdd(A + d.y, ga);
          atomicAdd(A + d.z, gb);
        }
        if constexpr (HESS) {
          const double s2a = quad_rs(na2), s2b = quad_rs(nb2);  // all lanes take part in the shuffles
          const double ha2 = warp_sum(valid ? w * (s2a * inv - r1a * r1a) : 0.0);
          const double hb2 = warp_sum(valid ? w * (s2b * inv - r1b * r1b) : 0.0);
          if (lane == 0) {
            atomicAdd(A + p.B + d.y, ha2);
            atomicAdd(A + p.B + d.z, hb2);
          }
        }
        handed = d.w;
        d = dn;
      }
      cpa_wait_all();
      __syncwarp();
    }
  }
}

}  // namespace pgk
