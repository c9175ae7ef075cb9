// K2 specialised for 4-state models with 4 rate categories (the HBM-bound
// C2/C3 path): one lane = one pattern with all categories (16 fp64 per
// vector), 32 patterns per warp tile, persistent warps.
//
// Differences from the generic walk_kernel (pg_walk.cuh):
//  * software pipeline: while step i computes, step i+1's memory operands
//    (edge-message / pre-partial slots, the TC blocks of the nodes involved)
//    are in flight into a per-warp shared-memory stage via cp.async, and its
//    tip codes via plain loads, so no load sits on the step's critical path;
//  * step descriptors are held 32 at a time in a register window and
//    broadcast with shuffles;
//  * compile-time column count NC, homogeneous generator Q and pi as direct
//    constant-bank operands, optional Hessian compiled out;
//  * pre-order step processed category by category (registers: q, e_a, e_b
//    for one category at a time + the two outgoing pre-partials);
//  * per-pattern normalisation from the integer max of the high words;
//  * gradient contributions go to the warp's accumulator row with RED
//    (fire-and-forget, single writer per address -> deterministic).
#pragma once

#include <type_traits>

#include "pg_walk.cuh"

// 1: the pre-partial of the child visited next is held in registers
// (qreg) instead of the next stage's shared q slot
#ifndef PG_WALK4_QREG
#define PG_WALK4_QREG 0
#endif

namespace pgk {

__device__ __forceinline__ void cp16_cg(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp16_ca(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp16_cg_hint(void* smem, const void* gmem, unsigned long long pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol)
               : "memory");
}
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
// The line's data is dead: drop it from L2 without a DRAM write-back.
__device__ __forceinline__ void discard_l2(const void* gmem) {
  asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Exponent of the peak of non-negative values from the max high word, as the
// power of two that brings the peak into [0.5, 1).  Returns 0 for all-zero,
// inf/NaN and subnormal-only blocks (left unscaled; reported at the root).
__device__ __forceinline__ int peak_exponent(int hmax) {
  const int bexp = (hmax >> 20) & 0x7ff;
  if (hmax <= 0 || bexp == 0x7ff || bexp == 0) return 0;
  return bexp - 1022;
}
// 2^-ex as a double (exact; ex in [-1021, 1022]).
__device__ __forceinline__ double pow2_neg(int ex) { return __hiloint2double((1023 - ex) << 20, 0); }

// double2 per shared-memory stage of one warp: 3 operand slots, 3 TC blocks,
// 2 x 32 B code rows, rounded up to 128 bytes so every warp-wide 512-byte slot
// access is 4 wavefronts (an odd 64-byte offset made it 5: 23 % excessive
// shared wavefronts in the C3 capture, profiles/r23_walk4_C3_100k_smem.txt)
__host__ __device__ constexpr int walk4_stage_d2(int LCV, int LT, int NC) {
  return (3 * (32 * LCV * 4 / 2) + 3 * (LT * NC * 4 / 2) + 4 + 7) & ~7;
}

// LT = rate categories (4, 2 or 1); LCV = categories per lane (LT: one lane
// per pattern, 32 patterns per warp tile; LT/2: two lanes per pattern, 16
// patterns per tile, half the registers and shared memory per warp -> more
// resident warps).
template <bool HOMOG, bool HESS, int NC, int LCV, int LT = 4>
__global__ void __launch_bounds__(kWarpsPerBlock * 32,
                                  (LCV >= 3 || (LCV == 2 && LT == 2 && !HOMOG) ? 2 : LCV == 2 ? 3 : 4))
    walk4_kernel(const __grid_constant__ Walk4Params P4) {
  static_assert(LT % LCV == 0, "categories split evenly over a pattern's lanes");
  constexpr int MP = 4, L = LT;
  constexpr int G = LT / LCV;                // lanes per pattern
  constexpr int TP = 32 / G;                 // patterns per warp tile
  constexpr int TCB = L * NC * MP;           // doubles per node TC block
  constexpr int TCC = TCB / 2;               // double2 chunks per TC block
  constexpr int VEC = 32 * LCV * MP;         // doubles per node slot of one warp
  constexpr int SD2 = VEC / 2;               // double2 per node slot
  constexpr int STAGE = walk4_stage_d2(LCV, LT, NC);  // double2 per stage (128-byte aligned)
  static_assert(STAGE >= 3 * SD2 + 3 * TCC + 4, "stage holds 3 slots, 3 TC blocks and the code rows");
  static_assert(TCC <= SD2, "a TC block fits in an operand slot");
  const WalkParams& p = P4.p;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int warp = blockIdx.x * kWarpsPerBlock + wib;
  const int TW = gridDim.x * kWarpsPerBlock;
  const int N = p.N, root = 2 * N - 1;
  double2* wsm = reinterpret_cast<double2*>(smem_raw) + size_t(wib) * 2 * STAGE;

  const int g = lane & (G - 1), pl = lane / G;
  double cw[LCV], crw[LCV], cr2w[LCV];
#pragma unroll
  for (int j = 0; j < LCV; ++j) {
    const double w = p.probs[g * LCV + j], r = p.rates[g * LCV + j];
    cw[j] = w;
    crw[j] = r * w;
    cr2w[j] = r * r * w;
  }
  auto gsum = [&](double v) {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
  };
  auto gmaxi = [&](int v) {
#pragma unroll
    for (int o = 1; o < G; o <<= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
    return v;
  };
  // lane-offset bases of this warp's scratch (slot k at + (k - N - 1) * VEC)
  const double2* Eb = reinterpret_cast<const double2*>(p.escr + size_t(warp) * size_t(N - 1) * VEC) + lane -
                      size_t(SD2) * size_t(N + 1);
  double2* Ew = reinterpret_cast<double2*>(p.escr + size_t(warp) * size_t(N - 1) * VEC) + lane -
                size_t(SD2) * size_t(N + 1);
  double2* Qw = reinterpret_cast<double2*>(p.qscr + size_t(warp) * size_t(N - 1) * VEC) + lane -
                size_t(SD2) * size_t(N + 1);
  double* A = p.acc + size_t(warp) * p.accw;
  for (int i = lane; i < p.accw; i += 32) A[i] = 0.0;
  __syncwarp();

  auto opp = [&](int stage, int slot) -> double2* { return wsm + stage * STAGE + slot * SD2 + lane; };
  auto tcp = [&](int stage, int slot) -> const double* {
    return reinterpret_cast<const double*>(wsm + stage * STAGE + 3 * SD2 + slot * TCC);
  };
  const unsigned long long pol_first = policy_evict_first();
  auto stage_slot = [&](int stage, int slot, const double2* gs) {
    double2* d = opp(stage, slot);
#pragma unroll
    for (int q = 0; q < 2 * LCV; ++q) cp16_cg(d + q * 32, gs + q * 32);
  };
  // edge messages are read once in the pre pass: evict-first
  auto stage_slot_once = [&](int stage, int slot, const double2* gs) {
    double2* d = opp(stage, slot);
#pragma unroll
    for (int q = 0; q < 2 * LCV; ++q) cp16_cg_hint(d + q * 32, gs + q * 32, pol_first);
  };
  // the tile's TP code bytes of one tip (16 B chunks)
  auto stage_codes = [&](int stage, int which, const uint8_t* row) {
    if (lane < TP / 16) cp16_cg(wsm + stage * STAGE + 3 * SD2 + 3 * TCC + which * 2 + lane, row + 16 * lane);
  };
  auto code_of = [&](int stage, int which) -> int {
    return reinterpret_cast<const uint8_t*>(wsm + stage * STAGE + 3 * SD2 + 3 * TCC + which * 2)[pl];
  };
  // a tip child's Q P column table (same layout as its TC block) goes into the
  // operand slot a tip does not use (pre-order pass), replacing the 16-FMA
  // Q e per category: one lane per pattern only (C3 153.9 -> 151.9 ms; with
  // two lanes per pattern it costs C2 1.33 -> 1.39 ms)
  const bool tipq = LCV >= 4 && p.qtc != nullptr;
  auto stage_qtc = [&](int stage, int slot, int node) {
    const double2* gs = reinterpret_cast<const double2*>(p.qtc) + size_t(node - 1) * TCC;
    double2* d = wsm + stage * STAGE + slot * SD2;
#pragma unroll
    for (int c = 0; c < (TCC + 31) / 32; ++c)
      if (c * 32 + lane < TCC) cp16_cg(d + c * 32 + lane, gs + c * 32 + lane);
  };
  auto qtp = [&](int stage, int slot) -> const double* {
    return reinterpret_cast<const double*>(wsm + stage * STAGE + slot * SD2);
  };
  auto stage_tc = [&](int stage, int slot, int node) {
    const double2* gs = reinterpret_cast<const double2*>(p.tc) + size_t(node - 1) * TCC;
    double2* d = wsm + stage * STAGE + 3 * SD2 + slot * TCC;
#pragma unroll
    for (int c = 0; c < (TCC + 31) / 32; ++c)
      if (c * 32 + lane < TCC) cp16_cg(d + c * 32 + lane, gs + c * 32 + lane);
  };
  // one category (4 doubles) of a lane's slot: double2 q = 2j, 2j+1
  auto read_cat = [&](const double2* src, int j, double (&v)[4]) {
    const double2 a = src[(2 * j) * 32], b = src[(2 * j + 1) * 32];
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  };
  auto gather_cat = [&](const double* tcs, int code, int j, double (&v)[4]) {
    const double2* c = reinterpret_cast<const double2*>(tcs + ((g * LCV + j) * NC + code) * MP);
    const double2 a = c[0], b = c[1];
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  };
  auto qm = [&](int x, int r, int c) -> double {
    if constexpr (HOMOG) return P4.q[r * 4 + c];
    else return __ldg(p.qtab + size_t(p.qidx[x]) * 16 + r * 4 + c);
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
    const int s = t * TP + pl;
    const bool valid = s < p.P;
    const bool owner = valid && g == 0;
    const int sc = valid ? s : p.P - 1;
    const double w = valid ? p.weights[sc] : 0.0;
    const uint8_t* codes = p.codes + size_t(t) * TP;  // tile base; row stride Pc
    const size_t P = size_t(p.Pc);

    // ------------------------------------------------ post-order pass (a)
    {
      int S = 0;
      double keep[LCV][4];
      auto issue = [&](int j, const int4 d, int last) {
        const int st = j & 1;
        if (d.y <= N) {
          stage_codes(st, 0, codes + size_t(d.y - 1) * P);
          stage_tc(st, 1, d.y);
        } else if (d.y != last) {
          stage_slot(st, 0, Eb + size_t(d.y) * SD2);
        }
        if (d.z <= N) {
          stage_codes(st, 1, codes + size_t(d.z - 1) * P);
          stage_tc(st, 2, d.z);
        } else if (d.z != last) {
          stage_slot(st, 0, Eb + size_t(d.z) * SD2);
        }
        if (d.x != root) stage_tc(st, 0, d.x);
      };
      int4 win = lane < n ? p.post[lane] : make_int4(0, 0, 0, 0);
      int4 winn = 32 + lane < n ? p.post[32 + lane] : make_int4(0, 0, 0, 0);
      int4 dnext = shfl4(win, 0);
      issue(0, dnext, -1);
      cp_commit();
      int last = -1;
      for (int i = 0; i < n; ++i) {
        const int4 d = dnext;
        if (i + 1 < n) {
          const int li = (i + 1) & 31;
          if (li == 0) {
            win = winn;
            winn = i + 33 + lane < n ? p.post[i + 33 + lane] : make_int4(0, 0, 0, 0);
          }
          dnext = shfl4(win, li);
          issue(i + 1, dnext, d.x);
        }
        cp_commit();
        cp_wait1();
        __syncwarp();
        const int st = i & 1;
        const int code0 = d.y <= N ? code_of(st, 0) : 0;
        const int code1 = d.z <= N ? code_of(st, 1) : 0;
        // p_k = e_c0 o e_c1 for all categories, then exponent normalisation
        double x[LCV][4];
        int hm = 0;
        // child operand kinds: 0 tip (column gather), 1 the previous step's
        // edge message (registers), 2 staged slot.  In the heavy-child-first
        // order an internal child is either the previous step's node or its
        // sibling is, so (tip, tip), (tip, kept), (kept, tip), (kept, slot)
        // and (slot, kept) are the only combinations; for LCV <= 2 the loop
        // is compiled per combination (no operand branches)
        auto cat_loop = [&](auto ka, auto kb) {
          const int KA = ka, KB = kb;
#pragma unroll
          for (int j = 0; j < LCV; ++j) {
            double a[4], b[4];
            if (KA == 0) gather_cat(tcp(st, 1), code0, j, a);
            else if (KA == 1) {
#pragma unroll
              for (int r = 0; r < 4; ++r) a[r] = keep[j][r];
            } else read_cat(opp(st, 0), j, a);
            if (KB == 0) gather_cat(tcp(st, 2), code1, j, b);
            else if (KB == 1) {
#pragma unroll
              for (int r = 0; r < 4; ++r) b[r] = keep[j][r];
            } else read_cat(opp(st, 0), j, b);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              x[j][r] = a[r] * b[r];
              hm = max(hm, __double2hiint(x[j][r]));
            }
          }
        };
        if constexpr (LCV >= 4) {
          // one lane per pattern: a single copy with the operand tests inside
          // (specialising costs C3 ~1 %)
#pragma unroll
          for (int j = 0; j < LCV; ++j) {
            double a[4], b[4];
            if (d.y <= N) gather_cat(tcp(st, 1), code0, j, a);
            else if (d.y == last) {
#pragma unroll
              for (int r = 0; r < 4; ++r) a[r] = keep[j][r];
            } else read_cat(opp(st, 0), j, a);
            if (d.z <= N) gather_cat(tcp(st, 2), code1, j, b);
            else if (d.z == last) {
#pragma unroll
              for (int r = 0; r < 4; ++r) b[r] = keep[j][r];
            } else read_cat(opp(st, 0), j, b);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              x[j][r] = a[r] * b[r];
              hm = max(hm, __double2hiint(x[j][r]));
            }
          }
        } else {
          const int ka = d.y <= N ? 0 : d.y == last ? 1 : 2;
          const int kb = d.z <= N ? 0 : d.z == last ? 1 : 2;
          using K0 = std::integral_constant<int, 0>;
          using K1 = std::integral_constant<int, 1>;
          using K2 = std::integral_constant<int, 2>;
          if (ka == 0) {
            if (kb == 0) cat_loop(K0{}, K0{});
            else cat_loop(K0{}, K1{});
          } else if (ka == 1) {
            if (kb == 0) cat_loop(K1{}, K0{});
            else cat_loop(K1{}, K2{});
          } else {
            cat_loop(K2{}, K1{});
          }
        }
        if (!p.disable) {
          const int ex = peak_exponent(gmaxi(hm));
          if (ex != 0) {
            S += ex;
            if (ex <= 1022) {
              const double sc2 = pow2_neg(ex);
#pragma unroll
              for (int j = 0; j < LCV; ++j)
#pragma unroll
                for (int r = 0; r < 4; ++r) x[j][r] *= sc2;
            } else {
#pragma unroll
              for (int j = 0; j < LCV; ++j)
#pragma unroll
                for (int r = 0; r < 4; ++r) x[j][r] = ldexp(x[j][r], -ex);
            }
          }
        }
        if (d.x == root) {
          double mix = 0.0;
#pragma unroll
          for (int j = 0; j < LCV; ++j) {
            double dd = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r) dd = fma(P4.pi[r], x[j][r], dd);
            mix = fma(cw[j], dd, mix);
          }
          mix = gsum(mix);
          const double ll = log(mix) + double(S) * 0.6931471805599453;
          if (owner) {
            if (!isfinite(mix)) atomicMin(&p.err[0], s);
            else if (mix <= 0.0) atomicMin(&p.err[1], s);
            if (p.site_ll) p.site_ll[s] = ll;
          }
          const double v = warp_sum(owner ? w * ll : 0.0);
          if (lane == 0) atomicAdd(A, v);
        } else {
          const double* T = tcp(st, 0);
          double2* dst = Ew + size_t(d.x) * SD2;
#pragma unroll
          for (int j = 0; j < LCV; ++j) {
            const double2* Tl = reinterpret_cast<const double2*>(T + (g * LCV + j) * NC * MP);
            double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const double2 a = Tl[2 * c], b = Tl[2 * c + 1];
              const double xc = x[j][c];
              e0 = fma(a.x, xc, e0);
              e1 = fma(a.y, xc, e1);
              e2 = fma(b.x, xc, e2);
              e3 = fma(b.y, xc, e3);
            }
            keep[j][0] = e0;
            keep[j][1] = e1;
            keep[j][2] = e2;
            keep[j][3] = e3;
            __stcs(dst + (2 * j) * 32, make_double2(e0, e1));
            __stcs(dst + (2 * j + 1) * 32, make_double2(e2, e3));
          }
          last = d.x;
        }
        __syncwarp();
      }
    }
    if (!p.do_pre) continue;

    // ----------------------------------- pre-order pass + gradient (b)+(c)
    {
      auto issue = [&](int j, const int4 d, int prev_next) {
        const int st = j & 1;
        if (d.x != root && prev_next != d.x) stage_slot(st, 2, Qw + size_t(d.x) * SD2);
        if (d.y <= N) {
          stage_codes(st, 0, codes + size_t(d.y - 1) * P);
          if (tipq) stage_qtc(st, 0, d.y);
        } else {
          stage_slot_once(st, 0, Eb + size_t(d.y) * SD2);
        }
        if (d.z <= N) {
          stage_codes(st, 1, codes + size_t(d.z - 1) * P);
          if (tipq) stage_qtc(st, 1, d.z);
        } else {
          stage_slot_once(st, 1, Eb + size_t(d.z) * SD2);
        }
        stage_tc(st, 0, d.y);
        stage_tc(st, 1, d.z);
      };
#if PG_WALK4_QREG
      double qreg[LCV][4];
#endif
      int4 win = lane < n ? p.pre[lane] : make_int4(0, 0, 0, 0);
      int4 winn = 32 + lane < n ? p.pre[32 + lane] : make_int4(0, 0, 0, 0);
      int4 dnext = shfl4(win, 0);
      issue(0, dnext, 0);
      cp_commit();
#if !PG_WALK4_QREG
      // the pre-partial operand always comes from the stage's q slot: the
      // root's is pi, written here (the first step is the root's)
#pragma unroll
      for (int j = 0; j < LCV; ++j) {
        double2* qd = opp(0, 2);
        qd[(2 * j) * 32] = make_double2(P4.pi[0], P4.pi[1]);
        qd[(2 * j + 1) * 32] = make_double2(P4.pi[2], P4.pi[3]);
      }
#endif
      int prev_next = 0;
      for (int i = 0; i < n; ++i) {
        const int4 d = dnext;
        if (i + 1 < n) {
          const int li = (i + 1) & 31;
          if (li == 0) {
            win = winn;
            winn = i + 33 + lane < n ? p.pre[i + 33 + lane] : make_int4(0, 0, 0, 0);
          }
          dnext = shfl4(win, li);
          issue(i + 1, dnext, d.w);
        }
        cp_commit();
        cp_wait1();
        __syncwarp();
        const int st = i & 1;
        const bool q_in_reg = prev_next == d.x;
        const int code0 = d.y <= N ? code_of(st, 0) : 0;
        const int code1 = d.z <= N ? code_of(st, 1) : 0;
        // consumed scratch is dead: drop it from L2 without write-back
        if (lane < VEC / 16) {
          const char* base_e = reinterpret_cast<const char*>(p.escr + size_t(warp) * size_t(N - 1) * VEC);
          const char* base_q = reinterpret_cast<const char*>(p.qscr + size_t(warp) * size_t(N - 1) * VEC);
          if (d.y > N) discard_l2(base_e + size_t(d.y - N - 1) * (VEC * 8) + lane * 128);
          if (d.z > N) discard_l2(base_e + size_t(d.z - N - 1) * (VEC * 8) + lane * 128);
          if (d.x != root && !q_in_reg) discard_l2(base_q + size_t(d.x - N - 1) * (VEC * 8) + lane * 128);
        }
        const bool a_int = d.y > N, b_int = d.z > N;
        double qa[LCV][4], qb[LCV][4];
        double den = 0.0, na = 0.0, nb = 0.0, na2 = 0.0, nb2 = 0.0;
        int ha = 0, hb = 0;
        const double* Ta = tcp(st, 0);
        const double* Tb = tcp(st, 1);
        // the category loop, compiled per child kind (internal / tip) for
        // LCV <= 2 so its operand selection and outgoing-partial code carry no
        // branches (C2 1.48 -> 1.36 ms); one lane per pattern (LCV = 4) keeps
        // one copy with runtime tests (C3 154 vs 157 ms specialised)
        auto cat_loop = [&](auto ai, auto bi) {
          const bool AI = ai, BI = bi;  // compile-time constants when given as std::integral_constant
#pragma unroll
          for (int j = 0; j < LCV; ++j) {
            double q[4], ea[4], eb[4];
#if PG_WALK4_QREG
            if (d.x == root) {
#pragma unroll
              for (int r = 0; r < 4; ++r) q[r] = P4.pi[r];
            } else if (q_in_reg) {
#pragma unroll
              for (int r = 0; r < 4; ++r) q[r] = qreg[j][r];
            } else {
              read_cat(opp(st, 2), j, q);
            }
#else
            read_cat(opp(st, 2), j, q);
#endif
            if (AI) read_cat(opp(st, 0), j, ea);
            else gather_cat(Ta, code0, j, ea);
            if (BI) read_cat(opp(st, 1), j, eb);
            else gather_cat(Tb, code1, j, eb);
            double ta[4], tb[4], dd = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              ta[r] = q[r] * eb[r];  // top for child a
              tb[r] = q[r] * ea[r];  // top for child b
              dd = fma(ta[r], ea[r], dd);
            }
            den = fma(cw[j], dd, den);
            // gradient numerators: top . (Q e), Hessian: top . (Q^2 e)
            // Q e: a mat-vec for an internal child; for a tip the column of
            // the staged Q P table (P and Q commute, engine.hpp:260)
            double qea[4], qeb[4];
            if constexpr (LCV < 4) {
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                double u = 0.0, v = 0.0;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  u = fma(qm(d.y, r, c), ea[c], u);
                  v = fma(qm(d.z, r, c), eb[c], v);
                }
                qea[r] = u;
                qeb[r] = v;
              }
            } else {
              if (AI || !tipq) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                  double u = 0.0;
#pragma unroll
                  for (int c = 0; c < 4; ++c) u = fma(qm(d.y, r, c), ea[c], u);
                  qea[r] = u;
                }
              } else {
                gather_cat(qtp(st, 0), code0, j, qea);
              }
              if (BI || !tipq) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                  double v = 0.0;
#pragma unroll
                  for (int c = 0; c < 4; ++c) v = fma(qm(d.z, r, c), eb[c], v);
                  qeb[r] = v;
                }
              } else {
                gather_cat(qtp(st, 1), code1, j, qeb);
              }
            }
            double d1a = 0.0, d1b = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              d1a = fma(ta[r], qea[r], d1a);
              d1b = fma(tb[r], qeb[r], d1b);
            }
            na = fma(crw[j], d1a, na);
            nb = fma(crw[j], d1b, nb);
            if constexpr (HESS) {
              double d2a = 0.0, d2b = 0.0;
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
              na2 = fma(cr2w[j], d2a, na2);
              nb2 = fma(cr2w[j], d2b, nb2);
            }
            // outgoing pre-partials q_x = P_x^T top (engine.hpp:249-250)
            if (AI) {
              const double2* Tl = reinterpret_cast<const double2*>(Ta + (g * LCV + j) * NC * MP);
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const double2 u = Tl[2 * c], v = Tl[2 * c + 1];
                qa[j][c] = fma(u.x, ta[0], fma(u.y, ta[1], fma(v.x, ta[2], v.y * ta[3])));
                ha = max(ha, __double2hiint(qa[j][c]));
              }
            }
            if (BI) {
              const double2* Tl = reinterpret_cast<const double2*>(Tb + (g * LCV + j) * NC * MP);
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const double2 u = Tl[2 * c], v = Tl[2 * c + 1];
                qb[j][c] = fma(u.x, tb[0], fma(u.y, tb[1], fma(v.x, tb[2], v.y * tb[3])));
                hb = max(hb, __double2hiint(qb[j][c]));
              }
            }
          }
        };
        using T_ = std::true_type;
        using F_ = std::false_type;
        if constexpr (LCV >= 4) {
          cat_loop(a_int, b_int);
        } else if (a_int) {
          if (b_int) cat_loop(T_{}, T_{});
          else cat_loop(T_{}, F_{});
        } else {
          if (b_int) cat_loop(F_{}, T_{});
          else cat_loop(F_{}, F_{});
        }
        den = gsum(den);
        na = gsum(na);
        nb = gsum(nb);
        if constexpr (HESS) {
          na2 = gsum(na2);
          nb2 = gsum(nb2);
        }
        ha = gmaxi(ha);
        hb = gmaxi(hb);
        const double inv = 1.0 / den;
        {
          const double r1a = na * inv, r1b = nb * inv;
          const double ga = warp_sum(owner ? w * r1a : 0.0);
          const double gb = warp_sum(owner ? w * r1b : 0.0);
          if (lane == 0) {
            atomicAdd(A + d.y, ga);
            atomicAdd(A + d.z, gb);
          }
          if constexpr (HESS) {
            const double ha2 = warp_sum(owner ? w * (na2 * inv - r1a * r1a) : 0.0);
            const double hb2 = warp_sum(owner ? w * (nb2 * inv - r1b * r1b) : 0.0);
            if (lane == 0) {
              atomicAdd(A + p.B + d.y, ha2);
              atomicAdd(A + p.B + d.z, hb2);
            }
          }
        }
        // normalise and hand on the pre-partials of internal children: the one
        // visited next goes straight into the next stage's q slot (not staged
        // from memory for that step), the other to its scratch slot
        auto emit = [&](const int x, double(&qx)[LCV][4], const int hx) {
          const int ex = peak_exponent(hx);
          const double scl = (ex != 0 && ex <= 1022) ? pow2_neg(ex) : 1.0;
          if (x == d.w) {
#if PG_WALK4_QREG
#pragma unroll
            for (int j = 0; j < LCV; ++j)
#pragma unroll
              for (int r = 0; r < 4; ++r) qreg[j][r] = qx[j][r] * scl;
#else
            double2* qd = opp(st ^ 1, 2);
#pragma unroll
            for (int j = 0; j < LCV; ++j) {
              qd[(2 * j) * 32] = make_double2(qx[j][0] * scl, qx[j][1] * scl);
              qd[(2 * j + 1) * 32] = make_double2(qx[j][2] * scl, qx[j][3] * scl);
            }
#endif
          } else {
            double2* dst = Qw + size_t(x) * SD2;
#pragma unroll
            for (int j = 0; j < LCV; ++j) {
              __stcg(dst + (2 * j) * 32, make_double2(qx[j][0] * scl, qx[j][1] * scl));
              __stcg(dst + (2 * j + 1) * 32, make_double2(qx[j][2] * scl, qx[j][3] * scl));
            }
          }
        };
        if (a_int) emit(d.y, qa, ha);
        if (b_int) emit(d.z, qb, hb);
        prev_next = d.w;
        __syncwarp();
      }
    }
  }
}

}  // namespace pgk
