// K2a'' — the 4-state, 4-category walk (one lane = one pattern, 32 patterns
// per warp tile, persistent warps) laid out for occupancy.
//
// walk4_kernel (pg_walk4.cuh) holds every vector of a step in registers (the
// kept edge message, the normalised product, both outgoing pre-partials: 64
// fp64 per lane) and double-buffers its shared-memory stage, so it runs at
// 255 registers and 114 KB per 4-warp CTA: 8 warps per SM.  Its C3 profile
// (profiles/r22_walk_C3_full_source.txt) is latency-bound -- fixed-latency and
// shared-memory dependency stalls with two warps per scheduler, 39 % issue
// utilisation, memory waits ~2 % -- so this variant trades the prefetch stage
// for warps:
//  * one shared-memory stage per warp: slots Q (the step's pre-partial), A
//    and B (the
//    children's staged edge messages), two TC
//    blocks (13.6 KB per warp, 128-byte aligned); tip codes go straight to
//    registers;
//  * results are written in place: a pre-order step's outgoing pre-partial
//    for the child visited next goes to slot Q category by category after
//    that category's q was read, the other one to its scratch slot -- no
//    per-lane vector arrays survive the category loop of the pre-order pass
//    (the post-order pass, below that register peak, keeps the previous
//    step's edge message in registers);
//  * the pre-partials' power-of-two normalisation is applied by the consumer
//    (the producer knows the peak only after the last category): the scale
//    of the handed-on one travels in a register, a deferred one's exponent
//    is stored next to its scratch slot ([TW][N-1][32] ints) -- the same
//    values as walk4_kernel's, multiplied at read instead of at write;
//  * a step's loads are issued once the previous step has consumed its
//    operands and waited on at the top of the step; latency is hidden by the
//    other warps (up to 16 per SM).  Measured neutral and removed: an L2
//    prefetch of the edge messages the pre-order pass reads, 2 or 3 steps
//    ahead (C3 145.2 / 146.8 / 147.7 ms at distance 0 / 2 / 3), and the step
//    list in the kernel parameters (constant bank) instead of the shuffled
//    register window (133.0 / 133.4 vs 133.7 / 132.8 ms).
// The per-pattern arithmetic is walk4_kernel's; the warp and grid reductions
// run in another fixed order (warp_sum2, twice the accumulator rows), so the
// two agree to rounding and each is bit-reproducible run to run.
#pragma once

#include "pg_walk4.cuh"

#ifndef PG_WALK4S_MINB
#define PG_WALK4S_MINB 4
#endif
// The cherry-table instances run 3 CTAs (12 warps) per SM at up to 168
// registers: with a third of the steps and of the DRAM traffic gone, the
// spill-free code beats the four extra warps (C3 115.0 vs 117.0 ms unfused;
// the fused cherry steps need the registers: 111.5 ms vs 123.5 ms at 128)
#ifndef PG_WALK4S_MINB_CH
#define PG_WALK4S_MINB_CH 3
#endif

namespace pgk {

// table copies (TC blocks, cherry blocks): .cg by default -- with the shared
// memory carve-out this kernel needs, almost no L1 is left to allocate into
// (C3 100.1 / 101.8 ms vs 103.0 / 103.7 ms with .ca on one box)
#ifndef PG_W4S_TABLE_CG
#define PG_W4S_TABLE_CG 1
#endif
__device__ __forceinline__ void cp16_tab(void* smem, const void* gmem) {
#if PG_W4S_TABLE_CG
  cp16_cg(smem, gmem);
#else
  cp16_ca(smem, gmem);
#endif
}

// WT: slots A and B also hold a cherry child's three tables + tip ids (below)
template <int NC, bool WT = false>
struct Walk4SGeom {
  static constexpr int MP = 4, L = 4;
  static constexpr int TCB = L * NC * MP;  // doubles per node TC block
  static constexpr int TCC = TCB / 2;      // double2 chunks per TC block
  static constexpr int VEC = 32 * L * MP;  // doubles per node slot of one warp
  static constexpr int SD2 = VEC / 2;      // double2 per node slot
  static constexpr int SDA = WT ? 392 : SD2;  // double2 per slot A / B (WT: 3 x 128 + ids, 128-byte multiple)
  // per warp: slots Q, A, B; TC blocks 0, 1; exponent row (32 ints)
  // (rounded up to 128 bytes: a 64-byte offset makes every 512-byte slot access 5 wavefronts)
  static constexpr int WARP = (SD2 + 2 * SDA + 2 * TCC + 8 + 7) & ~7;  // double2
};

// Cherry tables (CH instances; NC = 4, no missing / ambiguous tip codes): the
// edge message of a cherry -- an internal node whose two children are tips --
// depends on its pattern only through the two tip codes, so K1's epilogue
// (cherry_tc_kernel) tabulates e_k = P_k (P_a[:, ca] o P_b[:, cb]) for the 16
// code pairs and the cherry becomes a "tip" with 16 columns, addressed by the
// combined code row 4 ca + cb: its post-order step, its stored edge message
// (a third of the edge scratch traffic on a Yule tree) and the 4 KB operand
// copy of its parent's pre-order step disappear; the parent stages the 2 KB
// table into a free operand slot and gathers.  The table is left unnormalised
// (the parent's own power-of-two normalisation absorbs the scale exactly).
// Step descriptors carry the children's cherry flags in bits 29 / 30 of x.
// The cherry's pre-order step (the gradients of its tips u, v) is fused into
// its parent's, against the parent's own denominator (Eq. 8: q_k . (e_u o e_v)
// = top_k . e_k), so a third of the pre-order steps and every hand-off or
// scratch round trip of q_k go away too:
//  * gradient instances (WT): the tips' numerators q_k . (e_v o Q e_u) with
//    q_k = P_k^T top_k are top_k . W_u for the tabulated W_u = P_k (e_v o Q e_u)
//    (and W_v alike; Q e of a tip from K1's Q P columns, so per-branch
//    generators are covered): two more gathers and 8 FMAs per category, no
//    P_k^T mat-vec, no P_k^T block; slots A / B grow to 6.1 KB for the three
//    tables (12 warps per SM);
//  * Hessian instances with one shared generator: q_k = P_k^T top_k stays in
//    registers and the tips' terms are formed from their TC blocks (behind the
//    table in the cherry block); with per-branch generators the cherry keeps
//    its own step.
// A cherry block (kCherryBlk double2) is [e_k | TC_u | TC_v | ids | W_u | W_v].

// Table layout: the 32 bytes of a (category, code pair) entry as two 16-byte
// halves [category][half][code pair] (PG_W4S_CT_SOA, default) -- a lane's two
// LDS.128 then fall into bank group (code pair mod 8) instead of (code pair
// mod 4) of the entry-major layout, halving the gathers' bank conflicts.
#ifndef PG_W4S_CT_SOA
#define PG_W4S_CT_SOA 1
#endif
// double offset of element r of entry (l, combo) in a table of ncc code pairs
__host__ __device__ constexpr int cherry_elem(int l, int combo, int r, int ncc) {
#if PG_W4S_CT_SOA
  return ((l * 2 + (r >> 1)) * ncc + combo) * 2 + (r & 1);
#else
  return (l * ncc + combo) * 4 + r;
#endif
}

// one thread per (cherry, category, code pair); TC is [B][4][4][4]
static __global__ void cherry_tc_kernel(const int4* __restrict__ cherries, int ncherry, int N, const double* __restrict__ tc,
                                        const double* __restrict__ qtc, double* __restrict__ ct) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncherry * 64) return;
  const int ci = i >> 6, l = (i >> 4) & 3, combo = i & 15;
  const int4 ch = cherries[ci];  // {k, a, b, 0}
  const double* Ta = tc + (size_t(ch.y - 1) * 4 + l) * 16 + (combo >> 2) * 4;
  const double* Tb = tc + (size_t(ch.z - 1) * 4 + l) * 16 + (combo & 3) * 4;
  const double* Tk = tc + (size_t(ch.x - 1) * 4 + l) * 16;
  // Q e of the tips (K1's Q P columns, same layout as TC)
  const double* Qa = qtc + (Ta - tc);
  const double* Qb = qtc + (Tb - tc);
  double e[4] = {0.0, 0.0, 0.0, 0.0}, wu[4] = {0.0, 0.0, 0.0, 0.0}, wv[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double xc = Ta[c] * Tb[c], xu = Tb[c] * Qa[c], xv = Ta[c] * Qb[c];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      e[r] = fma(Tk[c * 4 + r], xc, e[r]);
      wu[r] = fma(Tk[c * 4 + r], xu, wu[r]);
      wv[r] = fma(Tk[c * 4 + r], xv, wv[r]);
    }
  }
  double* blk = ct + size_t(ch.x - N - 1) * (2 * kCherryBlk);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int o = cherry_elem(l, combo, r, 16);
    blk[o] = e[r];
    blk[2 * 200 + o] = wu[r];
    blk[2 * 328 + o] = wv[r];
  }
  // the tips' own TC blocks (32 double2 each) and node ids behind the table
  const int t64 = i & 63;
  const double2* src = reinterpret_cast<const double2*>(tc + size_t((t64 < 32 ? ch.y : ch.z) - 1) * 64) + (t64 & 31);
  reinterpret_cast<double2*>(blk)[128 + t64] = *src;
  if (t64 == 0) *reinterpret_cast<int4*>(blk + 2 * 192) = make_int4(ch.y, ch.z, 0, 0);
}

// Data with missing characters (NC = 5: the four states + the all-ones column):
// the e_k table alone, 25 code pairs (3.2 KB, it fits the 4 KB operand slots);
// the cherry keeps its own pre-order step.  One thread per (cherry, category,
// code pair); TC is [B][4][5][4].
static __global__ void cherry_tc5_kernel(const int4* __restrict__ cherries, int ncherry, int N,
                                         const double* __restrict__ tc, double* __restrict__ ct) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncherry * 100) return;
  const int ci = i / 100, l = (i % 100) / 25, combo = i % 25;
  const int4 ch = cherries[ci];
  const double* Ta = tc + (size_t(ch.y - 1) * 4 + l) * 20 + (combo / 5) * 4;
  const double* Tb = tc + (size_t(ch.z - 1) * 4 + l) * 20 + (combo % 5) * 4;
  const double* Tk = tc + (size_t(ch.x - 1) * 4 + l) * 20;
  double e[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double xc = Ta[c] * Tb[c];
#pragma unroll
    for (int r = 0; r < 4; ++r) e[r] = fma(Tk[c * 4 + r], xc, e[r]);
  }
  double* blk = ct + size_t(ch.x - N - 1) * (2 * kCherryBlk);
#pragma unroll
  for (int r = 0; r < 4; ++r) blk[cherry_elem(l, combo, r, 25)] = e[r];
}

// combined code rows of the cherries: cc[k - N - 1][s] = nc code_a[s] + code_b[s]
static __global__ void cherry_codes_kernel(const int4* __restrict__ cherries, int ncherry, int N, long long Pc, int nc,
                                    const uint8_t* __restrict__ codes, uint8_t* __restrict__ cc) {
  const int4 ch = cherries[blockIdx.y];
  const uint8_t* a = codes + size_t(ch.y - 1) * Pc;
  const uint8_t* b = codes + size_t(ch.z - 1) * Pc;
  uint8_t* o = cc + size_t(ch.x - N - 1) * Pc;
  for (long long s = blockIdx.x * blockDim.x + threadIdx.x; s < Pc; s += (long long)gridDim.x * blockDim.x)
    o[s] = uint8_t(nc * min(int(a[s]), nc - 1) + min(int(b[s]), nc - 1));
}

template <bool HOMOG, bool HESS, int NC, bool CH = false>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, CH ? PG_WALK4S_MINB_CH : PG_WALK4S_MINB)
    walk4s_kernel(const __grid_constant__ Walk4SParams PS) {
  static_assert(!CH || NC == 4 || NC == 5, "cherry tables: 4 x 4 or 5 x 5 code pairs");
  constexpr bool WT = CH && !HESS && NC == 4;               // fused cherry steps through the W tables
  constexpr bool FUSE_TC = CH && HESS && HOMOG && NC == 4;  // fused through the tips' TC blocks
  constexpr int NCC = NC * NC;         // code pairs of a cherry
  constexpr int TBLC = 4 * NCC * 2;    // double2 per e_k table
  constexpr bool FUSE = WT || FUSE_TC;
  using Gm = Walk4SGeom<NC, WT>;
  constexpr int L = 4, TCC = Gm::TCC, VEC = Gm::VEC, SD2 = Gm::SD2, SDA = Gm::SDA;
  static_assert(TCC <= SD2, "a TC block fits in an operand slot");
  const Walk4Params& P4 = PS.w;
  const WalkParams& p = P4.p;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int warp = blockIdx.x * kWarpsPerBlock + wib;
  const int TW = gridDim.x * kWarpsPerBlock;
  const int N = p.N, root = 2 * N - 1;
  double2* const wsm = reinterpret_cast<double2*>(smem_raw) + size_t(wib) * Gm::WARP;
  double2* const sQ = wsm;
  double2* const sA = wsm + SD2;
  double2* const sB = sA + SDA;
  double2* const sT0 = sB + SDA;
  double2* const sT1 = sT0 + TCC;
  double2* const sX = sT1 + TCC;  // exponent row of a staged pre-partial

  const size_t wbase = size_t(warp) * size_t(N - 1);
  const double2* Eb = reinterpret_cast<const double2*>(p.escr + wbase * VEC) + lane - size_t(SD2) * size_t(N + 1);
  double2* Ew = reinterpret_cast<double2*>(p.escr + wbase * VEC) + lane - size_t(SD2) * size_t(N + 1);
  double2* Qw = reinterpret_cast<double2*>(p.qscr + wbase * VEC) + lane - size_t(SD2) * size_t(N + 1);
  int* Xw = PS.qexp + wbase * 32 + lane - size_t(32) * size_t(N + 1);
  const int* Xb = PS.qexp + wbase * 32 - size_t(32) * size_t(N + 1);
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
  auto stage_blk = [&](double2* d, const double* table, int node) {
    const double2* gs = reinterpret_cast<const double2*>(table) + size_t(node - 1) * TCC;
#pragma unroll
    for (int c = 0; c < (TCC + 31) / 32; ++c)
      if (c * 32 + lane < TCC) cp16_tab(d + c * 32 + lane, gs + c * 32 + lane);
  };
  const size_t Pc = size_t(p.Pc);
  auto read_cat = [&](const double2* slot, int j, double (&v)[4]) {
    const double2 a = slot[lane + (2 * j) * 32], b = slot[lane + (2 * j + 1) * 32];
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  };
  auto write_cat = [&](double2* slot, int j, const double (&v)[4]) {
    slot[lane + (2 * j) * 32] = make_double2(v[0], v[1]);
    slot[lane + (2 * j + 1) * 32] = make_double2(v[2], v[3]);
  };
  auto gather_cat = [&](const double2* tcs, int code, int j, double (&v)[4]) {
    const double2* c = tcs + (j * NC + code) * 2;
    const double2 a = c[0], b = c[1];
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  };
  // a cherry's table [category][code pair][4] staged in an operand slot
  auto gather_ct = [&](const double2* tbl, int code, int j, double (&v)[4]) {
#if PG_W4S_CT_SOA
    const double2 a = tbl[(j * 2) * NCC + code], b = tbl[(j * 2 + 1) * NCC + code];
#else
    const double2* c = tbl + (j * NCC + code) * 2;
    const double2 a = c[0], b = c[1];
#endif
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  };
  auto stage_ct = [&](double2* d, int node) {
    const double2* gs = reinterpret_cast<const double2*>(PS.ct) + size_t(node - N - 1) * kCherryBlk + lane;
#pragma unroll
    for (int c = 0; c < (TBLC + 31) / 32; ++c)
      if (c * 32 + lane < TBLC) cp16_tab(d + c * 32 + lane, gs + c * 32);
  };
  static_assert(!CH || (TBLC <= SD2 && TCC + TBLC <= SD2), "an e_k table fits slot Q and the tail of slot B");
  // the whole cherry block (table, the tips' TC blocks, their node ids)
  auto stage_cb = [&](double2* d, int node) {
    const double2* gs = reinterpret_cast<const double2*>(PS.ct) + size_t(node - N - 1) * kCherryBlk + lane;
#pragma unroll
    for (int c = 0; c < 6; ++c) cp16_tab(d + c * 32 + lane, gs + c * 32);
    if (lane == 0) cp16_tab(d + 192, gs + 192);
  };
  // (WT) e_k, W_u, W_v and the ids: slot [0,128) [128,256) [256,384) [384]
  auto stage_cw = [&](double2* d, int node) {
    const double2* gs = reinterpret_cast<const double2*>(PS.ct) + size_t(node - N - 1) * kCherryBlk + lane;
#pragma unroll
    for (int c = 0; c < 4; ++c) cp16_tab(d + c * 32 + lane, gs + c * 32);
#pragma unroll
    for (int c = 0; c < 8; ++c) cp16_tab(d + 128 + c * 32 + lane, gs + 200 + c * 32);
    if (lane == 0) cp16_tab(d + 384, gs + 192);
  };
  constexpr int kIdsAt = WT ? 384 : 192;
  // descriptor -> node ids + the children's cherry flags (bit 0: y, bit 1: z)
  auto unflag = [&](int4& d) -> int {
    if constexpr (!CH) return 0;
    const int f = (d.x >> 29) & 3;
    d.x &= kNodeMask;
    return f;
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
  // 2^-ex applied by the consumer of a pre-partial (walk4_kernel's emit scale)
  auto qscale = [](int ex) -> double { return (ex != 0 && ex <= 1022) ? pow2_neg(ex) : 1.0; };

  const int n = p.nsteps;
  for (int t = warp; t < p.ntiles; t += TW) {
    const int s = t * 32 + lane;
    const bool valid = s < p.P;
    const int sc = valid ? s : p.P - 1;
    const double w = valid ? p.weights[sc] : 0.0;
    const uint8_t* codes = p.codes + size_t(t) * 32;  // tile base; row stride Pc
    // a tip's code for the lane's pattern, loaded into a register when the
    // step is issued (consumed one step later; cheaper than staging the
    // 32-byte row through shared memory: C3 18 instructions per step)
    auto code_ld = [&](int tip) -> int { return __ldg(codes + size_t(tip - 1) * Pc + lane); };
    // a cherry's combined code 4 ca + cb ([N-1][Pc] rows by node - N - 1)
    const uint8_t* ccodes = CH ? PS.ccodes + size_t(t) * 32 : nullptr;
    auto ccode_ld = [&](int node) -> int { return __ldg(ccodes + size_t(node - N - 1) * Pc + lane); };
    int cn0 = 0, cn1 = 0;  // the next step's tip codes

    // ------------------------------------------------ post-order pass (a)
    {
      int S = 0;
      // the previous step's edge message stays in registers (the post-order
      // pass is under the pre-order pass's register peak: 127 registers,
      // no occupancy cost; C3 128.3 / 128.7 vs 131.2 / 131.1 ms through slot Q)
      double keep[L][4];
      // operands: tip -> TC block 0/1 + its code (register); the previous
      // step's node -> its edge message in registers; else slot A
      // (CH) a cherry child: its combined code + its table into slot Q
      // (child 0; unused by this pass) or behind the node's own block in slot B
      auto issue_ops = [&](const int4 d, int f, int last) {
        if (CH && (f & 1)) {
          cn0 = ccode_ld(d.y);
          stage_ct(sQ, d.y);
        } else if (d.y <= N) {
          cn0 = code_ld(d.y);
          stage_blk(sT0, p.tc, d.y);
        } else if (d.y != last) {
          stage_slot(sA, Eb + size_t(d.y) * SD2);
        }
        if (CH && (f & 2)) {
          cn1 = ccode_ld(d.z);
          stage_ct(sB + TCC, d.z);
        } else if (d.z <= N) {
          cn1 = code_ld(d.z);
          stage_blk(sT1, p.tc, d.z);
        } else if (d.z != last) {
          stage_slot(sA, Eb + size_t(d.z) * SD2);
        }
      };
      auto issue_own = [&](const int4 d) {
        if (d.x != root) stage_blk(sB, p.tc, d.x);
      };
      const int n = CH ? PS.npost : p.nsteps;  // (CH) the cherries' own steps are gone
      int4 win = lane < n ? p.post[lane] : make_int4(0, 0, 0, 0);
      int4 winn = 32 + lane < n ? p.post[32 + lane] : make_int4(0, 0, 0, 0);
      int4 d = shfl4(win, 0);
      int f = unflag(d);
      issue_ops(d, f, -1);
      issue_own(d);
      cp_commit();
      int last = -1;
      for (int i = 0; i < n; ++i) {
        int4 dn = make_int4(0, 0, 0, 0);
        int fn = 0;
        if (i + 1 < n) {
          const int li = (i + 1) & 31;
          if (li == 0) {
            win = winn;
            winn = i + 33 + lane < n ? p.post[i + 33 + lane] : make_int4(0, 0, 0, 0);
          }
          dn = shfl4(win, li);
          fn = unflag(dn);
        }
        cpa_wait_all();
        __syncwarp();
        const int ka = (CH && (f & 1)) ? 3 : d.y <= N ? 0 : d.y == last ? 1 : 2;
        const int kb = (CH && (f & 2)) ? 3 : d.z <= N ? 0 : d.z == last ? 1 : 2;
        const int code0 = cn0, code1 = cn1;
        double x[L][4];
        int hm = 0;
#pragma unroll
        for (int j = 0; j < L; ++j) {
          double a[4], b[4];
          if (ka == 3) gather_ct(sQ, code0, j, a);
          else if (ka == 0) gather_cat(sT0, code0, j, a);
          else if (ka == 1) {
#pragma unroll
            for (int r = 0; r < 4; ++r) a[r] = keep[j][r];
          } else read_cat(sA, j, a);
          if (kb == 3) gather_ct(sB + TCC, code1, j, b);
          else if (kb == 0) gather_cat(sT1, code1, j, b);
          else if (kb == 1) {
#pragma unroll
            for (int r = 0; r < 4; ++r) b[r] = keep[j][r];
          } else read_cat(sA, j, b);
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            x[j][r] = a[r] * b[r];
            hm = max(hm, __double2hiint(x[j][r]));
          }
        }
        __syncwarp();
        // slot A and the TC blocks are free: the next step's operands
        if (i + 1 < n) issue_ops(dn, fn, d.x);
        if (!p.disable) {
          const int ex = peak_exponent(hm);
          if (ex != 0) {
            S += ex;
            if (ex <= 1022) {
              const double sc2 = pow2_neg(ex);
#pragma unroll
              for (int j = 0; j < L; ++j)
#pragma unroll
                for (int r = 0; r < 4; ++r) x[j][r] *= sc2;
            } else {
#pragma unroll
              for (int j = 0; j < L; ++j)
#pragma unroll
                for (int r = 0; r < 4; ++r) x[j][r] = ldexp(x[j][r], -ex);
            }
          }
        }
        if (d.x == root) {
          double mix = 0.0;
#pragma unroll
          for (int j = 0; j < L; ++j) {
            double dd = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r) dd = fma(P4.pi[r], x[j][r], dd);
            mix = fma(PS.cw[j], dd, mix);
          }
          const double ll = log(mix) + double(S) * 0.6931471805599453;
          if (valid) {
            if (!isfinite(mix)) atomicMin(&p.err[0], s);
            else if (mix <= 0.0) atomicMin(&p.err[1], s);
            if (p.site_ll) p.site_ll[s] = ll;
          }
          const double v = warp_sum(valid ? w * ll : 0.0);
          if (lane == 0) atomicAdd(A, v);
        } else {
          double2* dst = Ew + size_t(d.x) * SD2;
#pragma unroll
          for (int j = 0; j < L; ++j) {
            const double2* Tl = sB + j * NC * 2;
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
            // in place: the kept operand of this category was read above
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
        if (i + 1 < n) issue_own(dn);
        cp_commit();
        d = dn;
        f = fn;
      }
      cpa_wait_all();
      __syncwarp();
    }
    if (!p.do_pre) continue;

    // ----------------------------------- pre-order pass + gradient (b)+(c)
    {
      // the step's pre-partial is in slot Q: handed on in place by the
      // previous step (scale in qs_next) or staged from its scratch slot with
      // its exponent row; child 0 -> TC 0 + slot A (its edge message when
      // internal; a tip needs only its TC block and code); child 1 -> TC 1,
      // slot B
      // (CH) a cherry child's edge message: its table in the slot + its combined code
      auto issue = [&](const int4 d, int f, int handed) {
        if (d.x != root && handed != d.x) {
          stage_slot(sQ, Qw + size_t(d.x) * SD2);
          if (lane < 8) cp16_cg(sX + lane, Xb + size_t(d.x) * 32 + 4 * lane);
        }
        if (d.y <= N) {
          cn0 = code_ld(d.y);
        } else if (CH && (f & 1)) {
          cn0 = ccode_ld(d.y);
          if constexpr (WT) stage_cw(sA, d.y);
          else if constexpr (FUSE_TC) stage_cb(sA, d.y);
          else stage_ct(sA, d.y);
        } else {
          stage_slot_once(sA, Eb + size_t(d.y) * SD2);
        }
        if (d.z <= N) {
          cn1 = code_ld(d.z);
        } else if (CH && (f & 2)) {
          cn1 = ccode_ld(d.z);
          if constexpr (WT) stage_cw(sB, d.z);
          else if constexpr (FUSE_TC) stage_cb(sB, d.z);
          else stage_ct(sB, d.z);
        } else {
          stage_slot_once(sB, Eb + size_t(d.z) * SD2);
        }
        // (WT) a cherry child needs no P^T block
        if (!(WT && (f & 1))) stage_blk(sT0, p.tc, d.y);
        if (!(WT && (f & 2))) stage_blk(sT1, p.tc, d.z);
      };
      const char* base_e = reinterpret_cast<const char*>(p.escr + wbase * VEC);
      const int n = FUSE ? PS.npost : p.nsteps;  // (FUSE) the cherries' own steps are gone
      int4 win = lane < n ? p.pre[lane] : make_int4(0, 0, 0, 0);
      int4 winn = 32 + lane < n ? p.pre[32 + lane] : make_int4(0, 0, 0, 0);
      int4 d = shfl4(win, 0);
      int f = unflag(d);
      issue(d, f, 0);
      cp_commit();
      // the root's pre-partial is pi
#pragma unroll
      for (int j = 0; j < L; ++j) {
        sQ[lane + (2 * j) * 32] = make_double2(P4.pi[0], P4.pi[1]);
        sQ[lane + (2 * j + 1) * 32] = make_double2(P4.pi[2], P4.pi[3]);
      }
      double qs = 1.0, qs_next = 1.0;
      int handed = 0;
      for (int i = 0; i < n; ++i) {
        int4 dn = make_int4(0, 0, 0, 0);
        int fn = 0;
        if (i + 1 < n) {
          const int li = (i + 1) & 31;
          if (li == 0) {
            win = winn;
            winn = i + 33 + lane < n ? p.pre[i + 33 + lane] : make_int4(0, 0, 0, 0);
          }
          dn = shfl4(win, li);
          fn = unflag(dn);
        }
        cpa_wait_all();
        __syncwarp();
        if (d.x == root) qs = 1.0;
        else if (handed == d.x) qs = qs_next;
        else qs = qscale(reinterpret_cast<const int*>(sX)[lane]);
        const bool a_int = d.y > N, b_int = d.z > N;
        const bool a_ch = CH && (f & 1), b_ch = CH && (f & 2);
        const int code0 = cn0, code1 = cn1;
        // consumed scratch is dead: drop it from L2 without write-back
        if (lane < VEC / 16) {
          const char* base_q = reinterpret_cast<const char*>(p.qscr + wbase * VEC);
          if (a_int && !a_ch) discard_l2(base_e + size_t(d.y - N - 1) * (VEC * 8) + lane * 128);
          if (b_int && !b_ch) discard_l2(base_e + size_t(d.z - N - 1) * (VEC * 8) + lane * 128);
          if (d.x != root && handed != d.x) discard_l2(base_q + size_t(d.x - N - 1) * (VEC * 8) + lane * 128);
        }
        double den = 0.0, na = 0.0, nb = 0.0, na2 = 0.0, nb2 = 0.0;
        // (FUSE) a cherry child's tips u, v: gradient (and Hessian) numerators
        double cau = 0.0, cav = 0.0, cbu = 0.0, cbv = 0.0, cau2 = 0.0, cav2 = 0.0, cbu2 = 0.0, cbv2 = 0.0;
        const bool a_fuse = FUSE && a_ch, b_fuse = FUSE && b_ch;
        auto fused_tips = [&](const double2* blk, int code, int j, const double (&o)[4], double& nu, double& nv,
                              double& nu2, double& nv2) {
          double eu[4], ev[4];
          gather_cat(blk + 128, code >> 2, j, eu);
          gather_cat(blk + 160, code & 3, j, ev);
          double qu[4], qv[4], du = 0.0, dv = 0.0;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            double x = 0.0, y = 0.0;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              x = fma(P4.q[r * 4 + c], eu[c], x);
              y = fma(P4.q[r * 4 + c], ev[c], y);
            }
            qu[r] = x;
            qv[r] = y;
          }
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            du = fma(o[r] * ev[r], qu[r], du);
            dv = fma(o[r] * eu[r], qv[r], dv);
          }
          nu = fma(PS.crw[j], du, nu);
          nv = fma(PS.crw[j], dv, nv);
          if constexpr (HESS) {
            double du2 = 0.0, dv2 = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              double x = 0.0, y = 0.0;
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                x = fma(P4.q[r * 4 + c], qu[c], x);
                y = fma(P4.q[r * 4 + c], qv[c], y);
              }
              du2 = fma(o[r] * ev[r], x, du2);
              dv2 = fma(o[r] * eu[r], y, dv2);
            }
            nu2 = fma(PS.cr2w[j], du2, nu2);
            nv2 = fma(PS.cr2w[j], dv2, nv2);
          }
        };
        int ha = 0, hb = 0;
        double2* qa_dst = Qw + size_t(d.y) * SD2;  // lane offset included
        double2* qb_dst = Qw + size_t(d.z) * SD2;
#pragma unroll
        for (int j = 0; j < L; ++j) {
          double q[4], ea[4], eb[4];
          read_cat(sQ, j, q);
#pragma unroll
          for (int r = 0; r < 4; ++r) q[r] *= qs;
          if (a_ch) gather_ct(sA, code0, j, ea);
          else if (a_int) read_cat(sA, j, ea);
          else gather_cat(sT0, code0, j, ea);
          if (b_ch) gather_ct(sB, code1, j, eb);
          else if (b_int) read_cat(sB, j, eb);
          else gather_cat(sT1, code1, j, eb);
          double ta[4], tb[4], dd = 0.0;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            ta[r] = q[r] * eb[r];  // top for child a
            tb[r] = q[r] * ea[r];  // top for child b
            dd = fma(ta[r], ea[r], dd);
          }
          den = fma(PS.cw[j], dd, den);
          // gradient numerators top . (Q e) (engine.hpp:258-262): a 4x4
          // mat-vec with Q from the constant bank for tips too -- cheaper here
          // than gathering the tip's Q P column from shared memory (the
          // shared pipe, not the fp64 pipe, bounds this kernel: C3 131.3 vs
          // 132.8 ms with the gather)
          double qea[4], qeb[4];
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
          double d1a = 0.0, d1b = 0.0;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            d1a = fma(ta[r], qea[r], d1a);
            d1b = fma(tb[r], qeb[r], d1b);
          }
          na = fma(PS.crw[j], d1a, na);
          nb = fma(PS.crw[j], d1b, nb);
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
            na2 = fma(PS.cr2w[j], d2a, na2);
            nb2 = fma(PS.cr2w[j], d2b, nb2);
          }
          // outgoing pre-partials q_x = P_x^T top (engine.hpp:249-250),
          // unnormalised: the child visited next in place into slot Q (this
          // category's q was read above), the other to its scratch slot
          if (WT && a_ch) {
            double wu[4], wv[4];
            gather_ct(sA + 128, code0, j, wu);
            gather_ct(sA + 256, code0, j, wv);
            double du = 0.0, dv = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              du = fma(ta[r], wu[r], du);
              dv = fma(ta[r], wv[r], dv);
            }
            cau = fma(PS.crw[j], du, cau);
            cav = fma(PS.crw[j], dv, cav);
          } else if (a_int) {
            const double2* Tl = sT0 + j * NC * 2;
            double o[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const double2 u = Tl[2 * c], v = Tl[2 * c + 1];
              o[c] = fma(u.x, ta[0], fma(u.y, ta[1], fma(v.x, ta[2], v.y * ta[3])));
              ha = max(ha, __double2hiint(o[c]));
            }
            if (FUSE_TC && a_ch) fused_tips(sA, code0, j, o, cau, cav, cau2, cav2);
            else if (d.y == d.w) write_cat(sQ, j, o);
            else {
              __stcg(qa_dst + (2 * j) * 32, make_double2(o[0], o[1]));
              __stcg(qa_dst + (2 * j + 1) * 32, make_double2(o[2], o[3]));
            }
          }
          if (WT && b_ch) {
            double wu[4], wv[4];
            gather_ct(sB + 128, code1, j, wu);
            gather_ct(sB + 256, code1, j, wv);
            double du = 0.0, dv = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              du = fma(tb[r], wu[r], du);
              dv = fma(tb[r], wv[r], dv);
            }
            cbu = fma(PS.crw[j], du, cbu);
            cbv = fma(PS.crw[j], dv, cbv);
          } else if (b_int) {
            const double2* Tl = sT1 + j * NC * 2;
            double o[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const double2 u = Tl[2 * c], v = Tl[2 * c + 1];
              o[c] = fma(u.x, tb[0], fma(u.y, tb[1], fma(v.x, tb[2], v.y * tb[3])));
              hb = max(hb, __double2hiint(o[c]));
            }
            if (FUSE_TC && b_ch) fused_tips(sB, code1, j, o, cbu, cbv, cbu2, cbv2);
            else if (d.z == d.w) write_cat(sQ, j, o);
            else {
              __stcg(qb_dst + (2 * j) * 32, make_double2(o[0], o[1]));
              __stcg(qb_dst + (2 * j + 1) * 32, make_double2(o[2], o[3]));
            }
          }
        }
        // (FUSE) the fused tips' node ids (lane 0: u, lane 16: v) before the slots are refilled
        int ida = 0, idb = 0;
        if (a_fuse) ida = reinterpret_cast<const int*>(sA + kIdsAt)[lane >> 4];
        if (b_fuse) idb = reinterpret_cast<const int*>(sB + kIdsAt)[lane >> 4];
        __syncwarp();
        // the next step's operands (slots A, B, TC blocks; slot Q
        // unless its pre-partial was just handed on there)
        if (i + 1 < n) issue(dn, fn, d.w);
        cp_commit();
        const double inv = 1.0 / den;
        {
          const double r1a = na * inv, r1b = nb * inv;
          // both children's sums in one butterfly: lane 0 gets child a's, lane 16 child b's
          const double g2 = warp_sum2(valid ? w * r1a : 0.0, valid ? w * r1b : 0.0);
          if ((lane & 15) == 0) atomicAdd(A + (lane == 0 ? d.y : d.z), g2);
          if constexpr (HESS) {
            const double h2 = warp_sum2(valid ? w * (na2 * inv - r1a * r1a) : 0.0,
                                        valid ? w * (nb2 * inv - r1b * r1b) : 0.0);
            if ((lane & 15) == 0) atomicAdd(A + p.B + (lane == 0 ? d.y : d.z), h2);
          }
          if (a_fuse) {
            const double ru = cau * inv, rv = cav * inv;
            const double g3 = warp_sum2(valid ? w * ru : 0.0, valid ? w * rv : 0.0);
            if ((lane & 15) == 0) atomicAdd(A + ida, g3);
            if constexpr (HESS) {
              const double h3 = warp_sum2(valid ? w * (cau2 * inv - ru * ru) : 0.0, valid ? w * (cav2 * inv - rv * rv) : 0.0);
              if ((lane & 15) == 0) atomicAdd(A + p.B + ida, h3);
            }
          }
          if (b_fuse) {
            const double ru = cbu * inv, rv = cbv * inv;
            const double g3 = warp_sum2(valid ? w * ru : 0.0, valid ? w * rv : 0.0);
            if ((lane & 15) == 0) atomicAdd(A + idb, g3);
            if constexpr (HESS) {
              const double h3 = warp_sum2(valid ? w * (cbu2 * inv - ru * ru) : 0.0, valid ? w * (cbv2 * inv - rv * rv) : 0.0);
              if ((lane & 15) == 0) atomicAdd(A + p.B + idb, h3);
            }
          }
        }
        // normalisation exponents of the emitted pre-partials
        if (a_int && !a_fuse) {
          const int ex = peak_exponent(ha);
          if (d.y == d.w) qs_next = qscale(ex);
          else Xw[size_t(d.y) * 32] = ex;
        }
        if (b_int && !b_fuse) {
          const int ex = peak_exponent(hb);
          if (d.z == d.w) qs_next = qscale(ex);
          else Xw[size_t(d.z) * 32] = ex;
        }
        handed = d.w;
        d = dn;
        f = fn;
      }
      cpa_wait_all();
      __syncwarp();
    }
  }
}

}  // namespace pgk
