// K2 for large state spaces (m = 9..64: amino acids, codons) on the fp64
// tensor cores (mma.sync m8n8k4 f64 -> DMMA; tcgen05 has no f64 kind).
//
// Work unit: a CTA of WPC warps (8 patterns per warp) walks the tree in
// lock-step, one (node, rate category) at a time, so each P(t) block is
// staged once in shared memory and reused by all of the CTA's patterns.
// Every mat-vec  y^T = x^T M  over a warp's 8 patterns is a chain of DMMA
// tiles: A = x^T (8 patterns x 4 states), B = 4 x 8 slice of M, D = y^T.
// Vectors live in the A-fragment layout (pattern = lane/4, states 4k +
// lane%4).  K1 writes P, P^T and Q in exact B-fragment order with the output
// columns permuted (sigma(ni, g) = 4(2ni + g%2) + g/2) so that D tile ni holds
// A-layout entries 2ni and 2ni+1: chained mat-vecs need no shuffles, staging
// is a contiguous copy and shared-memory reads are conflict free.  With an
// odd number of k-steps (20 states: K = 5) the last D entry is padding and
// is dropped.
//
// Staging (MP <= 32): scratch is CTA-major, so each operand of the lock-step
// CTA — an internal child's edge-message slots, the parent's pre-partial
// slots, or a tip child's whole column table — is one 1-D bulk copy into
// shared memory, issued while the previous unit computes; a tip's Q P table
// goes into the P^T buffer the tip does not need.  MP = 64 (codons) has no
// room for staged operands next to its 32 KB matrix blocks and loads them
// at use.
//
// Scaling: categories are processed one at a time, so each (pattern,
// category) vector carries its own power-of-two exponent (stored in the tail
// of its scratch slot); mixtures over categories (root likelihood, gradient
// numerator/denominator) are combined with those exponents.  Post partials are
// normalised per category at every node (exact), pre partials when produced.
#pragma once

#include "pg_walk.cuh"

namespace pgk {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cpa8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
// D (8 patterns x 8 NT states) = x^T M over K k-steps, one accumulator chain
// per n-tile (NT independent chains in flight; the other resident warps cover
// the 26-cycle dependent-DMMA latency, profiles/dmma_latency_b200.jsonl).
// Codon-size tables store B fragments in pairs (frag_pos): one 16-byte load
// per two DMMAs.
// (measured and removed: an even/odd k-step accumulator split, C4 176 vs 179 ms)
template <int K, int NT, bool GLOBAL>
__device__ __forceinline__ void dmma_chain(const double (&x)[K], double (&d)[NT][2], const double* frag, int lane) {
  constexpr int F = K * NT;
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) d[ni][0] = d[ni][1] = 0.0;
  if constexpr (F < kFragPairMin) {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      const double* fp = frag + f * 32 + lane;
      dmma(d[f % NT][0], d[f % NT][1], x[f / NT], GLOBAL ? __ldg(fp) : *fp);
    }
    return;
  }
  const double2* f2 = reinterpret_cast<const double2*>(frag) + lane;
#pragma unroll
  for (int h = 0; h < F / 2; ++h) {
    const double2 b = GLOBAL ? __ldg(f2 + h * 32) : f2[h * 32];
    const int f0 = 2 * h, f1 = 2 * h + 1;
    dmma(d[f0 % NT][0], d[f0 % NT][1], x[f0 / NT], b.x);
    dmma(d[f1 % NT][0], d[f1 % NT][1], x[f1 / NT], b.y);
  }
  if constexpr (F & 1) {
    const double* f1p = frag + (F / 2) * 64 + lane;
    const double b = GLOBAL ? __ldg(f1p) : *f1p;
    dmma(d[(F - 1) % NT][0], d[(F - 1) % NT][1], x[(F - 1) / NT], b);
  }
}

// Resident CTAs per SM for MP <= 32: 4 caps registers at 128 (C4: 204 ms vs
// 211 ms at 3 CTAs / 168 registers).
#ifndef PG_WALKM_MINB_SMALL
#define PG_WALKM_MINB_SMALL 4
#endif
#ifndef PG_WALKM_WPC_SMALL
#define PG_WALKM_WPC_SMALL 4
#endif

#ifndef PG_WALKM_WPC_LARGE
#define PG_WALKM_WPC_LARGE 4
#endif

template <int MP>
struct WalkMGeom {
  static_assert(MP % 4 == 0, "MP: whole k-steps");
  static constexpr int K = MP / 4;         // k-steps (A fragments per vector per lane)
  static constexpr int NT = (K + 1) / 2;   // n-tiles (D fragments per vector per lane); odd K drops
                                           // the last D entry (padded output columns)
  static constexpr int FRAG = K * NT * 32;  // doubles of one matrix in B-fragment order
  // small state spaces double-buffer the P(t) blocks across units and stage
  // the next unit's operands in shared memory (SOP)
  static constexpr bool PIPE = MP <= 32;
  static constexpr int NPB = PIPE ? 4 : 2;
  static constexpr bool SOP = PIPE;
  // warps per CTA (lock-step group sharing each staged matrix).  Measured on
  // C5: 8 warps with double-buffered 32 KB codon blocks (one CTA per SM) is
  // slower than two 4-warp CTAs (432 vs 423 ms).
  static constexpr int WPC = MP <= 32 ? PG_WALKM_WPC_SMALL : PG_WALKM_WPC_LARGE;
  // one (node, category) scratch slot: K x 32 doubles of the warp's 8 vectors
  // followed by their 8 int exponents (one bulk copy moves both)
  static constexpr int SL = K * 32 + 4;
  // per warp: 2 stages x 3 operand slots
  static constexpr int SOPD = SOP ? 6 * SL : 0;
  // P(t) blocks (two children of a pre-order step, x2 parities if PIPE) + Q
  // + SOP + two mbarriers (one per buffer parity) for the bulk copies
  // + two mbarriers, pi (MP) and up to kSmemCats category weights and rates
  static constexpr int kSmemCats = 16;
  static constexpr size_t smem_bytes() {
    return size_t((NPB + 1) * FRAG + WPC * SOPD + 2 + MP + 2 * kSmemCats) * sizeof(double);
  }
};

// HESS: Hessian-diagonal variant (a template parameter so the gradient-only
// kernel does not carry the Q^2 e terms in its register allocation)
// FAST: the launch-invariant switches of the common case folded at compile
// time -- one shared generator, rescaling on, L = 4 categories (weights and
// rates in shared memory), operands and tip tables staged (the host checks
// walkm_fast_ok) -- so the unit body carries no branches or index
// multiplications for them
template <int MP, bool HESS, bool FAST>
__global__ void __launch_bounds__(32 * WalkMGeom<MP>::WPC, (MP <= 32 ? PG_WALKM_MINB_SMALL : 2)) walkm_kernel(const __grid_constant__ WalkMParams PM) {
  using Gm = WalkMGeom<MP>;
  constexpr int K = Gm::K, NT = Gm::NT, FRAG = Gm::FRAG;
  // lane 0 of the last warp issues the P-block copies (warps 0..2 issue the
  // staged operand slots), spreading the copy issue over the CTA's warps
  constexpr int kPIssuer = 32 * (Gm::WPC - 1);
  // (measured and removed: register prefetch of the next unit's operands,
  // interleaved mat-vecs of the two children -- both cost registers at the
  // 128-register cap of 4 CTAs per SM)
  const WalkParams& p = PM.p;
  constexpr bool PIPE = Gm::PIPE;
  constexpr bool DESC2 = MP > 32;  // step descriptors two ahead (see below)
  extern __shared__ __align__(16) double smd[];
  auto pbuf = [&](int slot, int par) -> double* { return smd + size_t(PIPE ? slot * 2 + par : slot) * FRAG; };
  double* Qsm = smd + size_t(Gm::NPB) * FRAG;  // homogeneous generator in B-fragment order
  // staged operands of the whole CTA: [stage][operand][warp][slot]
  double* sop_cta = smd + size_t(Gm::NPB + 1) * FRAG;
  // P blocks and operand slots are staged with 1-D bulk copies (TMA engine)
  // that complete on these mbarriers
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smd + size_t(Gm::NPB + 1) * FRAG + size_t(Gm::WPC) * Gm::SOPD);
  if (threadIdx.x == 0) {
    mbar_init(mbar, Gm::WPC + 1);  // lane 0 of every warp + the P-block issuer
    mbar_init(mbar + 1, Gm::WPC + 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned txP = 0, txW = 0, mphase = 0;  // pending transaction bytes; parity bit per buffer
  // all staging for a buffer is issued: arm its mbarrier with the bytes
  auto stage_done = [&](int sb) {
    if ((threadIdx.x & 31) == 0) mbar_arrive_tx(mbar + sb, txW);
    if (threadIdx.x == kPIssuer) mbar_arrive_tx(mbar + sb, txP);
    txP = txW = 0;
  };
  // wait for a buffer's bulk copies (and every thread's cp.async), then the
  // CTA barrier (cross-thread visibility, and no one still reads the other buffer)
  auto stage_wait = [&](int sb) {
    // this thread's earlier scratch stores (generic proxy) must be ordered
    // before the bulk copies (async proxy) that other threads issue after the
    // barrier below and that may read them
    fence_proxy_async_global();
    cpa_wait_all();
    if constexpr (Gm::PIPE) {
      mbar_wait(mbar + sb, (mphase >> sb) & 1u);
      mphase ^= 1u << sb;
    }
    __syncthreads();
  };
  // unbuffered (large MP): the current unit's blocks are staged after the
  // unit-top barrier and awaited here, right before their first use
  auto unit_blocks_wait = [&]() {
    mbar_wait(mbar, mphase & 1u);
    mphase ^= 1u;
  };
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  const int q = lane >> 2, t = lane & 3;  // pattern within the warp, state phase
  const int N = p.N, L = FAST ? 4 : p.L, root = 2 * N - 1, NC = p.NC;
  const bool rescale = FAST || !p.disable;
  constexpr int WPC = Gm::WPC, CT = 32 * WPC;  // warps / threads per CTA
  const int warp = blockIdx.x * WPC + wib;
  const int ntile_cta = (p.P + 8 * WPC - 1) / (8 * WPC);
  // 32-bit element offsets inside the per-warp scratch and the K1 tables
  // (the host guarantees they fit) keep the index math to one IMAD.WIDE
  constexpr int SL = Gm::SL;
  // CTA-major scratch: [CTA][node][category][warp][slot], so one (node,
  // category) operand of the whole lock-step CTA is one contiguous bulk copy
  const int slotd = L * WPC * SL;  // doubles per node of the CTA
  double* E = p.escr + size_t(blockIdx.x) * size_t(N - 1) * slotd;
  double* Qs = p.qscr + size_t(blockIdx.x) * size_t(N - 1) * slotd;
  double* Acc = p.acc + size_t(warp) * p.accw;
  for (int i = lane; i < p.accw; i += 32) Acc[i] = 0.0;
  __syncwarp();

  // stage one (node, category) matrix in B-fragment order (contiguous copy)
  auto stage_P = [&](double* buf, const double* tab, int node, int l, int sb) {
    if (tid == kPIssuer) {
      bulk_g2s(buf, tab + ((node - 1) * L + l) * FRAG, FRAG * sizeof(double), mbar + sb);
      txP += FRAG * sizeof(double);
    }
  };
  // y = M x over the warp's 8 patterns: B fragment (ki, ni) for this lane is
  // frag[frag_pos(ki * NT + ni, lane, K * NT)]; with the permuted columns baked into the
  // fragment tables, D tile ni holds y's A-layout entries 2ni and 2ni+1.
  auto matvec = [&](const double* frag, const double (&x)[K], double (&y)[K]) {
    double d[NT][2];
    dmma_chain<K, NT, false>(x, d, frag, lane);
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      y[2 * ni] = d[ni][0];
      if (2 * ni + 1 < K) y[2 * ni + 1] = d[ni][1];
    }
  };
  auto matvec_g = [&](const double* frag, const double (&x)[K], double (&y)[K]) {
    double d[NT][2];
    dmma_chain<K, NT, true>(x, d, frag, lane);
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      y[2 * ni] = d[ni][0];
      if (2 * ni + 1 < K) y[2 * ni + 1] = d[ni][1];
    }
  };
  auto unpack = [&](double (&d)[NT][2], double (&y)[K]) {
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      y[2 * ni] = d[ni][0];
      if (2 * ni + 1 < K) y[2 * ni + 1] = d[ni][1];
    }
  };
  auto matvec_P = [&](const double* buf, const double (&x)[K], double (&y)[K]) { matvec(buf, x, y); };
  auto matvec_PT = [&](const double* buf, const double (&x)[K], double (&y)[K]) { matvec(buf, x, y); };
  // homogeneous Q staged in smem; per-branch generators read in fragment order from global
  const bool homog = FAST || PM.homogeneous != 0;
  // y = Q_x x for the generator of node x's branch (shared generator staged
  // in shared memory; per-branch ones in fragment order from global)
  auto matvec_Q = [&](int x_node, const double (&x)[K], double (&y)[K]) {
    if (homog) matvec(Qsm, x, y);
    else matvec_g(PM.fq + size_t(p.qidx[x_node]) * FRAG, x, y);
  };
  auto quad_sum = [&](double v) {
    v += __shfl_xor_sync(kFull, v, 1);
    v += __shfl_xor_sync(kFull, v, 2);
    return v;
  };
  // exponent of the per-pattern peak (quad reduction) of K non-negative values
  auto quad_peak_exp = [&](const double (&v)[K]) {
    int h = 0;
#pragma unroll
    for (int ki = 0; ki < K; ++ki) h = max(h, __double2hiint(v[ki]));
    h = max(h, __shfl_xor_sync(kFull, h, 1));
    h = max(h, __shfl_xor_sync(kFull, h, 2));
    const int bexp = (h >> 20) & 0x7ff;
    if (h <= 0 || bexp == 0x7ff || bexp == 0) return 0;
    return bexp - 1022;
  };
  auto scale_by = [&](double (&v)[K], int ex) {
    if (ex == 0) return;
    if (ex > -1021 && ex < 1022) {
      const double sc = __hiloint2double((1023 - ex) << 20, 0);
#pragma unroll
      for (int ki = 0; ki < K; ++ki) v[ki] *= sc;
    } else {
#pragma unroll
      for (int ki = 0; ki < K; ++ki) v[ki] = ldexp(v[ki], -ex);
    }
  };
  // 2^e for e <= 0 (exact down to the subnormal range; 0 below)
  auto pow2 = [](int e) -> double {
    if (e >= -1022) return __hiloint2double((1023 + e) << 20, 0);
    return e >= -1074 ? ldexp(1.0, e) : 0.0;
  };
  // running mixture over categories with exponents: value = acc * 2^ref
  constexpr int NR = HESS ? 5 : 3;  // mixture terms: den, num_a, num_b (, num2_a, num2_b)
  struct Mix {
    double v[NR];
    int ref;
  };

  // pi and the category weights / rates in shared memory (read every unit)
  double* pism = reinterpret_cast<double*>(mbar + 2);
  double* probsm = pism + MP;
  double* ratesm = probsm + Gm::kSmemCats;
  const bool cats_sm = FAST || p.L <= Gm::kSmemCats;
  for (int i = tid; i < MP; i += CT) pism[i] = p.pi[i];
  if (cats_sm)
    for (int i = tid; i < p.L; i += CT) {
      probsm[i] = p.probs[i];
      ratesm[i] = p.rates[i];
    }
  if (homog)
    for (int i = tid; i < FRAG; i += CT) Qsm[i] = PM.fq[i];
  __syncthreads();

  for (int tile = blockIdx.x; tile < ntile_cta; tile += gridDim.x) {
    const int s = tile * (8 * WPC) + wib * 8 + q;
    const bool valid = s < p.P;
    const bool owner = valid && t == 0;
    const int sc = valid ? s : p.P - 1;
    const double w = valid ? p.weights[sc] : 0.0;
    const uint8_t* codes = p.codes + sc;
    const int Pc = int(p.Pc);
    const int n = p.nsteps, U = n * L;
    const bool sop = Gm::SOP && (FAST || L > 1);

    // slot layout: [category][k-step pair][lane] double2 (512 B per warp access),
    // an odd last k-step as [lane] double, then the 8 patterns' exponents
    auto slot_ptr = [&](const double* base, int node, int l) {
      return reinterpret_cast<const double2*>(base + ((node - N - 1) * slotd + (l * WPC + wib) * SL)) + lane;
    };
    auto xslot = [&](double* base, int node, int l) -> int* {
      return reinterpret_cast<int*>(base + ((node - N - 1) * slotd + (l * WPC + wib) * SL + K * 32)) + q;
    };
    auto load_slot = [&](const double* base, int node, int l, double (&v)[K]) {
      const double2* src = slot_ptr(base, node, l);
#pragma unroll
      for (int kp = 0; kp < K / 2; ++kp) {
        const double2 d = __ldcg(src + kp * 32);
        v[2 * kp] = d.x;
        v[2 * kp + 1] = d.y;
      }
      if constexpr (K & 1) v[K - 1] = __ldcg(reinterpret_cast<const double*>(src - lane + (K / 2) * 32) + lane);
    };
    auto store_slot = [&](double* base, int node, int l, const double (&v)[K]) {
      double2* dst = const_cast<double2*>(slot_ptr(base, node, l));
#pragma unroll
      for (int kp = 0; kp < K / 2; ++kp) __stcg(dst + kp * 32, make_double2(v[2 * kp], v[2 * kp + 1]));
      if constexpr (K & 1) __stcg(reinterpret_cast<double*>(dst - lane + (K / 2) * 32) + lane, v[K - 1]);
    };
    // ---- staged operands (SOP): the next unit's operands are copied into the
    // CTA's shared stage (bulk copies of slots and tip column tables; per-lane
    // cp.async gathers when a table does not fit) while this unit computes
    auto opbuf = [&](int stage, int which) -> double* { return sop_cta + ((stage * 3 + which) * WPC + wib) * SL; };
    auto xpbuf = [&](int stage, int which) -> int* { return reinterpret_cast<int*>(opbuf(stage, which) + K * 32); };
    // the CTA's slots of one operand (WPC x (K x 32 doubles + 8 exponents)):
    // one bulk copy, issued by lane 0 of warp `which` (operands spread over warps)
    auto stage_slot_op = [&](int stage, int which, const double* base, int node, int l) {
      if (lane == 0 && wib == which % WPC) {
        bulk_g2s(sop_cta + (stage * 3 + which) * WPC * SL, base + ((node - N - 1) * slotd + l * WPC * SL),
                 WPC * SL * sizeof(double), mbar + stage);
        txW += WPC * SL * sizeof(double);
      }
    };
    // a tip operand: the child's whole column table (NC x MP) is one bulk copy
    // into the operand's CTA region when it fits (each lane then reads its
    // pattern's column); otherwise per-lane 8-byte gathers of the column
    const bool tstage = Gm::SOP && (FAST || NC * MP <= WPC * SL);
    auto opblk = [&](int stage, int which) -> double* { return sop_cta + (stage * 3 + which) * WPC * SL; };
    auto stage_gather_op = [&](int stage, int which, int node, int code, int l) {
      if (tstage) {
        if (lane == 0 && wib == which % WPC) {
          bulk_g2s(opblk(stage, which), p.tc + size_t((node - 1) * L + l) * (NC * MP), NC * MP * sizeof(double),
                   mbar + stage);
          txW += NC * MP * sizeof(double);
        }
        return;
      }
      const double* col = p.tc + (((node - 1) * L + l) * NC + code) * MP + t;
      double* dst = opbuf(stage, which);
#pragma unroll
      for (int ki = 0; ki < K; ++ki)
        cpa8(dst + (ki < 2 * (K / 2) ? ((ki >> 1) * 32 + lane) * 2 + (ki & 1) : (K / 2) * 64 + lane), col + ki * 4);
      if (t == 0) xpbuf(stage, which)[q] = 0;
    };
    auto read_op = [&](int stage, int which, double (&v)[K], int& x) {
      const double2* src = reinterpret_cast<const double2*>(opbuf(stage, which)) + lane;
#pragma unroll
      for (int kp = 0; kp < K / 2; ++kp) {
        const double2 d = src[kp * 32];
        v[2 * kp] = d.x;
        v[2 * kp + 1] = d.y;
      }
      if constexpr (K & 1) v[K - 1] = reinterpret_cast<const double*>(src - lane + (K / 2) * 32)[lane];
      x = xpbuf(stage, which)[q];
    };
    auto read_tip = [&](int stage, int which, int code, double (&v)[K], int& x) {
      const double* col = opblk(stage, which) + code * MP + t;
#pragma unroll
      for (int ki = 0; ki < K; ++ki) v[ki] = col[ki * 4];
      x = 0;
    };
    auto gather = [&](int node, int code, int l, double (&v)[K]) {
      const double* col = p.tc + (((node - 1) * L + l) * NC + code) * MP + t;
#pragma unroll
      for (int ki = 0; ki < K; ++ki) v[ki] = __ldg(col + ki * 4);
    };
    // Q e of a tip = the same column of Q P (built by K1): a gather, not a mat-vec
    auto gather_q = [&](int node, int code, int l, double (&v)[K]) {
      const double* col = p.qtc + (((node - 1) * L + l) * NC + code) * MP + t;
#pragma unroll
      for (int ki = 0; ki < K; ++ki) v[ki] = __ldg(col + ki * 4);
    };
    auto tipcode = [&](int node) -> int { return node <= N ? int(codes[int64_t(node - 1) * Pc]) : 0; };

    // ------------------------------------------------ post-order pass (a)
    // Units (step i, category l) in lock-step.  PIPE: the next unit's P(t)
    // block (and, with SOP, its operands) is staged into the other buffer
    // parity while this unit computes.
    {
      auto load_post = [&](const int4 st, int c0, int c1, int l, double (&a)[K], double (&b)[K], int& xa, int& xb) {
        xa = xb = 0;
        if (st.y <= N) gather(st.y, c0, l, a);
        else {
          load_slot(E, st.y, l, a);
          xa = *xslot(E, st.y, l);
        }
        if (st.z <= N) gather(st.z, c1, l, b);
        else {
          load_slot(E, st.z, l, b);
          xb = *xslot(E, st.z, l);
        }
      };
      int4 stc = p.post[0];
      int4 stn = n > 1 ? p.post[1] : stc;
      // large MP: descriptors run two steps ahead (no load-use stall at the
      // step boundary; measured C5 412 -> 405 ms); small MP keeps the
      // registers (C4 at the 128-register cap: 203 vs 213 ms)
      int4 stn2 = DESC2 && n > 2 ? p.post[2] : stn;
      int cc0 = tipcode(stc.y), cc1 = tipcode(stc.z);
      int cn0 = tipcode(stn.y), cn1 = tipcode(stn.z);
      auto stage_post_ops = [&](const int4 st, int c0, int c1, int l, int stage) {
        if (st.y <= N) stage_gather_op(stage, 0, st.y, c0, l);
        else stage_slot_op(stage, 0, E, st.y, l);
        if (st.z <= N) stage_gather_op(stage, 1, st.z, c1, l);
        else stage_slot_op(stage, 1, E, st.z, l);
      };
      if (PIPE && stc.x != root) stage_P(pbuf(0, 0), PM.fpp, stc.x, 0, 0);
      if (sop) stage_post_ops(stc, cc0, cc1, 0, 0);
      if (PIPE) stage_done(0);
      cpa_commit();
      Mix mix{{}, INT_MIN};
      int i = 0, l = 0;
      for (int u = 0; u < U; ++u) {
        const int par = PIPE ? (u & 1) : 0;
        stage_wait(par);
        int l2 = l + 1;
        const bool step_end = l2 == L;
        if (step_end) l2 = 0;
        const bool has_next = u + 1 < U;
        const int4 st2 = step_end ? stn : stc;
        if (PIPE) {
          if (has_next) {
            if (st2.x != root) stage_P(pbuf(0, (u + 1) & 1), PM.fpp, st2.x, l2, (u + 1) & 1);
            if (sop) stage_post_ops(st2, step_end ? cn0 : cc0, step_end ? cn1 : cc1, l2, (u + 1) & 1);
            stage_done((u + 1) & 1);
          }
        } else if (stc.x != root) {
          stage_P(pbuf(0, 0), PM.fpp, stc.x, l, 0);
          stage_done(0);  // awaited below (non-root units only)
        }
        cpa_commit();
        double a[K], b[K];
        int xa = 0, xb = 0;
        if (sop) {
          if (tstage && stc.y <= N) read_tip(u & 1, 0, cc0, a, xa);
          else read_op(u & 1, 0, a, xa);
          if (tstage && stc.z <= N) read_tip(u & 1, 1, cc1, b, xb);
          else read_op(u & 1, 1, b, xb);
        } else {
          load_post(stc, cc0, cc1, l, a, b, xa, xb);
        }
#pragma unroll
        for (int ki = 0; ki < K; ++ki) a[ki] *= b[ki];
        const int ex = rescale ? quad_peak_exp(a) : 0;
        scale_by(a, ex);
        const int Sk = xa + xb + ex;
        if (stc.x == root) {
          double d = 0.0;
#pragma unroll
          for (int ki = 0; ki < K; ++ki) d = fma(pism[ki * 4 + t], a[ki], d);
          d = quad_sum(d) * (cats_sm ? probsm[l] : p.probs[l]);
          if (Sk > mix.ref) {
            mix.v[0] = mix.ref == INT_MIN ? 0.0 : mix.v[0] * pow2(mix.ref - Sk);
            mix.ref = Sk;
          }
          mix.v[0] += d * pow2(Sk - mix.ref);
          if (step_end) {
            const double m = mix.v[0];
            const double ll = log(m) + double(mix.ref) * 0.6931471805599453;
            if (owner) {
              if (!isfinite(m)) atomicMin(&p.err[0], s);
              else if (m <= 0.0) atomicMin(&p.err[1], s);
              if (p.site_ll) p.site_ll[s] = ll;
            }
            const double v = warp_sum(owner ? w * ll : 0.0);
            if (lane == 0) atomicAdd(Acc, v);
          }
        } else {
          if (!PIPE) unit_blocks_wait();
          double e[K];
          matvec_P(pbuf(0, par), a, e);
          store_slot(E, stc.x, l, e);
          if (t == 0) *xslot(E, stc.x, l) = Sk;
        }
        l = l2;
        if (step_end) {
          ++i;
          mix = Mix{{}, INT_MIN};
          stc = stn;
          cc0 = cn0;
          cc1 = cn1;
          if (i + 1 < n) {
            stn = DESC2 ? stn2 : p.post[i + 1];
            cn0 = tipcode(stn.y);
            cn1 = tipcode(stn.z);
            if (DESC2 && i + 2 < n) stn2 = p.post[i + 2];
          }
        }
      }
    }
    if (!p.do_pre) continue;

    // ----------------------------------- pre-order pass + gradient (b)+(c)
    {
      auto load_pre = [&](const int4 st, int c0, int c1, int l, double (&qv)[K], double (&ea)[K], double (&eb)[K],
                          int& xq, int& xa, int& xb) {
        xq = xa = xb = 0;
        if (st.x == root) {
#pragma unroll
          for (int ki = 0; ki < K; ++ki) qv[ki] = pism[ki * 4 + t];
        } else {
          load_slot(Qs, st.x, l, qv);
          xq = *xslot(Qs, st.x, l);
        }
        if (st.y > N) {
          load_slot(E, st.y, l, ea);
          xa = *xslot(E, st.y, l);
        } else gather(st.y, c0, l, ea);
        if (st.z > N) {
          load_slot(E, st.z, l, eb);
          xb = *xslot(E, st.z, l);
        } else gather(st.z, c1, l, eb);
      };
      // a tip child has no outgoing pre-partial, so its P^T buffer instead
      // receives the child's Q P column table (NC x MP) when it fits: the
      // tip's Q e is then a shared-memory read instead of a dependent global
      // gather in the middle of the unit
      const bool qstage = PIPE && (FAST || NC * MP <= FRAG);
      auto stage_qtc = [&](double* buf, int node, int l, int sb) {
        if (tid == kPIssuer) {
          bulk_g2s(buf, p.qtc + size_t((node - 1) * L + l) * (NC * MP), NC * MP * sizeof(double), mbar + sb);
          txP += NC * MP * sizeof(double);
        }
      };
      auto stage_pre = [&](const int4 st, int l, int par) {
        if (st.y > N) stage_P(pbuf(0, par), PM.fpt, st.y, l, par);
        else if (qstage) stage_qtc(pbuf(0, par), st.y, l, par);
        if (st.z > N) stage_P(pbuf(1, par), PM.fpt, st.z, l, par);
        else if (qstage) stage_qtc(pbuf(1, par), st.z, l, par);
      };
      auto staged_q = [&](const double* buf, int code, double (&v)[K]) {
        const double* col = buf + code * MP + t;
#pragma unroll
        for (int ki = 0; ki < K; ++ki) v[ki] = col[ki * 4];
      };
      int4 stc = p.pre[0];
      int4 stn = n > 1 ? p.pre[1] : stc;
      // large MP: descriptors run two steps ahead (no load-use stall at the
      // step boundary; measured C5 412 -> 405 ms); small MP keeps the
      // registers (C4 at the 128-register cap: 203 vs 213 ms)
      int4 stn2 = DESC2 && n > 2 ? p.pre[2] : stn;
      int cc0 = tipcode(stc.y), cc1 = tipcode(stc.z);
      int cn0 = tipcode(stn.y), cn1 = tipcode(stn.z);
      auto stage_pre_ops = [&](const int4 st, int c0, int c1, int l, int stage) {
        if (st.x != root) stage_slot_op(stage, 2, Qs, st.x, l);
        if (st.y > N) stage_slot_op(stage, 0, E, st.y, l);
        else stage_gather_op(stage, 0, st.y, c0, l);
        if (st.z > N) stage_slot_op(stage, 1, E, st.z, l);
        else stage_gather_op(stage, 1, st.z, c1, l);
      };
      if (PIPE) stage_pre(stc, 0, 0);
      if (sop) stage_pre_ops(stc, cc0, cc1, 0, 0);
      if (PIPE) stage_done(0);
      cpa_commit();
      // mixtures: [0] den, [1] num_a, [2] num_b, [3] num2_a, [4] num2_b
      Mix mix{{}, INT_MIN};
      int i = 0, l = 0;
      for (int u = 0; u < U; ++u) {
        const int par = PIPE ? (u & 1) : 0;
        const int ca = stc.y, cb = stc.z;
        const bool a_int = ca > N, b_int = cb > N;
        stage_wait(par);
        int l2 = l + 1;
        const bool step_end = l2 == L;
        if (step_end) l2 = 0;
        const bool has_next = u + 1 < U;
        const int4 st2 = step_end ? stn : stc;
        if (PIPE) {
          if (has_next) {
            stage_pre(st2, l2, (u + 1) & 1);
            if (sop) stage_pre_ops(st2, step_end ? cn0 : cc0, step_end ? cn1 : cc1, l2, (u + 1) & 1);
            stage_done((u + 1) & 1);
          }
        } else {
          stage_pre(stc, l, 0);
          stage_done(0);
        }
        cpa_commit();
        double qv[K], ea[K], eb[K];
        int xq = 0, xa = 0, xb = 0;
        if (sop) {
          if (stc.x == root) {
#pragma unroll
            for (int ki = 0; ki < K; ++ki) qv[ki] = pism[ki * 4 + t];
          } else {
            read_op(u & 1, 2, qv, xq);
          }
          if (tstage && !a_int) read_tip(u & 1, 0, cc0, ea, xa);
          else read_op(u & 1, 0, ea, xa);
          if (tstage && !b_int) read_tip(u & 1, 1, cc1, eb, xb);
          else read_op(u & 1, 1, eb, xb);
        } else {
          load_pre(stc, cc0, cc1, l, qv, ea, eb, xq, xa, xb);
        }
        const int El = xq + xa + xb;
        double ta[K], tb[K], dd = 0.0;
#pragma unroll
        for (int ki = 0; ki < K; ++ki) {
          ta[ki] = qv[ki] * eb[ki];
          tb[ki] = qv[ki] * ea[ki];
          dd = fma(ta[ki], ea[ki], dd);
        }
        const double wl = cats_sm ? probsm[l] : p.probs[l], cl = cats_sm ? ratesm[l] : p.rates[l];
        double term[NR];
        term[0] = wl * quad_sum(dd);
        {
          double ua[K], ub[K];
          if (a_int) matvec_Q(ca, ea, ua);
          else if (qstage) staged_q(pbuf(0, par), cc0, ua);
          else gather_q(ca, cc0, l, ua);
          if (b_int) matvec_Q(cb, eb, ub);
          else if (qstage) staged_q(pbuf(1, par), cc1, ub);
          else gather_q(cb, cc1, l, ub);
          double d1a = 0.0, d1b = 0.0;
#pragma unroll
          for (int ki = 0; ki < K; ++ki) {
            d1a = fma(ta[ki], ua[ki], d1a);
            d1b = fma(tb[ki], ub[ki], d1b);
          }
          term[1] = cl * wl * quad_sum(d1a);
          term[2] = cl * wl * quad_sum(d1b);
          if constexpr (HESS) {
            double u2a[K], u2b[K];
            matvec_Q(ca, ua, u2a);
            matvec_Q(cb, ub, u2b);
            double d2a = 0.0, d2b = 0.0;
#pragma unroll
            for (int ki = 0; ki < K; ++ki) {
              d2a = fma(ta[ki], u2a[ki], d2a);
              d2b = fma(tb[ki], u2b[ki], d2b);
            }
            term[3] = cl * cl * wl * quad_sum(d2a);
            term[4] = cl * cl * wl * quad_sum(d2b);
          }
        }
        if (El > mix.ref) {
          if (mix.ref != INT_MIN) {
            const double down = pow2(mix.ref - El);
            for (int r = 0; r < NR; ++r) mix.v[r] *= down;
          }
          mix.ref = El;
        }
        const double scl = pow2(El - mix.ref);
        for (int r = 0; r < NR; ++r) mix.v[r] = fma(term[r], scl, mix.v[r]);
        // outgoing pre-partials of internal children: q_x = P_x^T top
        if (!PIPE) unit_blocks_wait();
        auto emit_q = [&](int x, double (&qo)[K], int xbase) {
          const int ex = quad_peak_exp(qo);
          scale_by(qo, ex);
          store_slot(Qs, x, l, qo);
          if (t == 0) *xslot(Qs, x, l) = xbase + ex;
        };
        if (a_int) {
          double qo[K];
          matvec_PT(pbuf(0, par), ta, qo);
          emit_q(ca, qo, xq + xb);
        }
        if (b_int) {
          double qo[K];
          matvec_PT(pbuf(1, par), tb, qo);
          emit_q(cb, qo, xq + xa);
        }
        if (step_end) {
          const double inv = 1.0 / mix.v[0];
          const double r1a = mix.v[1] * inv, r1b = mix.v[2] * inv;
          const double ga = warp_sum(owner ? w * r1a : 0.0);
          const double gb = warp_sum(owner ? w * r1b : 0.0);
          if (lane == 0) {
            atomicAdd(Acc + ca, ga);
            atomicAdd(Acc + cb, gb);
          }
          if constexpr (HESS) {
            const double ha = warp_sum(owner ? w * (mix.v[3] * inv - r1a * r1a) : 0.0);
            const double hb = warp_sum(owner ? w * (mix.v[4] * inv - r1b * r1b) : 0.0);
            if (lane == 0) {
              atomicAdd(Acc + p.B + ca, ha);
              atomicAdd(Acc + p.B + cb, hb);
            }
          }
          ++i;
          mix = Mix{{}, INT_MIN};
          stc = stn;
          cc0 = cn0;
          cc1 = cn1;
          if (i + 1 < n) {
            stn = DESC2 ? stn2 : p.pre[i + 1];
            cn0 = tipcode(stn.y);
            cn1 = tipcode(stn.z);
            if (DESC2 && i + 2 < n) stn2 = p.pre[i + 2];
          }
        }
        l = l2;
      }
    }
  }
}

}  // namespace pgk
