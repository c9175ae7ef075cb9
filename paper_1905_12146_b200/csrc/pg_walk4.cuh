// K2 specialised for 4-state models with 3-4 rate categories (the HBM-bound
// C2/C3 path): one lane = one pattern with all categories (16 fp64 per
// vector), 32 patterns per warp tile, persistent warps.
//
// Differences from the generic walk_kernel (pg_walk.cuh):
//  * software pipeline: while step i computes, step i+1's memory operands
//    (edge-message / pre-partial slots, the TC blocks of the nodes involved)
//    are already in flight into a per-warp shared-memory stage via cp.async,
//    and its tip codes via plain loads — the per-step dependent-load chain of
//    the generic kernel disappears from the critical path;
//  * the homogeneous generator Q and pi live in the kernel-parameter
//    (constant) bank;
//  * per-pattern normalisation uses the integer max of the high words
//    (exponent only), one IMNMX per element instead of a DSETP/SEL triple;
//  * gradient contributions go to the warp's accumulator row with RED
//    (fire-and-forget, single writer per address -> deterministic).
#pragma once

#include "pg_walk.cuh"

namespace pgk {

struct Walk4Params {
  WalkParams p;
  double q[16];  // homogeneous generator (row-major)
  double pi[4];
  int homogeneous;
};

__device__ __forceinline__ void cp16_cg(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp16_ca(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Exponent-only normalisation of non-negative values: brings the per-pattern
// peak into [0.5, 1) by an exact power of two; returns the exponent removed.
template <int LC, int MP>
__device__ __forceinline__ int normalize_hi(double (&v)[LC][MP]) {
  int h = 0;
#pragma unroll
  for (int j = 0; j < LC; ++j)
#pragma unroll
    for (int i = 0; i < MP; ++i) h = max(h, __double2hiint(v[j][i]));
  const int bexp = (h >> 20) & 0x7ff;
  if (h <= 0 || bexp == 0x7ff) return 0;  // all zero (or subnormal-only), inf, NaN
  if (bexp == 0) {                        // subnormal peak: exact slow path
    double pk = 0.0;
#pragma unroll
    for (int j = 0; j < LC; ++j)
#pragma unroll
      for (int i = 0; i < MP; ++i) pk = fmax(pk, v[j][i]);
    int ex;
    frexp(pk, &ex);
#pragma unroll
    for (int j = 0; j < LC; ++j)
#pragma unroll
      for (int i = 0; i < MP; ++i) v[j][i] = ldexp(v[j][i], -ex);
    return ex;
  }
  const int ex = bexp - 1022;
  if (ex == 0) return 0;
  if (ex > 1022) {
#pragma unroll
    for (int j = 0; j < LC; ++j)
#pragma unroll
      for (int i = 0; i < MP; ++i) v[j][i] = ldexp(v[j][i], -ex);
    return ex;
  }
  const double sc = __hiloint2double((1023 - ex) << 20, 0);
#pragma unroll
  for (int j = 0; j < LC; ++j)
#pragma unroll
    for (int i = 0; i < MP; ++i) v[j][i] *= sc;
  return ex;
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32) walk4_kernel(const __grid_constant__ Walk4Params P4) {
  constexpr int MP = 4, LC = 4;
  const WalkParams& p = P4.p;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int warp = blockIdx.x * kWarpsPerBlock + wib;
  const int TW = gridDim.x * kWarpsPerBlock;
  const int N = p.N, root = 2 * N - 1, NC = p.NC, L = p.L;
  const int TCB = L * NC * MP;  // doubles per node TC block
  const int tc_chunks = TCB / 2;
  // per-warp smem: 2 stages x (3 operand slots of 256 double2 + 3 TC blocks)
  const int stage_d2 = 3 * 256 + 3 * (TCB / 2);
  double2* wsm = reinterpret_cast<double2*>(smem_raw) + size_t(wib) * 2 * stage_d2;

  int lc[LC];
  double cw[LC], crw[LC], cr2w[LC];
#pragma unroll
  for (int j = 0; j < LC; ++j) {
    const bool real = j < L;
    lc[j] = real ? j : L - 1;
    const double w = real ? p.probs[lc[j]] : 0.0, r = p.rates[lc[j]];
    cw[j] = w;
    crw[j] = r * w;
    cr2w[j] = r * r * w;
  }
  constexpr size_t VEC = size_t(32) * LC * MP;  // doubles per node slot (4 KB)
  double* E = p.escr + size_t(warp) * size_t(N - 1) * VEC;
  double* Qs = p.qscr + size_t(warp) * size_t(N - 1) * VEC;
  double* A = p.acc + size_t(warp) * p.accw;
  for (int i = lane; i < p.accw; i += 32) A[i] = 0.0;
  __syncwarp();

  auto op_ptr = [&](int stage, int slot) -> double2* { return wsm + stage * stage_d2 + slot * 256; };
  auto tc_ptr = [&](int stage, int slot) -> double* {
    return reinterpret_cast<double*>(wsm + stage * stage_d2 + 3 * 256 + slot * (TCB / 2));
  };
  auto stage_slot = [&](double2* dst, const double* gslot) {
    const double2* g = reinterpret_cast<const double2*>(gslot);
#pragma unroll
    for (int q = 0; q < 8; ++q) cp16_cg(dst + q * 32 + lane, g + q * 32 + lane);
  };
  auto stage_tc = [&](double* dst, int node) {
    const double2* g = reinterpret_cast<const double2*>(p.tc + size_t(node - 1) * TCB);
    double2* d = reinterpret_cast<double2*>(dst);
    for (int c = lane; c < tc_chunks; c += 32) cp16_ca(d + c, g + c);
  };
  auto read_slot = [&](const double2* src, double(&v)[LC][MP]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double2 d = src[q * 32 + lane];
      v[(2 * q) / MP][(2 * q) % MP] = d.x;
      v[(2 * q + 1) / MP][(2 * q + 1) % MP] = d.y;
    }
  };
  auto gather = [&](const double* tcs, int code, double(&v)[LC][MP]) {
#pragma unroll
    for (int j = 0; j < LC; ++j) {
      const double2* c = reinterpret_cast<const double2*>(tcs + (lc[j] * NC + code) * MP);
      const double2 a = c[0], b = c[1];
      v[j][0] = a.x;
      v[j][1] = a.y;
      v[j][2] = b.x;
      v[j][3] = b.y;
    }
  };
  auto qmat = [&](int x, int r, int c) -> double {
    return P4.homogeneous ? P4.q[r * 4 + c] : __ldg(p.qtab + size_t(p.qidx[x]) * 16 + r * 4 + c);
  };

  const int n = p.nsteps;
  for (int t = warp; t < p.ntiles; t += TW) {
    const int s = t * 32 + lane;
    const bool valid = s < p.P;
    const int sc = valid ? s : p.P - 1;
    const double w = valid ? p.weights[sc] : 0.0;

    // ------------------------------------------------ post-order pass (a)
    int S = 0;
    double keep[LC][MP];
    int code_n0 = 0, code_n1 = 0;
    auto issue_post = [&](int j, const int4 d, int last) {
      const int st = j & 1;
      int c0 = 0, c1 = 0;
      if (d.y <= N) {
        c0 = p.codes[size_t(d.y - 1) * p.P + sc];
        stage_tc(tc_ptr(st, 1), d.y);
      } else if (d.y != last) {
        stage_slot(op_ptr(st, 0), E + size_t(d.y - N - 1) * VEC);
      }
      if (d.z <= N) {
        c1 = p.codes[size_t(d.z - 1) * p.P + sc];
        stage_tc(tc_ptr(st, 2), d.z);
      } else if (d.z != last) {
        stage_slot(op_ptr(st, 0), E + size_t(d.z - N - 1) * VEC);
      }
      if (d.x != root) stage_tc(tc_ptr(st, 0), d.x);
      code_n0 = c0;
      code_n1 = c1;
    };
    int4 dcur = p.post[0];
    int4 dnext = n > 1 ? p.post[1] : dcur;
    issue_post(0, dcur, -1);
    cp_commit();
    int last = -1;
    for (int i = 0; i < n; ++i) {
      const int4 d = dcur;
      const int code0 = code_n0, code1 = code_n1;
      if (i + 1 < n) {
        dcur = dnext;
        if (i + 2 < n) dnext = p.post[i + 2];
        issue_post(i + 1, dcur, d.x);
      }
      cp_commit();
      cp_wait1();
      __syncwarp();
      const int st = i & 1;
      double x[LC][MP], y[LC][MP];
      if (d.y <= N) gather(tc_ptr(st, 1), code0, x);
      else if (d.y == last) {
#pragma unroll
        for (int j = 0; j < LC; ++j)
#pragma unroll
          for (int r = 0; r < MP; ++r) x[j][r] = keep[j][r];
      } else read_slot(op_ptr(st, 0), x);
      if (d.z <= N) gather(tc_ptr(st, 2), code1, y);
      else if (d.z == last) {
#pragma unroll
        for (int j = 0; j < LC; ++j)
#pragma unroll
          for (int r = 0; r < MP; ++r) y[j][r] = keep[j][r];
      } else read_slot(op_ptr(st, 0), y);
#pragma unroll
      for (int j = 0; j < LC; ++j)
#pragma unroll
        for (int r = 0; r < MP; ++r) x[j][r] *= y[j][r];
      if (!p.disable) S += normalize_hi<LC, MP>(x);
      if (d.x == root) {
        double mix = 0.0;
#pragma unroll
        for (int j = 0; j < LC; ++j) {
          double dd = 0.0;
#pragma unroll
          for (int r = 0; r < MP; ++r) dd = fma(P4.pi[r], x[j][r], dd);
          mix = fma(cw[j], dd, mix);
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
        const double* T = tc_ptr(st, 0);
#pragma unroll
        for (int j = 0; j < LC; ++j) {
          const double2* Tl = reinterpret_cast<const double2*>(T + lc[j] * NC * MP);
          double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll
          for (int c = 0; c < MP; ++c) {
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
        }
        double2* dst = reinterpret_cast<double2*>(E + size_t(d.x - N - 1) * VEC);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          double2 v;
          v.x = keep[(2 * q) / MP][(2 * q) % MP];
          v.y = keep[(2 * q + 1) / MP][(2 * q + 1) % MP];
          __stcg(dst + q * 32 + lane, v);
        }
        last = d.x;
      }
      __syncwarp();
    }
    if (!p.do_pre) continue;

    // ----------------------------------- pre-order pass + gradient (b)+(c)
    auto issue_pre = [&](int j, const int4 d, int prev_next) {
      const int st = j & 1;
      int c0 = 0, c1 = 0;
      if (d.x != root && prev_next != d.x) stage_slot(op_ptr(st, 2), Qs + size_t(d.x - N - 1) * VEC);
      if (d.y <= N) c0 = p.codes[size_t(d.y - 1) * p.P + sc];
      else stage_slot(op_ptr(st, 0), E + size_t(d.y - N - 1) * VEC);
      if (d.z <= N) c1 = p.codes[size_t(d.z - 1) * p.P + sc];
      else stage_slot(op_ptr(st, 1), E + size_t(d.z - N - 1) * VEC);
      stage_tc(tc_ptr(st, 0), d.y);
      stage_tc(tc_ptr(st, 1), d.z);
      code_n0 = c0;
      code_n1 = c1;
    };
    double qreg[LC][MP];
    dcur = p.pre[0];
    dnext = n > 1 ? p.pre[1] : dcur;
    issue_pre(0, dcur, 0);
    cp_commit();
    int prev_next = 0;
    for (int i = 0; i < n; ++i) {
      const int4 d = dcur;
      const int code0 = code_n0, code1 = code_n1;
      if (i + 1 < n) {
        dcur = dnext;
        if (i + 2 < n) dnext = p.pre[i + 2];
        issue_pre(i + 1, dcur, d.w);
      }
      cp_commit();
      cp_wait1();
      __syncwarp();
      const int st = i & 1;
      double q[LC][MP];
      if (d.x == root) {
#pragma unroll
        for (int j = 0; j < LC; ++j)
#pragma unroll
          for (int r = 0; r < MP; ++r) q[j][r] = P4.pi[r];
      } else if (prev_next == d.x) {
#pragma unroll
        for (int j = 0; j < LC; ++j)
#pragma unroll
          for (int r = 0; r < MP; ++r) q[j][r] = qreg[j][r];
      } else {
        read_slot(op_ptr(st, 2), q);
      }
      double ea[LC][MP], eb[LC][MP];
      if (d.y <= N) gather(tc_ptr(st, 0), code0, ea);
      else read_slot(op_ptr(st, 0), ea);
      if (d.z <= N) gather(tc_ptr(st, 1), code1, eb);
      else read_slot(op_ptr(st, 1), eb);

      double den = 0.0;
#pragma unroll
      for (int j = 0; j < LC; ++j) {
        double dd = 0.0;
#pragma unroll
        for (int r = 0; r < MP; ++r) dd = fma(q[j][r] * ea[j][r], eb[j][r], dd);
        den = fma(cw[j], dd, den);
      }
      const double inv_den = 1.0 / den;

      auto child = [&](const int x, const double(&ex_)[LC][MP], const double(&ey)[LC][MP], const double* T) {
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
            for (int c = 0; c < MP; ++c) a = fma(qmat(x, r, c), ex_[j][c], a);
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
              for (int c = 0; c < MP; ++c) a = fma(qmat(x, r, c), qe[c], a);
              d2 = fma(top[r], a, d2);
            }
            num2 = fma(cr2w[j], d2, num2);
          }
          if (x > N) {
            const double2* Tl = reinterpret_cast<const double2*>(T + lc[j] * NC * MP);
#pragma unroll
            for (int c = 0; c < MP; ++c) {
              const double2 a = Tl[2 * c], b = Tl[2 * c + 1];
              qx[j][c] = fma(a.x, top[0], fma(a.y, top[1], fma(b.x, top[2], b.y * top[3])));
            }
          }
        }
        const double r1 = num * inv_den;
        const double gv = warp_sum(valid ? w * r1 : 0.0);
        if (lane == 0) atomicAdd(A + x, gv);
        if (p.hess) {
          const double r2 = num2 * inv_den;
          const double hv = warp_sum(valid ? w * (r2 - r1 * r1) : 0.0);
          if (lane == 0) atomicAdd(A + p.B + x, hv);
        }
        if (x > N) {
          normalize_hi<LC, MP>(qx);
          if (x == d.w) {
#pragma unroll
            for (int j = 0; j < LC; ++j)
#pragma unroll
              for (int r = 0; r < MP; ++r) qreg[j][r] = qx[j][r];
          } else {
            double2* dst = reinterpret_cast<double2*>(Qs + size_t(x - N - 1) * VEC);
#pragma unroll
            for (int q8 = 0; q8 < 8; ++q8) {
              double2 v;
              v.x = qx[(2 * q8) / MP][(2 * q8) % MP];
              v.y = qx[(2 * q8 + 1) / MP][(2 * q8 + 1) % MP];
              __stcg(dst + q8 * 32 + lane, v);
            }
          }
        }
      };
      child(d.y, ea, eb, tc_ptr(st, 0));
      child(d.z, eb, ea, tc_ptr(st, 1));
      prev_next = d.w;
      __syncwarp();
    }
  }
}

}  // namespace pgk
