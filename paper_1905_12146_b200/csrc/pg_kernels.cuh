// phylograd-b200 device code: K1 (transition columns) and K3 (reduction).
// See pg_walk.cuh for K2.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "pg_walk.cuh"  // frag_pos

namespace pgk {

// Fixed-order reduction over warps (deterministic for a fixed grid), plus the
// clock chain rule: d/dr_i = dt_i d/db_i, d2/dr_i2 = dt_i^2 d2/db_i2.
// Block = 32 columns x kReduceGroups row groups: group r sums rows r, r + G,
// r + 2G, ... (coalesced 256-byte row segments, four independent chains),
// then the G partials are added in group order.  One thread per column
// summing all rows serially was latency-bound (C2: 163 us of a 1.56 ms
// evaluation).
constexpr int kReduceGroups = 16;
__global__ void __launch_bounds__(32 * kReduceGroups) reduce_kernel(const double* __restrict__ acc, int TW, int accw,
                                                                   int width, double* __restrict__ out,
                                                                   const double* __restrict__ dt, int B) {
  __shared__ double part[kReduceGroups][33];
  const int c = threadIdx.x & 31, r = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + c;
  double s = 0.0;
  if (i < width) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int w = r;
    constexpr int G = kReduceGroups;
    for (; w + 3 * G < TW; w += 4 * G) {
      s0 += acc[size_t(w) * accw + i];
      s1 += acc[size_t(w + G) * accw + i];
      s2 += acc[size_t(w + 2 * G) * accw + i];
      s3 += acc[size_t(w + 3 * G) * accw + i];
    }
    for (; w < TW; w += G) s0 += acc[size_t(w) * accw + i];
    s = (s0 + s1) + (s2 + s3);
  }
  part[r][c] = s;
  __syncthreads();
  if (r != 0 || i >= width) return;
#pragma unroll
  for (int g = 1; g < kReduceGroups; ++g) s += part[g][c];
  if (dt) {
    if (i >= 1 && i <= B) s *= dt[i - 1];
    else if (i > B) s *= dt[i - B - 1] * dt[i - B - 1];
  }
  out[i] = s;
}

// ------------------------------------------------------- clock chain rule
// clock.hpp:140-152 (likelihood part of RelaxedClockPosterior::gradient) and
// clock.hpp:199-213 (node_time_gradient) from one branch gradient g:
//   dlog_eps[i] = b_i g_i, dlog_mu = sum_i b_i g_i (fixed-order block
//   reduction), dnode[k] = r_k g_k (non-root) - sum_{c in children} r_c g_c
// with r_i = rates[i], or b_i / dt_i when rates is null.  One block.
constexpr int kClockThreads = 512;
__global__ void __launch_bounds__(kClockThreads)
    clock_kernel(const double* __restrict__ g, const double* __restrict__ b, const double* __restrict__ rates,
                 const double* __restrict__ dt, const int* __restrict__ children, int N,
                 double* __restrict__ out /* [1 + B + N-1]: dlog_mu, dlog_eps, dnode */) {
  __shared__ double part[kClockThreads];
  const int B = 2 * N - 2, root = 2 * N - 1;
  double s = 0.0;
  for (int i = threadIdx.x; i < B; i += kClockThreads) {
    const double v = b[i] * g[i];
    out[1 + i] = v;
    s += v;
  }
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = kClockThreads / 2; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = part[0];
  auto rg = [&](int node) {
    const double r = rates ? rates[node - 1] : b[node - 1] / dt[node - 1];
    return r * g[node - 1];
  };
  for (int k = threadIdx.x; k < N - 1; k += kClockThreads) {
    const int node = N + 1 + k;
    double v = 0.0;
    if (node != root) v += rg(node);
    v -= rg(children[2 * node]);
    v -= rg(children[2 * node + 1]);
    out[1 + B + k] = v;
  }
}

// Fixed rank-order sum of G shard outputs gathered on one device
// (bit-reproducible multi-device reduction: sum over shards 0, 1, ..., G-1).
__global__ void shard_sum_kernel(const double* __restrict__ parts, int G, int width, double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < width; i += gridDim.x * blockDim.x) {
    double s = parts[i];
    for (int r = 1; r < G; ++r) s += parts[size_t(r) * width + i];
    out[i] = s;
  }
}

// ------------------------------------------------------------------- K1
struct TcParams {
  const double* blen;   // [B] branch lengths (index node-1)
  const double* rates;  // [L]
  const double* qtab;   // [nq][MP][MP] row-major, padded
  const int* qidx;      // [2N] node -> generator index (0 = shared)
  const double* eig_u;  // [m][m] row-major U = D^{-1/2} V
  const double* eig_ui; // [m][m] U^{-1} = V^T D^{1/2}
  const double* eig_w;  // [m] eigenvalues
  const double* amb;    // [A][m] ambiguity partials
  double* tc;           // [B][L][NC][MP]
  double* qtc;          // optional [B][L][NC][MP]: the same columns of Q_branch * P (tip Q-e gathers)
  double* fpp;          // optional [B][L][MP*MP]: P in DMMA B-fragment order for y = P x (walkm)
  double* fpt;          // optional [B][L][MP*MP]: same for y = P^T x
  double* f4post;       // optional [B][L][32]: 4-state P in m8n8k4 B-fragment order for e = P x (walk4t)
  double* f4pre;        // optional [B][L+1][32]: [l] P^T x in the even, Q^T x in the odd output columns;
                        //   [L] (Q^2)^T x in the even columns (walk4t)
  int* err;             // err[2] <- 1 on a negative / non-finite branch length
  int m, MP, NC, A, L, have_eigen;
};

__device__ __forceinline__ void block_matmul(const double* a, const double* b, double* c, int m) {
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int i = e / m, j = e % m;
    double s = 0.0;
    for (int k = 0; k < m; ++k) s = fma(a[i * m + k], b[k * m + j], s);
    c[e] = s;
  }
  __syncthreads();
}

// Higham (2005) Pade scaling-and-squaring, the algorithm behind Eigen's
// MatrixBase::exp() used at substitution.hpp:71-75/:155-156.  Dynamic shared
// memory: 7 m x m buffers + m pivot factors.  Returns the buffer holding e^{arg}.
__device__ double* block_expm(const double* arg, int m, double* sm) {
  const int mm = m * m;
  double* A = sm;
  double* A2 = sm + mm;
  double* A4 = sm + 2 * mm;
  double* A6 = sm + 3 * mm;
  double* Ub = sm + 4 * mm;
  double* Vb = sm + 5 * mm;
  double* Tb = sm + 6 * mm;
  double* f = sm + 7 * mm;
  __shared__ double s_l1;
  __shared__ int s_piv;
  __shared__ int s_sq;
  if (threadIdx.x == 0) {
    double l1 = 0.0;
    for (int j = 0; j < m; ++j) {
      double c = 0.0;
      for (int i = 0; i < m; ++i) c += fabs(arg[i * m + j]);
      l1 = fmax(l1, c);
    }
    s_l1 = l1;
    int sq = 0;
    if (l1 >= 2.097847961257068e+000) {
      frexp(l1 / 5.371920351148152, &sq);
      if (sq < 0) sq = 0;
    }
    s_sq = sq;
  }
  __syncthreads();
  const double l1 = s_l1;
  const int sq = s_sq;
  for (int e = threadIdx.x; e < mm; e += blockDim.x) A[e] = ldexp(arg[e], -sq);
  __syncthreads();
  block_matmul(A, A, A2, m);
  auto eye = [&](int e) { return (e / m == e % m) ? 1.0 : 0.0; };
  if (l1 < 2.097847961257068e+000) {
    int deg;
    const double* b;
    static constexpr double b3[] = {120.0, 60.0, 12.0, 1.0};
    static constexpr double b5[] = {30240.0, 15120.0, 3360.0, 420.0, 30.0, 1.0};
    static constexpr double b7[] = {17297280.0, 8648640.0, 1995840.0, 277200.0, 25200.0, 1512.0, 56.0, 1.0};
    static constexpr double b9[] = {17643225600.0, 8821612800.0, 2075673600.0, 302702400.0, 30270240.0,
                                    2162160.0,     110880.0,     3960.0,       90.0,        1.0};
    if (l1 < 1.495585217958292e-002) { deg = 3; b = b3; }
    else if (l1 < 2.539398330063230e-001) { deg = 5; b = b5; }
    else if (l1 < 9.504178996162932e-001) { deg = 7; b = b7; }
    else { deg = 9; b = b9; }
    if (deg >= 5) block_matmul(A2, A2, A4, m);
    if (deg >= 7) block_matmul(A4, A2, A6, m);
    if (deg >= 9) block_matmul(A6, A2, Tb, m);  // A8 in Tb
    for (int e = threadIdx.x; e < mm; e += blockDim.x) {
      double u = b[1] * eye(e) + b[3] * A2[e], v = b[0] * eye(e) + b[2] * A2[e];
      if (deg >= 5) { u += b[5] * A4[e]; v += b[4] * A4[e]; }
      if (deg >= 7) { u += b[7] * A6[e]; v += b[6] * A6[e]; }
      if (deg >= 9) { u += b[9] * Tb[e]; v += b[8] * Tb[e]; }
      Ub[e] = u;
      Vb[e] = v;
    }
    __syncthreads();
    block_matmul(A, Ub, Tb, m);  // U = A * inner -> Tb
  } else {
    static constexpr double b[] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                                   1187353796428800.0,  129060195264000.0,   10559470521600.0,
                                   670442572800.0,      33522128640.0,       1323241920.0,
                                   40840800.0,          960960.0,            16380.0,
                                   182.0,               1.0};
    block_matmul(A2, A2, A4, m);
    block_matmul(A4, A2, A6, m);
    for (int e = threadIdx.x; e < mm; e += blockDim.x) Tb[e] = b[13] * A6[e] + b[11] * A4[e] + b[9] * A2[e];
    __syncthreads();
    block_matmul(A6, Tb, Ub, m);
    for (int e = threadIdx.x; e < mm; e += blockDim.x)
      Ub[e] += b[7] * A6[e] + b[5] * A4[e] + b[3] * A2[e] + b[1] * eye(e);
    __syncthreads();
    block_matmul(A, Ub, Tb, m);  // U -> Tb
    for (int e = threadIdx.x; e < mm; e += blockDim.x) Ub[e] = b[12] * A6[e] + b[10] * A4[e] + b[8] * A2[e];
    __syncthreads();
    block_matmul(A6, Ub, Vb, m);
    for (int e = threadIdx.x; e < mm; e += blockDim.x)
      Vb[e] += b[6] * A6[e] + b[4] * A4[e] + b[2] * A2[e] + b[0] * eye(e);
    __syncthreads();
  }
  // num = V + U (A2), den = V - U (A4); solve den R = num by partial-pivot LU.
  double* num = A2;
  double* den = A4;
  for (int e = threadIdx.x; e < mm; e += blockDim.x) {
    num[e] = Vb[e] + Tb[e];
    den[e] = Vb[e] - Tb[e];
  }
  __syncthreads();
  for (int k = 0; k < m; ++k) {
    if (threadIdx.x == 0) {
      int piv = k;
      for (int i = k + 1; i < m; ++i)
        if (fabs(den[i * m + k]) > fabs(den[piv * m + k])) piv = i;
      s_piv = piv;
    }
    __syncthreads();
    const int piv = s_piv;
    if (piv != k)
      for (int j = threadIdx.x; j < m; j += blockDim.x) {
        double t = den[k * m + j]; den[k * m + j] = den[piv * m + j]; den[piv * m + j] = t;
        t = num[k * m + j]; num[k * m + j] = num[piv * m + j]; num[piv * m + j] = t;
      }
    __syncthreads();
    for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) f[i] = den[i * m + k] / den[k * m + k];
    __syncthreads();
    for (int e = threadIdx.x; e < (m - k - 1) * m; e += blockDim.x) {
      const int i = k + 1 + e / m, j = e % m;
      if (j > k) den[i * m + j] -= f[i] * den[k * m + j];
      num[i * m + j] -= f[i] * num[k * m + j];
    }
    __syncthreads();
  }
  for (int i = m - 1; i >= 0; --i) {
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      double s = num[i * m + j];
      for (int k = i + 1; k < m; ++k) s -= den[i * m + k] * num[k * m + j];
      num[i * m + j] = s / den[i * m + i];
    }
    __syncthreads();
  }
  double* cur = num;
  double* other = A6;
  for (int r = 0; r < sq; ++r) {
    block_matmul(cur, cur, other, m);
    double* t = cur; cur = other; other = t;
  }
  return cur;
}

__global__ void tc_kernel(const __grid_constant__ TcParams p) {
  extern __shared__ double sm[];
  const int node = blockIdx.x + 1, l = blockIdx.y, m = p.m, mm = m * m;
  double* P = sm;        // result / arg buffer for the eigen path
  double* arg = sm;  // block_expm scales it in place into its A buffer
  const double b = p.blen[node - 1];
  const bool bad = !(b >= 0.0) || !isfinite(b);
  if (bad && threadIdx.x == 0) atomicExch(&p.err[2], 1);
  const double t = bad ? 0.0 : b * p.rates[l];
  const int qi = p.qidx[node];
  double* R = P;
  if (t == 0.0) {
    for (int e = threadIdx.x; e < mm; e += blockDim.x) P[e] = (e / m == e % m) ? 1.0 : 0.0;
    __syncthreads();
  } else if (p.have_eigen && qi == 0) {
    // P = U diag(e^{w t}) U^-1: the m exponentials once, then the contraction
    double* ew = sm + mm;
    for (int k = threadIdx.x; k < m; k += blockDim.x) ew[k] = exp(p.eig_w[k] * t);
    __syncthreads();
    for (int e = threadIdx.x; e < mm; e += blockDim.x) {
      const int i = e / m, j = e % m;
      double s = 0.0;
      for (int k = 0; k < m; ++k) s = fma(__ldg(p.eig_u + i * m + k) * ew[k], __ldg(p.eig_ui + k * m + j), s);
      P[e] = s;
    }
    __syncthreads();
  } else {
    const double* Q = p.qtab + size_t(qi) * p.MP * p.MP;
    for (int e = threadIdx.x; e < mm; e += blockDim.x) arg[e] = Q[(e / m) * p.MP + (e % m)] * t;
    __syncthreads();
    R = block_expm(arg, m, sm);
  }
  for (int e = threadIdx.x; e < mm; e += blockDim.x) R[e] = fmax(R[e], 0.0);  // cwiseMax(0), :158
  __syncthreads();
  double* out = p.tc + (size_t(node - 1) * p.L + l) * p.NC * p.MP;
  for (int e = threadIdx.x; e < p.NC * p.MP; e += blockDim.x) {
    const int c = e / p.MP, r = e % p.MP;
    double v = 0.0;
    if (r < m) {
      if (c < p.MP) {
        if (c < m) v = R[r * m + c];
      } else if (c - p.MP < p.A) {  // columns past the last class are zero padding
        const double* a = p.amb + size_t(c - p.MP) * m;
        for (int j = 0; j < m; ++j) v = fma(R[r * m + j], a[j], v);
      }
    }
    out[e] = v;
  }
  if (p.fpp) {
    // B fragments of mma.m8n8k4 for the walkm kernel: element (ki, ni, lane)
    // = M(k = 4ki + lane%4, n = sigma(ni, lane/4)), sigma(ni, g) =
    // 4(2ni + g%2) + g/2 — the column permutation that makes D land in the
    // A-fragment layout (no shuffles between chained mat-vecs)
    const int KK = p.MP / 4, NT = (KK + 1) / 2, frag = KK * NT * 32;
    double* fp = p.fpp + (size_t(node - 1) * p.L + l) * size_t(frag);
    double* ft = p.fpt + (size_t(node - 1) * p.L + l) * size_t(frag);
    for (int e = threadIdx.x; e < KK * NT * 32; e += blockDim.x) {
      const int lane = e & 31, f = e >> 5, ki = f / NT, ni = f % NT;
      const int k = 4 * ki + (lane & 3), g = lane >> 2, n = 4 * (2 * ni + (g & 1)) + (g >> 1);
      const bool in = k < m && n < m;
      const int at = frag_pos(f, lane, KK * NT);
      fp[at] = in ? R[n * m + k] : 0.0;  // y = P x: M(k, n) = P[n][k]
      ft[at] = in ? R[k * m + n] : 0.0;  // y = P^T x: M(k, n) = P[k][n]
    }
  }
  if (p.f4post && m <= 4) {
    // m8n8k4 B fragments for walk4t (lane t holds B[kk = t%4][n = t/4]); the
    // vector layout there is lane = (pattern, state kk), so output column
    // n = 2c lands on the lane of state c: even columns carry the result in
    // that layout, odd columns a second product of the same A
    const double* Q = p.qtab + size_t(qi) * p.MP * p.MP;
    double* fo = p.f4post + (size_t(node - 1) * p.L + l) * 32;
    double* fr = p.f4pre + (size_t(node - 1) * (p.L + 1) + l) * 32;
    for (int e = threadIdx.x; e < 32; e += blockDim.x) {
      const int kk = e & 3, n = e >> 2, c = n >> 1;
      const bool in = kk < m && c < m, odd = n & 1;
      fo[e] = (in && !odd) ? R[c * m + kk] : 0.0;                     // e[c] = sum_kk P[c][kk] x[kk]
      fr[e] = !in ? 0.0 : odd ? Q[kk * p.MP + c] : R[kk * m + c];     // q[c] = (P^T t)[c], u[c] = (Q^T t)[c]
    }
    if (l == 0) {
      double* fh = p.f4pre + (size_t(node - 1) * (p.L + 1) + p.L) * 32;
      for (int e = threadIdx.x; e < 32; e += blockDim.x) {
        const int kk = e & 3, n = e >> 2, c = n >> 1;
        double v = 0.0;
        if (kk < m && c < m && !(n & 1))
          for (int j = 0; j < m; ++j) v = fma(Q[kk * p.MP + j], Q[j * p.MP + c], v);  // (Q^2)[kk][c]
        fh[e] = v;
      }
    }
  }
  if (p.qtc) {
    // Q e for a tip is a column of Q P (P and Q commute, engine.hpp:260):
    // build QR = Q_branch * R once, then the same column table
    double* QR = sm + 5 * mm;  // dead expm buffer, disjoint from R
    const double* Q = p.qtab + size_t(qi) * p.MP * p.MP;
    for (int e = threadIdx.x; e < mm; e += blockDim.x) {
      const int i = e / m, j = e % m;
      double s = 0.0;
      for (int k = 0; k < m; ++k) s = fma(Q[i * p.MP + k], R[k * m + j], s);
      QR[e] = s;
    }
    __syncthreads();
    double* qout = p.qtc + (size_t(node - 1) * p.L + l) * p.NC * p.MP;
    for (int e = threadIdx.x; e < p.NC * p.MP; e += blockDim.x) {
      const int c = e / p.MP, r = e % p.MP;
      double v = 0.0;
      if (r < m) {
        if (c < p.MP) {
          if (c < m) v = QR[r * m + c];
        } else if (c - p.MP < p.A) {
          const double* a = p.amb + size_t(c - p.MP) * m;
          for (int j = 0; j < m; ++j) v = fma(QR[r * m + j], a[j], v);
        }
      }
      qout[e] = v;
    }
  }
}

}  // namespace pgk
