// Host side of the warp-specialised 4-state walk (pg_walk4x.cuh): per post-
// and pre-order step, the header (descriptor + hand-off flags) and the list of
// operand copies the producer warp issues.  Built once per topology /
// pattern layout (the tables depend on the schedule, L, NC and the tip-code
// row stride), uploaded next to the schedule.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "pg_walk.cuh"

namespace pgk {

struct Walk4xHdr {
  int4 d;
  int flags;
  int ncopy;
  int tx;
  int pad;
};
struct Walk4xCopy {
  long long src;
  int dst;
  int kb;
};
// Header flags.  Hand-off distances (0: none) are 2 bit fields: a value
// produced at step i and consumed at step i + dist (dist <= kW4xHand, one
// less than the stage count) is written by the consumer warps straight into
// that step's stage instead of going through scratch + a bulk copy.
//   post: bits 0-1 distance of this node's edge message (1 = kept in registers)
//   pre:  bit 0 q staged from scratch (drop it after use);
//         bits 1-2 / 3-4 distance of child y's / z's pre-partial
constexpr int kW4xPreQGlobal = 1;
constexpr int kW4xHand = 3;
constexpr int kW4xMaxCopies = 8;

struct Walk4xParams {
  Walk4Params p4;
  const Walk4xHdr* hdr;    // [2][n] post steps, then pre steps
  const Walk4xCopy* cpy;   // [2][n][kW4xMaxCopies]
};

// post / pre: the engine's schedules ({node, child, child, next}); N tips, L
// categories, NC table columns, Pc tip-code row stride.
inline void build_walk4x_tables(const std::vector<int4>& post, const std::vector<int4>& pre, int N, int L, int NC,
                                long long Pc, std::vector<Walk4xHdr>& hdr, std::vector<Walk4xCopy>& cpy) {
  const int n = int(post.size()), root = 2 * N - 1;
  const long long SLOT = 32LL * 4 * L, TCB = 4LL * L * NC;  // doubles
  const int SLOTB = int(SLOT * 8), TCBB = int(TCB * 8);
  // stage layout in bytes (pg_walk4x.cuh Walk4xGeom): header, 3 slots, 3 TC blocks, 2 x 32 code bytes
  auto OP = [&](int k) { return 32 + k * SLOTB; };
  auto TC = [&](int k) { return 32 + 3 * SLOTB + k * TCBB; };
  const int CODES = 32 + 3 * SLOTB + 3 * TCBB;
  hdr.assign(size_t(2 * n), Walk4xHdr{});
  cpy.assign(size_t(2 * n) * kW4xMaxCopies, Walk4xCopy{});
  auto add = [&](int k, int kind, long long src, int dst, int bytes) {
    Walk4xHdr& h = hdr[size_t(k)];
    Walk4xCopy& c = cpy[size_t(k) * kW4xMaxCopies + size_t(h.ncopy++)];
    c.src = src;
    c.dst = dst;
    c.kb = (kind << 24) | bytes;
    h.tx += bytes;
  };
  auto slot = [&](int node) { return (node - N - 1) * SLOT; };
  auto tcb = [&](int node) { return (node - 1) * TCB; };
  auto codes = [&](int node) { return (node - 1) * Pc; };
  // ---- post-order steps
  for (int s = 0; s < n; ++s) {
    const int4 d = post[size_t(s)];
    Walk4xHdr& h = hdr[size_t(s)];
    h.d = d;
    const int ch[2] = {d.y, d.z};
    for (int i = 0; i < 2; ++i) {
      const int c = ch[i];
      if (c <= N) {
        add(s, 4, codes(c), CODES + 32 * i, 32);
        add(s, 2, tcb(c), TC(1 + i), TCBB);
      } else {
        bool handed = false;  // produced within the last kW4xHand steps: in registers / handed on
        for (int dist = 1; dist <= kW4xHand && s - dist >= 0; ++dist) handed = handed || post[size_t(s - dist)].x == c;
        if (!handed) add(s, 0, slot(c), OP(0), SLOTB);
      }
    }
    if (d.x != root) add(s, 2, tcb(d.x), TC(0), TCBB);
    for (int dist = 1; dist <= kW4xHand && s + dist < n; ++dist)
      if (post[size_t(s + dist)].y == d.x || post[size_t(s + dist)].z == d.x) {
        h.flags |= dist;
        break;
      }
    add(s, 5, (long long)s * 32, 0, 32);
  }
  // ---- pre-order steps
  auto other = [&](const int4& d) {
    const int o = d.y == d.w ? d.z : d.y;
    return o > N ? o : -1;
  };
  for (int s = 0; s < n; ++s) {
    const int k = n + s;
    const int4 d = pre[size_t(s)];
    Walk4xHdr& h = hdr[size_t(k)];
    h.d = d;
    bool handed = d.x == root || (s >= 1 && pre[size_t(s - 1)].w == d.x);
    for (int dist = 2; dist <= kW4xHand && s - dist >= 0; ++dist) handed = handed || other(pre[size_t(s - dist)]) == d.x;
    if (!handed) {
      add(k, 1, slot(d.x), OP(2), SLOTB);
      h.flags |= kW4xPreQGlobal;
    }
    const int ch[2] = {d.y, d.z};
    for (int i = 0; i < 2; ++i) {
      const int c = ch[i];
      if (c <= N) {
        add(k, 4, codes(c), CODES + 32 * i, 32);
        add(k, 3, tcb(c), OP(i), TCBB);  // Q P table of the tip
      } else {
        add(k, 0, slot(c), OP(i), SLOTB);
        if (c != d.w)
          for (int dist = 2; dist <= kW4xHand && s + dist < n; ++dist)
            if (pre[size_t(s + dist)].x == c) {
              h.flags |= dist << (1 + 2 * i);
              break;
            }
      }
    }
    add(k, 2, tcb(d.y), TC(0), TCBB);
    add(k, 2, tcb(d.z), TC(1), TCBB);
    add(k, 5, (long long)k * 32, 0, 32);
  }
}

}  // namespace pgk
