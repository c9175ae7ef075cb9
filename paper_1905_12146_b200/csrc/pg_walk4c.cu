// Instantiations of the pipelined 4-state walk kernel for 1, 2, 3 and 8 rate
// categories (see pg_walk4.cuh): one lane per pattern holds all categories
// for L <= 3 (e.g. the C1 HKY85 configuration, L = 1); for L = 8 two lanes
// per pattern hold four categories each.
#include "pg_walk4.cuh"

#define PG_W4L(H, S, NC, LT) \
  if (homog == H && hess == S && nc == NC && L == LT) \
    return reinterpret_cast<void*>(&pgk::walk4_kernel<H, S, NC, (LT == 8 ? 4 : LT), LT>);

void* pg_walk4_kernel_l12(bool homog, bool hess, int nc, int L) {
  PG_W4L(true, false, 5, 1)
  PG_W4L(true, true, 5, 1)
  PG_W4L(false, false, 5, 1)
  PG_W4L(false, true, 5, 1)
  PG_W4L(true, false, 16, 1)
  PG_W4L(true, true, 16, 1)
  PG_W4L(false, false, 16, 1)
  PG_W4L(false, true, 16, 1)
  PG_W4L(true, false, 5, 2)
  PG_W4L(true, true, 5, 2)
  PG_W4L(false, false, 5, 2)
  PG_W4L(false, true, 5, 2)
  PG_W4L(true, false, 16, 2)
  PG_W4L(true, true, 16, 2)
  PG_W4L(false, false, 16, 2)
  PG_W4L(false, true, 16, 2)
  PG_W4L(true, false, 5, 3)
  PG_W4L(true, true, 5, 3)
  PG_W4L(false, false, 5, 3)
  PG_W4L(false, true, 5, 3)
  PG_W4L(true, false, 16, 3)
  PG_W4L(true, true, 16, 3)
  PG_W4L(false, false, 16, 3)
  PG_W4L(false, true, 16, 3)
  PG_W4L(true, false, 5, 8)
  PG_W4L(true, true, 5, 8)
  PG_W4L(false, false, 5, 8)
  PG_W4L(false, true, 5, 8)
  PG_W4L(true, false, 16, 8)
  PG_W4L(true, true, 16, 8)
  PG_W4L(false, false, 16, 8)
  PG_W4L(false, true, 16, 8)
  return nullptr;
}
