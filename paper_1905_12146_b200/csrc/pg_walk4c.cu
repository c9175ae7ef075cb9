// Instantiations of the pipelined 4-state walk kernel for one and two rate
// categories (one lane per pattern; see pg_walk4.cuh): models without or with
// a two-class rate mixture (e.g. the C1 HKY85 configuration).
#include "pg_walk4.cuh"

#define PG_W4L(H, S, NC, LT) \
  if (homog == H && hess == S && nc == NC && L == LT) \
    return reinterpret_cast<void*>(&pgk::walk4_kernel<H, S, NC, LT, LT>);

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
  return nullptr;
}
