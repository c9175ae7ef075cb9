// Instantiations of the pipelined 4-state walk kernel (pg_walk4.cuh) with
// 4 categories per lane: homogeneous / per-branch generators x with / without
// Hessian x padded column counts NC in {5, 16} (4 states + classes + missing).
#include "pg_walk4.cuh"

#define PG_W4(H, S, NC, LCV) \
  if (homog == H && hess == S && nc == NC) return reinterpret_cast<void*>(&pgk::walk4_kernel<H, S, NC, LCV>);

void* pg_walk4_kernel_lc4(bool homog, bool hess, int nc) {
  PG_W4(true, false, 5, 4)
  PG_W4(true, true, 5, 4)
  PG_W4(false, false, 5, 4)
  PG_W4(false, true, 5, 4)
  PG_W4(true, false, 16, 4)
  PG_W4(true, true, 16, 4)
  PG_W4(false, false, 16, 4)
  PG_W4(false, true, 16, 4)
  return nullptr;
}

int pg_walk4_nc(int nc) { return nc <= 5 ? 5 : nc <= 16 ? 16 : 0; }
