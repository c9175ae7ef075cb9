// Instantiations of the pipelined 4-state walk kernel (pg_walk4.cuh):
// homogeneous / per-branch generators x with / without Hessian x padded
// column counts NC in {5, 8, 16} (4 states + ambiguity classes + missing).
#include "pg_walk4.cuh"

#define PG_W4(H, S, NC) \
  if (homog == H && hess == S && nc == NC) return reinterpret_cast<void*>(&pgk::walk4_kernel<H, S, NC>);

void* pg_walk4_kernel(bool homog, bool hess, int nc) {
  PG_W4(true, false, 5)
  PG_W4(true, true, 5)
  PG_W4(false, false, 5)
  PG_W4(false, true, 5)
  PG_W4(true, false, 8)
  PG_W4(true, true, 8)
  PG_W4(false, false, 8)
  PG_W4(false, true, 8)
  PG_W4(true, false, 16)
  PG_W4(true, true, 16)
  PG_W4(false, false, 16)
  PG_W4(false, true, 16)
  return nullptr;
}

int pg_walk4_nc(int nc) { return nc <= 5 ? 5 : nc <= 8 ? 8 : nc <= 16 ? 16 : 0; }
