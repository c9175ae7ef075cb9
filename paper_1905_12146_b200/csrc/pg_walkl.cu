// Instantiations of the level-scheduled 4-state traversal (pg_walkl.cuh):
// rate categories L in {1, 2, 4, 8} (one lane per (pattern, category)) x
// homogeneous / per-branch generators x with / without Hessian.
#include "pg_walkl.cuh"

#define PG_WL(L_, H, S) \
  if (L == L_ && homog == H && hess == S) return reinterpret_cast<void*>(&pgk::walkl_kernel<L_, H, S>);
#define PG_WL_L(L_)       \
  PG_WL(L_, true, false)  \
  PG_WL(L_, true, true)   \
  PG_WL(L_, false, false) \
  PG_WL(L_, false, true)

void* pg_walkl_kernel(int L, bool homog, bool hess) {
  PG_WL_L(1)
  PG_WL_L(2)
  PG_WL_L(4)
  PG_WL_L(8)
  return nullptr;
}
