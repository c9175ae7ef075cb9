// Instantiations of the category-parallel 4-state walk (pg_walk4x.cuh):
// warps per CTA = rate categories (L = 1, 2, 4, 8) x homogeneous / per-branch
// generators x with / without Hessian x padded column counts NC in {5, 16}.
#include "pg_walk4x.cuh"

#define PG_W4X(H, S, NC_, LW_)                                                          \
  if (homog == H && hess == S && nc == NC_ && L == LW_) {                              \
    if (smem) *smem = pgk::Walk4xGeom<LW_, NC_, S>::smem_bytes();                      \
    return reinterpret_cast<void*>(&pgk::walk4x_kernel<H, S, NC_, LW_>);              \
  }
#define PG_W4X_L(LW_)            \
  PG_W4X(true, false, 5, LW_)    \
  PG_W4X(true, true, 5, LW_)     \
  PG_W4X(false, false, 5, LW_)   \
  PG_W4X(false, true, 5, LW_)    \
  PG_W4X(true, false, 16, LW_)   \
  PG_W4X(true, true, 16, LW_)    \
  PG_W4X(false, false, 16, LW_)  \
  PG_W4X(false, true, 16, LW_)

void* pg_walk4x_kernel(bool homog, bool hess, int nc, int L, size_t* smem) {
  PG_W4X_L(4)
  return nullptr;
}
