// Instantiations of the pipelined 4-state walk kernel with 2 categories per
// lane (two lanes per pattern; see pg_walk4.cuh).
#include "pg_walk4.cuh"

#define PG_W4(H, S, NC, LCV) \
  if (homog == H && hess == S && nc == NC) return reinterpret_cast<void*>(&pgk::walk4_kernel<H, S, NC, LCV>);

void* pg_walk4_kernel_lc2(bool homog, bool hess, int nc) {
  PG_W4(true, false, 5, 2)
  PG_W4(true, true, 5, 2)
  PG_W4(false, false, 5, 2)
  PG_W4(false, true, 5, 2)
  PG_W4(true, false, 16, 2)
  PG_W4(true, true, 16, 2)
  PG_W4(false, false, 16, 2)
  PG_W4(false, true, 16, 2)
  return nullptr;
}
