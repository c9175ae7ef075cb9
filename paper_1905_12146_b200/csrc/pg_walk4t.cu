// Instantiations of the tensor-core 4-state walk (pg_walk4t.cuh): 4 rate
// categories, with / without the Hessian, TC column counts NC in {5, 16}
// (per-branch generators need no variant: the B fragments carry them).
#include "pg_walk4t.cuh"

void* pg_walk4t_kernel(bool hess, int nc) {
  if (nc == 5) return hess ? reinterpret_cast<void*>(&pgk::walk4t_kernel<true, 5>)
                           : reinterpret_cast<void*>(&pgk::walk4t_kernel<false, 5>);
  if (nc == 16) return hess ? reinterpret_cast<void*>(&pgk::walk4t_kernel<true, 16>)
                            : reinterpret_cast<void*>(&pgk::walk4t_kernel<false, 16>);
  return nullptr;
}

size_t pg_walk4t_smem(int nc) {
  const size_t warp = nc <= 5 ? pgk::Walk4TGeom<5>::WARP : pgk::Walk4TGeom<16>::WARP;
  return size_t(pgk::kWarpsPerBlock) * warp * sizeof(double);
}
