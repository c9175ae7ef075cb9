// Instantiations of the single-buffered 4-state walk (pg_walk4s.cuh): 4 rate
// categories, one lane per pattern, homogeneous / per-branch generators x
// with / without the Hessian x TC column counts NC in {4 (no missing /
// ambiguous codes), 5, 16}.
#include <algorithm>

#include "pg_walk4s.cuh"

#define PG_W4S(H, S, NC) \
  if (homog == H && hess == S && nc == NC) return reinterpret_cast<void*>(&pgk::walk4s_kernel<H, S, NC>);

// cherry-table instances (NC = 4)
void* pg_walk4s_cherry_kernel(bool homog, bool hess) {
  if (homog) return hess ? reinterpret_cast<void*>(&pgk::walk4s_kernel<true, true, 4, true>)
                         : reinterpret_cast<void*>(&pgk::walk4s_kernel<true, false, 4, true>);
  return hess ? reinterpret_cast<void*>(&pgk::walk4s_kernel<false, true, 4, true>)
              : reinterpret_cast<void*>(&pgk::walk4s_kernel<false, false, 4, true>);
}

void pg_cherry_tables(const int4* cherries, int ncherry, int N, const double* tc, const double* qtc, double* ct,
                      cudaStream_t stream) {
  if (ncherry > 0)
    pgk::cherry_tc_kernel<<<(ncherry * 64 + 127) / 128, 128, 0, stream>>>(cherries, ncherry, N, tc, qtc, ct);
}

// dynamic shared memory of the cherry instances (the gradient ones hold three tables per cherry child)
size_t pg_walk4s_cherry_smem() {
  return size_t(pgk::kWarpsPerBlock) * pgk::Walk4SGeom<4, true>::WARP * sizeof(double2);
}

void pg_cherry_codes(const int4* cherries, int ncherry, int N, long long Pc, const uint8_t* codes, uint8_t* cc,
                     cudaStream_t stream) {
  if (ncherry <= 0) return;
  const unsigned gx = unsigned(std::min<long long>((Pc + 255) / 256, 64));
  pgk::cherry_codes_kernel<<<dim3(gx, unsigned(ncherry)), 256, 0, stream>>>(cherries, ncherry, N, Pc, codes, cc);
}

void* pg_walk4s_kernel(bool homog, bool hess, int nc) {
  PG_W4S(true, false, 4)
  PG_W4S(true, true, 4)
  PG_W4S(false, false, 4)
  PG_W4S(false, true, 4)
  PG_W4S(true, false, 5)
  PG_W4S(true, true, 5)
  PG_W4S(false, false, 5)
  PG_W4S(false, true, 5)
  PG_W4S(true, false, 16)
  PG_W4S(true, true, 16)
  PG_W4S(false, false, 16)
  PG_W4S(false, true, 16)
  return nullptr;
}

size_t pg_walk4s_smem(int nc) {
  const size_t warp = nc <= 4   ? pgk::Walk4SGeom<4>::WARP
                      : nc <= 5 ? pgk::Walk4SGeom<5>::WARP
                                : pgk::Walk4SGeom<16>::WARP;
  return size_t(pgk::kWarpsPerBlock) * warp * sizeof(double2);
}
