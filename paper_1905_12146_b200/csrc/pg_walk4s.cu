// Instantiations of the single-buffered 4-state walk (pg_walk4s.cuh): 4 rate
// categories, one lane per pattern, homogeneous / per-branch generators x
// with / without the Hessian x TC column counts NC in {4 (no missing /
// ambiguous codes), 5, 16}.
#include <algorithm>

#include "pg_walk4s.cuh"

#define PG_W4S(H, S, NC) \
  if (homog == H && hess == S && nc == NC) return reinterpret_cast<void*>(&pgk::walk4s_kernel<H, S, NC>);

// cherry-table instances (NC = 4: fused cherry steps; NC = 5: the e_k tables alone)
template <int NC>
static void* cherry_pick(bool homog, bool hess) {
  if (homog) return hess ? reinterpret_cast<void*>(&pgk::walk4s_kernel<true, true, NC, true>)
                         : reinterpret_cast<void*>(&pgk::walk4s_kernel<true, false, NC, true>);
  return hess ? reinterpret_cast<void*>(&pgk::walk4s_kernel<false, true, NC, true>)
              : reinterpret_cast<void*>(&pgk::walk4s_kernel<false, false, NC, true>);
}
void* pg_walk4s_cherry_kernel(bool homog, bool hess, int nc) {
  return nc == 4 ? cherry_pick<4>(homog, hess) : nc == 5 ? cherry_pick<5>(homog, hess) : nullptr;
}

void pg_cherry_tables(const int4* cherries, int ncherry, int N, int nc, const double* tc, const double* qtc, double* ct,
                      cudaStream_t stream) {
  if (ncherry <= 0) return;
  if (nc == 4) pgk::cherry_tc_kernel<<<(ncherry * 64 + 127) / 128, 128, 0, stream>>>(cherries, ncherry, N, tc, qtc, ct);
  else pgk::cherry_tc5_kernel<<<(ncherry * 100 + 127) / 128, 128, 0, stream>>>(cherries, ncherry, N, tc, ct);
}

// dynamic shared memory of the cherry instances (the gradient ones hold three tables per cherry child)
size_t pg_walk4s_cherry_smem() {
  return size_t(pgk::kWarpsPerBlock) * pgk::Walk4SGeom<4, true>::WARP * sizeof(double2);
}

void pg_cherry_codes(const int4* cherries, int ncherry, int N, long long Pc, int nc, const uint8_t* codes, uint8_t* cc,
                     cudaStream_t stream) {
  if (ncherry <= 0) return;
  const unsigned gx = unsigned(std::min<long long>((Pc + 255) / 256, 64));
  pgk::cherry_codes_kernel<<<dim3(gx, unsigned(ncherry)), 256, 0, stream>>>(cherries, ncherry, N, Pc, nc, codes, cc);
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
