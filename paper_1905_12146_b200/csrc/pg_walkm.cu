// Instantiations of the DMMA large-state walk kernel (pg_walkm.cuh).
#include "pg_walkm.cuh"

template <int MP>
static void* pick(bool hess) {
  return hess ? reinterpret_cast<void*>(&pgk::walkm_kernel<MP, true>)
              : reinterpret_cast<void*>(&pgk::walkm_kernel<MP, false>);
}

void* pg_walkm_kernel(int mp, bool hess) {
  if (mp == 8) return pick<8>(hess);
  if (mp == 16) return pick<16>(hess);
  if (mp == 20) return pick<20>(hess);
  if (mp == 24) return pick<24>(hess);
  if (mp == 32) return pick<32>(hess);
  if (mp == 64) return pick<64>(hess);
  return nullptr;
}

size_t pg_walkm_smem(int mp) {
  if (mp == 8) return pgk::WalkMGeom<8>::smem_bytes();
  if (mp == 16) return pgk::WalkMGeom<16>::smem_bytes();
  if (mp == 20) return pgk::WalkMGeom<20>::smem_bytes();
  if (mp == 24) return pgk::WalkMGeom<24>::smem_bytes();
  if (mp == 32) return pgk::WalkMGeom<32>::smem_bytes();
  if (mp == 64) return pgk::WalkMGeom<64>::smem_bytes();
  return 0;
}

int pg_walkm_wpc(int mp) {
  if (mp == 8) return pgk::WalkMGeom<8>::WPC;
  if (mp == 16) return pgk::WalkMGeom<16>::WPC;
  if (mp == 20) return pgk::WalkMGeom<20>::WPC;
  if (mp == 24) return pgk::WalkMGeom<24>::WPC;
  if (mp == 32) return pgk::WalkMGeom<32>::WPC;
  if (mp == 64) return pgk::WalkMGeom<64>::WPC;
  return 4;
}
