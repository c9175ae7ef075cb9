// Instantiations of the DMMA large-state walk kernel (pg_walkm.cuh).
#include "pg_walkm.cuh"

void* pg_walkm_kernel(int mp) {
  if (mp == 16) return reinterpret_cast<void*>(&pgk::walkm_kernel<16>);
  if (mp == 20) return reinterpret_cast<void*>(&pgk::walkm_kernel<20>);
  if (mp == 24) return reinterpret_cast<void*>(&pgk::walkm_kernel<24>);
  if (mp == 32) return reinterpret_cast<void*>(&pgk::walkm_kernel<32>);
  if (mp == 64) return reinterpret_cast<void*>(&pgk::walkm_kernel<64>);
  return nullptr;
}

size_t pg_walkm_smem(int mp) {
  if (mp == 16) return pgk::WalkMGeom<16>::smem_bytes();
  if (mp == 20) return pgk::WalkMGeom<20>::smem_bytes();
  if (mp == 24) return pgk::WalkMGeom<24>::smem_bytes();
  if (mp == 32) return pgk::WalkMGeom<32>::smem_bytes();
  if (mp == 64) return pgk::WalkMGeom<64>::smem_bytes();
  return 0;
}

int pg_walkm_wpc(int mp) {
  if (mp == 16) return pgk::WalkMGeom<16>::WPC;
  if (mp == 20) return pgk::WalkMGeom<20>::WPC;
  if (mp == 24) return pgk::WalkMGeom<24>::WPC;
  if (mp == 32) return pgk::WalkMGeom<32>::WPC;
  if (mp == 64) return pgk::WalkMGeom<64>::WPC;
  return 4;
}
