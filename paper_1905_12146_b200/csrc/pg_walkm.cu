// Instantiations of the DMMA large-state walk kernel (pg_walkm.cuh).
#include "pg_walkm.cuh"

// `fast`: the gradient kernel with the common case's switches folded at compile
// time (pg_walkm.cuh FAST).  Instantiated for the amino-acid size, where it
// pays (C4 141.4 / 141.7 vs 144.8 / 145.6 ms on one box); for codons the leaner
// unit body schedules worse (C5 407.2 / 408.6 vs 397.5 / 397.6 ms)
template <int MP>
static void* pick(bool hess, bool fast) {
  if constexpr (MP == 20) {
    if (fast && !hess) return reinterpret_cast<void*>(&pgk::walkm_kernel<MP, false, true>);
  }
  return hess ? reinterpret_cast<void*>(&pgk::walkm_kernel<MP, true, false>)
              : reinterpret_cast<void*>(&pgk::walkm_kernel<MP, false, false>);
}

void* pg_walkm_kernel(int mp, bool hess, bool fast) {
  if (mp == 8) return pick<8>(hess, fast);
  if (mp == 16) return pick<16>(hess, fast);
  if (mp == 20) return pick<20>(hess, fast);
  if (mp == 24) return pick<24>(hess, fast);
  if (mp == 32) return pick<32>(hess, fast);
  if (mp == 64) return pick<64>(hess, fast);
  return nullptr;
}

// FAST's assumptions about the staged tip tables (NC columns of MP doubles fit
// the CTA's operand region and a P^T buffer) for this MP
bool pg_walkm_fast_tables_fit(int mp, int nc) {
  auto fits = [&](auto g) {
    using G = decltype(g);
    return !G::SOP || (nc * mp <= G::WPC * G::SL && nc * mp <= G::FRAG);
  };
  if (mp == 20) return fits(pgk::WalkMGeom<20>{});
  return false;
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
