#include "pg_walk_inst.cuh"
void* pg_walk_kernel_large(int MP, int LC) {
  PG_WALK_CASE(32, 1)
  PG_WALK_CASE(64, 1)
  return nullptr;
}
