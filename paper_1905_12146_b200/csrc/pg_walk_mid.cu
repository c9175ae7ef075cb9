#include "pg_walk_inst.cuh"
void* pg_walk_kernel_mid(int MP, int LC) {
  PG_WALK_CASE(20, 1)
  return nullptr;
}
