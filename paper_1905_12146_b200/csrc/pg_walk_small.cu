#include "pg_walk_inst.cuh"
void* pg_walk_kernel_small(int MP, int LC) {
  PG_WALK_CASE(4, 1)
  PG_WALK_CASE(4, 2)
  PG_WALK_CASE(4, 4)
  PG_WALK_CASE(8, 1)
  PG_WALK_CASE(8, 2)
  return nullptr;
}
