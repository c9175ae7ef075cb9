// Explicit instantiation helpers: each pg_walk_*.cu translation unit compiles a
// subset of the (padded states MP, categories-per-lane LC) kernel variants so
// the build parallelises; pg_engine.cu fetches the launch pointers.
#pragma once
#include "pg_walk.cuh"

#define PG_WALK_CASE(MP_, LC_) \
  if (MP == MP_ && LC == LC_) return reinterpret_cast<void*>(&pgk::walk_kernel<MP_, LC_>);
