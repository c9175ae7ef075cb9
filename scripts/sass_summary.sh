#!/bin/bash
# Static SASS evidence per kernel: DMMA (fp64 tensor core), UBLKCP (1-D bulk
# copy / TMA engine), LDGSTS (cp.async), SYNCS (mbarrier), and register use.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}/paper_1905_12146_b200/_build"
for o in pg_walkm.o pg_walk4s.o pg_walk4.o pg_walk4b.o pg_walkl.o pg_compress.o pg_engine.o; do
  cuobjdump -sass "$o" | awk -v obj="$o" '
    /Function :/ { if (name != "") printf "%-12s %-70s DMMA %4d  UBLKCP %3d  LDGSTS %4d  SYNCS %3d  DFMA %5d  total %6d\n", obj, name, d, u, l, sy, f, n;
                   name = $3; d = u = l = sy = f = n = 0; next }
    /\/\*[0-9a-f]+\*\// { n++ }
    /DMMA/ { d++ } /UBLKCP/ { u++ } /LDGSTS/ { l++ } /SYNCS/ { sy++ } / DFMA/ { f++ }
    END { if (name != "") printf "%-12s %-70s DMMA %4d  UBLKCP %3d  LDGSTS %4d  SYNCS %3d  DFMA %5d  total %6d\n", obj, name, d, u, l, sy, f, n }'
done
