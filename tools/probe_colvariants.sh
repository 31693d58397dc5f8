#!/bin/bash
# A/B of column-major kernel variants (variants/*.so given as arguments): C2 geometry (one worker warp per
# sub-partition) and 8 warps per SM; three interleaved repetitions.
for rep in 1 2 3; do
for lib in "" "$@"; do
  echo "== rep $rep lib=${lib:-default}"
  MK2_LIB=$lib python tools/probe_one.py col 20 262144 0 0 2>&1 | tail -1
  MK2_LIB=$lib python tools/probe_one.py col 20 65536 256 1073741824 2>&1 | tail -1
done; done
