#!/bin/bash
# A/B of row-major kernel variants (variants/*.so passed as arguments), three interleaved repetitions
for rep in 1 2 3; do
for lib in "" "$@"; do
  echo "== rep $rep lib=${lib:-default}"
  MK2_LIB=$lib python tools/probe_one.py row 22 16384 0 0 2>&1 | tail -1
  MK2_LIB=$lib python tools/probe_one.py row 24 8192 0 0 2>&1 | tail -1
done; done
