#!/bin/bash
# Grain v1 keystream kernels, default library vs variants/*.so given as arguments; three interleaved repetitions
for rep in 1 2 3; do
for lib in "" "$@"; do
  echo "== rep $rep lib=${lib:-default}"
  MK2_LIB=$lib python tools/probe_grain.py col 22 65536 2>&1 | tail -1
  MK2_LIB=$lib python tools/probe_grain.py row 22 65536 2>&1 | tail -1
done; done
