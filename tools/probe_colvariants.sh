#!/bin/bash
# A/B of the column-major loop's output addressing (a: 0 = 64-bit pointer bump, 1 = 32-bit index) and
# checksum (s: 0 = mad.wide accumulate, 1 = IDP.2A half sums); three repetitions, interleaved.
for rep in 1 2 3; do
for lib in "" variants/libmk2_a0s0.so variants/libmk2_a0s1.so variants/libmk2_a1s0.so; do
  echo "== rep $rep lib=${lib:-default(a1s1)}"
  MK2_LIB=$lib python tools/probe_one.py col 20 262144 0 0 2>&1 | tail -1
  MK2_LIB=$lib python tools/probe_one.py col 20 65536 256 1073741824 2>&1 | tail -1
done; done
