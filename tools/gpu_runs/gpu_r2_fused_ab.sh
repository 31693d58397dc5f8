#!/bin/bash
# fused bulk kernel: scheduling variants (variants/libmk2_f*.so), config-5 batch
for rep in 1 2; do
for lib in "" $(ls variants/libmk2_f*.so); do
  echo "== lib=${lib:-default}"; MK2_LIB=$lib python tools/probe_fused.py time 2>&1 | grep "fused" | head -1
done; done
MK2_LIB=variants/libmk2_f3.so python tools/probe_fused.py parity 2>&1 | tail -3
