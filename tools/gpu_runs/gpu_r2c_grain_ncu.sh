#!/bin/bash
# ncu --set full of the default Grain v1 row-major kernel after the last session's changes (top-of-window copies,
# in-register transposes, line-completing evict_first sector) and of the column-major kernel with the 32-clock window.
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:gen_rowmajor_kernel --launch-skip 1 --launch-count 1 -f -o /tmp/grow \
    python tools/probe_grain_row_once.py 0 0 2 > /dev/null 2> /tmp/ncu_grow.err; echo "ncu rc=$?"; tail -3 /tmp/ncu_grow.err
python tools/ncu_summary.py /tmp/grow.ncu-rep gpurun_out/r02c_ncu_grain_rowmajor.txt "grain v1 row-major default kernel (7 warps/SM, fused transposes, policy 3), 2^22 x 65536" | tail -70
cp /tmp/grow.ncu-rep gpurun_out/r02c_grain_rowmajor.ncu-rep
