#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:gen_rowmajor_l2 --launch-skip 1 --launch-count 1 -f -o /tmp/l2tile \
    python tools/probe_grain_row_once.py 3 0 2 > /dev/null 2> /tmp/ncu_l2.err; echo "ncu rc=$?"; tail -3 /tmp/ncu_l2.err
python tools/ncu_summary.py /tmp/l2tile.ncu-rep gpurun_out/r02_ncu_grain_l2tile.txt "grain row64 L2-scratch tile kernel, 2^22 x 65536" | tail -60
ncu -i /tmp/l2tile.ncu-rep --page raw --csv | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for k,x in zip(h,v):
    if any(s in k for s in ('lts__t_sector','lts__t_bytes','lts__throughput','l1tex__m_','lts__t_sectors_srcunit_tex_op','hit_rate','dram__')): print(k,x)
" | head -60
