#!/bin/bash
mkdir -p gpurun_out
python tools/probe_small_once.py 64 65536
python tools/probe_small_once.py 18944 16384
ncu --set full --clock-control none --import-source on -k regex:gen_colmajor_kernel --launch-skip 1 --launch-count 1 -f -o /tmp/coop \
    python tools/probe_small_once.py 64 65536 > /dev/null 2> /tmp/ncu_coop.err; echo "ncu rc=$?"; tail -2 /tmp/ncu_coop.err
python tools/ncu_summary.py /tmp/coop.ncu-rep gpurun_out/r02b_ncu_coop_gen_colmajor_64lanes.txt "coop::gen_colmajor_kernel, 64 instances (2 warps) x 65536 clocks: the reference's own calling unit; latency-bound by design" | tail -42
