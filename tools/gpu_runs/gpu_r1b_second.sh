#!/bin/bash
mkdir -p gpurun_out
timeout 1500 tools/probe_rblock.sh variants/libmk2_k5.so variants/libmk2_k6.so > gpurun_out/probe_rblock2.txt 2>&1; cat gpurun_out/probe_rblock2.txt
