#!/bin/bash
for rep in 1 2; do
for r in 1 8 4 16; do echo "== MK2_BULK_RAMP=$r"; MK2_BULK_RAMP=$r python tools/probe_e2e_row.py; done
done
timeout 900 python -m pytest tests -m gpu -q -x -k "bulk or c5 or pipelined" 2>&1 | tail -2
