#!/bin/bash
for rep in 1 2; do
echo "== old policy (8 warps per SM per block, 512 MiB tiles)"; MK2_ROW_WORKERS=8 MK2_ROW_TILE_FACTOR=16 python tools/probe_e2e_row.py
echo "== new policy (4 warps per SM per block, 256 MiB tiles)"; python tools/probe_e2e_row.py
done
