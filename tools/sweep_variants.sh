#!/bin/bash
for v in "" "FEM_SWEEP_COL=7x5" "FEM_SWEEP_COL=6x5"; do
  echo "== variant: $v"
  env $v timeout 300 python tools/time_asm.py c5 tiled 2>&1 | grep -E "tiled"
done
