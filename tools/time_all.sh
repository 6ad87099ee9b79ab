#!/bin/bash
for c in c2 c3 c4; do timeout 600 python tools/time_asm.py $c tiled,tiled_unordered,coloured 2>&1 | grep -E "tiled|coloured|E="; done
