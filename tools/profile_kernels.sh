#!/bin/bash
# ncu --set full of each table tier kernel in pass 1 (the first non-PL pass) of an R-MAT run.
# usage: tools/profile_kernels.sh SCALE OUTNAME
SCALE=${1:-24}; OUT=${2:-prof}
ncu --set full --clock-control none --import-source on \
    -k regex:"k_(wtab|block|cluster|group|thread)" -s 14 -c 7 \
    -o gpurun_out/$OUT python tools/profile_run.py $SCALE
