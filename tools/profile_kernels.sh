#!/bin/bash
# ncu --set full of the team-table kernels of one R-MAT lpa() run.
# usage: tools/profile_kernels.sh SCALE OUTNAME SKIP COUNT
SCALE=${1:-24}; OUT=${2:-prof}; SKIP=${3:-0}; COUNT=${4:-8}
ncu --set full --clock-control none --import-source on \
    -k regex:"k_(wtab|block|cluster)" -s $SKIP -c $COUNT \
    -o gpurun_out/$OUT python tools/profile_run.py $SCALE
