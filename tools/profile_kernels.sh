#!/bin/bash
# ncu --set full of the shared-table team kernels of one R-MAT lpa() run.
# usage: tools/profile_kernels.sh SCALE OUTNAME SKIP COUNT [REGEX]
SCALE=${1:-24}; OUT=${2:-prof}; SKIP=${3:-0}; COUNT=${4:-8}; RE=${5:-"k_team|k_cluster|k_hub_accum"}
ncu --set full --clock-control none --import-source on \
    -k regex:"$RE" -s $SKIP -c $COUNT \
    -o gpurun_out/$OUT python tools/profile_run.py $SCALE
