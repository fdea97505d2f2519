#!/bin/bash
# usage (on the GPU box): tools/ncu_top.sh <tag> <kernel regex> <launch skip> <launch count> [bench args]
# Runs the bench once plainly (must exit 0), then one ncu --set full capture.
set -e
tag=$1; regex=$2; skip=$3; count=$4; shift 4
args=${@:-"--steps 1 --warmup 0 --no-e2e --no-cpu"}
mkdir -p gpurun_out
python bench.py $args > gpurun_out/plain_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$regex" -s $skip -c $count \
    -o gpurun_out/prof_$tag python bench.py $args > gpurun_out/ncu_$tag.log 2>&1
echo "ncu done: gpurun_out/prof_$tag.ncu-rep"
