#!/bin/bash
# K5 / K3 captures only (the first two of tools/round_profile.sh), for a re-run.
set -x
mkdir -p gpurun_out
A="--steps 1 --warmup 0 --no-e2e --no-cpu"
for spec in "k5|pg_residual_tma_kernel<.int.3, .int.2" "k3|pg_residual_tma_kernel<.int.3, .int.0"; do
  tag=${spec%%|*}; rx=${spec#*|}
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$rx" -s 0 -c 1 \
      -o gpurun_out/rp_$tag python bench.py $A > gpurun_out/rp_ncu_$tag.log 2>&1
  python tools/ncu_summary.py gpurun_out/rp_$tag.ncu-rep 0.0 > gpurun_out/rp_${tag}_sum.txt 2>&1
  python tools/sass_hist.py gpurun_out/rp_$tag.ncu-rep "." 0 > gpurun_out/rp_${tag}_hist.txt 2>&1
done
