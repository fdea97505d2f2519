#!/bin/bash
# Round evidence on the GPU box: the bench line, the ncu launch list of the same
# command, and one ncu --set full capture per dominant kernel (first cycle).
# Each ncu command runs only after the same bench command exited 0 without ncu.
set -x
KEEP=${KEEP:-k5}
mkdir -p gpurun_out
python bench.py > gpurun_out/rp_bench.json 2> gpurun_out/rp_bench.err || exit 1
A="--steps 2 --warmup 1 --no-e2e --no-cpu --no-extra"
python bench.py $A > gpurun_out/rp_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/rp_launches.csv python bench.py $A \
    > gpurun_out/rp_ncu_launch.log 2>&1
B="--steps 1 --warmup 0 --no-e2e --no-cpu --no-extra"
python bench.py $B > gpurun_out/rp_plain1.json 2>&1 || exit 1
cap() {   # tag regex skip
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$2" -s $3 -c 1 \
      -o gpurun_out/rp_$1 python bench.py $B > gpurun_out/rp_ncu_$1.log 2>&1
  python tools/ncu_summary.py gpurun_out/rp_$1.ncu-rep 0.0 > gpurun_out/rp_$1_sum.txt 2>&1
  python tools/sass_hist.py gpurun_out/rp_$1.ncu-rep "." 0 > gpurun_out/rp_$1_hist.txt 2>&1
  [ "$KEEP" = "$1" ] || rm -f gpurun_out/rp_$1.ncu-rep    # gpurun_out returns <= 64 MiB
}
cap k5 "pg_residual_tma_kernel<.int.3, .int.3" 0 1   # fused sweep K5 (folded correction, 3 fields)
cap k3 "pg_residual_tma_kernel<.int.3, .int.0" 0 1   # K3 (live first cycle)
cap k2a "pg_grad_x2" 0 1
cap k2b "pg_kcoef_tma" 0 1
cap up "upwind_smooth_tma" 0 1                       # finest-level smoother (TMA columns)
cap rs "restrict_kernel" 0 1
echo done
