#!/bin/bash
# Round evidence on the GPU box: the bench line, the ncu launch list of the same
# command, and one ncu --set full capture per dominant kernel (first cycle).
set -x
KEEP=${KEEP:-k5}
mkdir -p gpurun_out
python bench.py > gpurun_out/rp_bench.json 2> gpurun_out/rp_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/rp_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
    > gpurun_out/rp_ncu_launch.log 2>&1
A="--steps 1 --warmup 0 --no-e2e --no-cpu"
cap() {   # tag regex skip
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$2" -s $3 -c 1 \
      -o gpurun_out/rp_$1 python bench.py $A > gpurun_out/rp_ncu_$1.log 2>&1
  python tools/ncu_summary.py gpurun_out/rp_$1.ncu-rep 0.0 > gpurun_out/rp_$1_sum.txt 2>&1
  python tools/sass_hist.py gpurun_out/rp_$1.ncu-rep "." 0 > gpurun_out/rp_$1_hist.txt 2>&1
  [ "$KEEP" = "$1" ] || rm -f gpurun_out/rp_$1.ncu-rep    # gpurun_out returns <= 64 MiB
}
cap k5 "pg_residual_tma_kernel<.int.3, .int.2" 0 1   # the fused sweep K5 (TMA kernel, SWEEP mode)
cap k3 "pg_residual_tma_kernel<.int.3, .int.0" 0 1   # K3 (live first cycle)
cap k2a "pg_grad_x2" 0 1
cap k2b "pg_kcoef_x2" 0 1
cap up "upwind_smooth" 9 1           # finest-level smoother of the first cycle
cap rs "restrict_kernel" 0 1
echo done
