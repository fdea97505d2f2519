B="--config c3 --steps 1 --warmup 0 --no-e2e --no-cpu --no-extra --graphs off"
python bench.py $B > gpurun_out/c3p_plain.json 2>&1 || exit 1
cap() {
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$2" -s $3 -c 1 \
      -o gpurun_out/c3p_$1 python bench.py $B > gpurun_out/c3p_ncu_$1.log 2>&1
  python tools/ncu_summary.py gpurun_out/c3p_$1.ncu-rep 0.0 > gpurun_out/c3p_$1_sum.txt 2>&1
  python tools/sass_hist.py gpurun_out/c3p_$1.ncu-rep "." 0 > gpurun_out/c3p_$1_hist.txt 2>&1
}
cap k5 "pg_residual_tma_kernel<.int.1, .int.3" 0
cap k3 "pg_residual_tma_kernel<.int.1, .int.0" 0
cap k2 "pg_diffusivity_x2" 0
cap up "upwind_smooth_x2" 1
