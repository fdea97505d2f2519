#!/bin/bash
# ncu --set full captures of the 7-group linear-PG kernels (C5-weak generator at n_a = 8: a quarter
# of the ordinates so ncu's replay save/restore stays small).  Each capture runs only after the
# same bench command exited 0 without ncu.
B="--config c5w --na 8 --steps 1 --warmup 0 --no-e2e --no-cpu --no-extra --graphs off"
mkdir -p gpurun_out
python bench.py $B > gpurun_out/c5p_plain.json 2> gpurun_out/c5p_plain.err || exit 1
cap() {
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$2" -s $3 -c 1 \
      -o gpurun_out/c5p_$1 python bench.py $B > gpurun_out/c5p_ncu_$1.log 2>&1
  python tools/ncu_summary.py gpurun_out/c5p_$1.ncu-rep 0.0 > gpurun_out/c5p_$1_sum.txt 2>&1
  python tools/sass_hist.py gpurun_out/c5p_$1.ncu-rep "." 0 > gpurun_out/c5p_$1_hist.txt 2>&1
  [ "$KEEP" = "$1" ] || [ "$KEEP" = "all" ] || rm -f gpurun_out/c5p_$1.ncu-rep
}
for k in ${KERNELS:-k5 k3 k2 up}; do
  case $k in
    k5) cap k5 "pg_residual_tma_kernel<.int.1, .int.3" 0 ;;
    k3) cap k3 "pg_residual_tma_kernel<.int.1, .int.0" 0 ;;
    k2) cap k2 "pg_diffusivity_x2" 0 ;;
    k2a) cap k2a "pg_grad_x2" 0 ;;
    k2b) cap k2b "pg_kcoef" 0 ;;
    up) cap up "upwind_smooth" 0 ;;
  esac
done
echo done
