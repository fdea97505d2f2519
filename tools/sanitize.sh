#!/bin/bash
# compute-sanitizer over the small GPU parity tests (memcheck, racecheck, synccheck,
# initcheck): the TMA/mbarrier PG kernels, the cp.async stagers, the packed smoother,
# transfers, boundary, generic convolution, and a ThreadComm domain decomposition with
# a ragged slab (nx % 8 != 0 beside a ghost side).  Logs land in gpurun_out/san_*.log,
# one rc line per tool in gpurun_out/san_summary.txt.  Run on the GPU box:
#   gpurun --timeout 3000 -- 'bash tools/sanitize.sh'
set -u
mkdir -p gpurun_out
: > gpurun_out/san_summary.txt
K="boundary or upwind_residual_and_sweeps or (pg_operators and (1 or 3)) or transfers_and_correction or tma_residual or split_diffusivities or kcoef_tma or upwind_x2 or generic_convolution or (pg_cycles_with_state and 3)"
SAN="compute-sanitizer --print-limit 40 --error-exitcode 9 --target-processes all"
for tool in memcheck racecheck synccheck initcheck; do
    extra=""
    [ "$tool" = "racecheck" ] && extra="--racecheck-report analysis"
    timeout 1500 $SAN --tool $tool $extra python -m pytest -q -x -p no:cacheprovider \
        tests/test_gpu_parity.py -m gpu -k "$K" > gpurun_out/san_$tool.log 2>&1
    echo "$tool parity-subset rc=$?" >> gpurun_out/san_summary.txt
done
timeout 1500 $SAN --tool memcheck python -m pytest -q -x -p no:cacheprovider \
    tests/test_dd_gpu.py -m gpu -k "ragged" > gpurun_out/san_memcheck_dd.log 2>&1
echo "memcheck dd-ragged rc=$?" >> gpurun_out/san_summary.txt
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed" gpurun_out/san_*.log >> gpurun_out/san_summary.txt
cat gpurun_out/san_summary.txt
