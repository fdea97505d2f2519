#!/bin/bash
# A/B timing of library variants on the GPU box: tools/ab_libs.sh name1 name2 ... (ablib/<name>.so; ablib/ is git-ignored but travels)
# Prints ms/step and per-kernel ms for each variant, two alternating rounds.
LIB=paper_2301_09991_b200/libconvsn_sm100.so
mkdir -p gpurun_out
cp $LIB gpurun_out/.orig.so
for r in 1 2; do
  for v in "$@"; do
    cp ${ABDIR:-ablib}/$v.so $LIB
    timeout 300 python bench.py --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/ab_${v}_$r.json 2> gpurun_out/ab_err_$v.txt
    python - "$v" gpurun_out/ab_${v}_$r.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
k = {n: round(v["ms_avg"], 3) for n, v in d["kernels"].items()}
print(sys.argv[1], round(d["ms_per_step"], 3), k)
PY
  done
done
cp gpurun_out/.orig.so $LIB
