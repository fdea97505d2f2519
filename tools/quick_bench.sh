#!/bin/bash
# usage: tools/quick_bench.sh "c3" "c2 --steps 17" ...  -> ms/step and per-stage ms of each config
for cfg in "$@"; do
  python bench.py --config $cfg --no-extra --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$cfg', round(d['ms_per_step'],4), {k:round(v['ms_avg'],4) for k,v in d['kernels'].items()})"
done
