#!/bin/bash
# A/B of the PG y-chunk count (csn_set_tuning pg_chunks): C4, C3 and a DD rank at N = 8
for n in 0 1 2 4; do echo "== pg_chunks=$n"; 
  python bench.py --config c4 --no-extra --no-e2e --no-cpu --tune pg_chunks=$n 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4', round(d['ms_per_step'],3), {k:round(v['ms_avg'],3) for k,v in d['kernels'].items()})"
done
for n in 0 1 2 4 8; do echo "== pg_chunks=$n"; CSN_DD_OVERLAP=0 CSN_TUNE=pg_chunks=$n python tools/dd_rank_cost.py 8 | tail -1; done
for n in 0 2 4 8; do echo "== pg_chunks=$n"; python bench.py --config c3 --no-extra --no-e2e --no-cpu --tune pg_chunks=$n 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3', round(d['ms_per_step'],3), {k:round(v['ms_avg'],3) for k,v in d['kernels'].items()})"
done
