# A/B of the K2 resident-CTA target (CSN_K2_MINB) on the GPU box: rebuild, bench C4 and C3
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr"
for m in 3 4 3 4; do   # the default is per order (see pg_kernels_x2.cuh)
  touch paper_2301_09991_b200/csrc/pg_part.cu
  make -s all NVFLAGS="$F -DCSN_K2_MINB=$m" > /dev/null 2>&1 || echo "build failed"
  for c in c4 c3; do
    python bench.py --config $c --no-e2e --no-cpu --graphs off > gpurun_out/ab_$c.log 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/ab_$c.log') if l.startswith('{')][-1]); print('minb=$m $c', round(d['ms_per_step'],3), {k:round(v['ms_avg'],3) for k,v in d['kernels'].items()})"
  done
done
