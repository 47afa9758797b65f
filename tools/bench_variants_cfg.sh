#!/bin/bash
# Bench each library variant on workload $1 (default c1).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=${1:-c1}
for lib in paper_1903_11521_b200/libydg.so variants/*.so; do
  name=$(basename $lib .so)
  YDG_LIB=$PWD/$lib timeout 600 python bench.py --config $CFG --steps 4 --warmup 2 --no-cpu-baseline --e2e-reps 1 > gpurun_out/v_$name.json 2> gpurun_out/v_$name.err
  python3 -c "
import json
d=json.loads(open('gpurun_out/v_$name.json').read().strip().splitlines()[-1])
k=d['kernels']; ks=list(k)
print('$name', round(d['ms_per_step'],2), ks[0], k[ks[0]]['ms_per_launch'], ks[1], k[ks[1]]['ms_per_launch'])
" || tail -3 gpurun_out/v_$name.err
done
