#!/bin/bash
# Fifth session: L2 re-prefetch bits of the local kernel (YDG_QPF) re-measured on the
# sparser-direction code; two alternating repetitions, c1.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do
for lib in paper_1903_11521_b200/libydg.so "$@"; do
  YDG_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-reps 1 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$lib',round(d['ms_per_step'],3),{k:v['ms_per_launch'] for k,v in d['kernels'].items()})" 2>&1 | tail -1
done
done
