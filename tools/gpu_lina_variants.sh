#!/bin/bash
# LinA variants: parity + bench of the default build and variants/NAME.so
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for name in "$@"; do
  YDG_LIB=$PWD/variants/$name.so timeout 300 python -m pytest tests/test_gpu_lina.py -x -q 2>&1 | tail -1
done
for rep in 1 2; do
for lib in paper_1903_11521_b200/libydg.so $(for n in "$@"; do echo variants/$n.so; done); do
  YDG_LIB=$PWD/$lib timeout 300 python bench.py --config lina --no-cpu-baseline --steps 10 --warmup 3 --e2e-reps 1 > gpurun_out/bl.json 2>&1
  echo "$rep $lib $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bl.json)"
done
done
