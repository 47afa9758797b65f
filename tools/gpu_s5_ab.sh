#!/bin/bash
# Fifth session: parity subset of the re-annealed build (ck0 61 tiles), A/B c1 timing of
# the previous build (variants/base62.so) vs the new default and variants, three alternating reps.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "orders_fp64 or c1_replica or vperm_c0 or vperm_orders" 2>&1 | tail -1
for lib in "$@"; do
YDG_LIB=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "orders_fp64 or c1_replica or vperm_c0" 2>&1 | tail -1
done
for r in 1 2 3; do
for lib in paper_1903_11521_b200/libydg.so variants/base62.so "$@"; do
  YDG_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-reps 1 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$lib',round(d['ms_per_step'],3),{k:v['ms_per_launch'] for k,v in d['kernels'].items()},d['max_abs_q'])" 2>&1 | tail -1
done
done
