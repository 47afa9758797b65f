#!/bin/bash
# DMMA chain microbenchmark; parity subset of a variant library; A/B c1 timing vs default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./tools/dmma_chains > gpurun_out/dmma_chains.jsonl 2>&1; echo chains_rc=$?
for lib in "$@"; do
YDG_LIB=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "orders_fp64 or c1_replica or vperm_c0 or vperm_orders or fused_step or local_time" 2>&1 | tail -1
done
for r in 1 2 3; do
for lib in paper_1903_11521_b200/libydg.so "$@"; do
  YDG_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-reps 1 > gpurun_out/ab.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$lib',round(d['ms_per_step'],3),{k:v['ms_per_launch'] for k,v in d['kernels'].items()})" 2>&1 | tail -1
done
done
