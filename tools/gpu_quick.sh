#!/bin/bash
# quick iteration: fp64 parity subset + c1 bench (kernel times)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "${KSEL:-orders_fp64 or c1_replica or vperm_c0 or vperm_orders or fused_step}" 2>&1 | tail -3
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --e2e-reps 1 > $O/q_bench_c1.json 2> $O/q_bench_c1.err; echo c1_rc=$?
python -c "import json;d=json.load(open('$O/q_bench_c1.json'));print('c1',d['ms_per_step'],d['roofline']['frac'],{k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
done
