#!/bin/bash
# Fresh-box check of the committed code: GPU tests, smoke, c1 / c2 / c3 bench lines.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -4 > $O/base_pytest.log; cat $O/base_pytest.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-reps 1 > $O/base_bench_$c.json 2> $O/base_bench_$c.err; echo ${c}_rc=$?
  python -c "import json;d=json.load(open('$O/base_bench_$c.json'));print('$c',d['ms_per_step'],{k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
done
