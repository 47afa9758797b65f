#!/bin/bash
# Sparser derivative directions: full GPU parity suite, smoke, c1/c2/c3 bench lines.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -rA -s -x 2>&1 | grep -E "parity|PASS|FAIL|Error|passed|failed|assert" > $O/kd_pytest_gpu.log; tail -4 $O/kd_pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 600 python bench.py > $O/kd_bench_c1.json 2> $O/kd_bench_c1.err; echo c1_rc=$?
python -c "import json;d=json.load(open('$O/kd_bench_c1.json'));print('c1',d['value'],d['ms_per_step'],d['roofline']['frac'],d['step_roofline_frac'],{k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
for c in c2 c3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-reps 1 > $O/kd_bench_$c.json 2> $O/kd_bench_$c.err; echo ${c}_rc=$?
  python -c "import json;d=json.load(open('$O/kd_bench_$c.json'));print('$c',d['value'],d['ms_per_step'],d['roofline']['frac'],{k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
done
