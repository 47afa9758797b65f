#!/bin/bash
# Re-entry check: full pytest -m gpu, smoke, default c1 bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests/ -q -m gpu -rA -s 2>&1 | grep -E "parity|PASS|FAIL|Error|passed|failed" > $O/chk_pytest_gpu.log; tail -3 $O/chk_pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 600 python bench.py > $O/chk_bench_c1.json 2> $O/chk_bench_c1.err; echo c1_rc=$?
python -c "import json;d=json.load(open('$O/chk_bench_c1.json'));print('c1',d['value'],d['ms_per_step'],d['roofline']['frac'],{k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
