#!/bin/bash
# Fourth-session final check of the committed code: pytest -m gpu, smoke, c1 bench line,
# reference arm, ncu launch list of the bench command.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests/ -q -m gpu -rA -s 2>&1 | grep -E "parity|PASS|FAIL|Error|passed|failed" > $O/s4_pytest_gpu.log; tail -2 $O/s4_pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 600 python bench.py > $O/s4_bench_c1.json 2> $O/s4_bench_c1.err; echo c1_rc=$?
python -c "import json;d=json.load(open('$O/s4_bench_c1.json'));print('c1',d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'],{k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/s4_bench_ref.json 2> $O/s4_bench_ref.err; echo ref_rc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-reps 1"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/s4_launches_c1.csv $CMD > $O/ncu_launch.log 2>&1
echo ncu_launch_rc=$?
