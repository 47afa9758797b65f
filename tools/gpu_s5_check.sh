#!/bin/bash
# Fifth session, after YDG_QPF 7 -> 6: pytest -m gpu, smoke, default bench line, launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu -rA -s 2>&1 | grep -E "parity|PASS|FAIL|Error|passed|failed" > $O/s5b_pytest_gpu.log; tail -2 $O/s5b_pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 600 python bench.py > $O/s5b_bench_c1.json 2> $O/s5b_bench_c1.err; echo c1_rc=$?
python -c "import json;d=json.load(open('$O/s5b_bench_c1.json'));print('c1',d['value'],d['ms_per_step'],d['roofline']['frac'],d['step_roofline_frac'],d['e2e']['value'],{k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-reps 1"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/s5b_launches_c1.csv $CMD > $O/ncu_launch.log 2>&1
echo ncu_launch_rc=$?
timeout 600 ncu --set full --clock-control none -k regex:dm_local -s 1 -c 1 -o $O/s5b_prof_c1 $CMD > $O/ncu_full_c1.log 2>&1
echo ncu_c1_rc=$?
timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 5 --warmup 3 --e2e-reps 1 > $O/s5b_bench_c4.json 2> $O/s5b_bench_c4.err; echo c4_rc=$?
python -c "import json;d=json.load(open('$O/s5b_bench_c4.json'));print('c4',d['value'],d['ms_per_step'],d['roofline']['frac'],{k:v['ms_per_launch'] for k,v in d.get('kernels',{}).items()})"
