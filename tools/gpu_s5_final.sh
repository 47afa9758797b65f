#!/bin/bash
# Fifth-session final evidence of the committed code: pytest -m gpu, smoke, c1 bench line,
# reference arm, ncu launch list + --set full of the c1 kernels, then c2/c3/c0/c4/LTS/sims lines.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests/ -q -m gpu -rA -s 2>&1 | grep -E "parity|PASS|FAIL|Error|passed|failed" > $O/s5_pytest_gpu.log; tail -2 $O/s5_pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 600 python bench.py > $O/s5_bench_c1.json 2> $O/s5_bench_c1.err; echo c1_rc=$?
python -c "import json;d=json.load(open('$O/s5_bench_c1.json'));print('c1',d['value'],d['ms_per_step'],d['roofline']['frac'],d['step_roofline_frac'],d['e2e']['value'],d['max_abs_q'],{k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/s5_bench_ref.json 2> $O/s5_bench_ref.err; echo ref_rc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-reps 1"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/s5_launches_c1.csv $CMD > $O/ncu_launch.log 2>&1
echo ncu_launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dm_ -s 2 -c 2 -o $O/s5_prof_c1 $CMD > $O/ncu_full_c1.log 2>&1
echo ncu_c1_rc=$?
for c in c2 c3 c0; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-reps 1 > $O/s5_bench_$c.json 2> $O/s5_bench_$c.err; echo ${c}_rc=$?
  python -c "import json;d=json.load(open('$O/s5_bench_$c.json'));print('$c',d['value'],d['ms_per_step'],d['roofline']['frac'],d.get('max_abs_q'),{k:v['ms_per_launch'] for k,v in d.get('kernels',{}).items()})"
done
timeout 600 python bench.py --lts --steps 10 --warmup 3 > $O/s5_bench_lts.json 2> $O/s5_bench_lts.err; echo lts_rc=$?; tail -c 400 $O/s5_bench_lts.json
timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 5 --warmup 3 --e2e-reps 1 > $O/s5_bench_c4.json 2> $O/s5_bench_c4.err; echo c4_rc=$?
python -c "import json;d=json.load(open('$O/s5_bench_c4.json'));print('c4',d['value'],d['ms_per_step'],d['roofline']['frac'],{k:v['ms_per_launch'] for k,v in d.get('kernels',{}).items()})"
timeout 900 python bench.py --sims 4 --no-cpu-baseline --steps 5 --warmup 3 --e2e-reps 1 > $O/s5_bench_sims4.json 2> $O/s5_bench_sims4.err; echo sims_rc=$?
python -c "import json;d=json.load(open('$O/s5_bench_sims4.json'));print('sims4',d['value'],d['ms_per_step'])"
