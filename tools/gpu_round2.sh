#!/bin/bash
# Round-2 evidence: GPU tests, smoke, bench lines of every workload, reference arm, ncu
# launch list + --set full of the c1 kernels.  Output -> gpurun_out/r2_*.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests/ -q -m gpu -rA -s 2>&1 | grep -E "parity|PASS|FAIL|Error|passed|failed" > $O/r2_pytest_gpu.log; tail -3 $O/r2_pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 600 python bench.py > $O/r2_bench_c1.json 2> $O/r2_bench_c1.err; echo c1_rc=$?; tail -c 300 $O/r2_bench_c1.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/r2_bench_ref.json 2> $O/r2_bench_ref.err; echo ref_rc=$?
for c in c0 c2 c3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-reps 1 > $O/r2_bench_$c.json 2> $O/r2_bench_$c.err; echo ${c}_rc=$?
done
timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 5 --warmup 3 --e2e-reps 1 > $O/r2_bench_c4.json 2> $O/r2_bench_c4.err; echo c4_rc=$?
timeout 600 python bench.py --config lina --e2e-reps 1 > $O/r2_bench_lina.json 2> $O/r2_bench_lina.err; echo lina_rc=$?
timeout 600 python bench.py --lts --steps 10 --warmup 3 > $O/r2_bench_lts.json 2> $O/r2_bench_lts.err; echo lts_rc=$?
timeout 900 python bench.py --sims 4 --no-cpu-baseline --steps 5 --warmup 3 --e2e-reps 1 > $O/r2_bench_sims4.json 2> $O/r2_bench_sims4.err; echo sims_rc=$?
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-reps 1"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_launches_c1.csv $CMD > $O/ncu_launch.log 2>&1
echo ncu_launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dm_ -s 2 -c 2 -o $O/r2_prof_c1 $CMD > $O/ncu_full.log 2>&1
echo ncu_full_rc=$?
