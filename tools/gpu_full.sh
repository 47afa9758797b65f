#!/bin/bash
# Full GPU pass: parity tests, smoke, default bench, launch list, ncu --set full of the top kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-reps 1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-dm_}" -s 2 -c 2 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_full.log
