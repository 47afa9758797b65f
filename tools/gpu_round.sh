#!/bin/bash
# Round evidence: GPU tests (incl. full-size sampled parity), smoke, default bench (c1, with the
# oracle CPU baseline), the reference arm, c2/c3 bench lines, ncu launch list + --set full.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/ -x -q -m gpu -rA 2>&1 | tail -30 > gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench_rc=$?; tail -c 400 gpurun_out/bench_c1.json
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 600 python bench.py --config c2 --no-cpu-baseline --e2e-reps 1 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2_rc=$?
timeout 600 python bench.py --config c3 --no-cpu-baseline --e2e-reps 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3_rc=$?
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-reps 1"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo ncu_launch_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dm_ -s 2 -c 2 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu_full_rc=$?
