#!/bin/bash
# Round-2 check: GPU tests, c0 (graph) / c1 bench lines, c4 at N=1 (capacity), host info.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
free -g | head -2; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests/ -x -q -m gpu -rA -s 2>&1 | grep -E "parity |PASS|FAIL|Error|passed|failed" > gpurun_out/pytest_gpu.log; tail -4 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config c0 --no-cpu-baseline > gpurun_out/bench_c0.json 2> gpurun_out/bench_c0.err; echo c0_rc=$?; tail -c 600 gpurun_out/bench_c0.json
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo c1_rc=$?; tail -c 300 gpurun_out/bench_c1.json
if [ "$1" == "c4" ]; then
timeout 1500 python bench.py --config c4 --no-cpu-baseline --steps 5 --warmup 3 --e2e-reps 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4_rc=$?; tail -c 600 gpurun_out/bench_c4.json; tail -5 gpurun_out/bench_c4.err
fi
