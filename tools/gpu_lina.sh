#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lina.py -x -q -rA -s 2>&1 | grep -E "lina parity|passed|failed|Error" | tail -12
timeout 600 python bench.py --config lina --steps 5 --warmup 2 --e2e-reps 1 > gpurun_out/bench_lina.json 2> gpurun_out/bench_lina.err; echo lina_rc=$?
tail -c 1500 gpurun_out/bench_lina.json; tail -3 gpurun_out/bench_lina.err
