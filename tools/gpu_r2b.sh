#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -x -q -m gpu -rA -s 2>&1 | grep -E "parity |PASS|FAIL|Error|passed|failed" > gpurun_out/pytest_gpu.log; tail -4 gpurun_out/pytest_gpu.log
for ro in 1 0 1 0; do
  YDG_REORDER=$ro timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-reps 1 > gpurun_out/bv.json 2>&1
  echo "reorder=$ro $(grep -o '"ms_per_step": [0-9.]*\|"dm_local": {"ms_per_launch": [0-9.]*\|"dm_flux": {"ms_per_launch": [0-9.]*' gpurun_out/bv.json | tr '\n' ' ')"
done
for ro in 1 0; do
  YDG_REORDER=$ro timeout 400 python bench.py --config c2 --no-cpu-baseline --steps 5 --warmup 3 --e2e-reps 1 > gpurun_out/bv.json 2>&1
  echo "c2 reorder=$ro $(grep -o '"ms_per_step": [0-9.]*\|"ader_local": {"ms_per_launch": [0-9.]*\|"ader_neigh": {"ms_per_launch": [0-9.]*' gpurun_out/bv.json | tr '\n' ' ')"
done
