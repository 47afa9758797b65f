#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-reps 1"
timeout 300 $CMD > gpurun_out/plain_fz.log 2>&1; echo plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dm_fused -s 2 -c 1 -o gpurun_out/prof_fused $CMD > gpurun_out/ncu_fused.log 2>&1
echo ncu_rc=$?; tail -3 gpurun_out/ncu_fused.log
