#!/bin/bash
# ncu --set full with source-level stalls of the c1 kernels (one capture each)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-reps 1"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-dm_}" -s 2 -c 2 -o gpurun_out/prof_src $CMD > gpurun_out/ncu_src.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_src.log
