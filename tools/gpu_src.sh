#!/bin/bash
# ncu source-level captures (SASS windows, stall reasons) of the c3 and c2 kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c3 c2; do
  CMD="python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --e2e-reps 1"
  timeout 300 $CMD > /dev/null 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ader_|vm_" -s 2 -c 2 -o gpurun_out/prof_src_$c $CMD > gpurun_out/ncu_src_$c.log 2>&1
  echo $c ncu_rc=$?
done
