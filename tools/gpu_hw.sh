#!/bin/bash
# ncu source-level captures (for tools/hw_flops.py) of the c2 / c3 kernels, the max|Q|
# diagnostic tests and one c1 bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_memcheck.py -q -k "max_abs" 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --e2e-reps 1 --no-cpu-baseline > gpurun_out/hw_c1.json 2> gpurun_out/hw_c1.err; tail -c 600 gpurun_out/hw_c1.json
for c in c2 c3; do
  CMD="python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --e2e-reps 1"
  timeout 300 $CMD > /dev/null 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ader_|vm_" -s 2 -c 2 -o gpurun_out/prof_src_$c $CMD > gpurun_out/ncu_src_$c.log 2>&1
  echo $c ncu_rc=$?
done
