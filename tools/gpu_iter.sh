#!/bin/bash
# One GPU iteration: parity tests, bench, optional full ncu capture of the dm_ kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -c 2500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ "$1" == "ncu" ]; then
  CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-reps 1"
  ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-dm_}" -s 2 -c 2 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
  echo ncu_rc=$?
fi
