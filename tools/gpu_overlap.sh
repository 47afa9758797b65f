#!/bin/bash
# EXPERIMENT: local and flux kernels concurrently (wrong numerics, timing only)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "order5_generic or coexist or step_graph" 2>&1 | tail -2
for v in "" "148,296" "148,592" "296,296"; do
  YDG_LIB=$PWD/variants/g11.so YDG_EXP_OVERLAP=$v timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-reps 1 > gpurun_out/ov.json 2>&1
  echo "g11 overlap=[$v]"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/ov.json
done
for v in "" ; do
  YDG_EXP_OVERLAP=$v timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-reps 1 > gpurun_out/ov.json 2>&1
  echo "default overlap=[$v]"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/ov.json
done
