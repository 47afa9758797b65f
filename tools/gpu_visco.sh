#!/bin/bash
# Viscoelastic iteration: parity tests of the P = 27 paths, c3 bench (tensor-core local
# kernel and, for comparison, the CSR kernel), optional ncu capture of vm_local.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "visco or c3" 2>&1 | tail -8
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_rc=$?
tail -c 1800 gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
if [ "$1" == "cmp" ]; then
  YDG_VISCO_GENERIC=1 timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bench_c3_csr.json 2>&1; echo csr_rc=$?
  tail -c 600 gpurun_out/bench_c3_csr.json
fi
if [ "$1" == "ncu" ]; then
  ncu --set full --clock-control none --import-source on -k regex:vm_local -s 1 -c 1 -o gpurun_out/prof_visco \
    python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --e2e-reps 1 > gpurun_out/ncu_visco.log 2>&1
  echo ncu_rc=$?
fi
