#!/bin/bash
# fused step kernel: parity + bitwise tests, c1 bench (fused and two-kernel)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_step or fused_kernel or orders_fp64 or c1_replica or vperm_c0 or graph" 2>&1 | tail -5
timeout 600 python bench.py --no-cpu-baseline --e2e-reps 1 > $O/fz_bench_c1.json 2> $O/fz_bench_c1.err; echo c1_rc=$?
tail -3 $O/fz_bench_c1.err
python -c "import json;d=json.load(open('$O/fz_bench_c1.json'));print('fused',d['ms_per_step'],d['roofline']['frac'],{k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
YDG_FUSED=0 timeout 600 python bench.py --no-cpu-baseline --e2e-reps 1 > $O/fz_bench_c1_off.json 2> $O/fz_bench_c1_off.err; echo c1off_rc=$?
python -c "import json;d=json.load(open('$O/fz_bench_c1_off.json'));print('two-kernel',d['ms_per_step'],d['roofline']['frac'],{k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
