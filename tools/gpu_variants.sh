#!/bin/bash
# tools/gpu_variants.sh NAME... : c1 parity of each variants/NAME.so, then c1 benches of the
# default build and every variant, interleaved twice (ms/step and per-kernel ms).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for name in "$@"; do
  YDG_LIB=$PWD/variants/$name.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_replica or c0_parity or vperm_c1" 2>&1 | tail -1
done
for rep in 1 2; do
for lib in paper_1903_11521_b200/libydg.so $(for n in "$@"; do echo variants/$n.so; done); do
  YDG_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-reps 1 > gpurun_out/bv.json 2>&1
  echo "$rep $lib $(grep -o '"ms_per_step": [0-9.]*\|"dm_local": {"ms_per_launch": [0-9.]*\|"dm_flux": {"ms_per_launch": [0-9.]*' gpurun_out/bv.json | tr '\n' ' ')"
done
done
