#!/bin/bash
# Variant experiment: tools/gpu_variant.sh NAME -- parity (incl. full size and multi-rank
# loopback) of variants/NAME.so, then a c1 bench of the default build and of the variant.
# Build the variant with YDG_NVFLAGS=... YDG_BUILD_DIR=variants/_b_NAME YDG_LIB=variants/NAME.so
# python -m paper_1903_11521_b200.build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
name=${1:?variant name}
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
YDG_LIB=$PWD/variants/$name.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_multirank_loopback.py -x -q 2>&1 | tail -2
for lib in paper_1903_11521_b200/libydg.so variants/$name.so; do
  YDG_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-reps 1 > gpurun_out/b_$(basename $lib .so).json 2>&1
  echo $lib; tail -c 1500 gpurun_out/b_$(basename $lib .so).json | grep -o '"ms_per_step": [0-9.]*\|"dm_local": {"ms_per_launch": [0-9.]*\|"dm_flux": {"ms_per_launch": [0-9.]*'
done
