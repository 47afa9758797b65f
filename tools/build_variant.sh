#!/bin/bash
# Build a library variant: tools/build_variant.sh NAME [ENV=VAL ...] (generator / nvcc env)
# e.g. tools/build_variant.sh ck4 YDG_GEN_CKROWS=4 ; YDG_NVFLAGS=-DYDG_DM_LANES=8
set -e
cd /root/repo
name=$1; shift
env "$@" python -m paper_1903_11521_b200.gen.dmma > /dev/null
env "$@" python -m paper_1903_11521_b200.gen.kernels > /dev/null
env "$@" YDG_BUILD_DIR=/root/repo/variants/_b_$name YDG_LIB=/root/repo/variants/$name.so python -m paper_1903_11521_b200.build > /dev/null
rm -rf /root/repo/variants/_b_$name
python -m paper_1903_11521_b200.gen.dmma > /dev/null   # restore the default generated sources
python -m paper_1903_11521_b200.gen.kernels > /dev/null
echo built variants/$name.so
