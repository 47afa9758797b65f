#!/bin/bash
# Parity tests + bench + phase timing of the local kernel (variants/ydg_phases.so).
cd $GRAFT_REPO_ROOT
bash tools/gpu_iter.sh $1
YDG_LIB=$PWD/variants/ydg_phases.so timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-reps 1 2>&1 | grep -E "PH tile" | head -4
