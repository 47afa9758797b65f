#!/bin/bash
# tools/gpu_sanitize.sh TOOL : one compute-sanitizer tool over tools/sanitize_cases.py
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tool=${1:?tool}
timeout 300 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo plain_rc=$?
timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
echo ${tool}_rc=$?
tail -12 gpurun_out/sanitize_$tool.log
