#!/bin/bash
# Runs the peak micro-benchmarks with a clock sampler; output in gpurun_out/.
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/peaks | tee gpurun_out/peaks.json
kill $SMI || true
