#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config lina --steps 3 --warmup 1 --e2e-reps 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/bench_lina.json 2>&1; echo rc=$?; grep -o '"ms_per_step": [0-9.]*\|"achieved": [0-9.]*' gpurun_out/bench_lina.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lina --csv --log-file gpurun_out/lina_launches.csv $CMD > /dev/null 2>&1; echo ncu1=$?
grep lina gpurun_out/lina_launches.csv | head -6 | cut -c1-300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lina -s 2 -c 2 -o gpurun_out/prof_lina $CMD > gpurun_out/ncu_lina.log 2>&1; echo ncu2=$?
