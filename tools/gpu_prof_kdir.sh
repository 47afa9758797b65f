#!/bin/bash
# ncu evidence of the sparser-direction kernels: c1 launch list, --set full with source of the
# c1 and c2 kernels (tools/hw_flops.py, tools/ncu_summary.py read them back here).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-reps 1"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/kd_launches_c1.csv $CMD > $O/ncu_launch.log 2>&1
echo ncu_launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dm_ -s 2 -c 2 -o $O/kd_prof_c1 $CMD > $O/ncu_full_c1.log 2>&1
echo ncu_c1_rc=$?
CMD2="python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --e2e-reps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ader_ -s 2 -c 2 -o $O/kd_prof_c2 $CMD2 > $O/ncu_full_c2.log 2>&1
echo ncu_c2_rc=$?
ls -la $O/*.ncu-rep
