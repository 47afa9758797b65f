#!/bin/bash
# Fifth session: ncu --set full with source of the c3 kernels (vm_local / vm_neigh) on the
# sparser-direction code, plus its launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out
CMD="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-reps 1"
timeout 300 $CMD > $O/plain_c3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/s5_launches_c3.csv $CMD > $O/ncu_launch_c3.log 2>&1
echo ncu_launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vm_ -s 2 -c 2 -o $O/s5_prof_c3 $CMD > $O/ncu_full_c3.log 2>&1
echo ncu_c3_rc=$?
ls -la $O/*.ncu-rep
