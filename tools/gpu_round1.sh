set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py --smoke 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-reps 1"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ader_ -s 2 -c 2 -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_full.log
