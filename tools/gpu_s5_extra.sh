#!/bin/bash
# Fifth session: LinA line on the committed code; wall-clock of the default bench command and
# of the reference arm (what the driver runs at round end).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out
timeout 600 python bench.py --config lina --e2e-reps 1 > $O/s5_bench_lina.json 2> $O/s5_bench_lina.err; echo lina_rc=$?
python -c "import json;d=json.load(open('$O/s5_bench_lina.json'));print('lina',d['value'],d['ms_per_step'],d['roofline']['frac'])"
s=$(date +%s.%N); timeout 900 python bench.py > $O/s5_bench_c1_b.json 2> $O/s5_bench_c1_b.err; echo c1_rc=$? wall=$(echo "$(date +%s.%N) - $s" | bc)
python -c "import json;d=json.load(open('$O/s5_bench_c1_b.json'));print('c1',d['value'],d['ms_per_step'],d['roofline']['frac'],d['clocks'])"
s=$(date +%s.%N); timeout 900 python bench.py --impl reference > $O/s5_bench_ref_b.json 2> $O/s5_bench_ref_b.err; echo ref_rc=$? wall=$(echo "$(date +%s.%N) - $s" | bc)
tail -c 300 $O/s5_bench_ref_b.json
