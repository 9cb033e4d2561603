# quick iteration: GPU parity tests, 2M-atom bench in three precisions, launch list
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -2
for p in double mixed single; do timeout 300 python bench.py --steps 20 --warmup 5 --precision $p --no-cpu-baseline --no-e2e > gpurun_out/bench_$p.json 2> gpurun_out/bench_$p.err; echo "$p rc=$?"; done
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f64.csv $B > /dev/null 2>&1; echo ncu rc=$?
