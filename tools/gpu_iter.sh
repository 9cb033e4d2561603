timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for f in 1 0; do for p in double mixed; do TSF_FUSE_FILTER=$f timeout 300 python bench.py --steps 20 --warmup 5 --precision $p --no-cpu-baseline --no-e2e > gpurun_out/bench_${p}_f$f.json 2> gpurun_out/bench_$p.err; echo "$p rc=$?"; done; done
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
TSF_FUSE_FILTER=0 $B > /dev/null 2>&1 && TSF_FUSE_FILTER=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f64.csv $B > /dev/null 2>&1; echo ncu rc=$?
