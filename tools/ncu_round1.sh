# ncu evidence for the force kernel (run under gpurun; one GPU).
set -x
mkdir -p gpurun_out/ncu
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/ncu/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_f64.csv $B > gpurun_out/ncu/ncu_l.log 2>&1
for P in double mixed; do
  B2="$B --precision $P"
  $B2 > gpurun_out/ncu/plain_$P.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_force -s 4 -c 1 -o /tmp/prof_force_$P $B2 > gpurun_out/ncu/ncu_$P.log 2>&1
  ncu -i /tmp/prof_force_$P.ncu-rep --page raw --csv > gpurun_out/ncu/raw_$P.csv
  ncu -i /tmp/prof_force_$P.ncu-rep --page details --csv > gpurun_out/ncu/details_$P.csv
  ncu -i /tmp/prof_force_$P.ncu-rep --page source --csv > gpurun_out/ncu/source_$P.csv 2>&1
  ls -la /tmp/prof_force_$P.ncu-rep
  cp /tmp/prof_force_$P.ncu-rep gpurun_out/ncu/ 2>/dev/null
done
du -sh gpurun_out/ncu/*
