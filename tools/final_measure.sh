# One-call refresh of the round's evidence (one GPU): bench lines per config,
# the ncu launch list, pipe/DRAM traffic per kernel, and ncu --set full of the
# f64 / mixed force kernels and the steady-state filter.  Outputs under
# gpurun_out/final/ (copied into profiles/ by hand).
set -u
mkdir -p gpurun_out/final
for C in si2m sic256k liquid512k; do
  timeout 900 python bench.py --config $C > gpurun_out/final/bench_$C.json 2> gpurun_out/final/bench_$C.err
  echo "bench $C rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/ref.json 2> gpurun_out/final/ref.err
echo "ref rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/final/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/final/launches_si2m_f64.csv $B > gpurun_out/final/ncu_launches.log 2>&1
echo "launches rc=$?"
bash tools/ncu_traffic.sh si2m sic256k liquid512k
bash tools/ncu_kernel.sh 'k_force<double, double, \(int\)4' f64c 0
bash tools/ncu_kernel.sh 'k_force<float, double, \(int\)4' mixed4c 0 --precision mixed
bash tools/ncu_kernel.sh 'k_filter' filt 1
