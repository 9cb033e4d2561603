# Round-2 evidence on one GPU box: the asymmetric-cutoff parity test, ncu
# traffic + pipe utilisation of the main force kernel and filter per config and
# precision (profiles/ncu_traffic.json), launch lists of a bench step per
# config, and full source-level captures of the f64 main kernels.
mkdir -p gpurun_out/r2ev
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k asymmetric > gpurun_out/r2ev/asym.log 2>&1; tail -1 gpurun_out/r2ev/asym.log
bash tools/ncu_traffic.sh si2m sic256k liquid512k > gpurun_out/r2ev/traffic.log 2>&1; tail -9 gpurun_out/r2ev/traffic.log
for C in si2m sic256k liquid512k si32k; do
  B="python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-md"
  ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_steps/" --csv \
      --log-file gpurun_out/r2ev/launches_$C.csv $B > /dev/null 2>&1
  echo "launches $C rc=$?"
done
bash tools/ncu_source.sh f64_si2m "k_force<double, double, \(int\)4, \(int\)0, \(bool\)0, \(bool\)0" --precision double > /dev/null 2>&1
bash tools/ncu_source.sh f64_liquid "k_force_packed<double, double, \(int\)0, \(bool\)0, \(bool\)0" --precision double --config liquid512k > /dev/null 2>&1
bash tools/ncu_source.sh mixed_si2m "k_force<float, double, \(int\)4, \(int\)0, \(bool\)0, \(bool\)0" --precision mixed > /dev/null 2>&1
ls gpurun_out/src_* | head -20
