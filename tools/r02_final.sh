# Round-2 evidence refresh (one GPU): bench lines per config, the reference
# arm, launch lists of the evaluation step per config and of 100 MD steps,
# pipe/DRAM traffic per main kernel (profiles/ncu_traffic.json), and
# source-level ncu captures of the f64 / mixed main kernels and the f64
# packed SiC kernel.  Outputs under gpurun_out/r02f/ (copied into profiles/).
set -u
O=gpurun_out/r02f
mkdir -p $O
timeout 900 python bench.py > $O/bench_si2m.json 2> $O/bench_si2m.err; echo "bench si2m rc=$?"
for C in sic256k liquid512k si32k; do
  timeout 900 python bench.py --config $C --no-cpu-baseline > $O/bench_$C.json 2> $O/bench_$C.err
  echo "bench $C rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_si2m.json 2> $O/ref.err
echo "ref rc=$?"
for C in si2m sic256k liquid512k si32k; do
  B="python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variants --no-md"
  ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_steps/" --csv \
      --log-file $O/launches_$C.csv $B > /dev/null 2>&1
  echo "launches $C rc=$?"
  python tools/launch_summary.py $O/launches_$C.csv 6 > $O/launches_$C.txt
done
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "md_steps/" --csv \
    --log-file $O/launches_md_si2m.csv python tools/md_launches.py double 100 > /dev/null 2>&1
echo "md launches rc=$?"
python tools/launch_summary.py $O/launches_md_si2m.csv 100 > $O/launches_md_si2m.txt
bash tools/ncu_traffic.sh si2m sic256k liquid512k > $O/traffic.log 2>&1
python tools/ncu_traffic.py > $O/traffic_fold.log 2>&1; cp profiles/ncu_traffic.json $O/ncu_traffic.json
bash tools/ncu_source.sh f64_si2m "k_force<double, double, \(int\)4, \(int\)0, \(bool\)0, \(bool\)0" --precision double --no-md > /dev/null 2>&1
bash tools/ncu_source.sh mixed_si2m "k_force<float, double, \(int\)4, \(int\)0, \(bool\)0, \(bool\)0" --precision mixed --no-md > /dev/null 2>&1
bash tools/ncu_source.sh f64_sic "k_force_packed<double, double, \(int\)1, \(bool\)0, \(bool\)0" --precision double --config sic256k --no-md > /dev/null 2>&1
bash tools/ncu_source.sh f64_liquid "k_force_packed<double, double, \(int\)0, \(bool\)0, \(bool\)0" --precision double --config liquid512k --no-md > /dev/null 2>&1
for T in f64_si2m mixed_si2m f64_sic f64_liquid; do
  python tools/sass_profile.py gpurun_out/src_$T > gpurun_out/src_$T/profile.txt 2>&1
done
echo done
