# usage: bash tools/ncu_traffic.sh [config...]
# DRAM bytes, duration and pipe utilisation per launch of the main force
# kernel (OVF = FOREIGN = false: not the tier launches) and the filter
# for each config x precision (tools/ncu_traffic.py folds the CSVs into
# profiles/ncu_traffic.json for bench.py's roofline.traffic).  One GPU; each
# bench command runs once without ncu first.
CFGS=${@:-si2m}
mkdir -p gpurun_out/traffic
for C in $CFGS; do
  for P in double mixed single; do
    B="python bench.py --config $C --precision $P --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variants"
    $B > gpurun_out/traffic/plain_${C}_$P.log 2>&1 || { echo "plain $C $P failed"; continue; }
    M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
    M=$M,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed
    M=$M,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_elapsed
    M=$M,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed
    M=$M,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_elapsed
    M=$M,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed
    M=$M,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_elapsed
    M=$M,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_elapsed
    M=$M,smsp__issue_active.avg.pct_of_peak_sustained_elapsed
    M=$M,sm__throughput.avg.pct_of_peak_sustained_elapsed
    ncu --metrics $M \
        --clock-control none --kernel-name-base demangled --nvtx --nvtx-include "bench_steps/" \
        -k 'regex:k_force<[^(]*\(int\)[0-9]+, \(int\)[0-9]+, \(bool\)[01], \(bool\)0|k_force_packed<[^(]*\(int\)[0-9]+, \(bool\)[01], \(bool\)0|k_filter' -s 2 -c 4 --csv \
        --log-file gpurun_out/traffic/${C}_$P.csv $B > gpurun_out/traffic/ncu_${C}_$P.log 2>&1
    echo "ncu $C $P rc=$?"
  done
done
