# usage: bash tools/ncu_source.sh <tag> <kernel-regex> [bench args...]
# One `ncu --set full --import-source on` capture of the first matching launch
# inside the steady state (NVTX range bench_steps), exported as raw / details /
# per-SASS-line source CSVs under gpurun_out/src_<tag>/ (TSF_LIBRARY is honoured).
TAG=$1; K=$2; shift 2
OUT=gpurun_out/src_$TAG
mkdir -p $OUT
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variants $@"
$B > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    --nvtx --nvtx-include "bench_steps/" -k "regex:$K" -c 1 -f -o /tmp/prof_$TAG $B > $OUT/ncu.log 2>&1
echo "ncu $TAG rc=$?"
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > $OUT/raw.csv
ncu -i /tmp/prof_$TAG.ncu-rep --page details --csv > $OUT/details.csv
ncu -i /tmp/prof_$TAG.ncu-rep --page source --print-source sass --csv > $OUT/sass.csv 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page source --print-source cuda,sass --csv > $OUT/cuda_sass.csv 2>&1
