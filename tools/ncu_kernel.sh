# usage: bash tools/ncu_kernel.sh <regex> <tag> [skip] [extra bench args...]
# ncu --set full on one kernel of a short bench run (one GPU); exports raw/details/source CSVs.
K=$1; TAG=$2; SKIP=${3:-0}; shift 3
mkdir -p gpurun_out/ncu_$TAG
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $@"
$B > gpurun_out/ncu_$TAG/plain.log 2>&1 && ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$K" -s $SKIP -c 1 -f -o /tmp/prof_$TAG $B > gpurun_out/ncu_$TAG/ncu.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_$TAG/raw.csv
ncu -i /tmp/prof_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_$TAG/details.csv
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv > gpurun_out/ncu_$TAG/source.csv 2>&1
