# ncu --set full on the list kernels (k_skin_list, k_filter); one GPU.
mkdir -p gpurun_out/ncu2
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
export TSF_FUSE_FILTER=0
$B > gpurun_out/ncu2/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_skin_list|k_filter" -c 2 -f -o /tmp/prof_lists $B > gpurun_out/ncu2/ncu.log 2>&1
echo rc=$?
ncu -i /tmp/prof_lists.ncu-rep --page raw --csv > gpurun_out/ncu2/raw_lists.csv
ncu -i /tmp/prof_lists.ncu-rep --page details --csv > gpurun_out/ncu2/details_lists.csv
ncu -i /tmp/prof_lists.ncu-rep --page source --csv > gpurun_out/ncu2/source_lists.csv 2>&1
