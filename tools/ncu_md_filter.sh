O=gpurun_out/src_md_filter
mkdir -p $O
rm -f /tmp/prof_md_filter.ncu-rep
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    --nvtx --nvtx-include "tier_eval/" -k "regex:k_filter" \
    -c 1 -o /tmp/prof_md_filter env TSF_PACKED_OVER4=100 python tools/md_tier_state.py double > $O/ncu.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_md_filter.ncu-rep --page raw --csv > $O/raw.csv
ncu -i /tmp/prof_md_filter.ncu-rep --page source --print-source sass --csv > $O/sass.csv 2>&1
ncu -i /tmp/prof_md_filter.ncu-rep --page source --print-source cuda,sass --csv > $O/cuda_sass.csv 2>&1
python tools/sass_profile.py $O > $O/profile.txt 2>&1
