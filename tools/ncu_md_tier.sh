# ncu --set full of one packed tier launch (the atoms over 4) in the middle of
# the 2M-atom 1600 K MD run (tools/md_launches.py), source-level export
O=gpurun_out/src_md_tier
rm -f /tmp/prof_md_tier.ncu-rep
mkdir -p $O
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    --nvtx --nvtx-include "tier_eval/" -k "regex:k_force_packed<double, double, \(int\)0, \(bool\)0, \(bool\)1" \
    -c 1 -o /tmp/prof_md_tier env TSF_PACKED_OVER4=100 python tools/md_tier_state.py double > $O/ncu.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_md_tier.ncu-rep --page raw --csv > $O/raw.csv
ncu -i /tmp/prof_md_tier.ncu-rep --page details --csv > $O/details.csv
ncu -i /tmp/prof_md_tier.ncu-rep --page source --print-source sass --csv > $O/sass.csv 2>&1
ncu -i /tmp/prof_md_tier.ncu-rep --page source --print-source cuda,sass --csv > $O/cuda_sass.csv 2>&1
python tools/sass_profile.py $O > $O/profile.txt 2>&1
