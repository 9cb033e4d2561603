set -u
python tools/ab.py _exp/lib_head.so "" 3 sic256k liquid512k si2m > gpurun_out/ab_fin.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "packed or numeric or nonfinite or tier or virial" > gpurun_out/pytest_packed.log 2>&1; echo "pytest rc=$?"
bash tools/ncu_source.sh f64_si2m "k_force<double, double, \(int\)4, \(int\)0, \(bool\)0, \(bool\)0" --precision double --no-md > /dev/null 2>&1
python tools/sass_profile.py gpurun_out/src_f64_si2m > gpurun_out/src_f64_si2m/profile.txt 2>&1
bash tools/ncu_md_tier.sh > /dev/null 2>&1
python tools/sass_profile.py gpurun_out/src_md_tier > gpurun_out/src_md_tier/profile.txt 2>&1
echo done
