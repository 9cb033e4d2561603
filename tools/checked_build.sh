# Build the bounds-checked library (device asserts, TSF_BOUNDS_CHECK) next to
# the product one and run the small-case sweep and the GPU parity suite on it.
# On a GPU box:  bash tools/checked_build.sh   (the .so is prebuilt here: make
# -C paper_1607_02904_b200/csrc OUT=../_checked/libtersoff_b200.so OBJ=../_checked/obj
# EXTRA=-DTSF_BOUNDS_CHECK)
LIB=paper_1607_02904_b200/_checked/libtersoff_b200.so
mkdir -p gpurun_out/checked
TSF_LIBRARY=$LIB python tools/sanitize_case.py > gpurun_out/checked/sanitize_case.log 2>&1
echo "sanitize_case rc=$?"
TSF_LIBRARY=$LIB timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not refverify and not engine_run" > gpurun_out/checked/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/checked/pytest_gpu.log
