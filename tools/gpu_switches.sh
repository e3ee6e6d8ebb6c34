# every run-time switch gives the same results: the design / assign parity tests under each setting
for env in "VQB_TC=0" "VQB_SMALL=0 VQB_DIFF=0" "VQB_DELTA=0 VQB_GRAPH=0" "VQB_PDL=0 VQB_DELTA_FRAC=1.0" "VQB_BATCH=1 VQB_SUMS_RED=0"; do
  echo "== $env"; env $env timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -q -x -k "design or incremental or teacher or adversarial or small_codebook or assign" 2>&1 | tail -2
done
