for c in "cfg3 2" "cfg3 8" "cfg3 16" "cfg3 32"; do
  for d in 0 1 0 1; do echo -n "$c diff=$d: "; VQB_DIFF=$d timeout 300 python tools/profile_step.py $c 2>&1 | tail -1; done
done
for d in 0 1; do echo "== VQB_DIFF=$d"; VQB_DIFF=$d timeout 600 python tools/design_levels.py cfg3; done
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py tests/test_gpu_storage.py -q -x 2>&1 | tail -3
