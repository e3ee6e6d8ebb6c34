P=paper_0910_4711_b200/libvqb200_prev.so; B=paper_0910_4711_b200/libvqb200.so
for c in "cfg4" "cfg4 1024" "cfg4 256" "cfg2" "cfg3"; do
  for lib in $P $B $P $B; do echo -n "$c $lib: "; VQB200_LIB=$lib timeout 300 python tools/profile_step.py $c 2>&1 | tail -1; done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -q -x 2>&1 | tail -3
