export A=${A:-paper_0910_4711_b200/libvqb200_prev.so} B=${B:-paper_0910_4711_b200/libvqb200.so}
for c in "cfg4" "cfg4 256" "cfg4 64" "cfg2" "cfg2 256" "cfg2 64" "cfg3" "cfg3 64"; do
  for lib in $A $B $A $B; do echo -n "$c $lib: "; VQB200_LIB=$lib timeout 300 python tools/profile_step.py $c 2>&1 | tail -1; done
done
if [ -n "$PARITY" ]; then timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log; fi
