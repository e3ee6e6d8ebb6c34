# A/B of two libvqb200.so builds: cfg2 bench step and cfg3/cfg4-style steps (profile_step), then GPU parity on B
export A=${A:-paper_0910_4711_b200/libvqb200_prev.so} B=${B:-paper_0910_4711_b200/libvqb200.so}
bash tools/ab_lib.sh
for c in ${CFGS:-cfg3}; do for lib in $A $B $A $B; do echo -n "$c $lib: "; VQB200_LIB=$lib timeout 300 python tools/profile_step.py $c 2>&1 | tail -1; done; done
if [ -n "$PARITY" ]; then timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log; fi
