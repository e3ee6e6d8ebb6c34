timeout 1200 python -m pytest tests/test_gpu_parity_r2.py -q -x -k "incremental" 2>&1 | tail -5
for c in cfg2 cfg3; do timeout 600 python tools/delta_ab.py $c 0.3 2>&1 | tail -14; done
timeout 900 python tools/delta_ab.py cfg4 0.3 2>&1 | tail -16
B=paper_0910_4711_b200/libvqb200.so
for c in "cfg4 2" "cfg4 8" "cfg4 32" "cfg2 8" "cfg3 8"; do
  for pf in 0 1 0 1; do echo -n "$c pf=$pf: "; VQB_FAST_PF=$pf timeout 300 python tools/profile_step.py $c 2>&1 | tail -1; done
done
P=paper_0910_4711_b200/libvqb200_prev.so
for c in "cfg4" "cfg4 256" "cfg3" "cfg3 64"; do
  for lib in $P $B $P $B; do echo -n "$c $lib: "; VQB200_LIB=$lib timeout 300 python tools/profile_step.py $c 2>&1 | tail -1; done
done
