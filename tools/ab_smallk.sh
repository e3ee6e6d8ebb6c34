export A=${A:-paper_0910_4711_b200/libvqb200_prev.so} B=${B:-paper_0910_4711_b200/libvqb200.so}
for k in 2 8 32; do for lib in $A $B $A $B; do echo -n "K=$k $lib: "; VQB200_LIB=$lib timeout 300 python tools/profile_step.py cfg2 $k 2>&1 | tail -1; done; done
