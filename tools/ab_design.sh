# A/B of two libvqb200.so builds on full device-resident designs (tools/profile_design.py)
export A=${A:-paper_0910_4711_b200/libvqb200_prev.so} B=${B:-paper_0910_4711_b200/libvqb200.so}
for c in ${CFGS:-cfg2}; do for lib in $A $B $A $B; do echo -n "$lib: "; VQB200_LIB=$lib timeout 600 python tools/profile_design.py $c 2>&1 | tail -1; done; done
