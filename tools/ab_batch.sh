for c in cfg1 cfg2; do for k in 1 2; do for b in 2 4 8 16; do echo -n "$c batch=$b: "; VQB_BATCH=$b python tools/profile_design.py $c | tail -1; done; done; done
