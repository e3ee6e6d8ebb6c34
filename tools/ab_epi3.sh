# three-way: P = previous, B = current, C = variant
P=paper_0910_4711_b200/libvqb200_prev.so; B=paper_0910_4711_b200/libvqb200.so; C=${C:-paper_0910_4711_b200/libvqb200_a2.so}
for c in ${CFGS:-"cfg4" "cfg4 256" "cfg4 64" "cfg2" "cfg2 256" "cfg2 64"}; do
  for lib in $P $B $C $P $B $C; do echo -n "$c $lib: "; VQB200_LIB=$lib timeout 300 python tools/profile_step.py $c 2>&1 | tail -1; done
done
