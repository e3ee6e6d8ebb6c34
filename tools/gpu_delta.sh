# incremental sums A/B (designs), then step segments A/B (P = HEAD, B = current)
for c in cfg1 cfg2 cfg3; do timeout 600 python tools/delta_ab.py $c 0.3 2>&1 | tail -20; done
timeout 900 python tools/delta_ab.py cfg4 0.2 0.4 2>&1 | tail -40
P=paper_0910_4711_b200/libvqb200_prev.so; B=paper_0910_4711_b200/libvqb200.so
for c in "cfg4" "cfg4 256" "cfg4 64" "cfg2" "cfg2 256" "cfg3" "cfg3 64"; do
  for lib in $P $B $P $B; do echo -n "$c $lib: "; VQB200_LIB=$lib timeout 300 python tools/profile_step.py $c 2>&1 | tail -1; done
done
