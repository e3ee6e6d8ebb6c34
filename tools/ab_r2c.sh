# A/B: P = HEAD build, B = current; step segments at several sizes, then the role profile of the TC pass
P=paper_0910_4711_b200/libvqb200_prev.so; B=paper_0910_4711_b200/libvqb200.so
for c in ${CFGS:-"cfg4" "cfg4 1024" "cfg4 256" "cfg4 64" "cfg2" "cfg2 256" "cfg3" "cfg3 64"}; do
  for lib in $P $B $P $B; do echo -n "$c $lib: "; VQB200_LIB=$lib timeout 300 python tools/profile_step.py $c 2>&1 | tail -1; done
done
if [ -f paper_0910_4711_b200/libvqb200_prof.so ]; then
  for c in "cfg4" "cfg4 256" "cfg4 64" "cfg2 256"; do echo "== role profile $c"; VQB_TC_PROF=1 VQB200_LIB=paper_0910_4711_b200/libvqb200_prof.so timeout 300 python tools/profile_step.py $c 2>&1 | tail -6; done
fi
