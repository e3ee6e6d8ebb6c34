# ncu full captures: FFMA pass at cfg4 K=8, TC pass at cfg4 K=256 (plain runs first)
set -x
timeout 300 python tools/profile_step.py cfg4 8 > gpurun_out/plain_step8.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_fast -s 2 -c 1 \
  -o gpurun_out/fast_cfg4_k8 python tools/profile_step.py cfg4 8 > gpurun_out/ncu_fast.log 2>&1
timeout 300 python tools/profile_step.py cfg4 256 > gpurun_out/plain_step256.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_tc -s 4 -c 1 \
  -o gpurun_out/tc_cfg4_k256 python tools/profile_step.py cfg4 256 > gpurun_out/ncu_tc256.log 2>&1
python tools/ncu_summary.py gpurun_out/fast_cfg4_k8.ncu-rep > gpurun_out/fast_cfg4_k8.txt 2>&1
python tools/ncu_summary.py gpurun_out/tc_cfg4_k256.ncu-rep > gpurun_out/tc_cfg4_k256.txt 2>&1
cat gpurun_out/fast_cfg4_k8.txt gpurun_out/tc_cfg4_k256.txt
P=paper_0910_4711_b200/libvqb200_prev.so; B=paper_0910_4711_b200/libvqb200.so
for c in "cfg4" "cfg4 256"; do
  for lib in $P $B $P $B; do echo -n "$c $lib: "; VQB200_LIB=$lib timeout 300 python tools/profile_step.py $c 2>&1 | tail -1; done
done
