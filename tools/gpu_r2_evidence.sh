# round-2 evidence at HEAD: ncu launch list of the bench step, full captures of the dominant kernel, per-level design times
set -x
timeout 600 python bench.py --profile-steps --steps 3 --warmup 3 > gpurun_out/plain_profile.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv \
  python bench.py --profile-steps --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
timeout 300 python tools/profile_step.py cfg4 > gpurun_out/plain_step.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:assign_tc -s 2 -c 1 \
  -o gpurun_out/tc_full_cfg4_final python tools/profile_step.py cfg4 > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
timeout 300 python tools/profile_step.py cfg2 > gpurun_out/plain_step2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_tc -s 2 -c 1 \
  -o gpurun_out/tc_full_cfg2_final python tools/profile_step.py cfg2 > gpurun_out/ncu_full2.log 2>&1
echo full2 rc=$?
timeout 300 python tools/profile_step.py cfg4 8 > gpurun_out/plain_step8.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_small -s 2 -c 1 \
  -o gpurun_out/small_cfg4_k8 python tools/profile_step.py cfg4 8 > gpurun_out/ncu_small.log 2>&1
echo small rc=$?
for c in cfg1 cfg2 cfg3 cfg4; do timeout 600 python tools/design_levels.py $c; done > gpurun_out/design_levels_final.txt 2>&1
cat gpurun_out/design_levels_final.txt
