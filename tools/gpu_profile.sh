# ncu evidence for the round: launch list of the bench step + full capture of the top kernel
set -x
timeout 600 python bench.py --profile-steps --steps 3 --warmup 3 > gpurun_out/plain_profile.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --profile-steps --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
timeout 300 python tools/profile_step.py ${CFG:-cfg2} > gpurun_out/plain_step.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-assign_tc} -s 2 -c 1 \
  -o gpurun_out/${REPNAME:-tc_full} python tools/profile_step.py ${CFG:-cfg2} > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
