# round 2: headline bench (cfg4) + reference arm + ncu launch list + full capture of assign_tc at cfg4
set -x
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 600 python bench.py --profile-steps --steps 3 --warmup 3 > gpurun_out/plain_profile.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv \
  python bench.py --profile-steps --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
timeout 300 python tools/profile_step.py cfg4 > gpurun_out/plain_step.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:assign_tc -s 2 -c 1 \
  -o gpurun_out/tc_full_cfg4 python tools/profile_step.py cfg4 > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
