# round evidence at HEAD: parity suite, smoke, every bench line, ncu launch list + full capture
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
for w in cfg1 cfg3 cfg5 formats cfg4; do timeout 1500 python bench.py --workload $w --steps 5 --warmup 2 > gpurun_out/wl_$w.json 2> gpurun_out/wl_$w.err; echo $w rc=$?; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --profile-steps --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_tc -s 2 -c 1 \
  -o gpurun_out/tc_full python tools/profile_step.py cfg2 > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assign_tc -s 2 -c 1 \
  -o gpurun_out/tc64_full python tools/profile_step.py cfg3 > gpurun_out/ncu_full64.log 2>&1; echo full64 rc=$?
tail -2 gpurun_out/pytest_gpu.log
for c in cfg2 cfg3; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/launches_${c}_step.csv python tools/profile_step.py $c > /dev/null 2>&1; echo step_$c rc=$?
done
python tools/design_levels.py cfg2 > gpurun_out/design_levels.txt 2>&1; python tools/design_levels.py cfg4 >> gpurun_out/design_levels.txt 2>&1; echo levels rc=$?
