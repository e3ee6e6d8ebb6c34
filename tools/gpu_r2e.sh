# round-2 checkpoint: smoke, GPU parity suite, headline bench + reference arm, cfg2/cfg3 lines
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
for w in cfg1 cfg3; do timeout 900 python bench.py --workload $w --steps 5 --warmup 2 > gpurun_out/wl_$w.json 2> gpurun_out/wl_$w.err; echo $w rc=$?; cat gpurun_out/wl_$w.json; done
timeout 900 python tools/delta_ab.py cfg4 0.3 2>&1 | tail -16
