# parity suite + the headline bench + the L=64 / large-K workload lines
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
for w in ${WORKLOADS:-cfg3}; do timeout 600 python bench.py --workload $w --steps 3 --warmup 1 > gpurun_out/wl_$w.json 2>gpurun_out/wl_$w.err; echo $w rc=$?; done
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
