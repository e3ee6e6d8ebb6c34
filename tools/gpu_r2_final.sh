# final round-2 run at HEAD: smoke, GPU parity suite, the reference's own suite through the shim,
# every bench line, sanitize probe
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python -m pytest baseline/_ref/pkg_tests -q -rfE -p no:cacheprovider > gpurun_out/reference_suite.log 2>&1; echo refsuite rc=$?; tail -6 gpurun_out/reference_suite.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
for w in cfg1 cfg3 cfg5 formats; do timeout 1500 python bench.py --workload $w --steps 5 --warmup 2 > gpurun_out/wl_$w.json 2> gpurun_out/wl_$w.err; echo $w rc=$?; done
timeout 300 python tools/sanitize_probe.py > gpurun_out/sanitize_probe.log 2>&1; echo probe rc=$?; tail -2 gpurun_out/sanitize_probe.log
timeout 120 compute-sanitizer --tool memcheck python tools/sanitize_probe.py > gpurun_out/sanitizer.log 2>&1; echo sanitizer rc=$?; tail -3 gpurun_out/sanitizer.log
