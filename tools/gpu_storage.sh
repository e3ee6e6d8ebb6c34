set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests/test_gpu_storage.py -x -q > gpurun_out/pytest_storage.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_storage.log; tail -3 gpurun_out/smoke.log
