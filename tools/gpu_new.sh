set -x
timeout 900 python -m pytest tests/test_gpu_storage.py tests/test_cli.py tests/test_gpu_sweep.py -m gpu -x -q > gpurun_out/pytest_new.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_new.log
