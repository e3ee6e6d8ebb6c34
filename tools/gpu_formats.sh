# storage parity + formats workload line + ncu launch list of the imaging kernels
set -x
timeout 900 python -m pytest tests/test_gpu_storage.py -x -q > gpurun_out/pytest_storage.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_storage.log
timeout 600 python bench.py --workload formats > gpurun_out/formats.json 2> gpurun_out/formats.err; echo formats rc=$?
tail -5 gpurun_out/formats.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"pixels|blocks|decode|pair_rows|quantize" \
  --log-file gpurun_out/formats_ncu.csv python bench.py --workload formats --steps 1 > /dev/null 2>&1; echo ncu rc=$?
