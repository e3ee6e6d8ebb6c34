timeout 1800 python -m pytest tests/test_gpu_parity_r2.py -q -x -k "small_codebook or incremental" 2>&1 | tail -5
