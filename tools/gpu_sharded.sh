# the multi-GPU code path on one GPU: 2-rank gloo Lloyd test + torchrun world-1 sharded bench
set -x
timeout 900 python -m pytest tests/test_gpu_distributed.py -q -x > gpurun_out/pytest_dist.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_dist.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --sharded > gpurun_out/bench_sharded.json 2> gpurun_out/bench_sharded.err; echo sharded rc=$?
tail -3 gpurun_out/bench_sharded.err
python -c "import json; d=json.loads(open('gpurun_out/bench_sharded.json').read().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['config'])"
