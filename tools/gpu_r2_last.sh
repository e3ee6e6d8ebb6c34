# bench lines of the contract with their wall times (default run, reference arm, torchrun at one rank)
t0=$SECONDS; timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$? wall $((SECONDS-t0)) s"
t0=$SECONDS; timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$? wall $((SECONDS-t0)) s"
t0=$SECONDS; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err; echo "torchrun rc=$? wall $((SECONDS-t0)) s"
t0=$SECONDS; timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_default.json 2> gpurun_out/bench_ref_default.err; echo "ref default rc=$? wall $((SECONDS-t0)) s"
