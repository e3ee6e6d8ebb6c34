# every BASELINE config on one B200 (bench.py --workload), one JSON line each
for w in cfg1 cfg3 cfg5 cfg4; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 1 > gpurun_out/wl_$w.json 2> gpurun_out/wl_$w.err; echo "$w rc=$?"
done
