for c in cfg2 cfg3; do
timeout 300 python tools/profile_step.py $c > gpurun_out/plain_$c.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sums_kernel -s 2 -c 1 -o gpurun_out/sums_$c python tools/profile_step.py $c > /dev/null 2>&1; echo $c rc=$?
done
