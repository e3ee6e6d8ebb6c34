# per-kernel device times of one Lloyd step (tools/profile_step.py) for each config in $CFGS
for c in ${CFGS:-cfg2}; do
  timeout 300 python tools/profile_step.py $c > gpurun_out/plain_$c.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python tools/profile_step.py $c > /dev/null 2>&1
  echo "$c rc=$?"
done
