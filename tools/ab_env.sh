# A/B of an environment switch (${VAR}=0 vs default) on the bench step and a design
for k in 1 2; do
for v in 0 1; do
  echo -n "$VAR=$v step: "; env $VAR=$v timeout 300 python bench.py --steps 30 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['segments_ms'].items()})"
  echo -n "$VAR=$v design: "; env $VAR=$v timeout 300 python tools/profile_design.py ${CFG:-cfg2} | tail -1
done; done
