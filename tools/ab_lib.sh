# A/B of two builds of libvqb200.so on the headline step: ${A} vs ${B} (paths), alternating
for k in 1 2; do
for lib in ${A} ${B}; do
  VQB200_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$lib', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['segments_ms'].items()}, d['rerank_rows_per_step'])"
done; done
