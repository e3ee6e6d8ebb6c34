for k in 1 2; do for mb in 2 4 8 16; do echo -n "piece ${mb}MB: "; VQB_PIECE_MB=$mb timeout 300 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['e2e']['ms_per_step'],4), round(d['e2e']['value'],1))"; done; done
