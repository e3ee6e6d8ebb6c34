# A/B of two builds on encode() of 2^25 pageable float32 rows and lbg_train from numpy (cfg2)
export A=${A:-paper_0910_4711_b200/libvqb200_prev.so} B=${B:-paper_0910_4711_b200/libvqb200.so}
for lib in $A $B $A $B; do echo -n "$lib: "; VQB200_LIB=$lib python - <<'PY'
import time, numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import paper_0910_4711_b200 as vq
from paper_0910_4711_b200 import synthetic
cb, q = synthetic.make_encode_case(1 << 25)
C = vq.Codebook(cb.astype(np.float64))
t = []
for _ in range(4):
    t0 = time.perf_counter(); vq.encode(q, C); t.append(time.perf_counter() - t0)
x = synthetic.make_training("cfg2")
conf = vq.LbgConfig(target_size=1024, epsilon=1e-4, delta=0.01)
d = []
for _ in range(3):
    t0 = time.perf_counter(); vq.lbg_train(vq.TrainingSet(x), conf); d.append(time.perf_counter() - t0)
print("encode 2^25", round(min(t[1:]), 4), "design e2e", round(min(d[1:]), 4))
PY
done
