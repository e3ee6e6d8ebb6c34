# ncu --set full of the small-K pass kernels (sums + FFMA candidate pass) at K=${K:-2}
timeout 300 python tools/profile_step.py cfg2 ${K:-2} > gpurun_out/plain_k.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sums_kernel|assign_fast" -s 4 -c 2 \
  -o gpurun_out/smallk_${K:-2} python tools/profile_step.py cfg2 ${K:-2} > gpurun_out/ncu_smallk.log 2>&1; echo rc=$?
