# FMNMX3 microbenchmarks + ncu full capture of the TC candidate pass at cfg4 (after a plain run exits 0)
set -x
MB_ONLY=7,8,17,18 python tools/microbench.py > gpurun_out/microbench_fmnmx3.json 2>&1; cat gpurun_out/microbench_fmnmx3.json
timeout 300 python tools/profile_step.py cfg4 > gpurun_out/plain_step.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:assign_tc -s 2 -c 1 \
  -o gpurun_out/tc_full_cfg4_r2b python tools/profile_step.py cfg4 > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
python tools/ncu_summary.py gpurun_out/tc_full_cfg4_r2b.ncu-rep > gpurun_out/tc_full_cfg4_r2b.txt 2>&1; cat gpurun_out/tc_full_cfg4_r2b.txt
